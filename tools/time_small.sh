#!/bin/bash
# cfg1 / cfg2 device cycle (bench.py, CUDA graph) for library builds given as arguments
for L in "$@"; do
  for c in cfg1 cfg2; do
    echo -n "$(basename $(dirname $L))/$(basename $L) $c: "
    GC_LIB_PATH=$PWD/$L python bench.py --config $c --steps 20 --no-cpu-baseline --no-ref-mode --lat-cycles 200 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms' % d['ms_per_step'])"
  done
done
