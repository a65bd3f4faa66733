#!/bin/bash
# A/B the K2 of library builds on one GPU, interleaved.  Default: A = _lib/ab/libA.so
# (tools/ab_build.sh <git-rev>) vs B = the working-tree build; or pass the libraries.
LIBS=("$@")
[ ${#LIBS[@]} -eq 0 ] && LIBS=(paper_2603_01122_b200/_lib/ab/libA.so paper_2603_01122_b200/_lib/libgridcast_b200.so)
for r in 1 2 3; do
  for lib in "${LIBS[@]}"; do
    echo -n "$(basename $lib): "; GC_LIB_PATH=$PWD/$lib timeout 300 python tools/profile_predict.py --steps ${STEPS:-250} --cycles 6 --summary
  done
done
