for cfgs in "${@:-8 1.0}"; do set -- $cfgs
 echo -n "chunks $1 taper $2: "; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-mode --chunks $1 --chunk-taper $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dev %.3f ms  e2e %.3f ms p99 %.3f' % (d['ms_per_step'], 1000/d['e2e']['hz'], d['e2e']['p99_latency_ms']))"
done
