#!/bin/bash
# ncu evidence for profiles/: launch list of one bench run + full captures of K2/K3/K1 and
# of the f-row kernels (collision field, MPPI, exact enumeration).  Then, here:
#   python tools/write_profiles.py --tag rNN   (profiles/ + ncu_summary.json)
set -x
# PART=a|b splits the captures over two gpurun calls (each call brings back <= 64 MiB)
PART=${PART:-all}
# launch list of the bench's cycle (latency percentiles over --steps only: under ncu every
# launch is serialised and replayed, so the default 1000 latency cycles would take an hour)
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ref-mode --lat-cycles 0"
if [ "$PART" != b ]; then
$B > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $B > gpurun_out/ncu_launch.log 2>&1
python tools/profile_predict.py --steps 250 --cycles 3 > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_predict|k_epilogue|k_belief" -s 3 -c 3 \
    -o gpurun_out/cycle_cfg3 python tools/profile_predict.py --steps 250 --cycles 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_predict -s 1 -c 1 \
    -o gpurun_out/k2_cfg3 python tools/profile_predict.py --steps 250 --cycles 2 > gpurun_out/ncu_k2.log 2>&1
fi
[ "$PART" = a ] && exit 0
python tools/profile_predict.py --mode reference --steps 20 --cycles 2 > gpurun_out/plain_ref.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_predict -s 1 -c 1 \
    -o gpurun_out/k2_refmode python tools/profile_predict.py --mode reference --steps 20 --cycles 2 > gpurun_out/ncu_ref.log 2>&1
python tools/profile_extras.py > gpurun_out/plain_extras.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_collision|k_mppi|k_exact" -s 2 -c 6 \
    -o gpurun_out/extras python tools/profile_extras.py > gpurun_out/ncu_extras.log 2>&1
# every other kernel of the library (unions, time union, naive, emplace, smooth, sampling,
# propagate_step) at the small sizes of tools/sanitize_run.py
python tools/sanitize_run.py > gpurun_out/plain_aux.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"k_(union|time_union|naive|emplace|smooth|sample_hyp|propagate_step)" -c 12 \
    -o gpurun_out/aux python tools/sanitize_run.py > gpurun_out/ncu_aux.log 2>&1
# the tile-sparse D2H publication of the e2e cycle (f64 union)
timeout 900 ncu --set full --clock-control none -k regex:k_publish -s 8 -c 4 -o gpurun_out/publish \
    $B --no-e2e-alt > gpurun_out/ncu_publish.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log gpurun_out/ncu_publish.log gpurun_out/ncu_full.log gpurun_out/ncu_k2.log gpurun_out/ncu_ref.log gpurun_out/ncu_extras.log
