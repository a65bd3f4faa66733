#!/bin/bash
# one GPU iteration: parity tests, K2 timing at cfg3, ncu capture of K2 (T=60)
TAG=${1:-iter}
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/profile_predict.py --steps 250 --cycles 3 2>&1 | tail -2
timeout 300 python tools/profile_predict.py --steps 60 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_predict -s 1 -c 1 \
    -o gpurun_out/k2_$TAG python tools/profile_predict.py --steps 60 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
