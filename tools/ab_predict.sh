#!/bin/bash
# A/B the K2 of two library builds on one GPU, interleaved: A = paper_.../_lib/ab/libA.so
# (build it with tools/ab_build.sh <git-rev>), B = the working-tree build.
A=paper_2603_01122_b200/_lib/ab/libA.so
B=paper_2603_01122_b200/_lib/libgridcast_b200.so
for r in 1 2 3; do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    echo -n "$v: "; GC_LIB_PATH=$PWD/$lib timeout 300 python tools/profile_predict.py --steps ${STEPS:-250} --cycles 6 --summary
  done
done
