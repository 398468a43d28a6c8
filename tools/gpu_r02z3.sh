#!/bin/bash
TAG=${1:-r02z3}
mkdir -p gpurun_out
bash tools/ab_bench_wl.sh $TAG subset ab/base.so ab/w2fs.so ab/w2fsu6.so ab/w2fsu8.so ab/w2.so ab/fs.so ab/base.so
bash tools/ab_bench_wl.sh $TAG kal ab/base.so ab/w2fs.so ab/w2fsu8.so
