#!/bin/bash
TAG=${1:-r02z5}
mkdir -p gpurun_out
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset ab/u4.so ab/u5.so ab/u6.so; done
bash tools/ab_bench_wl.sh $TAG kal ab/u4.so ab/u5.so ab/u6.so
bash tools/ab_bench_wl.sh $TAG refseq8 ab/u4.so ab/u5.so ab/u6.so
