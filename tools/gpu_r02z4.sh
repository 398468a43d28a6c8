#!/bin/bash
TAG=${1:-r02z4}
mkdir -p gpurun_out
for rep in 1 2 3; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset ab/base.so ab/fs.so ab/w2fs.so ab/w2fsu6.so; done
