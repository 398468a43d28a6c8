#!/bin/bash
TAG=${1:-r02z2}
mkdir -p gpurun_out
bash tools/ab_bench_wl.sh $TAG subset ab/base.so ab/pc4.so ab/pc8.so ab/pc4l4.so ab/base.so
bash tools/ab_bench_wl.sh $TAG kal ab/base.so ab/pc4l4.so
MC_LIB_PATH=$PWD/ab/qprof_pc4.so timeout 600 python tools/qprof.py subset 2>&1 | tail -20
