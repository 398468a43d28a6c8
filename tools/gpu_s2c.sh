#!/bin/bash
# round-2 session-2 A/B: 8-char sketch loop (MC_HALF_ITER), rolled feature loop, CE on FMA pipe, direct scatter
TAG=${1:-s2c}
mkdir -p gpurun_out
for v in h1 h1d; do
  MC_LIB_PATH=$PWD/build_ab/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch_parity or db_parity or classify_parity_tiny or low_complexity or heavy_keys or spill" > gpurun_out/${TAG}_pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 gpurun_out/${TAG}_pytest_$v.log
done
V="build_ab/base.so build_ab/ce1.so build_ab/h0.so build_ab/h1.so build_ab/h5.so build_ab/h1d.so build_ab/h0d.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
MC_LIB_PATH=$PWD/build_ab/h1.so bash tools/ncu_kernel.sh ${TAG}_sk k_sketch_partition 1 1 --no-cpu-baseline --no-e2e
