#!/bin/bash
# round-2 session-2 A/B of the build sketch: candidate filter (MC_SKETCH_FILTER), merge of 16 (MC_MERGE16),
# compare-exchange max on the FMA pipe (MC_CE_FMA / MC_SORT_FMA_N), threshold (MC_THR0); parity first
TAG=${1:-s2b}
mkdir -p gpurun_out
for v in f1 f1s20 m16s20; do
  MC_LIB_PATH=$PWD/build_ab/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch_parity or db_parity or classify_parity_tiny or low_complexity or heavy_keys" > gpurun_out/${TAG}_pytest_$v.log 2>&1; echo "pytest $v rc=$?"; tail -1 gpurun_out/${TAG}_pytest_$v.log
done
V="build_ab/base.so build_ab/ce1.so build_ab/m16s20.so build_ab/f0.so build_ab/f1.so build_ab/f1s20.so build_ab/f1t28.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
MC_LIB_PATH=$PWD/build_ab/f1.so bash tools/ncu_kernel.sh ${TAG}_sk k_sketch_partition 1 1 --no-cpu-baseline --no-e2e
