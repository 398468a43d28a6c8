#!/bin/bash
# round-2 session-2 A/B: sketch_partition at 4 CTAs/SM (64 registers, region recomputed at write-out instead of
# staged), span staged with all loads in flight (MC_STAGE_WIDE)
TAG=${1:-s2d}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/k4.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest_k4.log 2>&1; echo "pytest k4 rc=$?"; tail -1 gpurun_out/${TAG}_pytest_k4.log
V="build_ab/cur.so build_ab/k4n.so build_ab/k4.so build_ab/k3w.so build_ab/k4c0.so build_ab/k4c5.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 build_ab/cur.so build_ab/k4.so build_ab/k3w.so
MC_LIB_PATH=$PWD/build_ab/k4.so bash tools/ncu_kernel.sh ${TAG}_sk k_sketch_partition 1 1 --no-cpu-baseline --no-e2e
