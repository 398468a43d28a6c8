#!/bin/bash
# round-2 session-2 query A/B: branch-free small-bin gather (MC_QS_BF), 8-char checked sketch loop (MC_HALF_ITER_SLOT)
TAG=${1:-s2k}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/qbfhs.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/qbf0.so build_ab/qbf.so build_ab/hs1.so build_ab/qbfhs.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} kal $V
bash tools/ab_bench_wl.sh ${TAG} hiseq $V
