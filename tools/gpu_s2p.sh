#!/bin/bash
# round-2 session-2 query A/B: read-sketch loop stops at the warp's longest window (q1), + even / odd windows
# of a tile in separate warps so full read windows take the fast sketch path (q2)
TAG=${1:-s2p}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/q2.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_multigpu.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/q0.so build_ab/q1.so build_ab/q2.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} kal $V
bash tools/ab_bench_wl.sh ${TAG} hiseq $V
bash tools/ab_bench_wl.sh ${TAG} miseq $V
