#!/bin/bash
# round-2 session-2: finalize rank parking (values range, staged sub-regions) + sketch tile of 384 windows
TAG=${1:-s2j}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_refseq.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
MC_LIB_PATH=$PWD/build_ab/t384.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest_t384.log 2>&1; echo "pytest t384 rc=$?"; tail -1 gpurun_out/${TAG}_pytest_t384.log
V="build_ab/fin0.so build_ab/fin1.so build_ab/cur.so build_ab/t384.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 build_ab/cur.so build_ab/t384.so
