#!/bin/bash
# round-2 session-2 A/B: k_sub_finalize rank placement (fin1), + batched first probe (fin2), probe only (fin3)
TAG=${1:-s2g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_refseq.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/fin0.so build_ab/fin1.so build_ab/fin2.so build_ab/fin3.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 $V
bash tools/ab_bench_wl.sh ${TAG} afs31x8 $V
