#!/bin/bash
# round-2 session-2 A/B: k_sub_finalize rank parking for sub-regions beyond the staging (per-CTA tail scratch)
TAG=${1:-s2m}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_refseq.py tests/test_gpu_multigpu.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/fu1.so build_ab/ft.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep refseq8 $V; done
bash tools/ab_bench_wl.sh ${TAG} subset $V
bash tools/ab_bench_wl.sh ${TAG} afs31x8 $V
