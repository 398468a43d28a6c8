#!/bin/bash
# round-2 session-2 A/B: k_sub_finalize places values by the count pass's ranks (MC_FIN_RANK)
TAG=${1:-s2f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "invariants or feature_lists or deterministic" > gpurun_out/${TAG}_pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -1 gpurun_out/${TAG}_pytest_full.log
V="build_ab/fin0.so build_ab/fin1.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 $V
bash tools/ab_bench_wl.sh ${TAG} afs31x8 $V
