#!/bin/bash
# round-2 session-2: k_sub_finalize ranks parked in the regrouped pairs (all sub-regions) + branch-free sketch
# feature loop / staging / write-out (HyperLogLog moved to the write-out); parity + A/B
TAG=${1:-s2h}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_refseq.py tests/test_gpu_afs31.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/fin0.so build_ab/fin1.so build_ab/cur.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 $V
bash tools/ab_bench_wl.sh ${TAG} afs31x8 $V
