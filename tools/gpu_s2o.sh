#!/bin/bash
# round-2 session-2 A/B: k_sub_scatter ranking branch-free up to the shared atomics (MC_SCATTER_BF)
TAG=${1:-s2o}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/sbf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "db_parity or heavy or spill or low_complexity or batched" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/cur.so build_ab/sbf.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 $V
