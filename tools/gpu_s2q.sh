#!/bin/bash
# round-2 session-2 A/B: staged pair regions (u16) instead of recomputing the hash at write-out (MC_SK_SREG2)
TAG=${1:-s2q}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/sr2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch or db_parity or heavy or low_complexity or spill or batched" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/cur.so build_ab/sr2.so"
for rep in 1 2 3; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ab_bench_wl.sh ${TAG} refseq8 $V
