#!/bin/bash
# round-2 session-2: k_sub_finalize rank parking: head in the value range + tail over dead keys (fin5) vs head only (fin6)
TAG=${1:-s2i}
mkdir -p gpurun_out
MC_LIB_PATH=$PWD/build_ab/fin5.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_refseq.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
V="build_ab/fin0.so build_ab/fin5.so build_ab/fin6.so"
bash tools/ab_bench_wl.sh ${TAG}_1 subset $V
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep refseq8 $V; done
bash tools/ab_bench_wl.sh ${TAG} afs31x8 $V
