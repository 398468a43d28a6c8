#!/bin/bash
TAG=${1:-r02p}
mkdir -p gpurun_out
bash tools/ab_bench.sh ${TAG}_ab ab/small_minb3.so ab/small_minb2.so
timeout 600 python tools/e2e_trace.py 262144 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"; grep read_batch gpurun_out/${TAG}_trace.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -x -q -k "pipelined or variable or backward or outlive" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
