#!/bin/bash
TAG=${1:-r02j}
mkdir -p gpurun_out
bash tools/ab_bench.sh ${TAG}_ab ab/probe1.so ab/probe2.so
timeout 600 python tools/host_trace.py afs31x8 > gpurun_out/${TAG}_host_afs31.log 2>&1; echo "host rc=$?"; tail -4 gpurun_out/${TAG}_host_afs31.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
