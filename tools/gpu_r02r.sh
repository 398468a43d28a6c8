#!/bin/bash
TAG=${1:-r02r}
mkdir -p gpurun_out
bash tools/ab_bench.sh ${TAG}_ab ab/pb8.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
