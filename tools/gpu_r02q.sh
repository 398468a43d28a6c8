#!/bin/bash
TAG=${1:-r02q}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/frc tools/fastrange_check.cu && /tmp/frc
bash tools/ab_bench.sh ${TAG}_ab ab/nofr.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
