#!/bin/bash
# parity of the select-chain bucket search + ncu source profile of the small bin
TAG=${1:-r02x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
bash tools/ncu_kernel.sh ${TAG}_qs k_query_small 2 1
