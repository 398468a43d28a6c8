#!/bin/bash
# A/B: small-bin gather fast claim (MC_FAST_CLAIM) and select-chain bucket search (MC_FIND4)
TAG=${1:-r02w}
mkdir -p gpurun_out
bash tools/ab_bench.sh ${TAG}_ab ab/nofc.so ab/fc.so ab/f4.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
