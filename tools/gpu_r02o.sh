#!/bin/bash
TAG=${1:-r02o}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_multigpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
bash tools/ab_bench.sh ${TAG}_ab ab/nomq.so
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "classify_parity_paired_strains and 1-4 or classify_parity_tiny" \
  > gpurun_out/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/${TAG}_racecheck.log
timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or classify_parity_tiny or pipelined or outlive or backward or rolls" \
  > gpurun_out/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/${TAG}_initcheck.log
