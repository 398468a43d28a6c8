#!/bin/bash
# compute-sanitizer passes over small GPU parity tests (memcheck + racecheck
# on the shared-memory kernels) and the torchrun / reference-arm launches of
# bench.py.  Usage: bash tools/gpu_sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or feature_zero or classify_parity_tiny or pipelined or variable_lengths" \
  > gpurun_out/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/${TAG}_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "classify_parity_paired_strains and 1-4 or db_parity_tiny and 1" \
  > gpurun_out/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/${TAG}_racecheck.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_torchrun.json 2> gpurun_out/${TAG}_torchrun.log
echo "torchrun rc=$?"; head -c 300 gpurun_out/${TAG}_torchrun.json; echo
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.log
echo "reference rc=$?"; head -c 400 gpurun_out/${TAG}_reference.json; echo
