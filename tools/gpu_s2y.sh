#!/bin/bash
# round-2 session-2 closing check of the final library: smoke, whole GPU suite, compute-sanitizer
# (memcheck / racecheck / initcheck on the build + query parity tests), the default bench line,
# ncu launch list and ncu --set full of one bench step's build and query kernels
TAG=${1:-s2y}
mkdir -p gpurun_out
K="sketch_parity or db_parity_tiny or heavy or feature_zero or low_complexity or spill or classify_parity_tiny or pipelined"
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/${TAG}_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/${TAG}_$tool.log
done
bash tools/gpu_check.sh $TAG 'k_sketch_partition|k_sub_|k_query_(small|medium|sketch_probe)' 10 10
