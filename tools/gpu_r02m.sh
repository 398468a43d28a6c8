#!/bin/bash
# ncu launch list + --set full of the top kernels of the default bench, initcheck re-run
TAG=${1:-r02m}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_launches.py gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_ncu_launches_subset.json "python bench.py --profile --steps 1 --warmup 1 (subset; ncu launch list, cold-cache serialised)"
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:'k_sketch_partition|k_sub_|k_query_(small|medium|sketch_probe)|k_merge' -s 7 -c 8 \
    -o gpurun_out/${TAG}_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep gpurun_out/${TAG}_ncu_full
timeout 1500 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or classify_parity_tiny or pipelined or outlive or backward or rolls" \
  > gpurun_out/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/${TAG}_initcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_robustness.py -m gpu -x -q -k "G-2-2 or 2-4 or pinned or device or outlive or backward or rolls or duplicate" \
  > gpurun_out/${TAG}_memcheck_mg.log 2>&1; echo "memcheck mg rc=$?"; tail -3 gpurun_out/${TAG}_memcheck_mg.log
