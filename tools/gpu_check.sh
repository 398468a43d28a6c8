#!/bin/bash
# One gpurun job: smoke, GPU parity tests, bench line, ncu launch list, ncu --set full
# of the build + query kernels.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_check.sh TAG [skip_full|KERNEL_REGEX] [MATCHING_LAUNCHES_TO_SKIP (default 7 = one bench step)]
TAG=${1:-check}
KRE=${2:-'k_sketch_partition|k_sub_|k_query_(small|medium|sketch_probe)'}
SKIP=${3:-7}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | head -c 600; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
if [ "$2" != "skip_full" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"$KRE" -s $SKIP -c ${4:-7} \
    -o gpurun_out/${TAG}_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
