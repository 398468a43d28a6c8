#!/bin/bash
# ncu --set full (with source) of single launches of the named kernels during
# bench.py --profile (the step after the warm-up).  Usage, under gpurun:
#   bash tools/ncu_kernel.sh TAG KERNEL_REGEX [SKIP (default 1)] [COUNT (default 1)] [extra bench args]
TAG=$1; KRE=$2; SKIP=${3:-1}; CNT=${4:-1}; shift 4
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT \
  -o gpurun_out/${TAG} python bench.py --profile --steps 1 --warmup 1 "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
