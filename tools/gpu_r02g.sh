#!/bin/bash
TAG=${1:-r02g}
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/mini_trace.py > gpurun_out/${TAG}_mini.log 2>&1; echo "mini rc=$?"; tail -5 gpurun_out/${TAG}_mini.log
timeout 600 python tools/host_trace.py afs31x8 > gpurun_out/${TAG}_host_afs31.log 2>&1; echo "host rc=$?"; tail -6 gpurun_out/${TAG}_host_afs31.log
timeout 600 python tools/host_trace.py subset > gpurun_out/${TAG}_host_subset.log 2>&1; echo "host rc=$?"; tail -6 gpurun_out/${TAG}_host_subset.log
timeout 600 python tools/e2e_trace.py 262144 131072 1048576 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"; grep read_batch gpurun_out/${TAG}_trace.log; tail -3 gpurun_out/${TAG}_trace.log | cut -c1-300
