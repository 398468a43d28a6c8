#!/bin/bash
TAG=${1:-r02l}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 600 python tools/host_trace.py afs31x8 > gpurun_out/${TAG}_host_afs31.log 2>&1; echo "host rc=$?"; tail -4 gpurun_out/${TAG}_host_afs31.log
timeout 3000 python -m pytest tests -m gpu -x -q -s --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/${TAG}_pytest.log
