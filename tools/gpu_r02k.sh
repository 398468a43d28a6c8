#!/bin/bash
TAG=${1:-r02k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_multigpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python tools/e2e_trace.py 262144 524288 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"; grep read_batch gpurun_out/${TAG}_trace.log
timeout 600 python tools/host_trace.py afs31x8 > gpurun_out/${TAG}_host_afs31.log 2>&1; echo "host rc=$?"; tail -4 gpurun_out/${TAG}_host_afs31.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("build ms", d["build"]["ms_per_step"], "query ms", d["query"]["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["build_ms_per_step"], d["e2e"]["query_ms_per_step"])
print({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})
PY
