#!/bin/bash
TAG=${1:-r02f}
mkdir -p gpurun_out
timeout 600 python tools/e2e_trace.py 262144 131072 1048576 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
grep -E "read_batch" gpurun_out/${TAG}_trace.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("build ms", d["build"]["ms_per_step"], "query ms", d["query"]["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["query_ms_per_step"])
print({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})
PY
