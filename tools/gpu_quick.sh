#!/bin/bash
# quick gpurun job: GPU tests (optionally filtered) + one bench line.  Usage: bash tools/gpu_quick.sh TAG [PYTEST_K] [bench args]
TAG=$1; K=${2:-}; shift 2
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; fi
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("build ms", d["build"]["ms_per_step"], "query ms", d["query"]["ms_per_step"], "e2e", d["e2e"]["value"] if d.get("e2e") else None)
print({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})
PY
