#!/bin/bash
# GPU tests (all), initcheck on the small parity tests, one bench line.  Usage: bash tools/gpu_r02b.sh TAG
TAG=${1:-r02b}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.log
timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or classify_parity_tiny or pipelined or robustness or outlive or backward" \
  > gpurun_out/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/${TAG}_initcheck.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("build ms", d["build"]["ms_per_step"], "query ms", d["query"]["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["query_ms_per_step"])
print(json.dumps(d["path_roofline"]))
print(json.dumps(d["cpu_baseline"]))
print({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})
PY
