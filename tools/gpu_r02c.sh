#!/bin/bash
# multi-GPU handle tests (rehearsed on one GPU), full GPU suite, bench N=1 and a rehearsed N=2 line
TAG=${1:-r02c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_robustness.py tests/test_gpu_bench_multigpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest_mg.log 2>&1; echo "pytest mg rc=$?"; tail -5 gpurun_out/${TAG}_pytest_mg.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
MC_BENCH_REHEARSE=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/${TAG}_bench_g2.json 2> gpurun_out/${TAG}_bench_g2.log; echo "bench g2 rc=$?"
python - <<PY
import json
for f in ("gpurun_out/${TAG}_bench.json", "gpurun_out/${TAG}_bench_g2.json"):
    try:
        d=json.load(open(f))
    except Exception as e:
        print(f, "no line", e); continue
    print(f, "n_gpus", d["n_gpus"], "build ms", d["build"]["ms_per_step"], "query ms", d["query"]["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["query_ms_per_step"])
    print({k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})
PY
tail -3 gpurun_out/${TAG}_bench_g2.log
