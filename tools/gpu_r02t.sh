#!/bin/bash
TAG=${1:-r02t}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('build', d['build']['ms_per_step'], 'query', d['query']['ms_per_step'], 'e2e', d['e2e']['query_ms_per_step'])"
for w in kal afs20; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$w.json')); print('$w query', d['query']['ms_per_step'])"; done
