#!/bin/bash
# end-of-round check: smoke, the whole GPU suite, the default bench line
TAG=${1:-final}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 3000 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('value', d['value'], 'build', d['build']['ms_per_step'], 'query', d['query']['ms_per_step'], d['query']['value'], 'e2e', d['e2e']['value'], d['e2e']['query_reads_per_s'], 'frac', d['roofline']['frac'], d['clocks'])"
