#!/bin/bash
TAG=${1:-r02v}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
bash tools/ab_bench.sh ${TAG}_ab ab/nows.so
for w in kal hiseq; do for lib in paper_2106_08150_b200/libmc.so ab/nows.so; do MC_LIB_PATH=$PWD/$lib timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$w.json')); print('$w $lib query', d['query']['ms_per_step'])"; done; done
