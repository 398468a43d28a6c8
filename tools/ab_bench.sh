#!/bin/bash
# A/B of library variants on the bench (device-resident step): bash tools/ab_bench.sh TAG LIB1.so LIB2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for lib in paper_2106_08150_b200/libmc.so "$@"; do
  MC_LIB_PATH=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$(basename $lib .so).json 2> gpurun_out/${TAG}_$(basename $lib .so).log
  python -c "
import json
d=json.load(open('gpurun_out/${TAG}_$(basename $lib .so).json'))
print('$lib', 'build', d['build']['ms_per_step'], 'query', d['query']['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if 'query' in k or 'sub' in k or 'sketch' in k})"
done
