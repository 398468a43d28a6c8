#!/bin/bash
# A/B of library variants on one workload's device-resident query: bash tools/ab_bench_wl.sh TAG WORKLOAD LIB1.so ...
TAG=$1; WL=$2; shift 2
mkdir -p gpurun_out
for lib in "$@"; do
  out=gpurun_out/${TAG}_${WL}_$(basename $lib .so)
  MC_LIB_PATH=$PWD/$lib timeout 600 python bench.py --workload $WL --no-cpu-baseline --no-e2e > $out.json 2> $out.log
  python -c "
import json
d=json.load(open('$out.json'))
print('$WL $lib', 'build', d['build']['ms_per_step'], 'query', d['query']['ms_per_step'])"
done
