#!/bin/bash
TAG=${1:-r02s}
mkdir -p gpurun_out
for rb in 1048576 524288 262144; do
  MC_DEV_BATCH_MIN=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --read-batch $rb > gpurun_out/${TAG}_rb$rb.json 2> gpurun_out/${TAG}_rb$rb.log
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_rb$rb.json')); print($rb, 'query', d['query']['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if 'query' in k})"
done
for w in afs20 kal; do for rb in 4194304 1048576 262144; do
  MC_DEV_BATCH_MIN=1 timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e --read-batch $rb > gpurun_out/${TAG}_${w}_rb$rb.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_${w}_rb$rb.json')); print('$w', $rb, 'query', d['query']['ms_per_step'])"
done; done
