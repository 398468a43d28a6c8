mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/randbw tools/randbw.cu
for sz in 1024 4096 24576; do for g in 0 32 128; do /tmp/randbw $sz $g | head -2; done; done > gpurun_out/exp1_randbw.jsonl 2>&1
for g in 0 32 64; do MC_L2_FETCH=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/exp1_bench_g$g.json 2>/dev/null; done
for g in 0 32 64; do python -c "
import json
d=json.load(open('gpurun_out/exp1_bench_g$g.json'))
print($g, 'build ms', d['build']['ms_per_step'], 'query ms', d['query']['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
cat gpurun_out/exp1_randbw.jsonl
