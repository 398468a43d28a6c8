bash tools/gpu_check.sh r01o skip_full
for rb in 1000000 131072; do timeout 600 python bench.py --read-batch $rb --no-cpu-baseline > gpurun_out/r01o_bench_rb$rb.json 2>/dev/null; done
