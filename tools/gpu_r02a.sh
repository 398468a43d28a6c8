#!/bin/bash
# Round-2 first GPU job: random-access ceilings at the kernels' working-set
# sizes (+ ncu DRAM bytes per op), compute-sanitizer synccheck / initcheck,
# and a baseline bench line of HEAD.  Usage (under gpurun): bash tools/gpu_r02a.sh TAG
TAG=${1:-r02a}
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/randbw tools/randbw.cu || exit 1
for mib in 2400 4096 24576; do
  timeout 300 /tmp/randbw $mib >> gpurun_out/${TAG}_randbw.jsonl 2>&1
done
echo "randbw rc=$?"; wc -l gpurun_out/${TAG}_randbw.jsonl
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_randbw_ncu.csv /tmp/randbw 4096 > /dev/null 2>&1; echo "randbw ncu rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or classify_parity_tiny or pipelined" \
  > gpurun_out/${TAG}_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/${TAG}_synccheck.log
timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
  -k "sketch_parity or db_parity_tiny or heavy or classify_parity_tiny or pipelined" \
  > gpurun_out/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/${TAG}_initcheck.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench rc=$?"
head -c 400 gpurun_out/${TAG}_bench.json; echo
