#!/bin/bash
TAG=${1:-r02y}
mkdir -p gpurun_out
for w in subset kal refseq8; do MC_LIB_PATH=$PWD/ab/qprof.so timeout 600 python tools/qprof.py $w 2>&1 | tail -20 > gpurun_out/${TAG}_qprof_$w.log; cat gpurun_out/${TAG}_qprof_$w.log; done
