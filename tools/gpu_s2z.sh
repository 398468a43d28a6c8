#!/bin/bash
# round-2 session-2 final measurement: smoke + whole GPU suite + default bench line + ncu launch list +
# ncu --set full of one bench step's build and query kernels, then every workload's bench line
TAG=${1:-s2z}
bash tools/gpu_check.sh $TAG 'k_sketch_partition|k_sub_|k_query_(small|medium|sketch_probe)' 10 10
bash tools/gpu_bench_all.sh $TAG
