#!/bin/bash
# round-2 session-2 A/B: sketch tiles of 128 / 192 windows (more, smaller CTAs per SM)
TAG=${1:-s2n}
mkdir -p gpurun_out
V="build_ab/cur.so build_ab/t128.so build_ab/t192.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
