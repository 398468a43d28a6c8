#!/bin/bash
# round-2 session-2: full GPU suite on the new default library, A/B of the unrolled write-out, ncu of sketch + finalize
TAG=${1:-s2e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
V="build_ab/h1.so build_ab/k3wu.so"
for rep in 1 2; do bash tools/ab_bench_wl.sh ${TAG}_$rep subset $V; done
bash tools/ncu_kernel.sh ${TAG}_sk 'k_sketch_partition|k_sub_finalize' 1 2 --no-cpu-baseline --no-e2e
