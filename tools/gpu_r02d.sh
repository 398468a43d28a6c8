#!/bin/bash
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.log
bash tools/ab_bench.sh ${TAG}_ab ab/minb3.so
