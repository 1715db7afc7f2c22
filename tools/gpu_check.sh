#!/bin/bash
# One GPU session: tests, smoke, bench line.  bash tools/gpu_check.sh <tag> [pytest-args]
TAG=${1:-r2}
shift
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo bench_rc=$?
tail -c 3000 gpurun_out/${TAG}_gpu_tests.log
