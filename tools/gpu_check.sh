#!/bin/bash
# One GPU round trip: tests, smoke, short bench. Each step under its own timeout.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q --timeout 300 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
echo "bench rc=$?"; tail -5 gpurun_out/bench.log
fi
