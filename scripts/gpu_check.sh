#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list.  Everything bounded.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
export CF_SPIN_TIMEOUT_MS=${CF_SPIN_TIMEOUT_MS:-5000}
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -rs ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/smoke.log
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
