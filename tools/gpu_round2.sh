#!/bin/bash
# one GPU session: the -m gpu suite, smoke(), and a bench line (gpurun_out/)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q --durations=25 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
tail -5 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.json
