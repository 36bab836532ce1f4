#!/bin/bash
# session 6: GPU suite, k_commit items A/B (warp-compacted commits), bench line
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/scan_probe.py > gpurun_out/scan_probe.log 2>&1
timeout 900 python tools/ab_round.py run c1 c4 c8 --rounds 40 > gpurun_out/ab_commit.log 2>&1
timeout 600 python tools/ab_round.py run c1 c4 --rounds 40 --workload C4 > gpurun_out/ab_commit_c4.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/ab_commit.log | cut -c1-200
