#!/bin/bash
# session 30: 32-cell direct box for full rounds -- tracker / full-size / slab parity
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 2400 python -m pytest tests/test_gpu_tracker.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py tests/test_gpu_slabs.py tests/test_gpu_bounds.py -q -x > gpurun_out/tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tests.log
tail -2 gpurun_out/tests.log
timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap.log 2>&1; tail -c 300 gpurun_out/snap.log
