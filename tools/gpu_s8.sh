#!/bin/bash
# session 8: A/B of the local-watermark far box; GPU suite
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python tools/ab_round.py run base lw0 --rounds 40 > gpurun_out/ab_s8_c5.log 2>&1
timeout 600 python tools/ab_round.py run base lw0 --rounds 40 --workload C4 > gpurun_out/ab_s8_c4.log 2>&1
AM_LIB_VARIANT=base timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_base.log 2>&1
AM_LIB_VARIANT=lw0 timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_lw0.log 2>&1
cut -c1-200 gpurun_out/ab_s8_c5.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
