#!/bin/bash
# session 11: the scan without statistics registers (no spills) x occupancy x direct box
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 python tools/ab_round.py run base mb4 d32 mb4d32 --rounds 40 > gpurun_out/ab_s11_c5.log 2>&1
timeout 600 python tools/ab_round.py run base mb4 d32 mb4d32 --rounds 40 --workload C4 > gpurun_out/ab_s11_c4.log 2>&1
for v in base d32; do AM_LIB_VARIANT=$v timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_s11_$v.log 2>&1; done
cut -c1-120 gpurun_out/ab_s11_c5.log
