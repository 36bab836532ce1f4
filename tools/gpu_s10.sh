#!/bin/bash
# session 10: scan register pressure (host lagcap, 32-bit Rc, cheaper half-warp mask),
# occupancy and direct-box A/B; ncu --set full of the scan
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 python tools/ab_round.py run base mb4 mb6 d32 d48 --rounds 40 > gpurun_out/ab_s10_c5.log 2>&1
timeout 600 python tools/ab_round.py run base d32 d48 --rounds 40 --workload C4 > gpurun_out/ab_s10_c4.log 2>&1
AM_LIB_VARIANT=base timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw" --profile-from-start off -c 1 \
  -o gpurun_out/full_s10 python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_s10.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_s10.ncu-rep --page raw --csv > gpurun_out/full_s10_raw.csv 2>/dev/null
cut -c1-120 gpurun_out/ab_s10_c5.log
