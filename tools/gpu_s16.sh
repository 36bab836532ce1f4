#!/bin/bash
# session 16: profiles of the final round-2 code: ncu --set full of the scan / commit /
# scatter (issue roofline, source lines), launch list of the slab round (G = 8)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw|k_commit|k_scatter" --profile-from-start off -c 3 \
  -o gpurun_out/full_s16 python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_s16.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_s16.ncu-rep --page raw --csv > gpurun_out/full_s16_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_slabs_s16.csv python tools/profile_slabs.py --G 8 --preroll 200 --rounds 2 \
  > gpurun_out/launches_slabs_s16.log 2>&1; echo "slab launch list rc=$?"
ls -la gpurun_out
