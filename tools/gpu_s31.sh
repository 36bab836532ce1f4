#!/bin/bash
# session 31: ncu --set full of the final code's scan / commit / scatter / finalize
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw|k_commit|k_scatter|k_finalize" --profile-from-start off -c 4 \
  -o gpurun_out/full_s31 python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_s31.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_s31.ncu-rep --page raw --csv > gpurun_out/full_s31_raw.csv 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs --no-snapshot > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
head -c 400 gpurun_out/bench_quick.json
