#!/bin/bash
# session 9: A/B of the lazy k_scatter loads; bench line; launch list of the replay
# round; ncu --set full of k_scan_hw / k_commit / k_scatter
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python tools/ab_round.py run base sl0 --rounds 40 > gpurun_out/ab_s9_c5.log 2>&1
cut -c1-150 gpurun_out/ab_s9_c5.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_s9.csv python tools/profile_round.py --preroll 400 --rounds 3 --range \
  > gpurun_out/launches_s9.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw|k_commit|k_scatter" --profile-from-start off -c 3 \
  -o gpurun_out/full_s9 python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_s9.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_s9.ncu-rep --page raw --csv > gpurun_out/full_s9_raw.csv 2>/dev/null
ncu -i gpurun_out/full_s9.ncu-rep --page source --csv -k regex:k_scan_hw > gpurun_out/full_s9_scan_source.csv 2>/dev/null
ls -la gpurun_out
