#!/bin/bash
# session 7: A/B of the single-pass scan classification, the witness re-check and the
# small-n sort (C5 and C4 replay rounds); launch lists of the replay round and the slab round
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 python tools/ab_round.py run base s0 w0 q0 c16 --rounds 40 > gpurun_out/ab_s7_c5.log 2>&1
timeout 900 python tools/ab_round.py run base w0 q0 --rounds 40 --workload C4 > gpurun_out/ab_s7_c4.log 2>&1
timeout 600 python tools/scan_probe.py > gpurun_out/scan_probe.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_slabs_s7.csv python tools/profile_slabs.py --G 8 --preroll 200 --rounds 2 \
  > gpurun_out/launches_slabs_s7.log 2>&1; echo "slab launch list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_s7.csv python tools/profile_round.py --preroll 400 --rounds 3 --range \
  > gpurun_out/launches_s7.log 2>&1; echo "launch list rc=$?"
cat gpurun_out/ab_s7_c5.log | cut -c1-150
