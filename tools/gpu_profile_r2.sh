# Round-2 profiles: launch lists of the C5 replay round and of the slab round (G = 8 on
# virtual slabs), ncu --set full of the scan.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_r2.csv python tools/profile_round.py --preroll 400 --rounds 3 --range \
  > gpurun_out/launches_r2.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_slabs_r2.csv python tools/profile_slabs.py --G 8 --preroll 200 --rounds 2 \
  > gpurun_out/launches_slabs_r2.log 2>&1; echo "slab launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw|k_commit|k_scatter" --profile-from-start off -c 3 \
  -o gpurun_out/full_r2 python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_r2.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_r2.ncu-rep --page raw --csv > gpurun_out/full_r2_raw.csv 2>/dev/null
tail -3 gpurun_out/launches_slabs_r2.log
