# Round profile for profiles/: ncu launch list (per-kernel time + DRAM bytes) of 3
# steady-state C5 replay rounds, and one ncu --set full capture of the scan kernel.
#   bash tools/gpu_profile.sh <tag>
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
# 15 launches per replay round, 2 for the replay's initial state
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -s 6002 -c 45 --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_round.py --preroll 400 --rounds 3 \
  > gpurun_out/launches_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_hw -s 401 -c 1 \
  -o gpurun_out/scan_$TAG python tools/profile_round.py --preroll 400 --rounds 2 > gpurun_out/scanfull_$TAG.log 2>&1; echo "full rc=$?"
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
