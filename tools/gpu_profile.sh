# Round profile for profiles/: ncu launch list (per-kernel time + DRAM bytes) of 3
# steady-state C5 replay rounds (profiler range = the measured rounds only), and one
# ncu --set full capture of every kernel of one steady-state round.
#   bash tools/gpu_profile.sh <tag>
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_round.py --preroll 400 --rounds 3 --range \
  > gpurun_out/launches_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -o gpurun_out/full_$TAG python tools/profile_round.py --preroll 400 --rounds 1 --range > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out/
