# ncu --set full on selected kernels of a steady-state C5 replay round:
#   bash tools/gpu_ncu_full.sh <tag> <regex> <kernels-per-round-matching>
set -x
cd $GRAFT_REPO_ROOT
TAG=$1; RX=$2; K=$3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || tail -20 gpurun_out/build_$TAG.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"$RX" --profile-from-start off -c $K -o gpurun_out/full_$TAG python tools/profile_round.py --preroll 400 --rounds 3 --stats --range > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/ncufull_$TAG.log
