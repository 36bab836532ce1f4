cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1500 python tools/ab_round.py run base:AM_CELL=32 base:AM_CELL=64 dir32:AM_CELL=32 dir128:AM_CELL=32 dir16:AM_CELL=64 dir32:AM_CELL=64 dir128:AM_CELL=64 --rounds 40 > gpurun_out/ab_cell2.log 2>&1
timeout 900 python tools/ab_round.py run base base:AM_CELL=16 base:AM_CELL=32 base:AM_CELL=64 --rounds 40 --workload C4 > gpurun_out/ab_cell_c4.log 2>&1
for c in 64 128; do
  AM_CELL=$c timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_cell$c.log 2>&1
done
