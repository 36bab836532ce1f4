#!/bin/bash
# session 13: size sweep of the replay round at C5 density (62.5k .. 4M agents)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 600 python tools/ab_round.py run base base:AM_DBG_NOSORT=1 --rounds 40 > gpurun_out/ab_nosort.log 2>&1
for n in 62500 250000 1000000 4000000; do
  timeout 900 python tools/ab_round.py run base --rounds 40 --agents $n > gpurun_out/sweep_$n.log 2>&1
done
timeout 600 python tools/ab_round.py run base --rounds 40 --workload C4 > gpurun_out/sweep_c4.log 2>&1
cut -c1-120 gpurun_out/sweep_*.log
