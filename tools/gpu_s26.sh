#!/bin/bash
# session 26: how much of the round the perception digests hold up (profiling knob)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python tools/ab_round.py run base base:AM_DBG_LATE_DIGEST=1 base:AM_DBG_NOSORT=1 --rounds 40 > gpurun_out/ab_digest.log 2>&1
cut -c1-140 gpurun_out/ab_digest.log
