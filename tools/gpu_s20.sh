#!/bin/bash
# session 20: the L2 prefetch spread over one warp per SM -- flushed A/B through bench.py
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
for rep in 1 2; do
  for v in base pf0 pf64; do
    AM_LIB_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-other-configs --no-snapshot \
      > gpurun_out/bench_${v}_${rep}.json 2> gpurun_out/bench_${v}_$rep.err
    python -c "import json,sys; d=json.load(open('gpurun_out/bench_${v}_${rep}.json')); print('$v', $rep, d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_share_warmup_us'].get('k_commit'), d['roofline']['avg_launch_us'])"
  done
done
