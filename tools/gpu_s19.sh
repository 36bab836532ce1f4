#!/bin/bash
# session 19: the round's L2 prefetch -- flushed A/B through bench.py (variants base /
# pf0, alternating), replay tests
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
for rep in 1 2; do
  for v in base pf0; do
    AM_LIB_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-other-configs --no-snapshot \
      > gpurun_out/bench_${v}_${rep}.json 2> gpurun_out/bench_${v}_$rep.err
    python -c "import json,sys; d=json.load(open('gpurun_out/bench_${v}_${rep}.json')); print('$v', $rep, d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_share_warmup_us'].get('k_scatter'), d['roofline']['avg_launch_us'])"
  done
done
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -x > gpurun_out/replay_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/replay_tests.log
tail -2 gpurun_out/replay_tests.log
