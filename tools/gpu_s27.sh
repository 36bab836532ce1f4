#!/bin/bash
# session 27: early loads before the PDL wait (k_commit, k_finalize): warm A/B, flushed
# A/B through bench.py, parity tests
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python tools/ab_round.py run base e0 --rounds 40 > gpurun_out/ab_early.log 2>&1
cut -c1-120 gpurun_out/ab_early.log
for rep in 1 2; do for v in base e0; do
  AM_LIB_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-other-configs --no-snapshot \
    > gpurun_out/bench_${v}_${rep}.json 2> gpurun_out/bench_${v}_$rep.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${v}_${rep}.json')); print('$v', $rep, d['ms_per_step'])"
done; done
timeout 1800 python -m pytest tests/test_gpu_tracker.py tests/test_gpu_replay.py tests/test_gpu_fullsize.py -q -x > gpurun_out/tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tests.log
tail -2 gpurun_out/tests.log
