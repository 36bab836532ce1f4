#!/bin/bash
# session 22: labels-only window rounds for the slabs (k_ready skipped; chg8 reset and
# DONE labels in k_finalize): the whole GPU suite (incl. the bounds-checked build) + bench
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], {k: v['rank_round_ms_max_over_ranks'] for k, v in d['virtual_slabs'].items()}, {k: v['rank_round_ms_max_over_ranks'] for k, v in d['virtual_slabs_weak'].items()})"
timeout 2400 python -m pytest tests -m gpu -q -rP --durations=10 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
