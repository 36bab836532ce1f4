#!/bin/bash
# session 25: slab restore and sort on two side streams: slab suites + bench
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_slabs_dist.py -q -x > gpurun_out/slab_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/slab_tests.log
tail -2 gpurun_out/slab_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], {k: v['rank_round_ms_max_over_ranks'] for k, v in d['virtual_slabs'].items()}, {k: v['rank_round_ms_max_over_ranks'] for k, v in d['virtual_slabs_weak'].items()})"
