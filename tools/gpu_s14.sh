#!/bin/bash
# session 14: tall maps over slabs (map beyond one tracker's 32768 rows): parity test and
# the weak-scaling virtual-slab measurement in the bench
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x -k "tall or random_state" > gpurun_out/tall_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tall_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/tall_tests.log; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['virtual_slabs_weak'])"
