#!/bin/bash
# session 21: the bounds-checked build test
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 2700 python -m pytest tests/test_gpu_bounds.py -q -x --durations=5 > gpurun_out/bounds.log 2>&1
echo "pytest rc=$?" >> gpurun_out/bounds.log
tail -15 gpurun_out/bounds.log
