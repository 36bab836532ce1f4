#!/bin/bash
# session 23: run-to-run determinism at full size
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k deterministic --durations=5 > gpurun_out/det.log 2>&1
echo "pytest rc=$?" >> gpurun_out/det.log
tail -8 gpurun_out/det.log
