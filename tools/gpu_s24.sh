#!/bin/bash
# session 24: full-round scan with the 3x3 min-step pre-test: snapshot A/B, parity tests
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
for rep in 1 2; do for v in base pre0; do
  AM_LIB_VARIANT=$v timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_${v}_$rep.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/snap_${v}_$rep.log').read().strip().splitlines()[-1]); print('$v', $rep, d['full_round_us_median'], d['kernels_us'].get('k_scan'))"
done; done
timeout 1800 python -m pytest tests/test_gpu_tracker.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py tests/test_gpu_slabs.py -q -x > gpurun_out/tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tests.log
tail -2 gpurun_out/tests.log
