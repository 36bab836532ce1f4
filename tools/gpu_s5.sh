cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python tools/repro_loose.py 4 > gpurun_out/repro_loose.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_slabs.py -k "stale" tests/test_gpu_slabs_dist.py -x -q --durations=10 > gpurun_out/stale_tests.log 2>&1
echo "rc=$?" >> gpurun_out/stale_tests.log
