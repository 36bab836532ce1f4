cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 python tools/repro_loose.py 5 > gpurun_out/repro_loose.log 2>&1
timeout 900 python -m pytest tests/test_gpu_slabs_dist.py -x -q > gpurun_out/stale_dist.log 2>&1
echo "rc=$?" >> gpurun_out/stale_dist.log
