# build, GPU parity suite, smoke, bench (+ optional ncu launch list):  bash tools/gpu_check.sh [tag] [ncu]
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-check}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || tail -20 gpurun_out/build_$TAG.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_round.py --preroll 400 --rounds 3 --range > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
fi
