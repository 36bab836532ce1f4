set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 ncu --set full --clock-control none -k regex:"k_ingest|k_bin|k_finalize|k_ready|k_cells|k_scatter|k_commit" -s 2808 -c 7 -o gpurun_out/stream_full python tools/profile_round.py --preroll 400 --rounds 3 > gpurun_out/ncu1.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu1.log
