cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/kernel_times.py --label r7
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline
