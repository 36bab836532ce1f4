cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/kernel_times.py --label hw
AM_SCAN=split python tools/kernel_times.py --label split
python tools/sort_probe.py
AM_CSORT_CTAS=8 python tools/sort_probe.py
AM_SORT=onesweep python tools/sort_probe.py
