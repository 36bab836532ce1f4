cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/kernel_times.py --label cs16
AM_CSORT_CTAS=8 python tools/kernel_times.py --label cs8
AM_CSORT_CTAS=4 python tools/kernel_times.py --label cs4
AM_CSORT_CTAS=1 python tools/kernel_times.py --label cs1
AM_SORT=onesweep python tools/kernel_times.py --label onesweep
