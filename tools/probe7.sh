cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/kernel_times.py --label efil
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan_hw|k_cells|k_ingest|k_commit|k_scatter|k_ready" -s $((6*402)) -c 6 -o gpurun_out/full_b python tools/profile_round.py --preroll 400 --rounds 3 > gpurun_out/ncufull_b.log 2>&1; echo "ncu rc=$?"
