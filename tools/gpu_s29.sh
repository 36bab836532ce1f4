#!/bin/bash
# session 29: knob sweep after the round's changes: k_finalize items (replay round),
# the full-round direct box and occupancy (snapshot round)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 900 python tools/ab_round.py run base fin1 fin4 --rounds 40 > gpurun_out/ab_fin.log 2>&1
python - <<'PY'
import json
for line in open('gpurun_out/ab_fin.log'):
    if line.startswith('{'):
        d = json.loads(line); print(d['variant'], d['pass'], round(d['round_us'], 1), d['kernels_us'].get('k_finalize'))
PY
for rep in 1 2; do for v in base df32 df64 mbf4; do
  AM_LIB_VARIANT=$v timeout 300 python tools/snapshot_round.py --reps 10 > gpurun_out/snap_${v}_$rep.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/snap_${v}_$rep.log').read().strip().splitlines()[-1]); print('$v', $rep, d['full_round_us_median'], d['kernels_us'].get('k_scan'))"
done; done
