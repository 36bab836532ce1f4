#!/bin/bash
# session 32: size sweep and e2e breakdown of the final code (informational)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
for n in 62500 250000 1000000 4000000; do
  timeout 900 python tools/ab_round.py run base --rounds 40 --agents $n > gpurun_out/sweep_$n.log 2>&1
done
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/sweep_*.log')):
    for line in open(f):
        if line.startswith('{'):
            d = json.loads(line)
            if d['pass'] == 0: print(f, round(d['round_us'], 1), round(d['agent_steps_per_round']))
PY
tail -5 gpurun_out/e2e_probe.log
