#!/bin/bash
# session 28: which kernels gain from loading before the PDL wait (bits 1 finalize,
# 2 commit, 4 scatter): warm A/B and flushed bench.py
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
export PYTHONPATH=$(pwd):$PYTHONPATH
timeout 1200 python tools/ab_round.py run e0 e1 e4 e5 e7 --rounds 40 > gpurun_out/ab_early2.log 2>&1
python - <<'PY'
import json
for line in open('gpurun_out/ab_early2.log'):
    if line.startswith('{'):
        d = json.loads(line); print(d['variant'], d['pass'], round(d['round_us'], 1))
PY
for rep in 1 2; do for v in e0 e1 e5; do
  AM_LIB_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-other-configs --no-snapshot \
    > gpurun_out/bench2_${v}_${rep}.json 2> gpurun_out/bench2_${v}_$rep.err
  python -c "import json; d=json.load(open('gpurun_out/bench2_${v}_${rep}.json')); print('$v', $rep, d['ms_per_step'])"
done; done
