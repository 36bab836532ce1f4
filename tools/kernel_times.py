"""Per-kernel event times of the steady-state C5 replay round (pre-roll, then R rounds
with every kernel bracketed by events).  Environment knobs (AM_SORT, AM_CSORT_CTAS ...)
are read by am_init."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C5")
ap.add_argument("--agents", type=int, default=None)
ap.add_argument("--preroll", type=int, default=400)
ap.add_argument("--rounds", type=int, default=10)
ap.add_argument("--label", default="")
a = ap.parse_args()
w = amgen.config(a.workload, n=a.agents)
rep = Replay.from_workload(w, amgen.latency_model(w.profile))
rep.run(a.preroll)
rep.profile((1 << 15) - 1)
for _ in range(a.rounds):
    rep.launch(1)
    rep.sync()
pr = rep.profile_read()
out = {k: round(v[0] / v[1] * 1000, 2) for k, v in pr.items() if v[1]}
out["_sum"] = round(sum(out.values()), 1)
print(a.label, json.dumps(out), flush=True)
rep.profile(0)
rep.launch(9)     # re-captured graphs: first launches upload them
rep.sync()
import torch  # noqa: E402
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(rep.stream_ptr())
s.record(st)
rep.launch(a.rounds)
e.record(st)
rep.sync()
print(a.label, "round_us", round(s.elapsed_time(e) * 1000 / a.rounds, 1), flush=True)
rep.close()
