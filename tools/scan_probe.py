"""Scan work of the incremental C5 replay round (AM_STATS): per round, the queued agents,
how many of them end blocked, cells listed and candidate records tested.
  python tools/scan_probe.py [--preroll 400] [--rounds 5] [--workload C5]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preroll", type=int, default=400)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--workload", default="C5")
a = ap.parse_args()
w = amgen.config(a.workload)
lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm, stats=True)
rep.run(a.preroll)
rep.sync()
rep.tracker.scan_stats()
for r in range(a.rounds):
    d0 = rep.dispatched()
    rep.launch(1)
    rep.sync()
    sc = rep.tracker.scan_stats()
    st = rep.tracker.stats()
    print(json.dumps({"round": r, "queued": st.get("n_work"), "dispatched": rep.dispatched() - d0,
                      "W": st.get("watermark"), "S": st.get("max_step"), **sc}), flush=True)
