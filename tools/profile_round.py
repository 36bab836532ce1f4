"""Profile the replay round at scale: per-round tracker statistics and scan work
counters (AM_STATS), per-kernel event times.  Used under ncu for launch lists:
  ncu --metrics gpu__time_duration.sum -s <skip> -c <n> python tools/profile_round.py
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--agents", type=int, default=None)
    ap.add_argument("--preroll", type=int, default=400)
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--cell", type=int, default=0)
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--prof", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--dbg", type=lambda v: int(v, 0), default=0, help="extra AM_* flag bits")
    ap.add_argument("--scan-thread", action="store_true")
    ap.add_argument("--range", action="store_true",
                    help="cudaProfilerStart/Stop around the measured rounds (ncu --profile-from-start off)")
    a = ap.parse_args()
    w = amgen.config(a.workload, n=a.agents)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm, stats=a.stats, cell=a.cell)
    if a.dbg or a.scan_thread:
        from paper_2411_03519_b200 import _lib
        # applied after the pre-roll so the replay state stays valid
        extra = a.dbg | (_lib.SCAN_THREAD if a.scan_thread else 0)
    else:
        extra = 0
    t0 = time.perf_counter()
    rep.run(a.preroll)
    t1 = time.perf_counter()
    print(f"preroll {a.preroll} rounds: {t1 - t0:.3f} s wall", flush=True)
    if a.stats:
        rep.tracker.scan_stats()
    if extra:
        L = rep.tracker.L
        rep.tracker.flags |= extra
        # graphs bake the flags: set them on the context and force a re-capture
        L.am_set_flags(rep.tracker.ctx, rep.tracker.flags | 0x4 | 0x8)   # + DIGEST | ASYNC
    if a.prof:
        rep.profile((1 << 15) - 1)
    rows = []
    if a.range:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    for k in range(a.rounds):
        rep.launch(1)
        act, nr = rep.sync()
        st = rep.tracker.stats()
        row = dict(round=k, ready=nr, active=act, running=st["n_running"], W=st["watermark"],
                   S=st["max_step"], clusters=st["n_clusters"], cell=st["cell"])
        if a.stats:
            sc = rep.tracker.scan_stats()
            row.update({k2: v / max(1, st["n_active"]) for k2, v in sc.items()})
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.range:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    if a.prof:
        pr = rep.profile_read()
        print(json.dumps({k: round(v[0] / v[1] * 1000, 2) for k, v in pr.items() if v[1]}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f)
    rep.close()


if __name__ == "__main__":
    main()
