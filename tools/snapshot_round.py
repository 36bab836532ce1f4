"""Full (non-incremental) tracker round on a C5 snapshot: the state after a replay
pre-roll is loaded with am_set_state (which forces every verdict, edge and cluster to
be recomputed) and am_ready(PEEK) is timed; per-kernel event times beside it.

  python tools/snapshot_round.py [--preroll 400] [--reps 20] [--workload C5]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay, Tracker  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--preroll", type=int, default=400)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--scan-thread", action="store_true", help="AM_SCAN_THREAD ablation scan")
    a = ap.parse_args()
    w = amgen.config(a.workload)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    rep.run(a.preroll)
    pos = rep.pos.clone()
    steps = rep.steps.clone()
    status = rep.tracker.status().clone()
    rep.close()
    n = pos.shape[0]
    tr = Tracker(w.map_w, w.map_h, 4, 1, n, target=w.steps, peek=True, validate=False, force="binned",
                 scan_thread=a.scan_thread)
    s = torch.cuda.current_stream()
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    order = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        tr.set_state(pos, steps, status)
        tr.ready(mask, order)
    ts = []
    for _ in range(a.reps):
        tr.set_state(pos, steps, status)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        tr.ready_async(mask, order)
        e1.record(s)
        tr.sync()
        ts.append(e0.elapsed_time(e1) * 1000)
    st = tr.stats()
    L = tr.L
    tr_prof = {}
    import ctypes as C
    L.am_profile_enable(tr.ctx, (1 << 15) - 1)
    for _ in range(a.reps):
        tr.set_state(pos, steps, status)
        tr.ready(mask, order)
    ms = (C.c_double * 32)()
    cnt = (C.c_int64 * 32)()
    k = L.am_profile_read(tr.ctx, ms, cnt, 32)
    for j in range(k):
        if cnt[j]:
            tr_prof[L.am_profile_name(j).decode()] = round(ms[j] / cnt[j] * 1000, 2)
    ts.sort()
    print(json.dumps({"workload": w.name, "agents": n, "full_round_us_median": ts[len(ts) // 2],
                      "full_round_us_min": ts[0], "ready": st["n_ready"], "W": st["watermark"],
                      "S": st["max_step"], "work": st["n_work"], "far": st["n_far"], "items": st["n_items"],
                      "edges": st["n_edges"], "kernels_us": tr_prof}))


if __name__ == "__main__":
    main()
