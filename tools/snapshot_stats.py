"""Scan work counters (AM_STATS) of a full (non-incremental) C5 round on the pre-rolled
state: cells visited, candidate pairs, far agents, pyramid blocks, blocked agents."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay, Tracker  # noqa: E402

w = amgen.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm)
rep.run(400)
pos, steps, status = rep.pos.clone(), rep.steps.clone(), rep.tracker.status().clone()
rep.close()
n = pos.shape[0]
tr = Tracker(w.map_w, w.map_h, 4, 1, n, target=w.steps, peek=True, validate=False, force="binned", stats=True)
tr.set_state(pos, steps, status)
tr.scan_stats()
tr.set_state(pos, steps, status)
mask, order = tr.ready()
sc = tr.scan_stats()
import ctypes as C  # noqa: E402
blk = torch.empty(n, dtype=torch.uint8, device="cuda")
tr.L.am_blocked(tr.ctx, C.c_void_p(blk.data_ptr()))
torch.cuda.synchronize()
sc["blocked_idle"] = int(blk.sum())
st = tr.stats()
idle = int((status == 0).sum())
print(json.dumps({"agents": n, "idle": idle, "running": int((status == 1).sum()), "ready": st["n_ready"],
                  "far": st["n_far"], "items": st["n_items"], "W": st["watermark"], "S": st["max_step"],
                  **{k: v for k, v in sc.items()}}))
