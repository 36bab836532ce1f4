"""Small workloads for compute-sanitizer (tests/test_gpu_sanitizer.py): every kernel of
the library runs at least once -- the fused per-simulation path (multi-kernel rounds and
the persistent replay kernel), the cell-binned round (full + incremental rounds, loose
cells, CUDA graphs and direct launches, the cluster sort), the host-buffer round and the
slab exchange (window trackers, merge, commit, apply)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay, Tracker, slabs  # noqa: E402


def case_small():
    w = amgen.config("C1", steps=40)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    for _ in range(5):
        rep.step()            # multi-kernel rounds
    rep.run(200)              # the persistent per-simulation kernel
    rep.close()
    w = amgen.config("C3", steps=20, n=32)
    rep = Replay.from_workload(w, lm)
    rep.run(100)
    rep.close()


def case_binned(graphs: bool):
    w = amgen.config("C4", steps=30, n=20000)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    if graphs:
        rep.run(12)           # CUDA graphs of rounds (incremental, loose cells, rebuilds)
    else:
        for _ in range(12):
            rep.step()        # direct launches
    n = rep.n
    h_pos = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
    h_steps = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_mask = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_order = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_pos.copy_(rep.pos)
    h_steps.copy_(rep.steps)
    for _ in range(2):
        rep.io(h_pos, h_steps, h_mask, h_order)
        rep.sync()
    rep.close()
    # a snapshot tracker: set_state + full round + incremental replica update
    x, y, s, st = amgen.random_state(5000, 300, 300, 7, max_step=5, p_running=0.3)
    tr = Tracker(300, 300, 4, 1, 5000, peek=True, force="binned")
    dev = torch.device("cuda")
    pos = torch.as_tensor(np.stack([x, y], 1), dtype=torch.int32, device=dev)
    tr.set_state(pos, torch.as_tensor(s, device=dev), torch.as_tensor(st, device=dev))
    tr.ready()
    pos[::7, 0] = (pos[::7, 0] + 1).clamp(max=299)
    tr.update_replica(pos, torch.as_tensor(s, device=dev), torch.as_tensor(st, device=dev))
    tr.ready()
    tr.close()


def case_slabs():
    w = amgen.config("C4", steps=20, n=6000)
    lm = amgen.latency_model(w.profile)
    wd = slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, slabs.Synth(lm), w.Q, 3,
                             check_rounds=4)
    for _ in range(3):
        for _ in range(4):
            wd.round()
        wd.check()
    wd.close()


if __name__ == "__main__":
    which = sys.argv[1]
    {"small": case_small, "binned": lambda: case_binned(True), "binned_direct": lambda: case_binned(False),
     "slabs": case_slabs}[which]()
    torch.cuda.synchronize()
    print("workload ok", which)
