"""Decompose the e2e replay round (am_replay_io) on C5: H2D + round only, + mask D2H,
+ order, + delta write-back of the committed state (events around each variant)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay  # noqa: E402

w = amgen.config("C5")
lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm)
rep.run(400)
n = rep.n
st = torch.cuda.ExternalStream(rep.stream_ptr())
h_pos = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
h_steps = torch.empty(n, dtype=torch.int32, pin_memory=True)
h_mask = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_order = torch.empty(n, dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize()
h_pos.copy_(rep.pos)
h_steps.copy_(rep.steps)
L = rep.L
P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
variants = {
    "h2d+round": (None, None, None, None),
    "+mask": (None, None, h_mask, None),
    "+order": (None, None, h_mask, h_order),
    "+state(delta)": (h_pos, h_steps, h_mask, h_order),
}
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda") if "--flush" in sys.argv else None
for name, (po, so, mo, oo) in variants.items():
    ts = []
    for k in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if flush is not None:
            with torch.cuda.stream(st):
                flush.fill_(k & 0xFF)
        a.record(st)
        L.am_replay_io(rep.h, P(h_pos), P(h_steps), P(po), P(so), P(mo), P(oo), None)
        b.record(st)
        rep.sync()
        ts.append(a.elapsed_time(b) * 1000)
        if po is None:   # keep the host state in step with the device
            h_pos.copy_(rep.pos)
            h_steps.copy_(rep.steps)
    ts.sort()
    print(f"{name:16s} median {ts[6]:.1f} us  min {ts[0]:.1f} us")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
rep.launch(10)
b.record(st)
rep.sync()
print(f"device round     {a.elapsed_time(b) * 100:.1f} us")
