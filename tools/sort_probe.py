"""Time the priority sort alone: a binned tracker of capacity N whose first k agents are
isolated and IDLE (ready), the rest DONE; rounds repeated under AM_PEEK with the sort
kernel bracketed by events."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_03519_b200 import Tracker  # noqa: E402

K_SORT_PASS, K_READY = 8, 6
N, side = 1_000_000, 16384
out = {}
for k in [0, 100, 1000, 10000, 42000, 100000, 300000]:
    ids = np.arange(N)
    g = 819
    x = np.where(ids < k, (ids % g) * 20, 0).astype(np.int32)
    y = np.where(ids < k, (ids // g) * 20, 0).astype(np.int32)
    s = np.where(ids < k, ids * 7919 % 5, 9).astype(np.int32)
    st = np.where(ids < k, 0, 2).astype(np.uint8)
    tr = Tracker(side, side, 4, 1, N, target=9, force="binned")
    dev = torch.device("cuda")
    tr.set_state(torch.as_tensor(np.stack([x, y], 1), device=dev), torch.as_tensor(s, device=dev),
                 torch.as_tensor(st, device=dev))
    tr.set_flags(peek=True)
    L = tr.L
    tr.ready()
    L.am_profile_enable(tr.ctx, (1 << K_SORT_PASS) | (1 << K_READY))
    for _ in range(20):
        m, o = tr.ready()
    ms = (C.c_double * 16)()
    cnt = (C.c_int64 * 16)()
    L.am_profile_read(tr.ctx, ms, cnt, 16)
    out[k] = {"sort_us": round(ms[K_SORT_PASS] / max(1, cnt[K_SORT_PASS]) * 1000, 2),
              "ready_us": round(ms[K_READY] / max(1, cnt[K_READY]) * 1000, 2), "n_ready": len(o)}
    tr.close()
print(os.environ.get("AM_SORT", "cluster"), os.environ.get("AM_CSORT_CTAS", "auto"), json.dumps(out), flush=True)
