"""Repeat tests/test_gpu_tracker.py::test_loose_cells_every_round_vs_oracle (default
knobs) and, at the first mismatch, print the round's diagnostics: counts, round stats,
the mismatching agents' state, and whether a fresh full round on the same state agrees."""
import sys

import numpy as np
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import Replay, Tracker

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = amgen.config("C4", n=5000)
lm = amgen.latency_model(w.profile)
p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
for it in range(reps):
    rep = Replay.from_workload(w, lm, force="binned")
    bad = None
    for r in range(300):
        x = rep.pos[:, 0].cpu().numpy().copy()
        y = rep.pos[:, 1].cpu().numpy().copy()
        s = rep.steps.cpu().numpy().copy()
        st = rep.tracker.status().cpu().numpy().copy()
        prev = rep.tracker.stats()
        mask_t, order_t, labels_t = rep.step()
        mask = mask_t.cpu().numpy()
        stt = rep.tracker.stats()
        ref = O.round_mt(p, x, y, s, st.copy(), peek=True)
        if not np.array_equal(mask, ref["mask"]):
            bad = r
            d = np.nonzero(mask != ref["mask"])[0]
            print(f"rep {it} round {r}: gpu ready {int(mask.sum())} oracle {int(ref['mask'].sum())} "
                  f"mismatch {len(d)} (gpu1/or0 {int((mask[d] == 1).sum())})", flush=True)
            print("  stats before", prev)
            print("  stats after ", stt)
            lab_ok = np.array_equal(labels_t.cpu().numpy(), ref["label"])
            print("  labels equal", lab_ok, " blocked gpu? n/a; oracle blocked", int(ref["blocked"].sum()))
            for i in d[:8]:
                print(f"   agent {i}: x {x[i]} y {y[i]} s {s[i]} st {st[i]} gpu {mask[i]} or {ref['mask'][i]} "
                      f"or_blk {ref['blocked'][i]} lab gpu {int(labels_t[i])} or {ref['label'][i]}")
            # a fresh full round on the same state
            tr = Tracker(w.map_w, w.map_h, w.r_p, w.v, len(x), peek=True, force="binned")
            pos = torch.as_tensor(np.stack([x, y], 1), dtype=torch.int32, device="cuda")
            tr.set_state(pos, torch.as_tensor(s, device="cuda"), torch.as_tensor(st, device="cuda"))
            m2, o2 = tr.ready()
            print("  fresh full round equals oracle:", np.array_equal(m2.cpu().numpy(), ref["mask"]), flush=True)
            try:
                rep.tracker.sync()
                print("  tracker sync ok")
            except Exception as e:
                print("  tracker sync error", e)
            break
    print(f"rep {it}: {'mismatch at round %d' % bad if bad is not None else 'all 300 rounds equal'}", flush=True)
    rep.close()
