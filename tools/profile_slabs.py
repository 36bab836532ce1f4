"""Profile the slab-distributed replay on virtual slabs (LoopbackWorld) for ncu launch
lists: pre-roll (outside the profiled range), then --rounds rounds inside
cudaProfilerStart/Stop.  Every rank's kernels run serialised on one GPU; per rank the
launch list gives its round's kernels (rank order = launch order)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import slabs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--agents", type=int, default=None)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--preroll", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    w = amgen.config(a.workload, n=a.agents)
    lm = amgen.latency_model(w.profile)
    wd = slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, slabs.Synth(lm), w.Q, a.G,
                             check_rounds=16)
    done = 0
    while done < a.preroll:
        for _ in range(min(wd.K, a.preroll - done)):
            wd.round()
            done += 1
        wd.check()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.rounds):
        wd.round()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    st = [slabs._lib.RoundStats() for _ in wd.ranks]
    for r, s in zip(wd.ranks, st):
        r.L.am_stats(r.tracker_ctx(), slabs.C.byref(s))
    print("window rebuilds", [s.n_rebuilds for s in st], "rebuilt last", [s.rebuilt for s in st],
          "n_work", [s.n_work for s in st])
    wd.close()


if __name__ == "__main__":
    main()
