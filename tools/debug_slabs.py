"""Debug: the slab replay (LoopbackWorld) against the single-GPU replay round by round;
reports the first round whose merged order / labels differ (gpurun_out/debug_slabs.txt)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay, slabs  # noqa: E402


def main(name="C1", steps=300, n=None, Gs=(1, 2)):
    out = open("gpurun_out/debug_slabs.txt", "a")
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    for G in Gs:
        rep = Replay.from_workload(w, lm, force="binned")
        wd = slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, slabs.Synth(lm, wall=w.wall),
                                 w.Q, G, check_rounds=4)
        bad = None
        for k in range(20000):
            x = rep.pos[:, 0].cpu().numpy().copy(); y = rep.pos[:, 1].cpu().numpy().copy()
            s = rep.steps.cpu().numpy().copy()
            mask, order, labels = rep.step()
            o1 = order.cpu().numpy(); l1 = labels.cpu().numpy()[o1]
            log = []
            wd.round(log)
            o2, l2 = slabs.merged_order(log[0])
            if not (np.array_equal(o1, o2) and np.array_equal(l1, l2)):
                bad = k
                print(f"{name} G={G}: round {k} differs", file=out)
                print(" single:", o1.tolist()[:40], l1.tolist()[:40], file=out)
                print(" slabs :", o2.tolist()[:40], l2.tolist()[:40], file=out)
                only1 = sorted(set(o1.tolist()) - set(o2.tolist())); only2 = sorted(set(o2.tolist()) - set(o1.tolist()))
                print(" only single:", only1[:20], " only slabs:", only2[:20], file=out)
                for i in (only1 + only2)[:6]:
                    print(f"  agent {i}: pos=({x[i]},{y[i]}) step={s[i]} label={labels.cpu().numpy()[i]}", file=out)
                    for r in wd.ranks:
                        gid = r.w_gid.cpu().numpy(); sl = np.flatnonzero(gid == i)
                        if len(sl):
                            j = sl[0]
                            print(f"    rank {r.k} [{r.lo},{r.hi}) win [{r.y0},{r.y1}) slot {j}: pos={r.w_pos[j].tolist()} "
                                  f"step={int(r.w_step[j])} stat={int(r.w_stat[j])} tc={int(r.w_tc[j])} "
                                  f"label={int(r.w_label[j])} ready={int(r.w_ready[j])}", file=out)
                st = rep.tracker.status().cpu().numpy()
                print(" t single:", None, " t slabs:", [int(r.counters[0]) for r in wd.ranks], file=out)
                break
            if (k + 1) % wd.K == 0:
                if wd.check():
                    print(f"{name} G={G}: slabs report all done at round {k}; single n_active "
                          f"{rep.tracker.stats()['n_active']}; last stats {wd._last_stats.tolist()}", file=out)
                    break
            if rep.tracker.stats()["n_active"] == 0 and len(o1) == 0:
                print(f"{name} G={G}: single done at round {k}", file=out)
                break
        print(f"{name} G={G}: first difference at round {bad} (rewindows {wd.rewindows}, halo {wd.halo})",
              file=out, flush=True)
        rep.close()
        wd.close()


if __name__ == "__main__":
    main("C1", 300)
    main("C2", 25, Gs=(1, 2, 4))
    main("C4", 12, 2000, Gs=(1, 2))
