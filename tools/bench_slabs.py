"""Spatial-slab tracker round (S7, include/am_slab.h) on a C5 steady-state snapshot.

  python tools/bench_slabs.py --virtual 4            # 4 virtual slabs on one GPU (loopback)
  torchrun --nproc-per-node N tools/bench_slabs.py   # one slab per GPU over NCCL

The snapshot is taken after --preroll replay rounds of C5 on every rank (identical,
seeded), split into horizontal slabs; each timed step is one distributed round
(watermark all-reduce, halo all-to-all, local round, link all-gather, merge) in
AM_PEEK mode, so every step does the same work.  Device time with CUDA events, max
over ranks.  Rank 0 prints one JSON line; the ready count is checked against the
single-GPU round on the same snapshot (rank 0).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay, Tracker, slabs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--agents", type=int, default=None)
    ap.add_argument("--preroll", type=int, default=400)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--virtual", type=int, default=0, help="G virtual slabs on one GPU (loopback)")
    a = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = amgen.config(a.workload, n=a.agents)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm, device=dev)
    rep.run(a.preroll)
    pos = rep.pos.clone()
    steps = rep.steps.clone()
    status = rep.tracker.status().clone()
    rep.close()
    n = pos.shape[0]
    gid = torch.arange(n, dtype=torch.int32, device=dev)
    G = a.virtual if a.virtual else ws
    part = slabs.partition(pos[:, 1], w.map_h, G)

    def mk(k):
        sel = torch.nonzero(part == k).flatten()
        return slabs.SlabRank(w.map_w, w.map_h, w.r_p, w.v, n, G, k, gid[sel], pos[sel], steps[sel],
                              status[sel], device=dev)

    if a.virtual:
        ranks = [mk(k) for k in range(G)]
        run = lambda: slabs.round_loopback(ranks)  # noqa: E731
    else:
        me = mk(rank)
        run = lambda: [slabs.round_distributed(me, dist)]  # noqa: E731
    for _ in range(a.warmup):
        run()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n_ready = 0
    for _ in range(a.steps):
        outs = run()
        n_ready = sum(o["n_ready"] for o in outs)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / a.steps
    if dist:
        t = torch.tensor([ms, float(n_ready)], dtype=torch.float64, device=dev)
        tm = t.clone()
        dist.all_reduce(tm[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms, n_ready = float(tm[0]), int(t[1])
    per_slab = None
    if a.virtual:   # every slab's local round (phase 3) alone: the per-GPU share of a round
        tl = []
        for _ in range(3):
            slabs.round_loopback(ranks, tl)
        per_slab = [round(min(tl[k::G]), 4) for k in range(G)]
    if rank == 0:
        # single-GPU reference round on the same snapshot
        tr = Tracker(w.map_w, w.map_h, w.r_p, w.v, n, peek=True, force="binned", device=dev)
        tr.set_state(pos, steps, status)
        _, order = tr.ready()
        ref_ready = int(order.numel())
        print(json.dumps({"metric": "distributed tracker round (spatial slabs)", "slabs": G,
                          "virtual": bool(a.virtual), "n_gpus": ws, "agents": n,
                          "ms_per_round": ms, "ready": n_ready, "ready_single_gpu": ref_ready,
                          "agent_steps_resolved_per_s": n_ready / (ms / 1000.0),
                          "match": n_ready == ref_ready,
                          "local_round_ms_per_slab": per_slab,
                          "local_rows_per_slab": [r.y1 - r.y0 for r in ranks] if a.virtual else None}),
              flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
