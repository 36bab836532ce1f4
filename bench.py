#!/usr/bin/env python
"""bench.py -- AI Metropolis dependency tracker on B200.

A STEP is one scheduling round of the GPU-resident trace replay of BASELINE config 5
(1M agents on a 16384x16384 map, hotspots, busy-hour latency profile, 50 ms quantum):
am_update (ingest + commit validation, S1) -> am_ready (binning S2, cell table S3,
time-dilated scan S4, cluster labelling S5, ready set + priority order S6) ->
dispatch + commit (driver, S8).  The replay is pre-rolled to steady state (untimed),
then W warm-up and K timed rounds; L2 is flushed (512 MB write) between timed rounds.

metric: agent-steps resolved per second (= agents dispatched by the tracker per second
of device time); rounds/s is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun, one process per GPU, NCCL): the same 1M-agent map split into N
horizontal slabs (slabs.DistWorld, strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-steps resolved/sec and scheduling rounds/sec; % of HBM roofline"
UNIT = "agent-steps/s"

# Algorithmic bytes per launch of each kernel: the bytes the
# kernel's definition must move at minimum, each input/output counted once.
# n = agents, a = active (not DONE) agents, c = Morton cells, r = ready agents,
# q = RUNNING agents, p = radix passes.
def algorithmic_bytes(kernel: str, s: dict) -> float:
    n, a, c, r, p = s["n"], s["n_active"], s["ncells"], s["n_ready"], s["passes"]
    table = {
        # replay rounds: k_replay_begin (timed as k_ingest) reads / resets the 64 post-commit
        # reduction stripes (128 B each); a host-buffer round's k_ingest reads pos 8 + step 4
        # (new) + old step 4 + status 1 + old pos 8 and writes pos 8 + step 4 + status 1
        "k_ingest": 64 * 128 * 2.0,
        # read status 1 + pos 8 + step 4; write key 4 + bad 1 + blkid 1; cell count + min 8
        "k_bin": 27.0 * n,
        # read count 4 + min 4; write start/min 8 + min reset 4 + pyramid 0.27
        "k_cells": 20.27 * c,
        # read key 4 + cell start 4 + count 4 + pos 8 + step 4 + status 1; write record 16
        "k_scatter": 41.0 * a,
        # k_efilter (timed as "k_near"): read last round's edge list 8 per edge, write the
        # kept ones 8 per edge (upper bound on the kept share: all)
        "k_near": 16.0 * s["n_edges"],
        # k_scan_hw, per re-scanned agent w: read queue entry 4 + pos 8 + step 4 + status 1
        # + own cell entry 8; write verdict 1 + witness 4 + a new edge 8; per far agent f:
        # 16x16 / 4x4 level words 4 + 64; per far item (surviving 4x4-cell block): its
        # 16 cell entries 136
        "k_scan": 38.0 * s["n_work"] + 68.0 * s["n_far"] + 136.0 * s["n_items"],
        # read record 16 + blocked bit 0.125 + parent 4; write label 4
        "k_finalize": 24.125 * a,
        # read status 1 + label 4 + bad 1; write mask 1 + status 1; ready: step 4 + key/id 12
        "k_ready": 8.0 * n + 16.0 * r,
        "k_sort_hist": 8.0 * r,
        # per pass read+write key 8 + id 4; last pass writes 4-byte order
        "k_sort_pass": 24.0 * r * p,
        # ready: order 4 + step 4 + label 4 + latency tables ~0 + cluster time 8
        "k_disp_a": 20.0 * r,
        # ready: order 4 + label 4 + cluster time 8 + step 4 + pos 8 + digest 8; write tcommit 8 + newpos 8
        "k_disp_b": 52.0 * r,
        # read status 1 (+ tcommit 8 for RUNNING, world step 4 for the post-commit W / S);
        # per commit (~ the ready count at steady state): world pos / step / traj r+w 32 +
        # move 8 + label 4 + slot 4 + key 4, tracker state 13, record 16, dirty 4, changed 1
        "k_commit": 1.0 * n + 12.0 * s["n_running"] + 4.0 * a + 86.0 * r,
        # read edge 8 + two parent words per edge
        "k_union": 16.0 * s["n_edges"],
    }
    return table.get(kernel, 0.0)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", pk
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu = gpu_id
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 5 + k and s[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ CPU oracle baseline
def oracle_sample(w, state, seconds: float, seed: int = 0):
    """The oracle as it stands (single-threaded C, brute force) on a bounded sample of
    the workload: sampled agents of ``state`` -- the pre-rolled round the GPU is timed
    on (``prerolled_state``) -- each resolved one by one (blocking test O(N), cluster
    walk O(N*|C|)).  Returns (ready agent-steps resolved per second, agents sampled,
    seconds)."""
    import numpy as np

    import oracle as O
    x, y, steps, status = state
    n = len(x)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    rng = np.random.default_rng(seed)
    ready = sampled = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        smp = rng.integers(0, n, 4).astype(np.int32)
        r = O.round_sampled(p, x, y, steps, status, smp)
        ready += int(r["mask"].sum())
        sampled += len(smp)
    dt = time.perf_counter() - t0
    return ready / dt, sampled, dt


def oracle_sample_threads(w, state, seconds: float, threads: int):
    """the same oracle, as it stands, on `threads` host cores at once --
    an outer loop over sampled agents split across threads (each thread its own seed;
    ctypes releases the GIL around every oracle.c call).  Returns (aggregate ready
    agent-steps per second, agents sampled, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(lambda k: oracle_sample(w, state, seconds, seed=1000 + k), range(threads)))
    return sum(r[0] for r in res), sum(r[1] for r in res), max(r[2] for r in res)


def take_round_state(rep):
    """Runs one replay round with its outputs and returns the state that round resolved:
    (x, y, steps, status) as the round saw them -- the world arrays after the last
    commits, and the statuses with the agents it dispatched still IDLE."""
    import numpy as np
    import torch
    x = rep.pos[:, 0].cpu().numpy().copy()
    y = rep.pos[:, 1].cpu().numpy().copy()
    s = rep.steps.cpu().numpy().copy()
    st = rep.tracker.status().cpu().numpy().copy()   # the last round's commits are applied in place
    rep.step()
    torch.cuda.synchronize()
    return x, y, s, st.astype(np.uint8)


def prerolled_state(w, lm, preroll: int):
    """The input state of the timed rounds, for the oracle arm: the workload's replay
    pre-rolled `preroll` rounds (deterministic: a pure function of the seeds), then the
    state of the next round.  The pre-roll itself is input preparation, untimed."""
    import torch

    from paper_2411_03519_b200 import Replay
    dev = torch.device("cuda", _dist()[2])
    torch.cuda.set_device(dev)
    rep = Replay.from_workload(w, lm, device=dev)
    rep.run(preroll)
    st = take_round_state(rep)
    rep.close()
    return st


def run_reference(args, w, lm):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle as O
    O.build()
    state = prerolled_state(w, lm, args.preroll)
    times, resolved, sampled = [], 0, 0
    nt = max(1, len(os.sched_getaffinity(0)))
    for k in range(args.warmup + args.steps):
        v, sm, dt = oracle_sample_threads(w, state, args.ref_step_seconds, nt)
        if k >= args.warmup:
            times.append(dt)
            resolved += v * dt
            sampled += sm
    total = sum(times)
    value = resolved / total if total else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": _config(w, ws),
        "cpu_baseline": {"kind": "oracle", "value": value, "unit": UNIT, "cores": nt,
                         "sample": f"{sampled} sampled agents of the {w.name} round after a "
                                   f"{args.preroll}-round pre-roll ({len(w.x)} agents; the state the GPU "
                                   f"arm times), resolved one by one by oracle.c on {nt} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(w, ws):
    return {"workload": f"{w.name}: {len(w.x)} agents, {w.map_w}x{w.map_h} open map, hotspots, "
                        f"busy-hour latencies, Q={w.Q // 1000} ms, T={w.steps}",
            "agents": len(w.x), "map": [w.map_w, w.map_h], "r_p": w.r_p, "v_max": w.v,
            "quantum_us": w.Q, "parallelism": "replicas" if ws > 1 else "single",
            "l2": "flushed between timed rounds (512 MB write)"}


# ------------------------------------------------------------------ the other configs
def other_configs(dev, budget_s: float = 2.0):
    """BASELINE configs 1-4 beside the headline (C5): the GPU-resident replay of each
    (C1/C2/C3 on the fused per-simulation kernel, C4 on the binned pipeline), timed on
    the device with CUDA events over whole launches of rounds (no L2 flush: these are
    latency-bound small rounds).  C1 and C3 run to completion (every agent at T=1000);
    C2 and C4 run a bounded number of rounds after a pre-roll."""
    import numpy as np
    import torch

    import amgen
    from paper_2411_03519_b200 import Replay
    out = {}
    plan = [("C1", 0, None), ("C3", 0, None), ("C2", 400, 4000), ("C4", 400, 2000)]
    for name, preroll, rounds in plan:
        w = amgen.config(name)
        lm = amgen.latency_model(w.profile)
        rep = Replay.from_workload(w, lm, device=dev)
        st = torch.cuda.ExternalStream(rep.stream_ptr(), device=dev)
        if preroll:
            rep.run(preroll)
        rep.run(8)
        d0 = rep.dispatched()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(st)
        done = 0
        if rounds is None:   # to completion
            while True:
                rep.launch(512)
                done += 512
                act, _ = rep.sync()
                if act == 0 or time.perf_counter() - t0 > 10 * budget_s:
                    break
        else:
            while done < rounds and time.perf_counter() - t0 < budget_s:
                rep.launch(256)
                done += 256
            rep.sync()
        b.record(st)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b)
        steps = rep.dispatched() - d0
        res = {"agents": len(w.x), "n_sims": w.n_sims, "rounds": done,
               "agent_steps_per_s": steps / (ms / 1e3), "rounds_per_s": done / (ms / 1e3),
               "path": "fused per-simulation kernel" if rep.tracker.stats()["path"] == 0 else "binned"}
        if rounds is None:
            r = rep.results()
            res["completed"] = bool(act == 0)
            res["sim_rounds_per_s"] = done * w.n_sims / (ms / 1e3)
            if act == 0:
                res["T_ooo_s_mean"] = float(r["T_ooo"].mean()) / 1e6
                # the paper's evaluation quantities under the synthetic model (context, not
                # targets): speedup over parallel-sync (Alg. 1) and the achieved
                # parallelism = average outstanding LLM requests
                llm = rep.llm_time().astype(np.float64)
                tsync = rep.lockstep_time(w.steps).astype(np.float64)
                tooo = r["T_ooo"].astype(np.float64)
                res["T_sync_s_mean"] = float(tsync.mean()) / 1e6
                res["speedup_vs_parallel_sync_mean"] = float((tsync / tooo).mean())
                res["achieved_parallelism_ooo_mean"] = float((llm / tooo).mean())
                res["achieved_parallelism_sync_mean"] = float((llm / tsync).mean())
        if name == "C4":   # C4 snapshot rounds (full recompute, AM_PEEK)
            fl = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
            sn = snapshot_rounds(rep, w, dev, fl, reps=20)
            res["snapshot_rounds_per_s"] = sn["rounds_per_s"]
            res["snapshot_ms_per_round"] = sn["ms_per_round_median"]
            del fl
        out[name] = res
        rep.close()
    # finite LLM capacity, C2 = 500 agents busy hour: the paper's
    # priority-scheduling breakdown (Table 1: 500 agents, 4 / 8 L4 GPUs,
    # +3.84% / +15.7% with priority) -- context, not a parity target
    w = amgen.config("C2", steps=200)   # 200 of the 1000 steps: a bounded run
    lm = amgen.latency_model(w.profile)
    cap = {}
    for K in (64,):
        row = {}
        for prio in (True, False):
            rep = Replay.from_workload(w, lm, device=dev, capacity=K, priority=prio)
            t0 = time.perf_counter()
            rep.run_to_end(chunk=4096)
            row["T_ooo_s_priority" if prio else "T_ooo_s_fifo"] = float(rep.results()["T_ooo"][0]) / 1e6
            row["wall_s_priority" if prio else "wall_s_fifo"] = time.perf_counter() - t0
            rep.close()
        row["priority_speedup_pct"] = (row["T_ooo_s_fifo"] / row["T_ooo_s_priority"] - 1.0) * 100.0
        cap[f"K={K}"] = row
    out["C2_capacity"] = {"capacity_unit": "agent-steps in service at once", "steps": w.steps, **cap}
    return out


def snapshot_rounds(rep, w, dev, flush, reps: int = 20):
    """SURVEY 8(d.1) C5 "snapshot rounds/s": the state the replay pre-roll reached is
    loaded into a fresh tracker with am_set_state (which forces every verdict, coupling
    edge and cluster to be recomputed: no incremental reuse) and one full am_ready
    round (AM_PEEK, nothing dispatched) is timed with CUDA events, L2 flushed before
    each.  Returns rounds/s, the full-round time and its per-round statistics."""
    import torch

    from paper_2411_03519_b200 import Tracker
    pos, steps = rep.pos.clone(), rep.steps.clone()
    status = rep.tracker.status().clone()
    n = pos.shape[0]
    tr = Tracker(w.map_w, w.map_h, 4, 1, n, target=w.steps, peek=True, validate=False,
                 force="binned", device=dev)
    s = torch.cuda.current_stream(dev)
    mask = torch.empty(n, dtype=torch.uint8, device=dev)
    order = torch.empty(n, dtype=torch.int32, device=dev)
    for _ in range(3):
        tr.set_state(pos, steps, status)
        tr.ready(mask, order)
    ts = []
    for k in range(reps):
        tr.set_state(pos, steps, status)
        flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        tr.ready_async(mask, order)
        e1.record(s)
        tr.sync()
        ts.append(e0.elapsed_time(e1))
    st = tr.stats()
    tr.close()
    ts.sort()
    med = ts[len(ts) // 2]
    return {"rounds_per_s": 1e3 / med, "ms_per_round_median": med, "ms_per_round_min": ts[0],
            "rounds": reps, "agents": n, "ready": st["n_ready"], "scanned": st["n_work"],
            "far": st["n_far"], "edges": st["n_edges"],
            "what": "full (non-incremental) am_ready round on the pre-rolled C5 state, AM_PEEK, "
                    "L2 flushed before each round"}


def virtual_slabs(w, lm, dev, slab_counts=((2, 1), (8, 1), (8, 4)), preroll=200, timed=8):
    """S7 + S8 on one GPU: the C5 replay split into G horizontal slabs
    (slabs.LoopbackWorld: the library calls of the NCCL run, exchanges as device copies),
    pre-rolled `preroll` rounds from t = 0, then `timed` rounds with every rank's own
    device time recorded (its library steps; the exchanges are NCCL's in a real run): the
    slowest rank's time is what one GPU of a G-GPU run computes per round.  (G, P): P > 1
    = stale-halo rounds (NEXT #3), a sync round every P rounds, reported as the mean over
    whole periods.  Synchronous runs are checked against the single-GPU replay after the
    same rounds (agent-steps dispatched)."""
    import torch

    from paper_2411_03519_b200 import Replay, slabs
    one = Replay.from_workload(w, lm, device=dev)
    one.run(preroll + timed)
    ref = one.dispatched()
    one.close()
    out = {}
    for G, P in slab_counts:
        sy = slabs.Synth(lm, device=dev)
        wd = slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, sy, w.Q, G, device=dev,
                                 check_rounds=16, stale_rounds=P)
        done = 0
        while done < preroll:
            k = min(wd.K, preroll - done)
            for _ in range(k):
                wd.round()
            done += k
            wd.check()
        tl = []
        for _ in range(timed):
            wd.round(timing=tl)
        wd.check()
        per = [max(r[k] for r in tl[1:] or tl) for k in range(G)]   # worst round per rank
        med = [sorted(r[k] for r in tl)[len(tl) // 2] for k in range(G)]
        mean = [sum(r[k] for r in tl) / len(tl) for k in range(G)]    # whole periods (timed % P == 0)
        disp = wd.dispatched()
        key = f"G={G}" if P == 1 else f"G={G},P={P}"
        out[key] = {"rank_round_ms_max_over_ranks": max(med) if P == 1 else max(mean),
                    "rank_round_ms_mean": sum(med) / G if P == 1 else sum(mean) / G,
                    "rank_round_ms_worst": max(per), "halo_rows": wd.halo, "rewindows": wd.rewindows,
                    "window_agents_max": max(int((r.w_gid >= 0).sum().item()) for r in wd.ranks),
                    "rounds": preroll + timed, "stale_rounds": P}
        if P == 1:
            out[key]["dispatched_equals_single_gpu"] = disp == ref
        else:
            out[key]["dispatched"] = disp
            out[key]["dispatched_single_gpu_same_rounds"] = ref
        wd.close()
    return out


def virtual_slabs_tall(lm, dev, slab_counts=(4, 16), preroll=200, timed=8):
    """Weak scaling on virtual slabs: C5's density and recipe on a tall map of G x 1M
    agents (16384 wide, G x 16384 rows: beyond one tracker's 32768 rows from G = 2, so
    only the slab decomposition holds it), one 1M-agent 16384^2 slab per rank.  Per rank:
    its own device time of a round (as in virtual_slabs); aggregate: the agent-steps all
    ranks dispatch per round over the slowest rank's round time -- what G GPUs would
    resolve per second, before the cost of the three collectives."""
    import amgen
    from paper_2411_03519_b200 import slabs
    out = {}
    for G in slab_counts:
        w = amgen.config("C5T", n=G * 1_000_000)
        sy = slabs.Synth(lm, device=dev)
        wd = slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, sy, w.Q, G, device=dev,
                                 check_rounds=16)
        done = 0
        while done < preroll:
            k = min(wd.K, preroll - done)
            for _ in range(k):
                wd.round()
            done += k
            wd.check()
        d0 = wd.dispatched()
        tl = []
        for _ in range(timed):
            wd.round(timing=tl)
        wd.check()
        per_round = (wd.dispatched() - d0) / timed
        med = [sorted(r[k] for r in tl)[len(tl) // 2] for k in range(G)]
        t = max(med)
        out[f"G={G}"] = {"agents": len(w.x), "map": [w.map_w, w.map_h], "rank_round_ms_max_over_ranks": t,
                         "rank_round_ms_mean": sum(med) / G, "agent_steps_per_round": per_round,
                         "agent_steps_per_s_if_one_gpu_per_slab": per_round / (t / 1000.0),
                         "halo_rows": wd.halo, "rewindows": wd.rewindows, "rounds": preroll + timed}
        wd.close()
        del w
    return out


# ------------------------------------------------------------------ N > 1: spatial slabs
def run_slabs(args, w, lm):
    """N GPUs (torchrun, one process per GPU, NCCL over NVLink): the ONE C5 map split into
    N horizontal slabs (slabs.DistWorld): every round = window tracker round
    + all-gather of merge records + merge/dispatch + all-reduce MIN of the event clock +
    commit + all-to-all of deltas + apply.  Strong scaling: the total work is the same 1M
    agents as N = 1.  value = agent-steps dispatched by all ranks / max over ranks of the
    summed device time of the timed rounds."""
    import torch
    import torch.distributed as dist

    from paper_2411_03519_b200 import slabs
    ws, rank, local = _dist()
    staged = os.environ.get("AM_SLAB_STAGED") == "1"   # test only: N ranks on ONE GPU over gloo
    if staged:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if staged:
        dist.init_process_group("gloo")
        ex = slabs.HostStagedDist(dist)
    else:
        dist.init_process_group("nccl", device_id=dev)
        ex = dist
    sy = slabs.Synth(lm, device=dev)
    wd = slabs.DistWorld(ex, w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, sy, w.Q, device=dev,
                         check_rounds=16, stale_rounds=args.slab_stale)
    done = 0
    while done < args.preroll:
        for _ in range(min(wd.K, args.preroll - done)):
            wd.round()
            done += 1
        wd.check()
    for _ in range(args.warmup):
        wd.round()
    wd.check()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    evs = []
    d0 = int(wd.rank.counters[2].item())
    try:
        gid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        gid = str(local)
    dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(gid) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            wd.round()
            b.record()
            evs.append((a, b))
            if (k + 1) % wd.K == 0:
                wd.check()   # (outside the event brackets)
    torch.cuda.synchronize(dev)
    dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    steps_local = int(wd.rank.counters[2].item()) - d0
    t = torch.tensor([total_ms, float(steps_local)], dtype=torch.float64, device=dev)
    tmax = t[:1].clone()
    ex.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = t[1:].clone()
    ex.all_reduce(tsum, op=dist.ReduceOp.SUM)
    total_ms, agent_steps = float(tmax.item()), int(tsum.item())
    value = agent_steps / (total_ms / 1e3) if total_ms > 0 else 0.0
    wd.check()
    # e2e: every round the rank's window state goes host -> device from page-locked
    # memory and back, and the rank's ready order + count come back to the host
    r = wd.rank
    L = r.cap_window
    h_pos = torch.empty((L, 2), dtype=torch.int32, pin_memory=True)
    h_step = torch.empty(L, dtype=torch.int32, pin_memory=True)
    h_order = torch.empty(L, dtype=torch.int32, pin_memory=True)
    h_n = torch.empty(1, dtype=torch.int32, pin_memory=True)
    h_pos.copy_(r.w_pos)
    h_step.copy_(r.w_step)
    torch.cuda.synchronize(dev)
    e_ms = []
    e0 = int(r.counters[2].item())
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r.w_pos.copy_(h_pos, non_blocking=True)
        r.w_step.copy_(h_step, non_blocking=True)
        wd.round()
        h_order.copy_(r.order, non_blocking=True)
        h_n.copy_(r.n_order, non_blocking=True)
        h_pos.copy_(r.w_pos, non_blocking=True)
        h_step.copy_(r.w_step, non_blocking=True)
        b.record()
        b.synchronize()
        e_ms.append(a.elapsed_time(b))
        if (k + 1) % wd.K == 0:
            wd.check()
            if wd.rank is not r:   # re-windowed: new buffers
                r = wd.rank
                L = r.cap_window
                h_pos = torch.empty((L, 2), dtype=torch.int32, pin_memory=True)
                h_step = torch.empty(L, dtype=torch.int32, pin_memory=True)
                h_order = torch.empty(L, dtype=torch.int32, pin_memory=True)
                h_pos.copy_(r.w_pos)
                h_step.copy_(r.w_step)
                torch.cuda.synchronize(dev)
    e_steps = int(r.counters[2].item()) - e0
    te = torch.tensor([sum(e_ms), float(e_steps)], dtype=torch.float64, device=dev)
    tem = te[:1].clone()
    ex.all_reduce(tem, op=dist.ReduceOp.MAX)
    tes = te[1:].clone()
    ex.all_reduce(tes, op=dist.ReduceOp.SUM)
    e_value = float(tes.item()) / (float(tem.item()) / 1e3) if float(tem.item()) > 0 else 0.0
    launches_round = 32   # library kernels of one rank's round (tracker ~14 + slab steps ~14 + sort)
    if rank == 0:
        cfg = _config(w, ws)
        cfg["parallelism"] = f"slabs{ws}" + ("-gloo-staged-one-gpu (test only)" if staged else "")
        cfg["halo_rows"] = wd.halo
        cfg["stale_rounds"] = args.slab_stale
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": cfg,
            "rounds_per_s": args.steps / (total_ms / 1e3) if total_ms > 0 else 0.0,
            "agent_steps_per_round": agent_steps / args.steps,
            "e2e": {"value": e_value, "unit": UNIT, "h2d_bytes_per_step": 12 * L * ws,
                    "d2h_bytes_per_step": (12 * L + 4 * L // 8) * ws, "ms_per_step": sum(e_ms) / args.steps,
                    "note": "per rank: window state H2D + round + window state, order and count D2H"},
            "gpu_launches": launches_round * args.steps,
            "clocks": clk.summary(), "roofline": None, "cpu_baseline": None,
            "rewindows": wd.rewindows,
        }
        print(json.dumps(line), flush=True)
    wd.close()
    dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, w, lm):
    import numpy as np
    import torch

    from paper_2411_03519_b200 import Replay

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    rep = Replay.from_workload(w, lm, device=dev)
    stream = torch.cuda.ExternalStream(rep.stream_ptr(), device=dev)
    names = ["k_ingest", "k_bin", "k_cells", "k_scatter", "k_scan", "k_finalize", "k_ready",
             "k_sort_hist", "k_sort_pass", "k_small", "k_commit", "k_disp_a", "k_disp_b", "k_union", "k_near"]
    ncells = None

    # pre-roll to steady state (untimed)
    rep.run(args.preroll)
    # warm-up with every kernel timed -> per-kernel shares, the dominant kernel
    rep.profile((1 << len(names)) - 1)
    for _ in range(args.warmup):
        rep.launch(1)
        rep.sync()
    prof_w = rep.profile_read()
    dom = max((k for k in prof_w if prof_w[k][1] > 0), key=lambda k: prof_w[k][0])
    # the state of the next round: the CPU oracle baseline samples exactly this state
    # (SURVEY 8(d.4) "same inputs, same run"); the round itself is one more warm-up
    rep.profile(0)
    cpu_state = take_round_state(rep)
    shares = {k: v[0] / v[1] for k, v in prof_w.items() if v[1] > 0}
    # timed region: only the dominant kernel bracketed by events
    rep.profile(1 << names.index(dom))
    rep.launch(1)
    rep.sync()
    rep.profile(1 << names.index(dom))
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    st_active, st_ready, st_running, st_work, st_far, st_items, st_edges, st_np = [], [], [], [], [], [], [], []
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    d0 = rep.dispatched()
    try:
        gid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        gid = str(local)
    with ClockSampler(gid) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
                ev[k][0].record(stream)
            rep.launch(1)
            ev[k][1].record(stream)
            act, nr = rep.sync()
            s = rep.tracker.stats()
            st_active.append(s["n_active"])
            st_ready.append(nr)
            st_running.append(s["n_running"])
            st_work.append(s["n_work"])
            st_far.append(s["n_far"])
            st_items.append(s["n_items"])
            st_edges.append(s["n_edges"])
            st_np.append(s["n_passes"])
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    d1 = rep.dispatched()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    prof_t = rep.profile_read()
    dom_ms, dom_cnt = prof_t[dom]
    agent_steps = d1 - d0
    # max over ranks of the timed device time; sum of work
    if pg:
        t = torch.tensor([total_ms, float(agent_steps)], dtype=torch.float64, device=dev)
        tmax = t.clone()
        pg.all_reduce(tmax[:1], op=pg.ReduceOp.MAX)
        pg.all_reduce(t[1:], op=pg.ReduceOp.SUM)
        total_ms, agent_steps = float(tmax[0]), int(t[1])
    value = agent_steps / (total_ms / 1000.0) if total_ms > 0 else 0.0
    rounds_per_s = args.steps / (total_ms / 1000.0) if total_ms > 0 else 0.0

    # ---- end to end: world state in pinned host memory, copies inside the timed region
    n = rep.n
    h_pos = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
    h_steps = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_mask = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_order = torch.empty(n, dtype=torch.int32, pin_memory=True)
    rep.profile(0)
    torch.cuda.synchronize(dev)
    h_pos.copy_(rep.pos)
    h_steps.copy_(rep.steps)
    # warm-up of the host-buffer path (its first call captures the round graph that
    # copies the mask out beside the round's tail)
    for _ in range(2):
        rep.io(h_pos, h_steps, h_mask, h_order)
        rep.sync()
    e_ms = []
    e0 = rep.dispatched()
    for k in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
            a.record(stream)
        rep.io(h_pos, h_steps, h_mask, h_order)
        b.record(stream)
        rep.sync()
        e_ms.append(a.elapsed_time(b))
    e_steps = rep.dispatched() - e0
    e_total = sum(e_ms)
    # D2H bytes of the delta write-back: counted on a few further (untimed) rounds by
    # diffing the host state -- touching the host arrays between timed rounds would put
    # them in the CPU caches and slow the device's PCIe accesses to them
    committed = groups = 0
    cnt_rounds = min(5, args.steps)
    for k in range(cnt_rounds):
        prev = h_steps.numpy().copy()
        rep.io(h_pos, h_steps, h_mask, h_order)
        rep.sync()
        chg = np.flatnonzero(h_steps.numpy() != prev)
        committed += len(chg)
        groups += len(np.unique(chg // 8))   # the write-back writes whole 8-agent groups
    e_value = e_steps / (e_total / 1000.0) if e_total > 0 else 0.0
    if pg:
        t = torch.tensor([e_total, float(e_steps)], dtype=torch.float64, device=dev)
        tm = t.clone()
        pg.all_reduce(tm[:1], op=pg.ReduceOp.MAX)
        pg.all_reduce(t[1:], op=pg.ReduceOp.SUM)
        e_value = float(t[1]) / (float(tm[0]) / 1000.0)

    snap = snapshot_rounds(rep, w, dev, flush) if not args.no_snapshot else None
    vslab = virtual_slabs(w, lm, dev) if (not args.no_snapshot and ws == 1) else None
    vtall = virtual_slabs_tall(lm, dev) if (not args.no_snapshot and ws == 1 and w.name == "C5") else None

    if rank != 0:
        rep.close()
        if pg:
            pg.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel
    L = rep.tracker.L
    stats = {"n": n, "n_active": statistics.mean(st_active), "n_ready": statistics.mean(st_ready),
             "n_running": statistics.mean(st_running), "n_work": statistics.mean(st_work),
             "n_far": statistics.mean(st_far), "n_items": statistics.mean(st_items),
             "n_edges": statistics.mean(st_edges), "passes": statistics.mean(st_np),
             "ncells": 0}
    # cell count of the binned path: (workspace layout) -- from the config the library chose
    cell = rep.tracker.stats()["cell"]
    g = 64
    while g * cell < max(w.map_w, w.map_h):
        g *= 2
    stats["ncells"] = g * g
    peak, peak_src, pk = _peaks()
    avg_dom_s = dom_ms / max(1, dom_cnt) / 1000.0
    alg = algorithmic_bytes(dom, stats)
    achieved = alg / avg_dom_s / 1e9 if avg_dom_s > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(dom)
            traffic = tr.get("dram_bytes_per_launch") if tr else None
    except Exception:
        pass
    # the dominant kernel against the SM issue rate (it is latency/issue-bound, not HBM
    # bound): warp instructions per launch from the committed ncu --set full capture
    # (profiles/ncu_instr.json) over the live average launch time
    issue = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_instr.json")) as f:
            ij = json.load(f)
        wi = ij[dom]["warp_instructions_per_launch"]
        pk_i = ij["issue_peak_warp_instr_per_s"]["value"]
        ach_i = wi / avg_dom_s if avg_dom_s > 0 else 0.0
        issue = {"kernel": dom, "achieved": ach_i, "peak": pk_i, "unit": "warp-instr/s", "frac": ach_i / pk_i,
                 "warp_instructions_per_launch": wi,
                 "peak_source": ij["issue_peak_warp_instr_per_s"]["derivation"]}
    except Exception:
        pass
    clocks = clk.summary()
    # round-level HBM traffic: ncu cold-cache DRAM bytes of every kernel of a round
    # (profiles/ncu_traffic.json) over the measured round time
    round_hbm = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        tot = sum(v["dram_bytes_per_launch"] * v.get("launches", 1) for k, v in tj.items()
                  if isinstance(v, dict) and "dram_bytes_per_launch" in v and k not in ("k_scan", "k_near"))
        gbs = tot / (total_ms / args.steps / 1e3) / 1e9
        round_hbm = {"dram_bytes_per_round": tot, "achieved_gbs": gbs, "frac": gbs / peak,
                     "compulsory_bytes_per_round": 18.0 * n,
                     "compulsory_frac": 18.0 * n / (total_ms / args.steps / 1e3) / 1e9 / peak,
                     "source": "ncu launch list (cold-cache DRAM bytes per kernel) / event-timed round"}
    except Exception:
        pass
    others = None
    if ws == 1 and not args.no_other_configs:
        others = other_configs(dev)
    # the oracle on the host cores, bounded sample (rank 0, N = 1 only)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        v, sm, dt = oracle_sample(w, cpu_state, args.cpu_seconds)
        nt = max(1, len(os.sched_getaffinity(0)))
        vt, smt, dtt = oracle_sample_threads(w, cpu_state, args.cpu_seconds / 2, nt) if nt > 1 else (v, sm, dt)
        cpu = {"value": vt, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"{smt} sampled agents of the pre-rolled {w.name} round the GPU is timed on "
                         f"({n} agents, after {args.preroll} + {args.warmup} rounds) resolved one by one "
                         f"by oracle.c in {dtt:.1f} s on {nt} threads (outer loop over sampled agents, "
                         f"one seed per thread)",
               "single_thread": {"value": v, "cores": 1,
                                 "sample": f"{sm} sampled agents in {dt:.1f} s"},
               "host_cores_available": os.cpu_count()}
    launches = rep.launches_per_round() * args.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        # the same C5 map at every N (N > 1: split into slabs, run_slabs): total work fixed
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": _config(w, ws),
        "rounds_per_s": rounds_per_s,
        "agent_steps_per_round": agent_steps / args.steps / ws,
        "round_stats": {"active": stats["n_active"], "ready": stats["n_ready"],
                        "running": stats["n_running"], "rescanned": stats["n_work"],
                        "far": stats["n_far"], "far_items": stats["n_items"], "edges": stats["n_edges"]},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg, "avg_launch_us": avg_dom_s * 1e6},
        "round_hbm": round_hbm,
        "issue_roofline": issue,
        "snapshot": snap,
        "virtual_slabs": vslab,
        "virtual_slabs_weak": vtall,
        "kernel_share_warmup_us": {k: round(v * 1000.0, 2) for k, v in sorted(shares.items())},
        # D2H (am_replay_io, page-locked host arrays, state outputs aliasing the inputs):
        # position + step of every aligned 8-agent group holding a committed agent (96 B
        # per group, delta write-back), the mask (n B) and the n_ready order entries
        # (4 B each), written by kernels / a copy into host memory
        "e2e": {"value": e_value, "unit": UNIT, "h2d_bytes_per_step": 12 * n,
                "d2h_bytes_per_step": int(n + 96 * groups / cnt_rounds + 4 * e_steps / args.steps),
                "committed_per_step": committed / cnt_rounds,
                "ms_per_step": e_total / args.steps},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "other_configs": others,
    }
    print(json.dumps(line), flush=True)
    rep.close()
    if pg:
        pg.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--agents", type=int, default=None, help="shrink the workload (same density)")
    ap.add_argument("--preroll", type=int, default=400)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--no-snapshot", action="store_true")
    ap.add_argument("--slab-stale", type=int, default=1, choices=[1, 2, 4, 8, 16],
                    help="N > 1: a sync round every P rounds (stale-halo rounds between)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    import amgen
    w = amgen.config(args.workload, n=args.agents)
    lm = amgen.latency_model(w.profile)
    if args.impl == "reference":
        return run_reference(args, w, lm)
    if _dist()[0] > 1:
        return run_slabs(args, w, lm)
    return run_ours(args, w, lm)


if __name__ == "__main__":
    sys.exit(main())
