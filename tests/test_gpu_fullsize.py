"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C5 (1M agents, 16384^2) and C4 (100k agents, 4096^2): the GPU-resident replay is
pre-rolled exactly as bench.py does it (incremental rounds from CUDA graphs), then one
round is taken with its outputs.  The brute-force oracle cannot run a whole round at
this size, so (tests/ note in DESIGN.md section 4):
  * sampled agents are resolved one by one by oracle.round_sampled (blocking by an
    O(N) scan, cluster by a BFS over the coupling graph): ready bit, cluster label
    (min id) and, for IDLE agents, the blocking verdict must match bit for bit;
  * properties that hold at any size are checked on the whole output: `order` is
    exactly the set of ready agents, sorted by (step, label, id); labels are the
    minimum id of their class (label[label[i]] == label[i] <= i); DONE agents have
    label -1; a ready agent's whole cluster is ready or RUNNING-free.
The same state is then recomputed from scratch by a fresh tracker (am_set_state, the
full non-incremental round of bench.py's "snapshot") and must equal the incremental
round on every output, element by element."""
import ctypes as C

import numpy as np
import pytest
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import Replay, Tracker

pytestmark = pytest.mark.gpu


def _sample(n, mask, blocked, labels, rng, k=60):
    """Uniform agents plus ready, blocked and clustered ones (the interesting cases)."""
    parts = [rng.integers(0, n, k)]
    for sel in (np.flatnonzero(mask), np.flatnonzero(blocked),
                np.flatnonzero((labels >= 0) & (labels != np.arange(n)))):
        if len(sel):
            parts.append(rng.choice(sel, min(k, len(sel)), replace=False))
    return np.unique(np.concatenate(parts)).astype(np.int32)


@pytest.mark.parametrize("name,preroll", [("C5", 400), ("C4", 400), ("C5", 150)])
def test_full_size_round_sampled_vs_oracle(name, preroll):
    w = amgen.config(name)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    rep.run(preroll)
    # the state the next round ingests (the world arrays after the last commits)
    x = rep.pos[:, 0].cpu().numpy().copy()
    y = rep.pos[:, 1].cpu().numpy().copy()
    s = rep.steps.cpu().numpy().copy()
    tr = rep.tracker
    # the statuses the round sees (the last round's commits were applied in place)
    st = tr.status().cpu().numpy().copy()
    mask_t, order_t, labels_t = rep.step()
    n = rep.n
    blk_t = torch.empty(n, dtype=torch.uint8, device="cuda")
    assert tr.L.am_blocked(tr.ctx, C.c_void_p(blk_t.data_ptr())) == 0
    torch.cuda.synchronize()
    mask = mask_t.cpu().numpy()
    order = order_t.cpu().numpy()
    labels = labels_t.cpu().numpy()
    blocked = blk_t.cpu().numpy()
    assert mask.sum() > 1000, "the pre-roll must reach a round that dispatches work"
    assert len(np.unique(s[st != O.DONE])) > 10, "expected a spread of steps"

    # ---- whole-output properties
    ready = np.flatnonzero(mask)
    assert np.array_equal(np.sort(order), ready)
    key = np.lexsort((order, labels[order], s[order]))
    assert np.array_equal(key, np.arange(len(order))), "order must be sorted by (step, label, id)"
    act = st != O.DONE
    assert np.all(labels[~act] == -1)
    la = labels[act]
    assert np.all(la <= np.flatnonzero(act))
    assert np.all(labels[la] == la), "a label is the id of its own class representative"
    assert np.all(st[ready] == O.IDLE)
    # every member of a ready cluster is ready (IDLE, unblocked, no RUNNING mate)
    rl = np.unique(labels[ready])
    members = np.isin(labels, rl)
    assert np.all(mask[members] == 1)

    # ---- sampled agents against the brute-force oracle
    rng = np.random.default_rng(7)
    smp = _sample(n, mask, blocked, labels, rng)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    r = O.round_sampled(p, x, y, s, st, smp)
    np.testing.assert_array_equal(mask[smp], r["mask"], err_msg=f"{name}: ready bits")
    np.testing.assert_array_equal(labels[smp], r["label"], err_msg=f"{name}: cluster labels")
    idle = st[smp] == O.IDLE
    np.testing.assert_array_equal(blocked[smp][idle], r["blocked"][idle], err_msg=f"{name}: blocking")

    # ---- the same state from scratch (full round) equals the incremental round
    ft = Tracker(w.map_w, w.map_h, w.r_p, w.v, n, target=w.steps, peek=True, validate=False,
                 force="binned")
    dev = torch.device("cuda")
    ft.set_state(torch.as_tensor(np.stack([x, y], 1), dtype=torch.int32, device=dev),
                 torch.as_tensor(s, device=dev), torch.as_tensor(st, device=dev))
    fmask, forder = ft.ready()
    flabels = ft.clusters()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(fmask.cpu().numpy(), mask)
    np.testing.assert_array_equal(forder.cpu().numpy(), order)
    np.testing.assert_array_equal(flabels.cpu().numpy(), labels)
    ft.close()
    rep.close()


@pytest.mark.parametrize("name,rounds", [("C4", 300), ("C5", 60)])
def test_replay_is_deterministic_at_full_size(name, rounds):
    """Run-to-run determinism at BASELINE sizes (the kernels order their work with
    atomics: slot count-downs, union-find hooks, stripe appends, sort ranks): two replays
    of the same workload from the same initial state, in the launch configuration bench.py
    times, dispatch the same agent-steps every round and end in the same world state
    (positions, steps, trajectory hashes) -- every output that the oracle fixes is unique,
    so any order dependence would show up here."""
    w = amgen.config(name)
    lm = amgen.latency_model(w.profile)
    runs = []
    for _ in range(2):
        rep = Replay.from_workload(w, lm)
        per_round = []
        for _r in range(rounds // 20):
            d0 = rep.dispatched()
            rep.launch(20)
            rep.sync()
            per_round.append(rep.dispatched() - d0)
        runs.append((per_round, rep.pos.cpu().numpy().copy(), rep.steps.cpu().numpy().copy(),
                     rep.results()["traj"].copy()))
        rep.close()
    (d1, p1, s1, t1), (d2, p2, s2, t2) = runs
    assert d1 == d2
    assert sum(d1) > 0
    np.testing.assert_array_equal(p1, p2)
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_array_equal(t1, t2)
