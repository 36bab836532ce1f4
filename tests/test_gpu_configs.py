"""GPU vs the CPU oracle on all five BASELINE configurations at their full sizes
(north_star: "bit-exact ready sets, clusters and final states against the CPU oracle
on all 5 configs"; SURVEY 8(d.1) parity scope).

* C2 (500 agents, 20 replicated maps, busy hour, T = 1000): every round's log (ids in
  priority order + cluster labels of the dispatched agents) of the whole replay, chained
  into blake2b checkpoints every 1000 rounds, against tests/golden/c2_replay_T1000.txt
  (written by tests/golden/make_c2_replay.py from oracle.replay, ~10 min of oracle time);
  round count, T_ooo and the final state; the binned path's final state too.
* C3 (4096 x 25-agent simulations, T = 1000): every simulation's final positions,
  trajectory hashes, T_ooo and round count against oracle.replay_mt and lock-step;
  the round logs of 64 sampled simulations against oracle.replay_sims_logged.
* C4 (100k agents, 4096^2, hotspots, Q = 50 ms, T = 1000): replay rounds 1, 50, 100,
  ..., 300, 500, 1000, 2000 compared element by element (mask, order, labels, blocking
  verdicts of IDLE agents) with the threaded brute-force round oracle.round_mt; the
  final state (positions, trajectory hashes) against the oracle's lock-step run
  (hash-grid perception, Alg. 1) -- OoO == lock-step.
* C5 (1M agents, 16384^2): three replay rounds with the label of EVERY agent
  (oracle.labels_steps, all same-step pairs) and >= 10k sampled agents' ready bits and
  blocking verdicts (oracle.round_at_scale); the final state at T = 200 against the
  oracle's lock-step run.
All integer: the bar is bit-exact everywhere."""
import ctypes as C
import hashlib
import os

import numpy as np
import pytest
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import Replay

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_replay_T1000.txt")


def _chain(rounds, every=1000):
    h = hashlib.blake2b(digest_size=16)
    marks, k = [], 0
    for ids, lab in rounds:
        h.update(np.int32(len(ids)).tobytes())
        h.update(np.ascontiguousarray(ids, np.int32).tobytes())
        h.update(np.ascontiguousarray(lab, np.int32).tobytes())
        k += 1
        if k % every == 0:
            marks.append(h.hexdigest())
    return k, marks, h.hexdigest()


def _state_hash(x, y, traj):
    h = hashlib.blake2b(digest_size=16)
    for a in (np.asarray(x, np.int32), np.asarray(y, np.int32), np.asarray(traj, np.uint64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


class _Stepper:
    """Round-by-round replay with the outputs kept on the device (few allocations)."""

    def __init__(self, rep):
        self.rep = rep
        n = rep.n
        self.mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        self.order = torch.empty(n, dtype=torch.int32, device="cuda")
        self.labels = torch.empty(n, dtype=torch.int32, device="cuda")

    def step(self):
        nr = C.c_int32(0)
        rc = self.rep.L.am_replay_step(self.rep.h, self.mask.data_ptr(), self.order.data_ptr(),
                                       self.labels.data_ptr(), C.byref(nr))
        assert rc == 0, self.rep.L.am_last_error(self.rep.tracker.ctx)
        return nr.value


def _round_state(rep):
    """The state the next round ingests: world arrays after the last commits (the
    replay commits at the end of a round) and the statuses."""
    x = rep.pos[:, 0].cpu().numpy().copy()
    y = rep.pos[:, 1].cpu().numpy().copy()
    s = rep.steps.cpu().numpy().copy()
    return x, y, s


def _take_round(rep):
    """Run one round with outputs; returns (x, y, s, st_seen, mask, order, labels, blocked).
    The state the round sees: the world arrays and the tracker's statuses before it (the
    last round's commits were applied in place at its end)."""
    x, y, s = _round_state(rep)
    tr = rep.tracker
    st = tr.status().cpu().numpy().copy()
    mask_t, order_t, labels_t = rep.step()
    n = rep.n
    blk_t = torch.empty(n, dtype=torch.uint8, device="cuda")
    assert tr.L.am_blocked(tr.ctx, C.c_void_p(blk_t.data_ptr())) == 0
    torch.cuda.synchronize()
    mask = mask_t.cpu().numpy()
    return x, y, s, st, mask, order_t.cpu().numpy(), labels_t.cpu().numpy(), blk_t.cpu().numpy()


# ------------------------------------------------------------------------------- C2
def _golden():
    g = {"marks": []}
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        if k == "log_mark":
            g["marks"].append((int(v[0]), v[1]))
        else:
            g[k] = v[0]
    return g


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden C2 replay not generated")
def test_c2_full_replay_round_logs_vs_oracle():
    g = _golden()
    w = amgen.config("C2")
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    st = _Stepper(rep)
    logs = []
    for _ in range(5 * 10**6):
        nr = st.step()
        if nr:
            logs.append((st.order[:nr].cpu().numpy(), st.labels[st.order[:nr].long()].cpu().numpy()))
        elif rep.tracker.stats()["n_active"] == 0:
            break
    nlog, marks, final = _chain(logs)
    assert nlog == int(g["logged_rounds"])
    for (k, m), mine in zip(g["marks"], marks):
        assert mine == m, f"C2 round log diverges before logged round {k}"
    assert final == g["log_final"]
    res = rep.results()
    assert int(res["rounds"][0]) == int(g["rounds"])
    assert int(res["T_ooo"][0]) == int(g["T_ooo"])
    assert _state_hash(res["x"], res["y"], res["traj"]) == g["state"]
    assert rep.dispatched() == len(w.x) * w.steps
    rep.close()
    # the persistent per-simulation kernel and the binned pipeline reach the same end
    for force in (None, "binned"):
        rep = Replay.from_workload(w, lm, force=force)
        rep.run_to_end(chunk=4096)
        res = rep.results()
        assert int(res["T_ooo"][0]) == int(g["T_ooo"]) and int(res["rounds"][0]) == int(g["rounds"])
        assert _state_hash(res["x"], res["y"], res["traj"]) == g["state"]
        rep.close()


# ------------------------------------------------------------------------------- C3
def test_c3_all_simulations_final_states():
    w = amgen.config("C3")
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    ref = O.replay_mt(p, sy, w.x, w.y)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(ref["traj"], ls["traj"])      # P:27 on the oracle side
    rep = Replay.from_workload(w, lm)
    rep.run_to_end(chunk=2048)
    res = rep.results()
    for k in ("x", "y", "traj", "T_ooo", "rounds"):
        np.testing.assert_array_equal(res[k], ref[k], err_msg=f"C3 {k}")
    assert np.all(res["T_ooo"] <= ls["T_sync"])
    rep.close()


def test_c3_sampled_simulations_round_logs():
    w = amgen.config("C3")
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    sims = sorted(np.random.default_rng(11).choice(w.n_sims, 64, replace=False).tolist())
    ref = O.replay_sims_logged(p, sy, w.x, w.y, sims)
    rep = Replay.from_workload(w, lm)
    st = _Stepper(rep)
    n = len(w.x)
    want = np.zeros(w.n_sims, bool)
    want[sims] = True
    logs = {b: [] for b in sims}
    for _ in range(10**6):
        nr = st.step()
        if nr:
            o = st.order[:nr].cpu().numpy()
            lab = st.labels.cpu().numpy()
            sim = (o.astype(np.int64) * w.n_sims + w.n_sims - 1) // n
            for b in np.unique(sim[want[sim]]):
                sel = o[sim == b]
                logs[int(b)].append((sel, lab[sel]))
        elif rep.tracker.stats()["n_active"] == 0:
            break
    for b in sims:
        r = ref[b]
        k = 0
        olog = []
        for nr in r["log_nready"]:
            if nr:
                olog.append((r["log_id"][k:k + nr], r["log_label"][k:k + nr]))
            k += nr
        assert len(logs[b]) == len(olog), (b, len(logs[b]), len(olog))
        for (gi, gl), (oi, ol) in zip(logs[b], olog):
            np.testing.assert_array_equal(gi, oi)
            np.testing.assert_array_equal(gl, ol)
    rep.close()


# ------------------------------------------------------------------------------- C4
C4_ROUNDS = [1, 50, 100, 150, 200, 250, 300, 500, 1000, 2000]


def test_c4_replay_rounds_full_vs_oracle_and_final_state():
    w = amgen.config("C4")
    lm = amgen.latency_model(w.profile)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    rep = Replay.from_workload(w, lm)
    done = 0
    compared = 0
    for r in C4_ROUNDS:
        if r - 1 > done:
            act = rep.run(r - 1 - done)
            done = r - 1
            if act == 0:
                break
        x, y, s, st, mask, order, labels, blocked = _take_round(rep)
        done += 1
        ref = O.round_mt(p, x, y, s, st.copy(), peek=True)
        np.testing.assert_array_equal(mask, ref["mask"], err_msg=f"C4 round {r}: mask")
        np.testing.assert_array_equal(order, ref["order"], err_msg=f"C4 round {r}: order")
        np.testing.assert_array_equal(labels, ref["label"], err_msg=f"C4 round {r}: labels")
        idle = st == O.IDLE
        np.testing.assert_array_equal(blocked[idle], ref["blocked"][idle], err_msg=f"C4 round {r}: blocking")
        compared += 1
    assert compared >= 8
    rep.run_to_end(chunk=1024)
    res = rep.results()
    assert np.all(res["steps"] == w.steps)
    sy = O.SynthTables.from_model(lm)
    ls = O.lockstep_grid(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["x"], ls["x"])
    np.testing.assert_array_equal(res["y"], ls["y"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert rep.dispatched() == len(w.x) * w.steps
    rep.close()


# ------------------------------------------------------------------------------- C5
@pytest.mark.parametrize("preroll", [1, 150, 400])
def test_c5_round_all_labels_and_sampled_agents(preroll):
    w = amgen.config("C5")
    lm = amgen.latency_model(w.profile)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    rep = Replay.from_workload(w, lm)
    if preroll > 1:
        rep.run(preroll - 1)
    x, y, s, st, mask, order, labels, blocked = _take_round(rep)
    rep.close()
    n = len(x)
    rng = np.random.default_rng(preroll)
    parts = [rng.choice(n, 8000, replace=False)]
    for sel in (np.flatnonzero(mask), np.flatnonzero(blocked), np.flatnonzero((labels >= 0) & (labels != np.arange(n)))):
        if len(sel):
            parts.append(rng.choice(sel, min(1500, len(sel)), replace=False))
    smp = np.unique(np.concatenate(parts)).astype(np.int32)
    assert len(smp) >= 10_000
    ref = O.round_at_scale(p, x, y, s, st, smp)
    np.testing.assert_array_equal(labels, ref["label"], err_msg="C5: labels of every agent")
    np.testing.assert_array_equal(mask[smp], ref["mask"], err_msg="C5: ready bits")
    idle = st[smp] == O.IDLE
    np.testing.assert_array_equal(blocked[smp][idle], ref["blocked"][idle], err_msg="C5: blocking")
    # the order is the ready set sorted by (step, label, id)
    ready = np.flatnonzero(mask)
    assert np.array_equal(np.sort(order), ready)
    assert np.array_equal(np.lexsort((order, labels[order], s[order])), np.arange(len(order)))


def test_c5_final_state_vs_lockstep_T200():
    w = amgen.config("C5", steps=200)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    rep.run_to_end(chunk=1024)
    res = rep.results()
    assert np.all(res["steps"] == w.steps)
    assert rep.dispatched() == len(w.x) * w.steps
    rep.close()
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    ls = O.lockstep_grid(p, O.SynthTables.from_model(lm), w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["x"], ls["x"])
    np.testing.assert_array_equal(res["y"], ls["y"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
