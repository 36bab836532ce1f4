"""GPU replay driver vs the oracle's OoO replay and lock-step simulator: per-round
logs (order and labels of every dispatched agent), final positions, per-agent
trajectory hashes, T_ooo and round counts -- all bit-exact."""
import numpy as np
import pytest
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import Replay

pytestmark = pytest.mark.gpu


def _oracle(w, lm, log=True, check=False):
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    cap_r = 10**6 if log else 0
    cap_e = len(w.x) * w.steps + 10 if log else 0
    return O.replay(p, sy, w.x, w.y, Q=w.Q, log_rounds=cap_r, log_entries=cap_e, check=check), \
        O.lockstep(p, sy, w.x, w.y, w.steps)


def _gpu_logged(rep, n_sims, n):
    """Step round by round; split the round's order per simulation (sim-major)."""
    logs = [[] for _ in range(n_sims)]
    for _ in range(10**7):
        mask, order, labels = rep.step()
        o = order.cpu().numpy()
        lab = labels.cpu().numpy()
        sims = (o.astype(np.int64) * n_sims + n_sims - 1) // n if n_sims > 1 else np.zeros(len(o), int)
        for b in np.unique(sims):
            sel = o[sims == b]
            logs[b].append((sel.copy(), lab[sel].copy()))
        if rep.tracker.stats()["n_active"] == 0 and len(o) == 0:
            break
    return logs


def _split_oracle_log(r, n_sims):
    logs = [[] for _ in range(n_sims)]
    k = 0
    for t, b, nr in zip(r["log_t"], r["log_sim"], r["log_nready"]):
        if nr:
            logs[b].append((r["log_id"][k:k + nr], r["log_label"][k:k + nr]))
        k += nr
    return logs


@pytest.mark.parametrize("name,steps,n_sims,path", [
    ("C1", 1000, 1, None),
    ("C1", 300, 1, "binned"),
    ("C3", 200, 16, None),
])
def test_replay_round_logs(name, steps, n_sims, path):
    w = amgen.config(name, steps=steps, n=n_sims if name == "C3" else None)
    lm = amgen.latency_model(w.profile)
    r, ls = _oracle(w, lm)
    assert r["log_complete"]
    rep = Replay.from_workload(w, lm, force=path)
    glogs = _gpu_logged(rep, w.n_sims, len(w.x))
    ologs = _split_oracle_log(r, w.n_sims)
    for b in range(w.n_sims):
        assert len(glogs[b]) == len(ologs[b]), (b, len(glogs[b]), len(ologs[b]))
        for (gi, gl), (oi, ol) in zip(glogs[b], ologs[b]):
            np.testing.assert_array_equal(gi, oi)
            np.testing.assert_array_equal(gl, ol)
    res = rep.results()
    np.testing.assert_array_equal(res["T_ooo"], r["T_ooo"])
    np.testing.assert_array_equal(res["rounds"], r["rounds"])
    np.testing.assert_array_equal(res["x"], r["x"])
    np.testing.assert_array_equal(res["y"], r["y"])
    np.testing.assert_array_equal(res["traj"], r["traj"])
    # outcome preservation: the OoO replay ends where lock-step ends
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert rep.dispatched() == len(w.x) * w.steps
    rep.close()


@pytest.mark.parametrize("name,steps,n,path", [
    ("C1", 1000, None, None),
    ("C2", 40, None, None),
    ("C2", 40, None, "binned"),
    ("C3", 300, 512, None),
    ("C4", 20, 2000, "binned"),
])
def test_replay_final_state(name, steps, n, path):
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    r, ls = _oracle(w, lm, log=False)
    rep = Replay.from_workload(w, lm, force=path)
    rep.run_to_end(chunk=512)
    res = rep.results()
    np.testing.assert_array_equal(res["T_ooo"], r["T_ooo"])
    np.testing.assert_array_equal(res["rounds"], r["rounds"])
    np.testing.assert_array_equal(res["traj"], r["traj"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert np.all(res["steps"] == w.steps)
    assert np.all(res["T_ooo"] <= ls["T_sync"]) if w.Q == 0 else True
    rep.close()


@pytest.mark.parametrize("x1,T,L0,L1,T_ooo", [
    (7, 2, [10, 1], [1, 10], 11), (6, 2, [10, 1], [1, 10], 20),
    (5, 2, [10, 1], [1, 10], 20), (7, 3, [1, 1, 1], [10, 10, 10], 30)])
def test_replay_closed_forms(x1, T, L0, L1, T_ooo):
    """D1/D2/D3/D5 on the GPU driver: stay policy, explicit durations."""
    rep = Replay(64, 8, 4, 1, [0, x1], [0, 0], T, dur_table=[L0, L1], policy=1)
    rep.run_to_end(chunk=8)
    assert int(rep.results()["T_ooo"][0]) == T_ooo
    rep.close()


@pytest.mark.parametrize("pinned", [True, False])
def test_host_io_round_equals_device_round(pinned):
    """am_replay_io (world state in host memory, the end-to-end user loop bench.py
    times) gives the same rounds as the device-resident replay: mask, the n_ready
    order entries and the committed state, round after round.  Page-locked host arrays
    take the kernel writes (n_ready order entries, delta write-back of the committed
    agents into the aliased state arrays), pageable ones the full copies."""
    w = amgen.config("C4", n=3000)
    lm = amgen.latency_model(w.profile)
    a = Replay.from_workload(w, lm)
    b = Replay.from_workload(w, lm)
    a.run(30)
    b.run(30)
    n = a.n
    h_pos = torch.empty((n, 2), dtype=torch.int32, pin_memory=pinned)
    h_steps = torch.empty(n, dtype=torch.int32, pin_memory=pinned)
    h_mask = torch.empty(n, dtype=torch.uint8, pin_memory=pinned)
    h_order = torch.full((n,), -7, dtype=torch.int32, pin_memory=pinned)
    torch.cuda.synchronize()
    h_pos.copy_(b.pos)
    h_steps.copy_(b.steps)
    for _ in range(25):
        mask, order, _ = a.step()
        b.io(h_pos, h_steps, h_mask, h_order)
        _, nr = b.sync()
        torch.cuda.synchronize()
        assert nr == order.numel()
        np.testing.assert_array_equal(h_mask.numpy(), mask.cpu().numpy())
        np.testing.assert_array_equal(h_order[:nr].numpy(), order.cpu().numpy())
        np.testing.assert_array_equal(h_pos.numpy(), a.pos.cpu().numpy())
        np.testing.assert_array_equal(h_steps.numpy(), a.steps.cpu().numpy())
    a.close()
    b.close()


@pytest.mark.parametrize("name,n_sims", [("C1", None), ("C3", 64), ("C2", None)])
def test_persistent_small_replay_equals_round_kernels(name, n_sims):
    """The persistent per-simulation replay kernel (am_replay_run / _launch on the fused
    path) and the multi-kernel rounds (am_replay_step) give identical states round for
    round, and the two can alternate: A runs 40 rounds persistently, B steps 40 rounds;
    then A steps 10 and B runs 10; then both run to the end."""
    w = amgen.config(name, steps=120, n=n_sims)
    lm = amgen.latency_model(w.profile)
    a = Replay.from_workload(w, lm)
    b = Replay.from_workload(w, lm)

    def same():
        torch.cuda.synchronize()
        np.testing.assert_array_equal(a.pos.cpu().numpy(), b.pos.cpu().numpy())
        np.testing.assert_array_equal(a.steps.cpu().numpy(), b.steps.cpu().numpy())
        ra, rb = a.results(), b.results()
        for k in ("T_ooo", "rounds", "traj"):
            np.testing.assert_array_equal(ra[k], rb[k], err_msg=k)
        assert a.dispatched() == b.dispatched()

    a.run(40)
    for _ in range(40):
        b.step()
    same()
    for _ in range(10):
        a.step()
    b.run(10)
    same()
    a.run_to_end()
    b.run_to_end()
    same()
    a.close()
    b.close()


@pytest.mark.parametrize("name,steps,n_sims,K,prio,path", [
    ("C1", 300, None, 1, True, None),
    ("C1", 300, None, 4, False, None),
    ("C1", 300, None, 8, True, None),
    ("C2", 60, None, 32, True, None),
    ("C2", 60, None, 32, False, None),
    ("C3", 120, 16, 3, True, None),
    ("C2", 60, None, 32, True, "binned"),
    ("C2", 60, None, 32, False, "binned"),
    ("C1", 200, None, 2, True, "binned"),
    ("C4", 15, 1500, 64, True, "binned"),
    ("C4", 15, 1500, 64, False, "binned"),
])
def test_capacity_replay_vs_oracle(name, steps, n_sims, K, prio, path):
    """Finite LLM capacity (am_replay_set_capacity: the persistent per-simulation kernel,
    or on the cell-binned path the device queue of ready clusters sorted by key and started
    while they fit) vs orc_replay_cap: T_ooo, round counts, final positions and trajectory
    hashes, bit for bit; the outcome equals lock-step's."""
    w = amgen.config(name, steps=steps, n=n_sims)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q, capacity=K, priority=prio)
    rep = Replay.from_workload(w, lm, capacity=K, priority=prio, force=path)
    rep.run_to_end()
    res = rep.results()
    for k in ("T_ooo", "rounds", "x", "y", "traj"):
        np.testing.assert_array_equal(res[k], r[k], err_msg=k)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert rep.dispatched() == len(w.x) * w.steps
    if path is None:
        with pytest.raises(Exception):
            rep.step()   # on the fused path finite capacity exists only in the persistent kernel


def test_capacity_binned_round_logs_vs_oracle():
    """The binned path with a finite capacity, round by round: the dispatched (queued)
    agents' ids and labels of every round equal orc_replay_cap's log."""
    w = amgen.config("C2", steps=30)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q, capacity=24, priority=True, log_rounds=10**6,
                 log_entries=len(w.x) * w.steps + 10)
    rep = Replay.from_workload(w, lm, capacity=24, priority=True, force="binned")
    glogs = _gpu_logged(rep, 1, len(w.x))
    ologs = _split_oracle_log(r, 1)
    assert len(glogs[0]) == len(ologs[0])
    for (gi, gl), (oi, ol) in zip(glogs[0], ologs[0]):
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gl, ol)
    res = rep.results()
    np.testing.assert_array_equal(res["traj"], r["traj"])
    rep.close()
    rep.close()


@pytest.mark.parametrize("path", [None, "binned"])
def test_linf_eight_connected_replay_vs_oracle(path):
    """NEXT #4 variant (L-infinity metric, 8-connected walk) on both GPU paths vs the
    oracle: T_ooo, rounds, final positions, trajectories; outcome == lock-step."""
    w = amgen.config("C1", steps=200)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall, policy=2)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, metric=O.LINF)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q)
    rep = Replay.from_workload(w, lm, policy=2, metric="linf", force=path)
    rep.run_to_end()
    res = rep.results()
    for k in ("T_ooo", "rounds", "x", "y", "traj"):
        np.testing.assert_array_equal(res[k], r[k], err_msg=k)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    rep.close()


def test_capacity_api_errors():
    """am_replay_set_capacity: only before the first round (AM_E_STATE) and with a
    non-negative capacity (AM_E_ARG); both paths accept it before the first round (the
    cell-binned path keeps its device queue)."""
    from paper_2411_03519_b200 import AmError, _lib
    w = amgen.config("C1", steps=20)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    rep.run(3)
    with pytest.raises(AmError) as e:
        _lib.check(rep.L.am_replay_set_capacity(rep.h, 4, 1), rep.tracker.ctx)
    assert e.value.code == _lib.E_STATE
    rep.close()
    rep = Replay.from_workload(w, lm, force="binned")
    with pytest.raises(AmError) as e:
        _lib.check(rep.L.am_replay_set_capacity(rep.h, -1, 1), rep.tracker.ctx)
    assert e.value.code == _lib.E_ARG
    _lib.check(rep.L.am_replay_set_capacity(rep.h, 4, 1), rep.tracker.ctx)
    rep.run(3)
    with pytest.raises(AmError) as e:
        _lib.check(rep.L.am_replay_set_capacity(rep.h, 8, 1), rep.tracker.ctx)
    assert e.value.code == _lib.E_STATE
    rep.close()


@pytest.mark.parametrize("name,steps,n_sims,K", [("C1", 300, None, 0), ("C2", 60, None, 0), ("C3", 120, 16, 0),
                                                 ("C1", 200, None, 4)])
def test_exclusive_tiles_replay_vs_oracle(name, steps, n_sims, K):
    """NEXT #4 exclusive tiles (per-cluster conflict resolution in the persistent kernel)
    vs the oracle, bit for bit; the outcome equals lock-step's with the rule applied over
    the whole simulation; also with a finite capacity."""
    w = amgen.config(name, steps=steps, n=n_sims)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall, conflict=1)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q, capacity=K)
    rep = Replay.from_workload(w, lm, conflict=1, capacity=K)
    rep.run_to_end()
    res = rep.results()
    for k in ("T_ooo", "rounds", "x", "y", "traj"):
        np.testing.assert_array_equal(res[k], r[k], err_msg=k)
    np.testing.assert_array_equal(res["traj"], O.lockstep(p, sy, w.x, w.y, w.steps)["traj"])
    rep.close()


@pytest.mark.parametrize("name,steps,n,path", [("C1", 300, None, None), ("C3", 120, 16, None),
                                               ("C4", 15, 2000, "binned"), ("C2", 30, None, "binned")])
def test_llm_time_and_lockstep_time(name, steps, n, path):
    """Achieved parallelism and the parallel-sync baseline: the LLM busy
    time the replay dispatched equals the schedule-independent sum over every agent-step
    of dur - base_us (each agent-step runs exactly once), and the device lock-step time
    equals the oracle's T_sync = sum_s max_i dur(i, s)."""
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm, force=path)
    rep.run_to_end(chunk=512)
    llm = rep.llm_time()
    tsync = rep.lockstep_time(w.steps)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    nn = len(w.x)
    durs = np.array([[O.duration(sy, i, s) for s in range(w.steps)] for i in range(nn)], np.int64)
    per_sim = (durs - lm.base_us).sum(1).reshape(w.n_sims, -1).sum(1)
    np.testing.assert_array_equal(llm, per_sim)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(tsync, ls["T_sync"])
    assert np.all(rep.results()["T_ooo"] <= tsync + (w.Q * w.steps if w.Q else 0))
    rep.close()


@pytest.mark.parametrize("Q", [0, 30_000])
def test_graph_metric_replay_vs_oracle(Q):
    """NEXT #4 variant, graph-distance dependencies: agents on the nodes of a
    600-node small-world graph, hop metric, the graph walk.  Every round's log (ids in
    priority order + labels) of the multi-kernel rounds, and the persistent kernel's
    final state, equal the oracle's replay; the outcome equals lock-step."""
    w = amgen.config("G1", steps=150)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, policy=3, graph=w.graph)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, graph_dist=w.gdist)
    r = O.replay(p, sy, w.x, w.y, Q=Q, log_rounds=10**6, log_entries=len(w.x) * w.steps + 10, check=True)
    assert r["violations"] == 0
    rep = Replay.from_workload(w, lm, quantum_us=Q)
    glogs = _gpu_logged(rep, 1, len(w.x))
    ologs = _split_oracle_log(r, 1)
    assert len(glogs[0]) == len(ologs[0])
    for (gi, gl), (oi, ol) in zip(glogs[0], ologs[0]):
        np.testing.assert_array_equal(gi, oi)
        np.testing.assert_array_equal(gl, ol)
    res = rep.results()
    for k in ("T_ooo", "rounds", "x", "traj"):
        np.testing.assert_array_equal(res[k], r[k], err_msg=k)
    rep.close()
    rep = Replay.from_workload(w, lm, quantum_us=Q)   # the persistent per-simulation kernel
    rep.run_to_end(chunk=4096)
    res = rep.results()
    for k in ("T_ooo", "rounds", "x", "traj"):
        np.testing.assert_array_equal(res[k], r[k], err_msg=k)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    rep.close()


def test_graph_metric_round_vs_oracle():
    """One round on random states of the graph (RUNNING / DONE mixes, a spread of steps)."""
    from paper_2411_03519_b200 import Tracker
    off, adj = amgen.social_graph(600, 4, 0.02, seed=5)
    gd = amgen.graph_distances(off, adj)
    rng = np.random.default_rng(4)
    n = 800
    x = rng.integers(0, 600, n).astype(np.int32)
    y = np.zeros(n, np.int32)
    s = rng.integers(0, 8, n).astype(np.int32)
    st = (rng.random(n) < 0.2).astype(np.uint8)
    st[rng.random(n) < 0.05] = O.DONE
    p = O.params(600, 1, 2, 1, graph_dist=gd)
    ref = O.round_(p, x, y, s, st.copy())
    tr = Tracker(600, 1, 2, 1, n, metric="graph",
                 graph_dist=torch.as_tensor(gd.view(np.int16)), device="cuda")
    dev = torch.device("cuda")
    tr.set_state(torch.as_tensor(np.stack([x, y], 1), dtype=torch.int32, device=dev), torch.as_tensor(s, device=dev),
                 torch.as_tensor(st, device=dev))
    mask, order = tr.ready()
    labels = tr.clusters()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(mask.cpu().numpy(), ref["mask"])
    np.testing.assert_array_equal(order.cpu().numpy(), ref["order"])
    np.testing.assert_array_equal(labels.cpu().numpy(), ref["label"])
    tr.close()
