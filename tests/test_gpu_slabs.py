"""S7 / S8 across spatial slabs (include/am_slab.h), run as virtual slabs on one GPU
(LoopbackWorld: the same library calls as the NCCL run, the exchanges are device copies).

* one distributed round on random and banded states equals the oracle's single round bit
  for bit: ready mask, cluster labels of every agent, and the global priority order (the
  ranks' orders merged), for G = 1 .. 16 slabs including multi-hop windows;
* the distributed REPLAY (incremental window trackers, deltas, migration across slab
  edges, arrivals / departures, cross-slab cluster completion times, the global event
  clock, re-windowing as the step spread grows) equals the oracle's replay round by round
  (every round's dispatched ids in priority order and their labels) and in its final
  state (positions, trajectory hashes, T_ooo, rounds) on C1, C2 and a C4-shaped map at
  G = 2 / 4 / 8;
* with stale-halo rounds (NEXT #3: a sync round every P rounds, the rounds between
  decided against the last exchange's ghosts) the replay equals the oracle's
  orc_replay_stale round by round and in its final state, and a long C4-shaped run
  (re-windows, migration) ends in the lock-step state."""
import numpy as np
import pytest
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import slabs

pytestmark = pytest.mark.gpu


def _world(w, lm, G, steps0=None, status0=None, **kw):   # kw: check_rounds, stale_rounds
    sy = slabs.Synth(lm, wall=w.wall)
    return slabs.LoopbackWorld(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, sy, w.Q, G, steps0=steps0,
                               status0=status0, **kw)


def _round_vs_oracle(x, y, s, st, W, H, G, r_p=4, v=1, metric="l2", check_rounds=4):
    n = len(x)
    lm = amgen.latency_model()
    w = amgen.Workload("rand", W, H, None, x, y, 1, 1000, r_p=r_p, v=v)
    sy = slabs.Synth(lm)
    wd = slabs.LoopbackWorld(W, H, r_p, v, x, y, 1000, sy, 0, G, steps0=s, status0=st, metric=metric,
                             check_rounds=check_rounds)
    log = []
    wd.round(log)
    outs = log[0]
    p = O.params(W, H, r_p, v, 1000, O.LINF if metric == "linf" else O.L2)
    ref = O.round_(p, x, y, s, st.copy(), peek=True)
    mask = np.zeros(n, np.uint8)
    lab = np.full(n, -7, np.int32)
    for o in outs:
        g = o["gid"].cpu().numpy()
        mask[g] = o["ready"].cpu().numpy()
        lab[g] = o["label"].cpu().numpy()
    np.testing.assert_array_equal(mask, ref["mask"])
    np.testing.assert_array_equal(lab, ref["label"])
    order, olab = slabs.merged_order(outs)
    np.testing.assert_array_equal(order, ref["order"])
    np.testing.assert_array_equal(olab, ref["label"][ref["order"]])
    wd.close()
    del w


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_random_state_round(G):
    n, m = 12000, 900
    x, y, s, st = amgen.random_state(n, m, m, 40 + G, max_step=6, p_running=0.3)
    st[np.random.default_rng(G).random(n) < 0.05] = O.DONE
    s[st == O.DONE] = 1000
    _round_vs_oracle(x, y, s, st, m, m, G)


@pytest.mark.parametrize("G", [2, 8, 16])
def test_banded_large_spread_multihop(G):
    """Spread ~60 steps: the window reaches past the neighbouring slabs for G = 16."""
    n, w = 10000, 1500
    x, y, s, st = amgen.banded_state(n, w, 480, 3, p_running=0.3)
    x, y = y.copy(), x.copy()          # the step gradient across the slabs
    _round_vs_oracle(x, y, s, st, 480, w, G)


def test_linf_and_coupled_chain_across_all_slabs():
    """A chain of coupled agents crossing every slab boundary: one global cluster."""
    H, G = 400, 8
    ys = np.arange(0, H, 5, dtype=np.int32)
    x = np.full(len(ys), 10, np.int32)
    s = np.zeros(len(ys), np.int32)
    st = np.zeros(len(ys), np.uint8)
    st[len(ys) // 2] = O.RUNNING        # poisons the whole chain
    _round_vs_oracle(x, ys, s, st, 64, H, G)
    _round_vs_oracle(x, ys, s, st, 64, H, G, metric="linf")


def _oracle_logs(r):
    logs, k = [], 0
    for nr in r["log_nready"]:
        if nr:
            logs.append((r["log_id"][k:k + nr], r["log_label"][k:k + nr]))
        k += nr
    return logs


def _replay_logged(wd, max_rounds=10**6):
    logs = []
    for k in range(max_rounds):
        log = []
        wd.round(log)
        ids, lab = slabs.merged_order(log[0])
        if len(ids):
            logs.append((ids, lab))
        if (k + 1) % wd.K == 0 and wd.check():
            break
    return logs


@pytest.mark.parametrize("name,steps,n,G", [
    ("C1", 300, None, 2), ("C1", 300, None, 4),
    ("C2", 25, None, 2), ("C2", 25, None, 4), ("C2", 25, None, 8),
    ("C4", 12, 2000, 2), ("C4", 12, 2000, 8),
])
def test_slab_replay_round_logs_vs_oracle(name, steps, n, G):
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    r = O.replay(p, sy, w.x, w.y, Q=w.Q, log_rounds=10**6, log_entries=len(w.x) * w.steps + 10)
    assert r["log_complete"]
    wd = _world(w, lm, G, check_rounds=4)
    glogs = _replay_logged(wd)
    ologs = _oracle_logs(r)
    assert len(glogs) == len(ologs), (len(glogs), len(ologs))
    for k, ((gi, gl), (oi, ol)) in enumerate(zip(glogs, ologs)):
        np.testing.assert_array_equal(gi, oi, err_msg=f"round {k}")
        np.testing.assert_array_equal(gl, ol, err_msg=f"round {k}")
    res = wd.results()
    np.testing.assert_array_equal(res["x"], r["x"])
    np.testing.assert_array_equal(res["y"], r["y"])
    np.testing.assert_array_equal(res["traj"], r["traj"])
    assert res["T_ooo"] == int(r["T_ooo"][0])
    assert res["rounds"] == int(r["rounds"][0])
    assert res["dispatched"] == len(w.x) * w.steps
    assert np.all(res["steps"] == w.steps)
    wd.close()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_slab_replay_c4_shape_final_state_vs_lockstep(G):
    """20k agents at C4 density over 120 steps (re-windows as the spread grows, agents
    migrate across slab edges): the final state equals the oracle's lock-step run
    and the single-GPU replay's completion time and round count."""
    from paper_2411_03519_b200 import Replay
    w = amgen.config("C4", steps=120, n=20000)
    lm = amgen.latency_model(w.profile)
    wd = _world(w, lm, G, check_rounds=8)
    wd.run(10**6)
    res = wd.results()
    assert wd.rewindows >= 1
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    ls = O.lockstep_grid(p, O.SynthTables.from_model(lm), w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["x"], ls["x"])
    np.testing.assert_array_equal(res["y"], ls["y"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    one = Replay.from_workload(w, lm)
    one.run_to_end(chunk=512)
    r1 = one.results()
    assert res["T_ooo"] == int(r1["T_ooo"][0]) and res["rounds"] == int(r1["rounds"][0])
    one.close()
    wd.close()


@pytest.mark.parametrize("G", [2, 4])
def test_slab_replay_tall_map_final_state_vs_lockstep(G):
    """A map taller than one tracker's 32768 rows (128 x 40000, 20k agents at C5 density in
    hotspots, 60 steps): split into G slabs whose windows fit 32768 rows (each window keeps
    its own row frame), the distributed replay ends in the oracle's lock-step state;
    a single slab cannot hold the map."""
    x, y = amgen.hotspot_positions(20000, 128, 40000, seed=3)
    w = amgen.Workload("tall", 128, 40000, None, x, y, 1, 60, profile="busy", Q=50_000)
    lm = amgen.latency_model(w.profile)
    with pytest.raises(ValueError):
        _world(w, lm, 1)
    wd = _world(w, lm, G, check_rounds=8)
    wd.run(10**6)
    res = wd.results()
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    ls = O.lockstep_grid(p, O.SynthTables.from_model(lm), w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["x"], ls["x"])
    np.testing.assert_array_equal(res["y"], ls["y"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert np.all(res["steps"] == w.steps)
    assert int(res["y"].max()) > 32767
    wd.close()


@pytest.mark.parametrize("name,steps,n,G,P", [
    ("C1", 300, None, 2, 2), ("C1", 300, None, 4, 4),
    ("C2", 8, None, 4, 2), ("C2", 8, None, 8, 4),
    ("C4", 6, 2000, 4, 4),
])
def test_stale_slab_replay_round_logs_vs_oracle(name, steps, n, G, P):
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    r = O.replay_stale(p, sy, w.x, w.y, G=G, P=P, Q=w.Q, log_rounds=10**6, log_entries=len(w.x) * w.steps + 10)
    assert r["log_complete"]
    wd = _world(w, lm, G, check_rounds=2 * P, stale_rounds=P)
    glogs = _replay_logged(wd)
    ologs = _oracle_logs(r)
    assert len(glogs) == len(ologs), (len(glogs), len(ologs))
    for k, ((gi, gl), (oi, ol)) in enumerate(zip(glogs, ologs)):
        np.testing.assert_array_equal(gi, oi, err_msg=f"round {k}")
        np.testing.assert_array_equal(gl, ol, err_msg=f"round {k}")
    res = wd.results()
    np.testing.assert_array_equal(res["x"], r["x"])
    np.testing.assert_array_equal(res["y"], r["y"])
    np.testing.assert_array_equal(res["traj"], r["traj"])
    assert res["T_ooo"] == int(r["T_ooo"][0])
    assert res["rounds"] == int(r["rounds"][0])
    assert res["dispatched"] == len(w.x) * w.steps
    wd.close()


@pytest.mark.parametrize("G,P", [(4, 2), (8, 4)])
def test_stale_slab_replay_c4_shape_final_state_vs_lockstep(G, P):
    """20k agents at C4 density over 120 steps with stale-halo rounds: re-windows at
    exchanges, agents handed over (RUNNING ones with their completion times) -- the final
    state is lock-step's."""
    w = amgen.config("C4", steps=120, n=20000)
    lm = amgen.latency_model(w.profile)
    wd = _world(w, lm, G, check_rounds=2 * P, stale_rounds=P)
    wd.run(10**6)
    res = wd.results()
    assert wd.rewindows >= 1
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    ls = O.lockstep_grid(p, O.SynthTables.from_model(lm), w.x, w.y, w.steps)
    np.testing.assert_array_equal(res["x"], ls["x"])
    np.testing.assert_array_equal(res["y"], ls["y"])
    np.testing.assert_array_equal(res["traj"], ls["traj"])
    assert res["dispatched"] == len(w.x) * w.steps
    wd.close()


def test_stale_period_must_divide_the_check_period():
    w = amgen.config("C1", steps=10)
    lm = amgen.latency_model(w.profile)
    with pytest.raises(ValueError):
        _world(w, lm, 2, check_rounds=6, stale_rounds=4)
