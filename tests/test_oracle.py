"""Pins for the CPU oracle (oracle/oracle.c) -- against the paper and the mathematics,
never against the CUDA path.  All run on CPU (``-m "not gpu"``)."""
import numpy as np
import pytest
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components
from scipy.spatial import cKDTree

import amgen
import oracle as O
from golden_io import load_vectors

VECTORS = load_vectors()


def _params(v, n):
    return O.params(1 << 12, 1 << 12, v["r_p"], v["v"], v["target"],
                    O.LINF if v["metric"] == "LINF" else O.L2, v["n_sims"])


@pytest.mark.parametrize("vec", VECTORS, ids=[v["name"] for v in VECTORS])
def test_hand_vectors(vec):
    """Hand-worked vectors (tests/golden/tracker_vectors.txt, each with its citation)."""
    p = _params(vec, len(vec["x"]))
    st = vec["status"].copy()
    r = O.round_(p, vec["x"], vec["y"], vec["step"], st, peek=False)
    np.testing.assert_array_equal(r["blocked"], vec["blocked"])
    np.testing.assert_array_equal(r["label"], vec["labels"])
    np.testing.assert_array_equal(r["mask"], vec["mask"])
    np.testing.assert_array_equal(r["order"], vec["order"])
    # dispatch: exactly the ready agents became RUNNING (Q12)
    exp = vec["status"].copy()
    exp[vec["mask"] == 1] = O.RUNNING
    np.testing.assert_array_equal(st, exp)
    # peek leaves the status alone and yields the same outputs
    st2 = vec["status"].copy()
    r2 = O.round_(p, vec["x"], vec["y"], vec["step"], st2, peek=True)
    np.testing.assert_array_equal(st2, vec["status"])
    np.testing.assert_array_equal(r2["order"], vec["order"])


def test_v10_two_round_protocol():
    """V10a -> commit of agent 0 -> V10b through the update protocol (Alg. 3 l.11)."""
    p = O.params(64, 64, 4, 1)
    s = O.State(p, 2)
    assert s.update([0, 6], [0, 0], [2, 3]) == O.OK
    r = s.round()                      # both ready? agent 1 is blocked by agent 0 (d=6, delta 1)
    assert list(r["order"]) == [0] and r["blocked"][1] == 1
    assert s.status[0] == O.RUNNING
    # agent 0 commits step 2 -> 3 moving to (1,0)
    assert s.update([1, 6], [0, 0], [3, 3]) == O.OK
    r = s.round()
    assert list(r["label"]) == [0, 0] and list(r["order"]) == [0, 1]


def test_splitmix64_published_values():
    """mix64 = splitmix64's output function: seed 0 yields 0xE220A8397B1DCDAF then
    0x6E789E6AA1B965F4 (Vigna's reference splitmix64.c)."""
    assert O.mix64(0) == 0xE220A8397B1DCDAF
    assert O.mix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def _kd_blocked(p, x, y, s, st, metric):
    """Independent: per step-gap layer, a k-d tree ball query (library routine)."""
    n = len(x)
    act = st != O.DONE
    pts = np.stack([x, y], 1).astype(np.float64)
    out = np.zeros(n, np.uint8)
    pnorm = np.inf if metric == O.LINF else 2
    for sb in np.unique(s[act]):
        layer = np.nonzero(act & (s == sb))[0]
        tree = cKDTree(pts[layer])
        for i in np.nonzero(act & (s > sb))[0]:
            R = (int(s[i]) - int(sb) + 1) * p.v + p.r_p
            # integer coordinates: d <= R  <=>  d < R + 1/(4R+4)
            hits = tree.query_ball_point(pts[i], R + 0.25 / (R + 1), p=pnorm)
            if hits:
                out[i] = 1
    return out


def _cc_labels(p, x, y, s, st, metric):
    """Independent: connected components (scipy.sparse.csgraph) of the coupling graph."""
    n = len(x)
    act = st != O.DONE
    pts = np.stack([x, y], 1).astype(np.float64)
    R = p.r_p + p.v
    rows, cols = [], []
    pnorm = np.inf if metric == O.LINF else 2
    tree = cKDTree(pts)
    for i, j in tree.query_pairs(R + 0.25 / (R + 1), p=pnorm):
        if act[i] and act[j] and s[i] == s[j]:
            rows.append(i)
            cols.append(j)
    g = coo_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
    _, comp = connected_components(g, directed=False)
    lab = np.full(n, -1, np.int32)
    for c in np.unique(comp):
        mem = np.nonzero(comp == c)[0]
        lab[mem] = mem.min()
    lab[~act] = -1
    return lab


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("metric", [O.L2, O.LINF])
def test_round_vs_library_routines(seed, metric):
    """blocked == k-d tree ball queries; labels == scipy connected components;
    mask/order from their definitions (Q9)."""
    n = 600
    x, y, s, st = amgen.random_state(n, 90, 90, seed, max_step=5, p_running=0.1)
    st[np.random.default_rng(seed).random(n) < 0.05] = O.DONE
    p = O.params(90, 90, 4, 1 + seed % 2, 0, metric)
    st0 = st.copy()
    r = O.round_(p, x, y, s, st, peek=True)
    np.testing.assert_array_equal(r["blocked"], _kd_blocked(p, x, y, s, st0, metric))
    lab = _cc_labels(p, x, y, s, st0, metric)
    np.testing.assert_array_equal(r["label"], lab)
    bad = {}
    for i in range(n):
        if st0[i] != O.DONE:
            bad[lab[i]] = bad.get(lab[i], False) or bool(r["blocked"][i]) or st0[i] == O.RUNNING
    mask = np.array([st0[i] == O.IDLE and not bad[lab[i]] for i in range(n)], np.uint8)
    np.testing.assert_array_equal(r["mask"], mask)
    ids = np.nonzero(mask)[0]
    exp = sorted(ids, key=lambda i: (s[i], lab[i], i))
    np.testing.assert_array_equal(r["order"], exp)


@pytest.mark.parametrize("seed", range(3))
def test_sampled_round_equals_full_round(seed):
    n = 400
    x, y, s, st = amgen.random_state(n, 70, 70, 100 + seed, max_step=3, p_running=0.2)
    p = O.params(70, 70, 4, 1)
    r = O.round_(p, x, y, s, st.copy(), peek=True)
    sample = np.arange(0, n, 7)
    q = O.round_sampled(p, x, y, s, st, sample)
    np.testing.assert_array_equal(q["blocked"], r["blocked"][sample])
    np.testing.assert_array_equal(q["label"], r["label"][sample])
    np.testing.assert_array_equal(q["mask"], r["mask"][sample])


def test_update_rejections():
    """I9: corrupt commits are rejected with the right code, all-or-nothing."""
    p = O.params(32, 32, 4, 1, target=5)
    s = O.State(p, 3)
    assert s.update([1, 10, 20], [1, 10, 20], [0, 0, 0]) == O.OK
    assert s.update([40, 10, 20], [1, 10, 20], [0, 0, 0]) == O.E_BOUNDS
    assert s.update([2, 10, 20], [1, 10, 20], [0, 0, 0]) == O.E_PROTOCOL   # IDLE agent moved
    assert s.update([1, 10, 20], [1, 10, 20], [1, 0, 0]) == O.E_PROTOCOL   # IDLE agent stepped
    r = s.round()
    assert list(r["order"]) == [0, 1, 2]
    assert s.update([1, 10, 20], [1, 10, 20], [2, 0, 0]) == O.E_PROTOCOL   # +2
    assert s.update([3, 10, 20], [1, 10, 20], [1, 0, 0]) == O.E_VELOCITY   # |dp| = 2 > v
    assert list(s.x) == [1, 10, 20] and list(s.step) == [0, 0, 0]        # nothing applied
    assert s.update([2, 10, 20], [1, 10, 20], [1, 0, 0]) == O.OK
    assert list(s.status) == [O.IDLE, O.RUNNING, O.RUNNING]


def test_done_at_target():
    p = O.params(32, 32, 4, 1, target=1)
    s = O.State(p, 2)
    assert s.update([1, 30], [1, 30], [0, 1]) == O.OK
    assert list(s.status) == [O.IDLE, O.DONE]
    r = s.round()
    assert list(r["label"]) == [0, -1] and list(r["order"]) == [0]
    assert s.update([1, 30], [2, 30], [1, 1]) == O.OK
    assert list(s.status) == [O.DONE, O.DONE]


# ------------------------------------------------------------------ driver closed forms
def _stay_synth(dur):
    lm = amgen.latency_model()
    return O.SynthTables.from_model(lm, dur_table=np.asarray(dur, np.int64), policy=1)


@pytest.mark.parametrize("name,x1,T,L0,L1,T_ooo,T_sync,rounds", [
    ("D1", 7, 2, [10, 1], [1, 10], 11, 20, 3),   # A1 runs ahead: d=7 > R_b(1)=6
    ("D2", 6, 2, [10, 1], [1, 10], 20, 20, 4),   # A1 blocked at delta 1 until t=10
    ("D3", 5, 2, [10, 1], [1, 10], 20, 20, 2),   # coupled pair = lock-step cluster
    ("D5", 7, 3, [1, 1, 1], [10, 10, 10], 30, 30, 6),  # delta 2 blocking (d=7=R_b(2))
])
def test_driver_closed_forms(name, x1, T, L0, L1, T_ooo, T_sync, rounds):
    """SURVEY 4.4, worked by hand from P:160/P:406 and Alg. 3 with exact events."""
    p = O.params(64, 8, 4, 1, target=T)
    sy = _stay_synth([L0, L1])
    r = O.replay(p, sy, [0, x1], [0, 0], log_rounds=100, log_entries=100, check=True)
    assert int(r["T_ooo"][0]) == T_ooo
    assert int(r["rounds"][0]) == rounds
    assert r["violations"] == 0
    ls = O.lockstep(p, sy, [0, x1], [0, 0], T)
    assert int(ls["T_sync"][0]) == T_sync


def test_driver_d1_log():
    """D1 round log: t=0 both ready, t=1 A1 again, t=10 A0."""
    p = O.params(64, 8, 4, 1, target=2)
    sy = _stay_synth([[10, 1], [1, 10]])
    r = O.replay(p, sy, [0, 7], [0, 0], log_rounds=10, log_entries=10)
    assert list(r["log_t"]) == [0, 1, 10]
    assert list(r["log_nready"]) == [2, 1, 1]
    assert list(r["log_id"]) == [0, 1, 1, 0]


def test_driver_d4_isolated():
    """D4: pairwise far-apart agents: T_ooo = max_i sum_s L, T_sync = sum_s max_i L."""
    rng = np.random.default_rng(7)
    n, T = 6, 5
    L = rng.integers(1, 50, size=(n, T))
    x = np.arange(n) * 40
    p = O.params(400, 4, 4, 1, target=T)
    sy = _stay_synth(L)
    r = O.replay(p, sy, x, np.zeros(n), check=True)
    assert int(r["T_ooo"][0]) == int(L.sum(1).max())
    ls = O.lockstep(p, sy, x, np.zeros(n), T)
    assert int(ls["T_sync"][0]) == int(L.max(0).sum())


@pytest.mark.parametrize("cfg,steps,Q", [("C1", 200, 0), ("C1", 120, 20_000)])
def test_ooo_equals_lockstep(cfg, steps, Q):
    """I4 (P:27 'without affecting the simulation's outcome'), I1/I2 checked at
    every dispatch/commit, I6 time bounds."""
    w = amgen.config(cfg, steps=steps)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    r = O.replay(p, sy, w.x, w.y, Q=Q, check=True)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert r["violations"] == 0
    np.testing.assert_array_equal(r["x"], ls["x"])
    np.testing.assert_array_equal(r["y"], ls["y"])
    np.testing.assert_array_equal(r["traj"], ls["traj"])
    durs = np.array([[O.duration(sy, i, s) for s in range(w.steps)] for i in range(len(w.x))])
    lower = durs.sum(1).max()
    assert lower <= r["T_ooo"][0] <= ls["T_sync"][0] + (Q * w.steps if Q else 0)
    assert ls["T_sync"][0] == durs.max(0).sum()
    if Q == 0:
        assert r["T_ooo"][0] <= ls["T_sync"][0]
    assert r["max_spread"] > 3          # the replay really ran out of order


def test_ooo_equals_lockstep_batched():
    """Batched independent sims (config 3 shape) replay == per-sim lock-step."""
    w = amgen.config("C3", steps=60, n=6)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    r = O.replay(p, sy, w.x, w.y, check=True)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert r["violations"] == 0
    np.testing.assert_array_equal(r["traj"], ls["traj"])
    assert np.all(r["T_ooo"] <= ls["T_sync"])


def test_degenerate_huge_radius_is_lockstep():
    """I7: r_p >= map diagonal => one cluster every round => OoO == parallel-sync."""
    w = amgen.config("C1", steps=30)
    lm = amgen.latency_model()
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, 200, 1, target=w.steps)
    r = O.replay(p, sy, w.x, w.y, log_rounds=1000, log_entries=10**5)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert r["T_ooo"][0] == ls["T_sync"][0]
    assert int(r["rounds"][0]) == w.steps
    assert np.all(r["log_nready"] == 25)
    assert np.all(r["log_label"] == 0)


def test_duration_table_statistics():
    """Latency model sanity (Q16): E[K] of the profiles and the LAT quantile table."""
    lat = amgen.lat_table()
    assert lat[511] < 600_000 < lat[512]
    assert np.all(np.diff(lat.astype(np.int64)) >= 0)
    lm = amgen.latency_model("fullday")
    sy = O.SynthTables.from_model(lm)
    d = np.array([O.duration(sy, i, s) for i in range(40) for s in range(100)])
    k_mean = ((d - amgen.BASE_US) > 0).mean()
    assert 0.07 < k_mean < 0.17         # P(K>0) = 0.12 for the full-day profile


# ------------------------------------------------------------------ finite capacity (NEXT #2)
def test_capacity_one_is_sequential():
    """K = 1 with pairwise far-apart (never coupled, never blocked) agents, exact events:
    one agent-step in service at a time, back to back -> T_ooo = sum of all durations."""
    rng = np.random.default_rng(11)
    n, T = 5, 4
    L = rng.integers(1, 50, size=(n, T))
    p = O.params(400, 4, 4, 1, target=T)
    sy = _stay_synth(L)
    for prio in (True, False):
        r = O.replay(p, sy, np.arange(n) * 40, np.zeros(n), capacity=1, priority=prio, check=True)
        assert int(r["T_ooo"][0]) == int(L.sum())
        assert r["violations"] == 0


def test_capacity_by_hand():
    """Worked by hand (exact events, far-apart agents, keys (step << 32) | label).
    K = 1, A0 = [3, 3], A1 = [1, 2]: t=0 A0 runs [0,3); t=3 A1 (step 0) before A0
    (step 1) [3,4); A0 [4,7); A1 [7,9) -> T = 9.
    K = 2, A0 = [1, 1], A1 = [10, 1], A2 = [1, 1]: t=0 A0 [0,1) and A1 [0,10), A2 waits;
    t=1 A2 (step 0) before A0 (step 1) [1,2); t=2 A0 [2,3); t=3 A2 [3,4); t=10 A1 [10,11)
    -> T = 11.  FIFO keys (round << 32) | label give the same orders here."""
    p = O.params(400, 4, 4, 1, target=2)
    for prio in (True, False):
        r = O.replay(p, _stay_synth([[3, 3], [1, 2]]), [0, 40], [0, 0], capacity=1, priority=prio)
        assert int(r["T_ooo"][0]) == 9
        r = O.replay(p, _stay_synth([[1, 1], [10, 1], [1, 1]]), [0, 40, 80], [0, 0, 0], capacity=2, priority=prio)
        assert int(r["T_ooo"][0]) == 11


@pytest.mark.parametrize("K", [1, 4, 16])
def test_capacity_keeps_the_outcome(K):
    """I4 with finite capacity: the schedule changes, the outcome does not; every
    agent's steps are sequential (T_ooo >= max_i sum_s L_is); with every cluster within
    the capacity (C1 clusters have <= 3 members) work conservation gives
    T_ooo >= sum of durations / K; K >= n equals infinite capacity bit for bit."""
    w = amgen.config("C1", steps=60)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    durs = np.array([[O.duration(sy, i, s) for s in range(w.steps)] for i in range(len(w.x))])
    for prio in (True, False):
        r = O.replay(p, sy, w.x, w.y, capacity=K, priority=prio, check=True)
        assert r["violations"] == 0
        np.testing.assert_array_equal(r["traj"], ls["traj"])
        assert r["T_ooo"][0] >= durs.sum(1).max()
        if K >= 3:
            assert r["T_ooo"][0] * K >= durs.sum()
    inf = O.replay(p, sy, w.x, w.y)
    big = O.replay(p, sy, w.x, w.y, capacity=len(w.x))
    for k in ("T_ooo", "rounds", "traj"):
        np.testing.assert_array_equal(inf[k], big[k])


def test_linf_eight_connected_walk_keeps_the_outcome():
    """NEXT #4 variant: L-infinity metric with the 8-connected walk (policy 2; a diagonal
    move is within v = 1 under L-infinity).  Diagonal moves happen, the OoO replay keeps
    the validity condition and ends exactly where lock-step ends."""
    w = amgen.config("C1", steps=120)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall, policy=2)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, metric=O.LINF)
    one = O.lockstep(O.params(w.map_w, w.map_h, w.r_p, w.v, target=1, metric=O.LINF), sy, w.x, w.y, 1)
    dx, dy = one["x"] - w.x, one["y"] - w.y
    assert np.any((dx != 0) & (dy != 0)), "some first move is diagonal"
    assert np.all(np.maximum(np.abs(dx), np.abs(dy)) <= 1)
    r = O.replay(p, sy, w.x, w.y, check=True)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert r["violations"] == 0
    np.testing.assert_array_equal(r["traj"], ls["traj"])


def test_exclusive_tiles_keep_the_outcome():
    """NEXT #4 variant: exclusive tiles (P:182 bathroom example; Alg. 3 l.20
    resolve_conflict_and_commit).  Lock-step resolves over the whole simulation, the
    out-of-order replay per cluster; the outcome is the same (P:27 + the cluster-locality
    argument in oracle.c), no two agents ever share a tile (checked after every step of
    a crowded run), and the rule does change the outcome against co-occupancy."""
    w = amgen.config("C1", steps=80)
    lm = amgen.latency_model(w.profile)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    ex = O.SynthTables.from_model(lm, wall=w.wall, conflict=1)
    co = O.SynthTables.from_model(lm, wall=w.wall, conflict=0)
    r = O.replay(p, ex, w.x, w.y, check=True)
    ls = O.lockstep(p, ex, w.x, w.y, w.steps)
    assert r["violations"] == 0
    np.testing.assert_array_equal(r["traj"], ls["traj"])
    assert not np.array_equal(ls["traj"], O.lockstep(p, co, w.x, w.y, w.steps)["traj"])
    # crowded: 60 agents in a 12 x 12 open room, every step's positions distinct
    rng = np.random.default_rng(5)
    cells = rng.choice(144, 60, replace=False)
    x0, y0 = (cells % 12).astype(np.int32), (cells // 12).astype(np.int32)
    lm0 = amgen.latency_model()
    ex0 = O.SynthTables.from_model(lm0, conflict=1)
    co0 = O.SynthTables.from_model(lm0, conflict=0)
    shared = 0
    for T in range(1, 25):
        pT = O.params(12, 12, 4, 1, target=T)
        a = O.lockstep(pT, ex0, x0, y0, T)
        assert len(set(zip(a["x"].tolist(), a["y"].tolist()))) == 60, T
        b = O.lockstep(pT, co0, x0, y0, T)
        shared += 60 - len(set(zip(b["x"].tolist(), b["y"].tolist())))
    assert shared > 0, "co-occupancy happens without the rule"
    pT = O.params(12, 12, 4, 1, target=24)
    r = O.replay(pT, ex0, x0, y0, check=True)
    np.testing.assert_array_equal(r["traj"], O.lockstep(pT, ex0, x0, y0, 24)["traj"])
