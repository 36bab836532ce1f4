"""Pins for the oracle functions the round-1 review found unpinned, and for the at-scale
oracle drivers (oracle/oracle_scale.c).  All CPU (``-m "not gpu"``); nothing here
touches the CUDA path.

* orc_validity_violations (the I2 checker, P:156 / App. A): exact counts on hand
  states at the strict boundary, for both metrics, and on states that do violate it.
* the synthetic driver model (the paper is silent, Q16): mix64 = the
  splitmix64 finaliser (Vigna's published outputs), key3, the perception digest, the
  random-walk move and the latency draw -- each against an independent pure-Python
  implementation of the c.4 definition (built on the pinned splitmix64), plus structural
  pins (which agents a digest includes, wall / off-map rejection, K = 0 -> BASE_US,
  the explicit-table path).
* the trajectory hash chained at every commit (lock-step, one agent).
* the at-scale drivers equal their plain counterparts of oracle.c element by element.
"""
import numpy as np
import pytest

import amgen
import oracle as O

M64 = (1 << 64) - 1


# ---------------------------------------------------------------- independent splitmix64
def py_mix64(z: int) -> int:
    """splitmix64 output function (Steele, Lea, Flood 2014; Vigna's splitmix64.c)."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def py_key3(s, a, b):
    return py_mix64((py_mix64((py_mix64((s + a) & M64) + b) & M64)))


def test_python_splitmix64_matches_published_stream():
    """Vigna's splitmix64 with state 0: the first outputs are 0xE220A8397B1DCDAF,
    0x6E789E6AA1B965F4, 0x06C45D188009454F (the state advances by the golden gamma)."""
    st = 0
    outs = []
    for _ in range(3):
        outs.append(py_mix64(st))
        st = (st + 0x9E3779B97F4A7C15) & M64
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("s,a,b", [(0, 0, 0), (3, 7, 11), (4, 2**31 + 5, 999), (M64, 1, M64)])
def test_key3_is_the_c4_chain(s, a, b):
    """key3(seed, a, b) = mix64(mix64(mix64(seed + a) + b))."""
    assert O.key3(s, a, b) == py_key3(s, a, b)
    # and the chain is order sensitive (a dropped or swapped term changes it)
    if a != b:
        assert O.key3(s, a, b) != O.key3(s, b, a)


# ---------------------------------------------------------------- validity (I2)
def test_validity_boundary_l2():
    """for Step_A != Step_B the pair is valid iff dist > r_p + (|dS| - 1) v.
    r_p = 4, v = 1: |dS| = 2 -> bound 5: d = 5 violates, d = 6 does not; |dS| = 1 ->
    bound 4: d = 4 violates, d = 5 does not; equal steps never violate (coupling)."""
    p = O.params(64, 64, 4, 1)
    assert O.validity_violations(p, [0, 5], [0, 0], [3, 1]) == 1
    assert O.validity_violations(p, [0, 6], [0, 0], [3, 1]) == 0
    assert O.validity_violations(p, [0, 4], [0, 0], [3, 2]) == 1
    assert O.validity_violations(p, [0, 5], [0, 0], [3, 2]) == 0
    # (0,1) and (0,2): |dS| = 1, d^2 = 25 > 16 valid; (1,2) co-located at equal steps -> 0
    assert O.validity_violations(p, [0, 3, 3], [0, 4, 4], [7, 6, 6]) == 0


def test_validity_exact_counts():
    """Exact violation counts of a hand state (r_p = 4, v = 1, L2):
    A0 (0,0,s0)  A1 (5,0,s1)  A2 (0,3,s2)  A3 (20,0,s0)
      A0-A1 |dS|=1 bound 4, d=5  -> valid
      A0-A2 |dS|=2 bound 5, d=3  -> violation
      A1-A2 |dS|=1 bound 4, d^2=34 (d~5.83) -> valid
      A0-A3 equal steps          -> never
      A1-A3 |dS|=1 bound 4, d=15 -> valid
      A2-A3 |dS|=2 bound 5, d^2=409 -> valid
    -> 1.  Moving A1 to (4,0): A0-A1 d=4 <= 4 -> +1, A1-A2 d=5 > 4 valid -> 2."""
    p = O.params(64, 64, 4, 1)
    x, y, s = [0, 5, 0, 20], [0, 0, 3, 0], [0, 1, 2, 0]
    assert O.validity_violations(p, x, y, s) == 1
    assert O.validity_violations(p, [0, 4, 0, 20], y, s) == 2
    # co-located at different steps: d = 0 <= any bound -> a violation
    assert O.validity_violations(p, [9, 9], [9, 9], [0, 50]) == 1
    assert O.validity_violations(p, [9, 9], [9, 9], [50, 50]) == 0
    # L-infinity: (4,4) at |dS| = 1: max = 4 <= 4 violates; under L2 d^2 = 32 > 16 does not
    assert O.validity_violations(O.params(64, 64, 4, 1, metric=O.LINF), [0, 4], [0, 4], [0, 1]) == 1
    assert O.validity_violations(p, [0, 4], [0, 4], [0, 1]) == 0
    # v = 0: the bound is r_p for every gap
    p0 = O.params(64, 64, 4, 0)
    assert O.validity_violations(p0, [0, 4], [0, 0], [0, 9]) == 1
    assert O.validity_violations(p0, [0, 5], [0, 0], [0, 9]) == 0
    # batched simulations: pairs across simulations never count
    pb = O.params(64, 64, 4, 1, n_sims=2)
    assert O.validity_violations(pb, [0, 0, 1, 1], [0, 0, 0, 0], [0, 5, 0, 5]) == 2
    assert O.validity_violations(pb, [0, 1, 0, 1], [0, 0, 0, 0], [0, 0, 5, 5]) == 0


def test_validity_counts_pairs_brute_force_small():
    """On tiny random states the count equals a pair enumeration written from P:156."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = 12
        x, y = rng.integers(0, 12, n), rng.integers(0, 12, n)
        s = rng.integers(0, 4, n)
        p = O.params(12, 12, 2, 1)
        cnt = 0
        for i in range(n):
            for j in range(i + 1, n):
                if s[i] == s[j]:
                    continue
                bound = 2 + (abs(int(s[i]) - int(s[j])) - 1) * 1
                d2 = (int(x[i]) - int(x[j])) ** 2 + (int(y[i]) - int(y[j])) ** 2
                cnt += not (d2 > bound * bound)
        assert O.validity_violations(p, x, y, s) == cnt


# ---------------------------------------------------------------- perception digest (c.4)
def py_digest(i, x, y, step, status, r_p, metric="l2"):
    d = 0
    for j in range(len(x)):
        if j == i or status[j] == O.DONE or step[j] != step[i]:
            continue
        dx, dy = int(x[j]) - int(x[i]), int(y[j]) - int(y[i])
        ok = (dx * dx + dy * dy <= r_p * r_p) if metric == "l2" else max(abs(dx), abs(dy)) <= r_p
        if ok:
            d = (d + py_mix64((j << 32) ^ ((dx & 0xFFFF) << 16) ^ (dy & 0xFFFF))) & M64
    return d


def test_digest_structure():
    """Which agents a digest includes (perception): same step, not DONE, not self,
    within radius_p inclusive -- an agent at exactly r_p counts, r_p + 1 does not."""
    p = O.params(64, 64, 4, 1)
    #            self  at r_p  r_p+1  other step  DONE   (3,4): d = 5 > 4   (0,-4)
    x = np.array([10, 14, 15, 11, 10, 13, 10], np.int32)
    y = np.array([10, 10, 10, 10, 11, 14, 6], np.int32)
    s = np.array([5, 5, 5, 4, 5, 5, 5], np.int32)
    st = np.array([0, 0, 0, 0, 2, 1, 0], np.uint8)
    dig = O.digest(p, x, y, s, st, 0)
    exp = (py_mix64((1 << 32) ^ (4 << 16) ^ 0) + py_mix64((6 << 32) ^ (0 << 16) ^ (0xFFFF & -4))) & M64
    assert dig == exp
    assert dig == py_digest(0, x, y, s, st, 4)
    # an empty perception digests to 0; a RUNNING same-step neighbour is perceived
    assert O.digest(p, [0, 30], [0, 30], [1, 1], np.zeros(2, np.uint8), 0) == 0
    assert O.digest(p, [0, 3], [0, 0], [1, 1], np.array([0, 1], np.uint8), 0) == py_mix64((1 << 32) ^ (3 << 16))


@pytest.mark.parametrize("seed", range(4))
def test_digest_random_states(seed):
    rng = np.random.default_rng(seed)
    n = 60
    x, y = rng.integers(0, 20, n).astype(np.int32), rng.integers(0, 20, n).astype(np.int32)
    s = rng.integers(0, 3, n).astype(np.int32)
    st = rng.integers(0, 3, n).astype(np.uint8)
    for metric, mname in ((O.L2, "l2"), (O.LINF, "linf")):
        p = O.params(20, 20, 4, 1, metric=metric)
        for i in range(0, n, 7):
            assert O.digest(p, x, y, s, st, i) == py_digest(i, x, y, s, st, 4, mname)
    # order independence: relabelling positions of the perceived set keeps the sum
    p = O.params(20, 20, 4, 1)
    perm = np.arange(n)
    assert O.digest(p, x[perm], y[perm], s[perm], st[perm], 3) == O.digest(p, x, y, s, st, 3)


# ---------------------------------------------------------------- policy (c.4)
MX = [0, 1, -1, 0, 0, 1, -1, 1, -1]
MY = [0, 0, 0, 1, -1, 1, 1, -1, -1]


def py_move(i, s, px, py, dig, policy_seed, W, H, wall=None, policy=0):
    h = py_mix64((py_key3(policy_seed, i, s) + dig) & M64)
    m = 0 if policy == 1 else (h % 9 if policy == 2 else h % 5)
    qx, qy = px + MX[m], py + MY[m]
    ok = 0 <= qx < W and 0 <= qy < H and not (wall is not None and wall[qy, qx])
    return (qx, qy) if ok else (px, py)


def test_policy_move_matches_definition():
    lm = amgen.latency_model()
    W, H = 16, 12
    wall = np.zeros((H, W), np.uint8)
    wall[5, :] = 1
    for policy in (0, 1, 2):
        sy = O.SynthTables.from_model(lm, wall=wall, policy=policy)
        p = O.params(W, H, 4, 1)
        seen = set()
        for i in range(40):
            for s in range(5):
                px, py = (i * 7) % W, (i * 3) % H
                if wall[py, px]:
                    continue
                dig = py_mix64(i * 1000 + s)
                got = O.policy_move(p, sy, i, s, px, py, dig)
                assert got == py_move(i, s, px, py, dig, lm.policy_seed, W, H, wall, policy)
                seen.add((got[0] - px, got[1] - py))
        if policy == 1:
            assert seen == {(0, 0)}
        elif policy == 0:
            assert seen == {(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)}
        else:
            assert len(seen) == 9


def test_policy_move_rejects_walls_and_off_map():
    """A move into a wall or off the map becomes stay (co-occupancy allowed, Q15)."""
    lm = amgen.latency_model()
    W, H = 3, 3
    wall = np.zeros((H, W), np.uint8)
    wall[1, 2] = 1
    sy = O.SynthTables.from_model(lm, wall=wall)
    p = O.params(W, H, 4, 1)
    hit = {"wall": 0, "off": 0}
    for i in range(200):
        # agent at (1, 1): +x hits the wall at (2, 1); agent at (0, 0): -x / -y leave the map
        h = py_mix64(py_key3(lm.policy_seed, i, 0))
        m = h % 5
        if m == 1:
            assert O.policy_move(p, sy, i, 0, 1, 1, 0) == (1, 1)
            hit["wall"] += 1
        if m in (2, 4):
            assert O.policy_move(p, sy, i, 0, 0, 0, 0) == (0, 0)
            hit["off"] += 1
    assert hit["wall"] > 5 and hit["off"] > 5


# ---------------------------------------------------------------- latency draw (c.4)
def py_duration(lm, i, s):
    u = py_key3(lm.lat_seed, i, s)
    hi = u >> 32
    m = 0
    while m < len(lm.vals) - 1 and not (hi < int(lm.cdf32[m])):
        m += 1
    K = int(lm.vals[m])
    d = lm.base_us
    for k in range(K):
        h = py_key3(lm.lat_seed ^ 0xC0FFEE, ((i << 20) ^ s) & M64, k)
        d += int(lm.lat[h >> 54])
    return d, K


def test_duration_matches_definition():
    lm = amgen.latency_model("busy")
    sy = O.SynthTables.from_model(lm)
    ks = set()
    for i in range(30):
        for s in range(30):
            d, K = py_duration(lm, i, s)
            assert O.duration(sy, i, s) == d
            ks.add(K)
            if K == 0:
                assert d == amgen.BASE_US     # no LLM call: the base cost only
    assert ks == {0, 1, 2, 3, 5}


def test_duration_explicit_table_path():
    lm = amgen.latency_model()
    tab = np.array([[7, 8, 9], [10, 11, 12]], np.int64)
    sy = O.SynthTables.from_model(lm, dur_table=tab)
    assert [O.duration(sy, i, s) for i in range(2) for s in range(3)] == [7, 8, 9, 10, 11, 12]


def test_trajectory_hash_chain():
    """traj = mix64(traj ^ (s << 32 | (u16)x << 16 | (u16)y)) after every committed step
    s = 1..T (one agent, stay policy -> the position is constant)."""
    lm = amgen.latency_model()
    sy = O.SynthTables.from_model(lm, policy=1)
    p = O.params(32, 32, 4, 1, target=3)
    r = O.lockstep(p, sy, [7], [9], 3)
    th = 0
    for s in range(1, 4):
        th = py_mix64(th ^ ((s << 32) | (7 << 16) | 9))
    assert int(r["traj"][0]) == th


# ---------------------------------------------------------------- at-scale drivers
@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("metric", [O.L2, O.LINF])
def test_round_mt_equals_round(seed, metric):
    n = 1500
    x, y, s, st = amgen.random_state(n, 120, 120, 50 + seed, max_step=6, p_running=0.2)
    st[np.random.default_rng(seed).random(n) < 0.05] = O.DONE
    p = O.params(120, 120, 4, 1 + seed % 2, 0, metric)
    a = O.round_(p, x, y, s, st.copy(), peek=False)
    st2 = st.copy()
    b = O.round_mt(p, x, y, s, st2, peek=False, threads=4)
    for k in ("blocked", "label", "mask", "order"):
        np.testing.assert_array_equal(a[k], b[k])
    exp = st.copy()
    exp[a["mask"] == 1] = O.RUNNING
    np.testing.assert_array_equal(st2, exp)
    lab = O.labels_steps(p, x, y, s, st, threads=3)
    np.testing.assert_array_equal(lab, a["label"])
    idx = np.arange(0, n, 5, dtype=np.int32)
    np.testing.assert_array_equal(O.blocked_list(p, x, y, s, st, idx, threads=3), a["blocked"][idx])
    smp = np.arange(1, n, 11, dtype=np.int32)
    r = O.round_at_scale(p, x, y, s, st, smp, threads=2)
    np.testing.assert_array_equal(r["label"], a["label"])
    np.testing.assert_array_equal(r["blocked"], a["blocked"][smp])
    np.testing.assert_array_equal(r["mask"], a["mask"][smp])


def test_round_mt_banded_valid_state():
    """A valid state with a large spread (far blocking at many gaps)."""
    x, y, s, st = amgen.banded_state(3000, 600, 300, 9, p_running=0.3)
    p = O.params(600, 300, 4, 1)
    a = O.round_(p, x, y, s, st.copy(), peek=True)
    b = O.round_mt(p, x, y, s, st.copy(), peek=True, threads=8)
    for k in ("blocked", "label", "mask", "order"):
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("name,steps,n", [("C1", 60, None), ("C2", 30, None), ("C4", 25, 3000)])
def test_lockstep_grid_equals_lockstep(name, steps, n):
    """The hash-grid perception changes nothing: positions, trajectory hashes and T_sync
    equal orc_lockstep's (walls on C1/C2; the open hotspot map of C4/C5 shrunk)."""
    w = amgen.config(name, steps=steps, n=n)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps)
    a = O.lockstep(p, sy, w.x, w.y, w.steps)
    b = O.lockstep_grid(p, sy, w.x, w.y, w.steps, threads=4)
    for k in ("x", "y", "traj", "T_sync"):
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("r_p,v,metric", [(0, 0, O.L2), (1, 1, O.L2), (6, 2, O.LINF)])
def test_lockstep_grid_radius_edge_cases(r_p, v, metric):
    """r_p = 0 (cell edge 1: only co-located agents are perceived), small and L-inf."""
    rng = np.random.default_rng(r_p + 10 * v)
    n, W = 400, 40
    x, y = rng.integers(0, W, n).astype(np.int32), rng.integers(0, W, n).astype(np.int32)
    lm = amgen.latency_model()
    sy = O.SynthTables.from_model(lm, policy=2 if metric == O.LINF else 0)
    p = O.params(W, W, r_p, v, target=12, metric=metric)
    a = O.lockstep(p, sy, x, y, 12)
    b = O.lockstep_grid(p, sy, x, y, 12, threads=3)
    for k in ("x", "y", "traj", "T_sync"):
        np.testing.assert_array_equal(a[k], b[k])


def test_replay_mt_equals_replay():
    """Concurrent simulations of a batch (C3 shape) give the sequential replay's results."""
    w = amgen.config("C3", steps=80, n=24)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    a = O.replay(p, sy, w.x, w.y)
    b = O.replay_mt(p, sy, w.x, w.y, threads=5)
    for k in ("x", "y", "traj", "T_ooo", "rounds"):
        np.testing.assert_array_equal(a[k], b[k])
    a = O.replay(p, sy, w.x, w.y, capacity=3, priority=False)
    b = O.replay_mt(p, sy, w.x, w.y, capacity=3, priority=False, threads=3)
    for k in ("traj", "T_ooo", "rounds"):
        np.testing.assert_array_equal(a[k], b[k])


def test_replay_sims_logged_equals_batched_log():
    """One simulation replayed alone logs exactly its part of the batched replay's log."""
    w = amgen.config("C3", steps=40, n=5)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, wall=w.wall)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, n_sims=w.n_sims)
    full = O.replay(p, sy, w.x, w.y, log_rounds=10**5, log_entries=10**5)
    one = O.replay_sims_logged(p, sy, w.x, w.y, [1, 3])
    k = 0
    per = {b: ([], [], []) for b in range(5)}
    for b, nr in zip(full["log_sim"], full["log_nready"]):
        per[b][0].append(nr)
        per[b][1].extend(full["log_id"][k:k + nr])
        per[b][2].extend(full["log_label"][k:k + nr])
        k += nr
    for b in (1, 3):
        np.testing.assert_array_equal(one[b]["log_nready"], per[b][0])
        np.testing.assert_array_equal(one[b]["log_id"], per[b][1])
        np.testing.assert_array_equal(one[b]["log_label"], per[b][2])
        assert one[b]["T_ooo"] == full["T_ooo"][b] and one[b]["rounds"] == full["rounds"][b]
        lo, hi = b * 125 // 5, (b + 1) * 125 // 5
        np.testing.assert_array_equal(one[b]["traj"], full["traj"][lo:hi])
