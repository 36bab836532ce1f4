"""GPU parity: the CUDA tracker (through the C ABI) vs the CPU oracle, element by element.
Bit-exact on every output (integer work): mask, order, labels, statuses."""
import numpy as np
import pytest
import torch

import amgen
import oracle as O
from golden_io import load_vectors
from paper_2411_03519_b200 import AmError, Tracker, _lib

pytestmark = pytest.mark.gpu
VECTORS = load_vectors()
PATHS = ["small", "binned"]


def _dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def _pos(x, y):
    return _dev(np.stack([np.asarray(x), np.asarray(y)], 1), torch.int32)


def _gpu_round(tr, x, y, s, st, peek=False):
    tr.set_state(_pos(x, y), _dev(s, torch.int32), _dev(st, torch.uint8))
    tr.set_flags(peek=peek)
    mask, order = tr.ready()
    labels = tr.clusters()
    torch.cuda.synchronize()
    return dict(mask=mask.cpu().numpy().copy(), order=order.cpu().numpy().copy(),
                label=labels.cpu().numpy().copy(), status=tr.status().cpu().numpy(),
                stats=tr.stats())


def _compare(g, r, st_after):
    np.testing.assert_array_equal(g["mask"], r["mask"])
    np.testing.assert_array_equal(g["label"], r["label"])
    np.testing.assert_array_equal(g["order"], r["order"])
    np.testing.assert_array_equal(g["status"], st_after)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("vec", VECTORS, ids=[v["name"] for v in VECTORS])
def test_hand_vectors(vec, path):
    n = len(vec["x"])
    if path == "binned" and vec["n_sims"] > 1:
        pytest.skip("binned path is single-simulation")
    tr = Tracker(64, 64, vec["r_p"], vec["v"], n, target=vec["target"], n_sims=vec["n_sims"],
                 metric=vec["metric"].lower(), force=path)
    g = _gpu_round(tr, vec["x"], vec["y"], vec["step"], vec["status"])
    exp_st = vec["status"].copy()
    exp_st[vec["mask"] == 1] = O.RUNNING
    np.testing.assert_array_equal(g["mask"], vec["mask"])
    np.testing.assert_array_equal(g["label"], vec["labels"])
    np.testing.assert_array_equal(g["order"], vec["order"])
    np.testing.assert_array_equal(g["status"], exp_st)


CASES = [
    # n, map, r_p, v, max_step, p_run, p_done, metric, seed
    (1, 16, 4, 1, 0, 0.0, 0.0, "l2", 0),
    (33, 40, 4, 1, 3, 0.2, 0.1, "l2", 1),
    (1000, 120, 4, 1, 4, 0.2, 0.05, "l2", 2),
    (1000, 120, 4, 2, 6, 0.1, 0.05, "linf", 3),
    (777, 90, 0, 0, 2, 0.1, 0.0, "l2", 4),
    (900, 300, 12, 3, 8, 0.3, 0.1, "l2", 5),
    (5000, 400, 4, 1, 5, 0.3, 0.05, "l2", 6),
    (20011, 1200, 4, 1, 6, 0.3, 0.05, "l2", 7),
    (20011, 700, 4, 1, 60, 0.3, 0.05, "l2", 8),
]


def _random_case(n, m, r_p, v, ms, pr, pd, seed, target):
    x, y, s, st = amgen.random_state(n, m, m, seed, max_step=ms, p_running=pr)
    rng = np.random.default_rng(seed + 1000)
    done = rng.random(n) < pd
    st[done] = O.DONE
    s[done] = target
    return x, y, s, st


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_m{c[1]}_rp{c[2]}_v{c[3]}_{c[7]}" for c in CASES])
def test_random_states_vs_oracle(case):
    n, m, r_p, v, ms, pr, pd, metric, seed = case
    target = ms + 1
    x, y, s, st = _random_case(n, m, r_p, v, ms, pr, pd, seed, target)
    p = O.params(m, m, r_p, v, target, O.LINF if metric == "linf" else O.L2)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o, peek=False)
    for path in PATHS:
        if path == "small" and n > 1024:
            continue
        tr = Tracker(m, m, r_p, v, n, target=target, metric=metric, force=path)
        g = _gpu_round(tr, x, y, s, st)
        _compare(g, r, st_o)
        assert g["stats"]["n_ready"] == len(r["order"])
        # determinism: the same round again gives the same bits
        g2 = _gpu_round(tr, x, y, s, st)
        _compare(g2, r, st_o)
        tr.close()


@pytest.mark.parametrize("case", CASES[5:], ids=[f"n{c[0]}_spread{c[4]}" for c in CASES[5:]])
def test_thread_scan_ablation_matches(case):
    """The one-thread-per-agent scan (AM_SCAN_THREAD, ablation baseline) gives the same bits."""
    n, m, r_p, v, ms, pr, pd, metric, seed = case
    target = ms + 1
    x, y, s, st = _random_case(n, m, r_p, v, ms, pr, pd, seed, target)
    p = O.params(m, m, r_p, v, target, O.LINF if metric == "linf" else O.L2)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o, peek=False)
    tr = Tracker(m, m, r_p, v, n, target=target, metric=metric, force="binned", scan_thread=True)
    _compare(_gpu_round(tr, x, y, s, st), r, st_o)


@pytest.mark.parametrize("cell", [1, 4, 8, 32])
def test_cell_size_does_not_change_results(cell):
    n, m = 3000, 256
    x, y, s, st = _random_case(n, m, 4, 1, 4, 0.2, 0.05, 11, 5)
    p = O.params(m, m, 4, 1, 5)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o, peek=True)
    tr = Tracker(m, m, 4, 1, n, target=5, cell=cell, force="binned", peek=True)
    g = _gpu_round(tr, x, y, s, st, peek=True)
    _compare(g, r, st)


RECT = [
    # n, map_w, map_h, r_p, v, max_step, seed: rectangular Morton grids (mkey), both orientations
    (3000, 2000, 64, 4, 1, 5, 21),
    (3000, 64, 2500, 4, 1, 5, 22),
    (8000, 5000, 300, 4, 1, 30, 23),
    (4000, 1000, 130, 12, 3, 8, 24),
]


@pytest.mark.parametrize("case", RECT, ids=[f"{c[1]}x{c[2]}" for c in RECT])
@pytest.mark.parametrize("cell", [0, 2, 16])
def test_rectangular_maps_vs_oracle(case, cell):
    n, w, h, r_p, v, ms, seed = case
    target = ms + 1
    x, y, s, st = amgen.random_state(n, w, h, seed, max_step=ms, p_running=0.2)
    p = O.params(w, h, r_p, v, target)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o, peek=False)
    tr = Tracker(w, h, r_p, v, n, target=target, cell=cell, force="binned")
    _compare(_gpu_round(tr, x, y, s, st), r, st_o)
    tr.close()


@pytest.mark.parametrize("seed", [0, 1])
def test_banded_wide_thin_map(seed):
    """A valid large-spread state on a 6000 x 96 map: the far phase walks the pyramid
    of a 1-block-high rectangular grid."""
    n, w, h = 12000, 6000, 96
    x, y, s, st = amgen.banded_state(n, w, h, seed, p_running=0.3)
    p = O.params(w, h, 4, 1, 0)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o)
    assert s.max() - s.min() > 50
    for cell in (0, 1):
        tr = Tracker(w, h, 4, 1, n, cell=cell, force="binned")
        _compare(_gpu_round(tr, x, y, s, st), r, st_o)
        tr.close()


@pytest.mark.parametrize("seed", [0, 1])
def test_banded_valid_state_large_spread(seed):
    """Valid states with a step spread of ~100: exercises the time-dilated
    scan's pyramid pruning over far cells."""
    n, w = 15000, 3000
    x, y, s, st = amgen.banded_state(n, w, w // 2, seed, p_running=0.3)
    p = O.params(w, w // 2, 4, 1, 0)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o)
    assert s.max() - s.min() > 50
    tr = Tracker(w, w // 2, 4, 1, n, force="binned")
    g = _gpu_round(tr, x, y, s, st)
    _compare(g, r, st_o)


def test_co_located_giant_cell():
    """All agents in one tile (>= 10k): one giant cluster, maximal root contention."""
    n = 12000
    x = np.full(n, 7, np.int32)
    y = np.full(n, 9, np.int32)
    s = np.zeros(n, np.int32)
    st = np.zeros(n, np.uint8)
    st[123] = O.RUNNING
    p = O.params(64, 64, 4, 1)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o)
    tr = Tracker(64, 64, 4, 1, n, force="binned")
    g = _gpu_round(tr, x, y, s, st)
    _compare(g, r, st_o)
    assert np.all(g["label"] == 0) and g["mask"].sum() == 0


def test_max_coordinates_and_huge_step_gap():
    """Map edge 16383 and step gaps up to 2^30 (radius clamp Q20)."""
    n = 4000
    rng = np.random.default_rng(5)
    m = 16384
    x = rng.integers(0, m, n).astype(np.int32)
    y = rng.integers(0, m, n).astype(np.int32)
    x[:10] = m - 1
    y[:10] = m - 1
    s = rng.integers(0, 3, n).astype(np.int32)
    s[:50] = 1 << 30
    st = np.zeros(n, np.uint8)
    p = O.params(m, m, 4, 1)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o)
    tr = Tracker(m, m, 4, 1, n, force="binned")
    g = _gpu_round(tr, x, y, s, st)
    _compare(g, r, st_o)
    assert np.all(g["mask"][:50] == 0)      # everything within any radius blocks them


@pytest.mark.parametrize("sims,per", [(2, 1), (7, 25), (64, 25), (3, 333), (2, 1024)])
def test_batched_sims_vs_oracle(sims, per):
    n = sims * per
    x, y, s, st = amgen.random_state(n, 50, 50, sims * 7 + per, max_step=3, p_running=0.2)
    p = O.params(50, 50, 4, 1, 0, O.L2, sims)
    st_o = st.copy()
    r = O.round_(p, x, y, s, st_o)
    tr = Tracker(50, 50, 4, 1, n, n_sims=sims)
    g = _gpu_round(tr, x, y, s, st)
    _compare(g, r, st_o)


def test_update_protocol_and_rejections():
    """I9 through the ABI: commits validated on the device, reported at the sync point,
    rejected updates leave the last good state."""
    tr = Tracker(32, 32, 4, 1, 3, target=5, force="binned")
    pos = _pos([1, 10, 20], [1, 10, 20])
    tr.update(pos, _dev([0, 0, 0], torch.int32))
    mask, order = tr.ready()
    assert order.tolist() == [0, 1, 2]
    bad = [([40, 10, 20], [1, 10, 20], [0, 0, 0], _lib.E_BOUNDS),
           ([1, 10, 20], [1, 10, 20], [2, 0, 0], _lib.E_PROTOCOL),
           ([3, 10, 20], [1, 10, 20], [1, 0, 0], _lib.E_VELOCITY)]
    for xs, ys, ss, code in bad:
        tr.update(_pos(xs, ys), _dev(ss, torch.int32))
        with pytest.raises(AmError) as e:
            tr.sync()
        assert e.value.code == code
    # the state is unchanged: everything is still RUNNING, nothing ready
    mask, order = tr.ready()
    assert len(order) == 0 and tr.status().tolist() == [1, 1, 1]
    tr.update(_pos([2, 10, 20], [1, 10, 20]), _dev([1, 0, 0], torch.int32))
    tr.sync()
    assert tr.status().tolist() == [0, 1, 1]
    # an error pending at am_ready is returned by am_ready and nothing is dispatched
    tr.update(_pos([2, 10, 20], [1, 10, 20]), _dev([3, 0, 0], torch.int32))
    with pytest.raises(AmError):
        tr.ready()
    assert tr.status().tolist() == [0, 1, 1]
    mask, order = tr.ready()
    assert order.tolist() == [0]


def test_protocol_sequence_matches_oracle_state_machine():
    """A few rounds of update/ready through both the ABI and oracle.State."""
    n, m = 400, 60
    rng = np.random.default_rng(3)
    x = rng.integers(0, m, n).astype(np.int32)
    y = rng.integers(0, m, n).astype(np.int32)
    s = np.zeros(n, np.int32)
    p = O.params(m, m, 4, 1, target=4)
    so = O.State(p, n)
    assert so.update(x, y, s) == O.OK
    for path in PATHS:
        tr = Tracker(m, m, 4, 1, n, target=4, force=path)
        so = O.State(p, n)
        so.update(x, y, s)
        tr.update(_pos(x, y), _dev(s, torch.int32))
        cx, cy, cs = x.copy(), y.copy(), s.copy()
        for rnd in range(12):
            ro = so.round()
            mask, order = tr.ready()
            np.testing.assert_array_equal(order.cpu().numpy(), ro["order"], err_msg=f"{path} round {rnd}")
            np.testing.assert_array_equal(tr.clusters().cpu().numpy(), ro["label"], err_msg=f"{path} round {rnd}")
            # commit half of the RUNNING agents, moving them by one tile
            run = np.nonzero(so.status == O.RUNNING)[0]
            pick = run[rng.random(len(run)) < 0.5]
            cx[pick] = np.clip(cx[pick] + rng.integers(-1, 2, len(pick)) * (rng.random(len(pick)) < 0.5), 0, m - 1)
            cs[pick] += 1
            assert so.update(cx, cy, cs) == O.OK
            tr.update(_pos(cx, cy), _dev(cs, torch.int32))
            tr.sync()
            np.testing.assert_array_equal(tr.status().cpu().numpy(), so.status)


def test_empty_and_all_done():
    tr = Tracker(16, 16, 4, 1, 0)
    tr.update(torch.zeros((0, 2), dtype=torch.int32, device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"))
    mask, order = tr.ready()
    assert len(order) == 0
    tr = Tracker(16, 16, 4, 1, 2000, target=3, force="binned")
    tr.update(_pos(np.arange(2000) % 16, np.arange(2000) // 16 % 16), _dev(np.full(2000, 3), torch.int32))
    mask, order = tr.ready()
    assert len(order) == 0 and int(mask.sum()) == 0
    assert (tr.clusters() == -1).all()


@pytest.mark.parametrize("path", ["binned"])
def test_large_ready_set_closed_form(path):
    """300k isolated agents (spacing 20 > R_b(6) = 11), steps 0..6: every agent is its own
    ready cluster, so order = agents sorted by (step, id) -- a closed form at a size whose
    ready set spans many radix tiles (the first replay round has this shape)."""
    side = 548
    n = side * side
    ids = np.arange(n)
    x = ((ids % side) * 20).astype(np.int32)
    y = ((ids // side) * 20).astype(np.int32)
    s = (ids * 7919 % 7).astype(np.int32)
    st = np.zeros(n, np.uint8)
    tr = Tracker(side * 20, side * 20, 4, 1, n, force=path)
    g = _gpu_round(tr, x, y, s, st)
    assert g["mask"].all()
    np.testing.assert_array_equal(g["label"], ids)
    np.testing.assert_array_equal(g["order"], np.lexsort((ids, s)))
    # a second round on the dispatched state: nothing is ready
    mask, order = tr.ready()
    assert len(order) == 0


@pytest.mark.parametrize("wide", [False, True], ids=["keys32", "keys64"])
@pytest.mark.parametrize("sort", ["cluster", "onesweep"])
@pytest.mark.parametrize("pairs", [1, 700, 21000, 150000])
def test_interleaved_pair_clusters_closed_form(pairs, sort, wide, monkeypatch):
    """Coupled pairs whose members are n/2 ids apart (clusters interleave in id space),
    isolated from each other (spacing 20 > R_b(4) = 9): label = min id of the pair, and
    order = ready agents sorted by (step, label, id) -- the priority rule P:143 / Q9 /
    Q10 as a closed form.  Sizes span the cluster sort's shared-memory-resident mode
    (<= 16 x ~8k ready agents) and its streaming mode, and the onesweep ablation.
    `wide`: v = 0 (R_b = r_p at any lag) with step gaps up to ~2^27, so the priority keys
    need more than 32 bits (the 16-byte element path of the cluster sort)."""
    if sort == "onesweep":
        monkeypatch.setenv("AM_SORT", "onesweep")
    n = 2 * pairs
    side = int(np.ceil(np.sqrt(pairs)))
    k = np.arange(pairs)
    px = ((k % side) * 20).astype(np.int32)
    py = ((k // side) * 20).astype(np.int32)
    x = np.concatenate([px, px + 1]).astype(np.int32)       # partner one tile east
    y = np.concatenate([py, py]).astype(np.int32)
    step = (k * 7919 % 5).astype(np.int32) * (33554467 if wide else 1)
    s = np.concatenate([step, step]).astype(np.int32)
    st = np.zeros(n, np.uint8)
    ids = np.arange(n)
    label = np.concatenate([k, k]).astype(np.int32)
    tr = Tracker(side * 20 + 2, side * 20 + 2, 4, 0 if wide else 1, n, force="binned")
    g = _gpu_round(tr, x, y, s, st)
    assert g["mask"].all()
    np.testing.assert_array_equal(g["label"], label)
    np.testing.assert_array_equal(g["order"], np.lexsort((ids, label, s)))
    tr.close()


@pytest.mark.parametrize("knobs", [{}, {"AM_REBUILD_D": "1000", "AM_REBUILD_K": "1000"},
                                   {"AM_REBUILD_D": "0", "AM_REBUILD_K": "0"}])
def test_loose_cells_every_round_vs_oracle(knobs, monkeypatch):
    """Incremental binning ("loose cells"): between rebuilds the
    records keep their cells, committed agents update theirs in place and every cell
    box is widened by the drift D.  A C4-shaped replay (5000 agents at C4 density,
    hotspots, busy hour, 50 ms quantum) compared with the brute-force oracle round by
    round for 300 rounds: default policy, never rebuilding (D grows to tens of tiles:
    the widening carries everything), and rebuilding every round."""
    import amgen
    from paper_2411_03519_b200 import Replay
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    w = amgen.config("C4", n=5000)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm, force="binned")
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, w.steps)
    rebuilt, loose, dmax = 0, 0, 0
    for r in range(300):
        x = rep.pos[:, 0].cpu().numpy().copy()
        y = rep.pos[:, 1].cpu().numpy().copy()
        s = rep.steps.cpu().numpy().copy()
        st = rep.tracker.status().cpu().numpy().copy()   # as the round sees them
        mask_t, order_t, labels_t = rep.step()
        mask = mask_t.cpu().numpy()
        ref = O.round_mt(p, x, y, s, st.copy(), peek=True)
        np.testing.assert_array_equal(mask, ref["mask"], err_msg=f"round {r}")
        np.testing.assert_array_equal(order_t.cpu().numpy(), ref["order"], err_msg=f"round {r}")
        np.testing.assert_array_equal(labels_t.cpu().numpy(), ref["label"], err_msg=f"round {r}")
        stt = rep.tracker.stats()
        rebuilt += stt["rebuilt"]
        loose += 1 - stt["rebuilt"]
        dmax = max(dmax, stt["drift"])
    if knobs.get("AM_REBUILD_K") == "0":
        assert loose == 0
    else:
        assert loose > 200 and rebuilt >= 1
    if knobs.get("AM_REBUILD_K") == "1000":
        assert dmax > 8, dmax          # the drift really grew past the cell edge
    rep.close()
