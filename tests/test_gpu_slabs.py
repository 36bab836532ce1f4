"""S7 multi-GPU spatial slabs, virtual slabs on one GPU (loopback exchange): the
distributed round equals the oracle's single round bit for bit (mask, labels,
per-rank order) for several slab counts, including multi-hop halos."""
import numpy as np
import pytest
import torch

import amgen
import oracle as O
from paper_2411_03519_b200 import slabs

pytestmark = pytest.mark.gpu


def _run(x, y, s, st, W, H, G, r_p=4, v=1, metric="l2"):
    n = len(x)
    gid = np.arange(n, dtype=np.int32)
    part = slabs.partition(torch.as_tensor(y), H, G).numpy()
    ranks = []
    for k in range(G):
        sel = np.nonzero(part == k)[0]
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a[sel]), dtype=dt, device="cuda")
        pos = torch.as_tensor(np.stack([x[sel], y[sel]], 1), dtype=torch.int32, device="cuda")
        ranks.append(slabs.SlabRank(W, H, r_p, v, n, G, k, t(gid, torch.int32), pos, t(s, torch.int32),
                                    t(st, torch.uint8), metric=metric))
    outs = slabs.round_loopback(ranks)
    mask = np.zeros(n, np.uint8)
    label = np.zeros(n, np.int32)
    orders = []
    for o in outs:
        g = o["gid"].cpu().numpy()
        mask[g] = o["mask"].cpu().numpy()
        label[g] = o["labels"].cpu().numpy()
        orders.append(o["order"].cpu().numpy())
    return mask, label, orders


def _check(x, y, s, st, W, H, G, **kw):
    p = O.params(W, H, kw.get("r_p", 4), kw.get("v", 1), 0,
                 O.LINF if kw.get("metric") == "linf" else O.L2)
    r = O.round_(p, x, y, s, st.copy(), peek=True)
    mask, label, orders = _run(x, y, s, st, W, H, G, **kw)
    np.testing.assert_array_equal(mask, r["mask"])
    np.testing.assert_array_equal(label, r["label"])
    # each rank's order = the global order restricted to its agents
    part = slabs.partition(torch.as_tensor(y), H, G).numpy()
    for k, ok in enumerate(orders):
        exp = np.array([i for i in r["order"] if part[i] == k], np.int32)
        np.testing.assert_array_equal(ok, exp)
    assert sum(len(o) for o in orders) == len(r["order"])


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_random_state_slabs(G):
    n, m = 12000, 900
    x, y, s, st = amgen.random_state(n, m, m, 40 + G, max_step=6, p_running=0.3)
    st[np.random.default_rng(G).random(n) < 0.05] = O.DONE
    _check(x, y, s, st, m, m, G)


@pytest.mark.parametrize("G", [2, 8, 16])
def test_banded_large_spread_multihop(G):
    """Spread ~60 steps -> halo radius > slab height for G=16 (multi-hop halo)."""
    n, w = 10000, 1500
    x, y, s, st = amgen.banded_state(n, w, 480, 3, p_running=0.3)
    # rotate so that the step gradient runs across the slabs (bands along y)
    x, y = y.copy(), x.copy()
    _check(x, y, s, st, 480, w, G)


def test_linf_and_coupled_chain_across_all_slabs():
    """A chain of coupled agents crossing every slab boundary: one global cluster."""
    H, G = 400, 8
    ys = np.arange(0, H, 5, dtype=np.int32)
    x = np.full(len(ys), 10, np.int32)
    s = np.zeros(len(ys), np.int32)
    st = np.zeros(len(ys), np.uint8)
    st[len(ys) // 2] = O.RUNNING        # poisons the whole chain
    mask, label, _ = _run(x, ys, s, st, 64, H, G)
    assert np.all(label == 0) and mask.sum() == 0
    _check(x, ys, s, st, 64, H, G, metric="linf")
