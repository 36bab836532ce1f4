"""NEXT #4 variant, graph-distance dependencies ("non-Euclidean spaces such as social
networks"): positions are graph nodes, dist = hop count.  Pins of the oracle's
graph metric: the BFS distance table against scipy's shortest paths (library routine),
hand-worked rule vectors on a path graph (App. A's rules with the hop metric), and the
out-of-order replay's outcome == lock-step with the validity condition checked at
every commit."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

import amgen
import oracle as O


def _path_graph(V):
    off = np.arange(V + 1, dtype=np.int32) * 2 - 1
    off[0] = 0
    adj = []
    for u in range(V):
        if u > 0:
            adj.append(u - 1)
        if u < V - 1:
            adj.append(u + 1)
    off = np.zeros(V + 1, np.int32)
    for u in range(V):
        off[u + 1] = off[u] + (u > 0) + (u < V - 1)
    return off, np.array(adj, np.int32)


def test_bfs_table_equals_scipy_shortest_paths():
    off, adj = amgen.social_graph(200, 4, 0.1, seed=5)
    V = len(off) - 1
    rows = np.repeat(np.arange(V), np.diff(off))
    g = csr_matrix((np.ones(len(adj)), (rows, adj)), shape=(V, V))
    ref = shortest_path(g, unweighted=True, directed=False)
    d = amgen.graph_distances(off, adj)
    assert np.isfinite(ref).all()
    np.testing.assert_array_equal(d.astype(np.int64), ref.astype(np.int64))
    assert np.array_equal(d, d.T) and (np.diag(d) == 0).all()


def test_graph_rules_on_a_path_graph():
    """Path graph 0-1-2-...-19, r_p = 2, v = 1 (hop metric): R_c = 3 hops, R_b(1) = 4,
    R_b(2) = 5.  Coupled iff same step and <= 3 hops (inclusive); A blocked by B iff
    s_B < s_A and hops <= (s_A - s_B + 1) + 2."""
    off, adj = _path_graph(20)
    gd = amgen.graph_distances(off, adj)
    p = O.params(20, 1, 2, 1, graph_dist=gd)
    assert O.coupled(p, (0, 0, 5), (3, 0, 5)) and not O.coupled(p, (0, 0, 5), (4, 0, 5))
    assert O.blocked_by(p, (0, 0, 6), (4, 0, 5)) and not O.blocked_by(p, (0, 0, 6), (5, 0, 5))
    assert O.blocked_by(p, (0, 0, 7), (5, 0, 5)) and not O.blocked_by(p, (0, 0, 7), (6, 0, 5))
    assert not O.blocked_by(p, (0, 0, 5), (1, 0, 6))          # future agents never block
    # a round: A0@0 s1, A1@3 s1 (coupled), A2@7 s0 blocks A1 (4 hops <= R_b(1) = 4)
    r = O.round_(p, [0, 3, 7], [0, 0, 0], [1, 1, 0], np.zeros(3, np.uint8), peek=True)
    assert list(r["label"]) == [0, 0, 2] and list(r["blocked"]) == [0, 1, 0] and list(r["order"]) == [2]
    # validity: |dS| = 2 -> bound r_p + v = 3 hops: 3 violates, 4 does not
    assert O.validity_violations(p, [0, 3], [0, 0], [0, 2]) == 1
    assert O.validity_violations(p, [0, 4], [0, 0], [0, 2]) == 0


@pytest.mark.parametrize("Q", [0, 30_000])
def test_graph_replay_equals_lockstep(Q):
    w = amgen.config("G1", steps=150)
    lm = amgen.latency_model(w.profile)
    sy = O.SynthTables.from_model(lm, policy=3, graph=w.graph)
    p = O.params(w.map_w, w.map_h, w.r_p, w.v, target=w.steps, graph_dist=w.gdist)
    r = O.replay(p, sy, w.x, w.y, Q=Q, check=True)
    ls = O.lockstep(p, sy, w.x, w.y, w.steps)
    assert r["violations"] == 0
    np.testing.assert_array_equal(r["traj"], ls["traj"])
    np.testing.assert_array_equal(r["x"], ls["x"])
    assert r["max_spread"] > 3
    # the walk moves along edges: every final node is reachable in <= T hops (sanity) and
    # some agents moved
    assert np.any(r["x"] != w.x)
    assert np.all(w.gdist[w.x, r["x"]] <= w.steps)
