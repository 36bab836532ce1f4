"""Seeded synthetic-input generators shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no blocking/coupling rule, no
clustering, no policy or latency hashing).  It only produces data:

* maps: the procedural SmallVille-shaped town (the paper gives only
  "SmallVille, a 100x140 grid"), its replica tiling (Q19, "concatenating
  multiple SmallVilles") and open maps for the large configs;
* initial agent positions (distinct free tiles, or Gaussian hotspots);
* the LLM-latency tables the synthetic driver indexes (Q16): LAT[1024] quantiles
  of LogNormal(median 600 ms, sigma 0.5) in integer microseconds, and the
  call-count CDF per load profile.  Calibration: 56.7k calls/day and the busy
  hour's ~5000 calls for 25 agents, 10 s per step.

Everything is computed with numpy's seeded ``default_rng`` / stdlib doubles on
the host once and handed to both sides as arrays (so neither side depends on a
libm).  The recipe is restated in DESIGN.md section 5.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from statistics import NormalDist

import numpy as np

TOWN_W, TOWN_H = 140, 100          # Q14: 100x140 grid, x = 140 wide
BASE_US = 5000                     # fixed per-step cost (Q16)
LAT_MEDIAN_US = 600_000            # LogNormal median 600 ms (Q16)
LAT_SIGMA = 0.5

# call-count distributions per agent-step (values, probabilities), Q16
PROFILES = {
    "fullday": ((0, 1, 2, 3, 5), (0.88, 0.05, 0.03, 0.02, 0.02)),
    "busy": ((0, 1, 2, 3, 5), (0.77, 0.08, 0.06, 0.05, 0.04)),
}


def lat_table(n: int = 1024) -> np.ndarray:
    """LAT[q] = round(exp(ln median + sigma * Phi^-1((q+0.5)/n))) microseconds."""
    nd = NormalDist()
    out = np.empty(n, np.uint32)
    for q in range(n):
        z = nd.inv_cdf((q + 0.5) / n)
        out[q] = int(round(float(np.exp(np.log(LAT_MEDIAN_US) + LAT_SIGMA * z))))
    return out


def cdf_table(profile: str):
    """(vals int32[m], cdf32 uint64[m]): cumulative probability scaled to 2^32; last = 2^32."""
    vals, probs = PROFILES[profile]
    c = np.cumsum(np.asarray(probs, np.float64))
    cdf = np.array([int(round(v * 2**32)) for v in c], np.uint64)
    cdf[-1] = np.uint64(2**32)
    return np.asarray(vals, np.int32), cdf


@dataclass
class LatencyModel:
    lat: np.ndarray
    vals: np.ndarray
    cdf32: np.ndarray
    base_us: int
    lat_seed: int
    policy_seed: int


def latency_model(profile: str = "fullday", lat_seed: int = 4, policy_seed: int = 3) -> LatencyModel:
    vals, cdf = cdf_table(profile)
    return LatencyModel(lat_table(), vals, cdf, BASE_US, lat_seed, policy_seed)


# ----------------------------------------------------------------------------- maps
def _connected(free: np.ndarray) -> bool:
    h, w = free.shape
    ys, xs = np.nonzero(free)
    if len(xs) == 0:
        return False
    seen = np.zeros_like(free, dtype=bool)
    dq = deque([(ys[0], xs[0])])
    seen[ys[0], xs[0]] = True
    cnt = 1
    while dq:
        cy, cx = dq.popleft()
        for dy, dx in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            ny, nx = cy + dy, cx + dx
            if 0 <= ny < h and 0 <= nx < w and free[ny, nx] and not seen[ny, nx]:
                seen[ny, nx] = True
                cnt += 1
                dq.append((ny, nx))
    return cnt == int(free.sum())


def town_map(seed: int = 1, w: int = TOWN_W, h: int = TOWN_H, n_buildings: int = 14) -> np.ndarray:
    """uint8[h, w] wall bitmap: border wall, rectangular buildings with 1-tile walls
    and a 2-tile door; the free space is 4-connected (BFS-verified)."""
    for attempt in range(1000):
        rng = np.random.default_rng([seed, attempt])
        wall = np.zeros((h, w), np.uint8)
        wall[0, :] = wall[-1, :] = 1
        wall[:, 0] = wall[:, -1] = 1
        occupied = np.zeros((h, w), bool)
        placed = 0
        for _ in range(400):
            if placed == n_buildings:
                break
            bw = int(rng.integers(8, 21))
            bh = int(rng.integers(6, 15))
            x0 = int(rng.integers(3, w - bw - 3))
            y0 = int(rng.integers(3, h - bh - 3))
            if occupied[y0 - 2:y0 + bh + 2, x0 - 2:x0 + bw + 2].any():
                continue
            occupied[y0:y0 + bh, x0:x0 + bw] = True
            wall[y0, x0:x0 + bw] = 1
            wall[y0 + bh - 1, x0:x0 + bw] = 1
            wall[y0:y0 + bh, x0] = 1
            wall[y0:y0 + bh, x0 + bw - 1] = 1
            side = int(rng.integers(0, 4))
            if side in (0, 1):
                dx = int(rng.integers(x0 + 1, x0 + bw - 2))
                yy = y0 if side == 0 else y0 + bh - 1
                wall[yy, dx:dx + 2] = 0
            else:
                dy = int(rng.integers(y0 + 1, y0 + bh - 2))
                xx = x0 if side == 2 else x0 + bw - 1
                wall[dy:dy + 2, xx] = 0
            placed += 1
        if placed == n_buildings and _connected(wall == 0):
            return wall
    raise RuntimeError("town generator failed")


def replicated_map(tile: np.ndarray, cols: int = 5, rows: int = 4) -> np.ndarray:
    """Q19: replicas side by side (5 columns x 4 rows -> 700x400), each keeps its own border."""
    return np.tile(tile, (rows, cols))


def distinct_free_positions(wall: np.ndarray, n: int, seed: int, x0: int = 0, y0: int = 0,
                            w: int | None = None, h: int | None = None):
    """n distinct free tiles, uniform without replacement, inside the window."""
    H, W = wall.shape
    w = W - x0 if w is None else w
    h = H - y0 if h is None else h
    sub = wall[y0:y0 + h, x0:x0 + w]
    ys, xs = np.nonzero(sub == 0)
    rng = np.random.default_rng(seed)
    pick = rng.choice(len(xs), size=n, replace=False)
    return (xs[pick] + x0).astype(np.int32), (ys[pick] + y0).astype(np.int32)


def hotspot_positions(n: int, w: int, h: int, seed: int, frac_hot: float = 0.6,
                      per_spot: int = 250, sigma: float = 40.0):
    """frac_hot of the agents in Gaussian hotspots of per_spot
    agents (sigma tiles, centres uniform), the rest uniform; rounded, clipped,
    co-location allowed."""
    rng = np.random.default_rng(seed)
    n_hot = int(round(n * frac_hot))
    n_spots = max(1, n_hot // per_spot)
    cx = rng.uniform(0, w, n_spots)
    cy = rng.uniform(0, h, n_spots)
    spot = np.arange(n_hot) % n_spots
    hx = np.rint(cx[spot] + rng.normal(0, sigma, n_hot))
    hy = np.rint(cy[spot] + rng.normal(0, sigma, n_hot))
    ux = rng.integers(0, w, n - n_hot)
    uy = rng.integers(0, h, n - n_hot)
    x = np.clip(np.concatenate([hx, ux]), 0, w - 1).astype(np.int32)
    y = np.clip(np.concatenate([hy, uy]), 0, h - 1).astype(np.int32)
    perm = rng.permutation(n)
    return x[perm], y[perm]


def random_state(n: int, w: int, h: int, seed: int, max_step: int = 4, p_running: float = 0.0):
    """Arbitrary (not necessarily valid) tracker state for kernel-robustness tests."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, w, n).astype(np.int32)
    y = rng.integers(0, h, n).astype(np.int32)
    s = rng.integers(0, max_step + 1, n).astype(np.int32)
    st = (rng.random(n) < p_running).astype(np.uint8)
    return x, y, s, st


# ----------------------------------------------------------------------------- graphs
def social_graph(V: int = 200, k: int = 4, p_rewire: float = 0.1, seed: int = 5):
    """A small-world "social network" (Watts-Strogatz: a ring where every node links to
    its k/2 nearest neighbours on each side, each link rewired with probability
    p_rewire; regenerated until connected) for the non-Euclidean variant.
    Returns (offsets int32 [V+1], neighbours int32 [E2]) -- CSR, neighbours sorted."""
    for attempt in range(100):
        rng = np.random.default_rng([seed, attempt])
        edges = set()
        for u in range(V):
            for j in range(1, k // 2 + 1):
                w = (u + j) % V
                if rng.random() < p_rewire:
                    w = int(rng.integers(0, V))
                    while w == u or (min(u, w), max(u, w)) in edges:
                        w = int(rng.integers(0, V))
                edges.add((min(u, w), max(u, w)))
        nbr = [[] for _ in range(V)]
        for a, b in edges:
            nbr[a].append(b)
            nbr[b].append(a)
        off = np.zeros(V + 1, np.int32)
        for u in range(V):
            off[u + 1] = off[u] + len(nbr[u])
        adj = np.concatenate([np.array(sorted(x), np.int32) for x in nbr]) if edges else np.zeros(0, np.int32)
        d = graph_distances(off, adj)
        if (d != 0xFFFF).all():
            return off, adj
    raise RuntimeError("social graph generator failed")


def graph_distances(off: np.ndarray, adj: np.ndarray) -> np.ndarray:
    """Hop distances between all node pairs by breadth-first search from every node:
    uint16 [V][V], 0xFFFF = unreachable.  Data for both sides (the metric's table)."""
    V = len(off) - 1
    out = np.full((V, V), 0xFFFF, np.uint16)
    for src in range(V):
        dist = out[src]
        dist[src] = 0
        frontier = [src]
        h = 0
        while frontier:
            h += 1
            nxt = []
            for u in frontier:
                for w in adj[off[u]:off[u + 1]]:
                    if dist[w] == 0xFFFF:
                        dist[w] = h
                        nxt.append(int(w))
            frontier = nxt
    return out


# ----------------------------------------------------------------------------- configs
@dataclass
class Workload:
    name: str
    map_w: int
    map_h: int
    wall: np.ndarray | None
    x: np.ndarray
    y: np.ndarray
    n_sims: int
    steps: int
    r_p: int = 4
    v: int = 1
    profile: str = "fullday"
    Q: int = 0
    graph: tuple | None = None        # (offsets, neighbours): the graph-metric variant
    gdist: np.ndarray | None = None   # uint16 [V][V] hop distances


def config(name: str, steps: int | None = None, n: int | None = None) -> Workload:
    """BASELINE.json configs C1..C5 as concrete synthetic inputs.
    ``n`` shrinks the agent count at the same density (tests only)."""
    if name == "C1":
        wall = town_map(1)
        x, y = distinct_free_positions(wall, 25, seed=2)
        return Workload("C1", TOWN_W, TOWN_H, wall, x, y, 1, steps or 1000)
    if name == "C2":
        wall = replicated_map(town_map(1))
        xs, ys = [], []
        for r in range(20):
            cx, cy = (r % 5) * TOWN_W, (r // 5) * TOWN_H
            x, y = distinct_free_positions(wall, 25, seed=2 + r, x0=cx, y0=cy, w=TOWN_W, h=TOWN_H)
            xs.append(x)
            ys.append(y)
        return Workload("C2", 5 * TOWN_W, 4 * TOWN_H, wall, np.concatenate(xs), np.concatenate(ys), 1,
                        steps or 1000, profile="busy")
    if name == "C3":
        wall = town_map(1)
        sims = n or 4096
        xs, ys = [], []
        for b in range(sims):
            x, y = distinct_free_positions(wall, 25, seed=2 + b)
            xs.append(x)
            ys.append(y)
        return Workload("C3", TOWN_W, TOWN_H, wall, np.concatenate(xs), np.concatenate(ys), sims,
                        steps or 1000)
    if name == "G1":
        # NEXT #4 variant ("non-Euclidean spaces such as social networks"): agents
        # on the nodes of a 600-node small-world graph (ring lattice k = 4, 2% of the links
        # rewired: diameter 39, mean distance 14 hops), hop metric, r_p = 2 hops, v = 1
        off, adj = social_graph(600, 4, 0.02, seed=5)
        V = len(off) - 1
        rng = np.random.default_rng(2)
        nodes = rng.integers(0, V, n or 60).astype(np.int32)
        return Workload("G1", V, 1, None, nodes, np.zeros(len(nodes), np.int32), 1, steps or 300, r_p=2, v=1,
                        graph=(off, adj), gdist=graph_distances(off, adj))
    if name in ("C4", "C5"):
        big = name == "C5"
        N = n or (1_000_000 if big else 100_000)
        side = 16384 if big else 4096
        full = 1_000_000 if big else 100_000
        # same density when shrunk: side scales with sqrt(N/full)
        side = max(64, int(round(side * (N / full) ** 0.5)))
        x, y = hotspot_positions(N, side, side, seed=2)
        return Workload(name, side, side, None, x, y, 1, steps or 1000, profile="busy", Q=50_000)
    if name == "C5T":
        # C5's density and recipe on a TALL map (width 16384, height 16384 * N / 1M): the
        # slab-distributed replay beyond one tracker's 32768 rows (weak scaling, one 1M-agent
        # 16384^2 slab per rank at N = G * 1M; each window keeps its own 16-bit row frame)
        N = n or 2_000_000
        w_ = 16384
        h_ = max(64, int(round(16384 * N / 1_000_000)))
        x, y = hotspot_positions(N, w_, h_, seed=2)
        return Workload(name, w_, h_, None, x, y, 1, steps or 1000, profile="busy", Q=50_000)
    raise KeyError(name)


def banded_state(n: int, w: int, h: int, seed: int, band: int = 24, gap: int = 6,
                 p_running: float = 0.3, p_done: float = 0.0, target: int = 0,
                 hot_frac: float = 0.5):
    """A state with a large step spread that satisfies the validity condition P:156
    by construction (for r_p < gap and v <= band + gap): agents only inside vertical
    bands of width ``band`` separated by empty gaps of width ``gap``; band k is at
    step k (steps change by one per band), so agents K bands apart are at least
    (K-1)(band+gap)+gap > r_p + (K-1)v apart.  Half the agents sit in hotspots.
    Statuses: RUNNING with p_running, DONE (step = target) with p_done."""
    rng = np.random.default_rng(seed)
    period = band + gap
    nb = max(1, w // period)
    n_hot = int(n * hot_frac)
    spots = max(1, n_hot // 250)
    cx = rng.uniform(0, w, spots)
    cy = rng.uniform(0, h, spots)
    sp = np.arange(n_hot) % spots
    x = np.concatenate([np.rint(cx[sp] + rng.normal(0, 40, n_hot)), rng.integers(0, w, n - n_hot)])
    y = np.concatenate([np.rint(cy[sp] + rng.normal(0, 40, n_hot)), rng.integers(0, h, n - n_hot)])
    x = np.clip(x, 0, nb * period - 1).astype(np.int64)
    y = np.clip(y, 0, h - 1).astype(np.int32)
    k = x // period
    off = x % period
    off = np.where(off >= band, band - 1, off)       # push gap agents to the band's edge
    x = (k * period + off).astype(np.int32)
    step = k.astype(np.int32)
    status = (rng.random(n) < p_running).astype(np.uint8)
    if p_done > 0 and target > 0:
        done = rng.random(n) < p_done
        status[done] = 2
        step[done] = target
    perm = rng.permutation(n)
    return x[perm], y[perm], step[perm], status[perm]
