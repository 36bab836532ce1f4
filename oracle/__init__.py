"""CPU oracle for the AI Metropolis dependency tracker -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2411_03519_b200``) never imports it and shares no code with it.

Thin ctypes marshalling over ``oracle/oracle.c`` (plain C, brute force, integer
arithmetic).  Every function cites the passage of /root/reference/PAPER.md it
restates in oracle.c.  Parity status per function:

* round / update / validity / sampled round: pinned (hand vectors V1-V14 in
  tests/golden, BFS components, invariants, brute force on tiny maps).
* replay / lockstep: pinned by the closed forms D1-D5 and the OoO == lock-step
  outcome invariant.
* replay_stale (stale-halo slabs, NEXT #3): pinned by P = 1 == replay round for round,
  zero I1/I2 violations and OoO == lock-step for every P and G, and hand states where a
  stale ghost must defer (tests/test_oracle_stale.py).
* duration / policy_move / digest / key3 / the trajectory hash (synthetic driver,
  Q16): the paper is silent -- our own constructs; pinned against an
  independent pure-Python implementation of the c.4 definitions built on splitmix64's
  published outputs, plus structural pins (tests/test_oracle_pins.py).
* round_mt / labels_steps / blocked_list / round_at_scale / lockstep_grid
  (oracle_scale.c, the same predicates with threaded outer loops for the 100k / 1M
  configs): pinned by equality with round_ / lockstep on random and workload states.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRC_SCALE = os.path.join(_HERE, "oracle_scale.c")   # the same definitions at BASELINE sizes
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

IDLE, RUNNING, DONE = 0, 1, 2
L2, LINF, GRAPH = 0, 1, 2
OK, E_ARG, E_BOUNDS, E_PROTOCOL, E_VELOCITY, E_LIVENESS = 0, -1, -2, -3, -4, -8


def build(force: bool = False) -> str:
    """Compile oracle.c + oracle_scale.c into liboracle.so with gcc (plain -O2, no
    vectorisation tricks; pthreads for the at-scale drivers' outer loops)."""
    with _lock:
        newest = max(os.path.getmtime(_SRC), os.path.getmtime(_SRC_SCALE))
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", "-o", tmp,
                                   _SRC, _SRC_SCALE])
            os.replace(tmp, _LIB)
    return _LIB


def host_threads() -> int:
    """Host cores this process may use (the at-scale oracle's thread count)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return max(1, os.cpu_count() or 1)


class Params(C.Structure):
    _fields_ = [("map_w", C.c_int32), ("map_h", C.c_int32), ("r_p", C.c_int32),
                ("v", C.c_int32), ("target", C.c_int32), ("metric", C.c_int32),
                ("n_sims", C.c_int32), ("gdist", C.c_void_p), ("gV", C.c_int32)]


class Synth(C.Structure):
    _fields_ = [("lat", C.c_void_p), ("cdf32", C.c_void_p), ("vals", C.c_void_p),
                ("n_vals", C.c_int32), ("base_us", C.c_int32), ("lat_seed", C.c_uint64),
                ("policy_seed", C.c_uint64), ("wall", C.c_void_p),
                ("dur_table", C.c_void_p), ("dur_T", C.c_int32), ("policy", C.c_int32),
                ("conflict", C.c_int32), ("graph_off", C.c_void_p), ("graph_adj", C.c_void_p)]


class Log(C.Structure):
    _fields_ = [("cap_rounds", C.c_int64), ("cap_entries", C.c_int64),
                ("round_t", C.c_void_p), ("round_sim", C.c_void_p),
                ("round_nready", C.c_void_p), ("entry_id", C.c_void_p),
                ("entry_label", C.c_void_p), ("n_rounds", C.c_int64),
                ("n_entries", C.c_int64), ("check", C.c_int32),
                ("violations", C.c_int64), ("max_spread", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.POINTER(Params)
        vp = C.c_void_p
        L.orc_round.argtypes = [P, C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, vp, vp, vp]
        L.orc_round_sampled.argtypes = [P, C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, vp, vp, vp]
        L.orc_update.argtypes = [P, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp, vp]
        L.orc_validity_violations.argtypes = [P, C.c_int32, vp, vp, vp]
        L.orc_validity_violations.restype = C.c_int64
        L.orc_coupled.argtypes = [P] + [C.c_int32] * 6
        L.orc_blocked_by.argtypes = [P] + [C.c_int32] * 6
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_key3.argtypes = [C.c_uint64] * 3
        L.orc_key3.restype = C.c_uint64
        L.orc_duration.argtypes = [C.POINTER(Synth), C.c_int32, C.c_int32]
        L.orc_duration.restype = C.c_int64
        L.orc_digest.argtypes = [P, C.c_int32, C.c_int32, vp, vp, vp, vp, C.c_int32]
        L.orc_digest.restype = C.c_uint64
        L.orc_policy_move.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_uint64, vp, vp]
        L.orc_lockstep.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.orc_replay.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int64, vp, vp, vp, vp, vp,
                                 C.POINTER(Log)]
        L.orc_replay_cap.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                     vp, vp, vp, vp, vp, C.POINTER(Log)]
        L.orc_replay_stale.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                       vp, vp, vp, vp, vp, C.POINTER(Log)]
        # oracle_scale.c
        L.orc_round_mt.argtypes = [P, C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, vp, vp, vp, C.c_int32]
        L.orc_labels_steps.argtypes = [P, C.c_int32, vp, vp, vp, vp, vp, C.c_int32]
        L.orc_blocked_list.argtypes = [P, C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, C.c_int32]
        L.orc_lockstep_grid.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int32, vp, vp, vp, vp, C.c_int32]
        L.orc_replay_sim_logged.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int64, C.c_int32, vp, vp, vp,
                                            vp, vp, C.POINTER(Log)]
        L.orc_replay_mt.argtypes = [P, C.POINTER(Synth), C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                    vp, vp, vp, vp, vp, C.c_int32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def params(map_w, map_h, r_p, v, target=0, metric=L2, n_sims=1, graph_dist=None) -> Params:
    """graph_dist: uint16 [V][V] hop distances (metric GRAPH; positions are nodes)."""
    if graph_dist is None:
        return Params(int(map_w), int(map_h), int(r_p), int(v), int(target), int(metric), int(n_sims), None, 0)
    gd = np.ascontiguousarray(graph_dist, np.uint16)
    p = Params(int(map_w), int(map_h), int(r_p), int(v), int(target), int(GRAPH), int(n_sims), _p(gd).value,
               int(gd.shape[0]))
    p._keep = gd
    return p


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def round_(p: Params, x, y, step, status, peek=False):
    """One scheduling round (oracle.c orc_round).  Returns dict; status is updated in
    place when peek is False (dispatch)."""
    x, y, step = _i32(x), _i32(y), _i32(step)
    n = len(x)
    assert status.dtype == np.uint8 and status.flags.c_contiguous
    blocked = np.zeros(n, np.uint8)
    label = np.zeros(n, np.int32)
    mask = np.zeros(n, np.uint8)
    order = np.zeros(max(n, 1), np.int32)
    nr = np.zeros(1, np.int32)
    rc = lib().orc_round(C.byref(p), n, _p(x), _p(y), _p(step), _p(status), int(bool(peek)),
                         _p(blocked), _p(label), _p(mask), _p(order), _p(nr))
    if rc != OK:
        raise RuntimeError(f"orc_round rc={rc}")
    return dict(blocked=blocked, label=label, mask=mask, order=order[: nr[0]].copy())


def round_sampled(p: Params, x, y, step, status, sample):
    x, y, step = _i32(x), _i32(y), _i32(step)
    status = np.ascontiguousarray(status, np.uint8)
    sample = _i32(sample)
    k = len(sample)
    blocked = np.zeros(k, np.uint8)
    label = np.zeros(k, np.int32)
    mask = np.zeros(k, np.uint8)
    csize = np.zeros(k, np.int32)
    rc = lib().orc_round_sampled(C.byref(p), len(x), _p(x), _p(y), _p(step), _p(status), k,
                                 _p(sample), _p(blocked), _p(label), _p(mask), _p(csize))
    if rc != OK:
        raise RuntimeError(f"orc_round_sampled rc={rc}")
    return dict(blocked=blocked, label=label, mask=mask, comp_size=csize)


class State:
    """Tracker state as the oracle keeps it (mirror of the am_* semantics)."""

    def __init__(self, p: Params, n: int):
        self.p = p
        self.x = np.zeros(n, np.int32)
        self.y = np.zeros(n, np.int32)
        self.step = np.zeros(n, np.int32)
        self.status = np.zeros(n, np.uint8)
        self.first = True

    def update(self, x, y, step) -> int:
        nx, ny, ns = _i32(x), _i32(y), _i32(step)
        rc = lib().orc_update(C.byref(self.p), len(self.x), int(self.first), _p(self.x), _p(self.y),
                              _p(self.step), _p(self.status), _p(nx), _p(ny), _p(ns))
        if rc == OK:
            self.first = False
        return rc

    def round(self, peek=False):
        return round_(self.p, self.x, self.y, self.step, self.status, peek)


def validity_violations(p: Params, x, y, step) -> int:
    x, y, step = _i32(x), _i32(y), _i32(step)
    return int(lib().orc_validity_violations(C.byref(p), len(x), _p(x), _p(y), _p(step)))


def coupled(p, a, b) -> bool:
    return bool(lib().orc_coupled(C.byref(p), *map(int, a), *map(int, b)))


def blocked_by(p, a, b) -> bool:
    return bool(lib().orc_blocked_by(C.byref(p), *map(int, a), *map(int, b)))


def mix64(x: int) -> int:
    return int(lib().orc_mix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def key3(seed: int, a: int, b: int) -> int:
    m = 0xFFFFFFFFFFFFFFFF
    return int(lib().orc_key3(seed & m, a & m, b & m))


class SynthTables:
    """Keeps the numpy arrays alive while the C struct points into them."""

    def __init__(self, lat, cdf32, vals, base_us, lat_seed, policy_seed, wall=None,
                 dur_table=None, policy=0, conflict=0, graph=None):
        self.lat = np.ascontiguousarray(lat, np.uint32)
        self.cdf32 = np.ascontiguousarray(cdf32, np.uint64)
        self.vals = np.ascontiguousarray(vals, np.int32)
        self.wall = None if wall is None else np.ascontiguousarray(wall, np.uint8)
        self.dur = None if dur_table is None else np.ascontiguousarray(dur_table, np.int64)
        self.goff = None if graph is None else np.ascontiguousarray(graph[0], np.int32)
        self.gadj = None if graph is None else np.ascontiguousarray(graph[1], np.int32)
        self.s = Synth(_p(self.lat).value, _p(self.cdf32).value, _p(self.vals).value,
                       len(self.vals), int(base_us), int(lat_seed), int(policy_seed),
                       None if self.wall is None else _p(self.wall).value,
                       None if self.dur is None else _p(self.dur).value,
                       0 if self.dur is None else self.dur.shape[1], int(policy), int(conflict),
                       None if graph is None else _p(self.goff).value,
                       None if graph is None else _p(self.gadj).value)

    @classmethod
    def from_model(cls, lm, wall=None, dur_table=None, policy=0, conflict=0, graph=None):
        """graph: (offsets, neighbours) CSR adjacency for the graph walk (policy 3)."""
        return cls(lm.lat, lm.cdf32, lm.vals, lm.base_us, lm.lat_seed, lm.policy_seed, wall,
                   dur_table, policy, conflict, graph)


def duration(sy: SynthTables, i: int, s: int) -> int:
    return int(lib().orc_duration(C.byref(sy.s), int(i), int(s)))


def digest(p: Params, x, y, step, status, i, lo=0, hi=None) -> int:
    x, y, step = _i32(x), _i32(y), _i32(step)
    status = np.ascontiguousarray(status, np.uint8)
    hi = len(x) if hi is None else hi
    return int(lib().orc_digest(C.byref(p), lo, hi, _p(x), _p(y), _p(step), _p(status), int(i)))


def policy_move(p: Params, sy: SynthTables, i, s, px, py, dig):
    nx = np.zeros(1, np.int32)
    ny = np.zeros(1, np.int32)
    lib().orc_policy_move(C.byref(p), C.byref(sy.s), int(i), int(s), int(px), int(py),
                          C.c_uint64(dig & 0xFFFFFFFFFFFFFFFF), _p(nx), _p(ny))
    return int(nx[0]), int(ny[0])


def lockstep(p: Params, sy: SynthTables, x0, y0, T: int):
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    traj = np.zeros(n, np.uint64)
    tsync = np.zeros(p.n_sims, np.int64)
    rc = lib().orc_lockstep(C.byref(p), C.byref(sy.s), n, int(T), _p(x), _p(y), _p(traj), _p(tsync))
    if rc != OK:
        raise RuntimeError(f"orc_lockstep rc={rc}")
    return dict(x=x, y=y, traj=traj, T_sync=tsync)


class _LogBufs:
    """The per-round log arrays of a replay (orc_log)."""

    def __init__(self, log_rounds: int, log_entries: int, check: bool):
        self.caps = (log_rounds, log_entries)
        self.rt = np.zeros(max(log_rounds, 1), np.int64)
        self.rs = np.zeros(max(log_rounds, 1), np.int32)
        self.rn = np.zeros(max(log_rounds, 1), np.int32)
        self.eid = np.zeros(max(log_entries, 1), np.int32)
        self.elab = np.zeros(max(log_entries, 1), np.int32)
        self.lg = Log(log_rounds, log_entries, _p(self.rt).value, _p(self.rs).value, _p(self.rn).value,
                      _p(self.eid).value, _p(self.elab).value, 0, 0, int(check), 0, 0)

    def result(self, **kw):
        lg, (cr, ce) = self.lg, self.caps
        nr, ne = min(lg.n_rounds, cr), min(lg.n_entries, ce)
        return dict(kw, log_t=self.rt[:nr].copy(), log_sim=self.rs[:nr].copy(), log_nready=self.rn[:nr].copy(),
                    log_id=self.eid[:ne].copy(), log_label=self.elab[:ne].copy(),
                    log_complete=(lg.n_rounds <= cr and lg.n_entries <= ce),
                    violations=int(lg.violations), max_spread=int(lg.max_spread))


def replay(p: Params, sy: SynthTables, x0, y0, Q: int = 0, log_rounds: int = 0,
           log_entries: int = 0, check: bool = False, capacity: int = 0, priority: bool = True):
    """Out-of-order replay (orc_replay; orc_replay_cap with a finite capacity of
    `capacity` agent-steps in service, clusters started in step-priority or FIFO order).
    p.target is the number of steps."""
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    traj = np.zeros(n, np.uint64)
    tooo = np.zeros(p.n_sims, np.int64)
    rounds = np.zeros(p.n_sims, np.int64)
    lb = _LogBufs(log_rounds, log_entries, check)
    rc = lib().orc_replay_cap(C.byref(p), C.byref(sy.s), n, int(Q), int(capacity), int(bool(priority)), _p(x),
                              _p(y), _p(traj), _p(tooo), _p(rounds), C.byref(lb.lg))
    if rc != OK:
        raise RuntimeError(f"orc_replay rc={rc}")
    return lb.result(x=x, y=y, traj=traj, T_ooo=tooo, rounds=rounds)


def replay_stale(p: Params, sy: SynthTables, x0, y0, G: int, P: int, Q: int = 0, log_rounds: int = 0,
                 log_entries: int = 0, check: bool = False):
    """Stale-halo replay over G horizontal slabs with a sync round every P rounds
    (orc_replay_stale).  One simulation; P = 1 is replay()."""
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    traj = np.zeros(n, np.uint64)
    tooo = np.zeros(1, np.int64)
    rounds = np.zeros(1, np.int64)
    lb = _LogBufs(log_rounds, log_entries, check)
    rc = lib().orc_replay_stale(C.byref(p), C.byref(sy.s), n, int(Q), int(G), int(P), _p(x), _p(y), _p(traj),
                                _p(tooo), _p(rounds), C.byref(lb.lg))
    if rc != OK:
        raise RuntimeError(f"orc_replay_stale rc={rc}")
    return lb.result(x=x, y=y, traj=traj, T_ooo=tooo, rounds=rounds)


# ------------------------------------------------------------------ at BASELINE sizes
# (oracle_scale.c: the same predicates of oracle.c with threaded outer loops)
def round_mt(p: Params, x, y, step, status, peek=False, threads: int | None = None):
    """orc_round (one simulation) with the outer loops over agents split across host
    threads; every pair is still tested.  Same outputs as round_()."""
    x, y, step = _i32(x), _i32(y), _i32(step)
    n = len(x)
    assert status.dtype == np.uint8 and status.flags.c_contiguous
    blocked = np.zeros(n, np.uint8)
    label = np.zeros(n, np.int32)
    mask = np.zeros(n, np.uint8)
    order = np.zeros(max(n, 1), np.int32)
    nr = np.zeros(1, np.int32)
    rc = lib().orc_round_mt(C.byref(p), n, _p(x), _p(y), _p(step), _p(status), int(bool(peek)),
                            _p(blocked), _p(label), _p(mask), _p(order), _p(nr), int(threads or host_threads()))
    if rc != OK:
        raise RuntimeError(f"orc_round_mt rc={rc}")
    return dict(blocked=blocked, label=label, mask=mask, order=order[: nr[0]].copy())


def labels_steps(p: Params, x, y, step, status, threads: int | None = None) -> np.ndarray:
    """Cluster label (min id, -1 DONE) of every agent: all same-step pairs tested."""
    x, y, step = _i32(x), _i32(y), _i32(step)
    status = np.ascontiguousarray(status, np.uint8)
    label = np.zeros(len(x), np.int32)
    rc = lib().orc_labels_steps(C.byref(p), len(x), _p(x), _p(y), _p(step), _p(status), _p(label),
                                int(threads or host_threads()))
    if rc != OK:
        raise RuntimeError(f"orc_labels_steps rc={rc}")
    return label


def blocked_list(p: Params, x, y, step, status, idx, threads: int | None = None) -> np.ndarray:
    """Blocking verdict of the listed agents, each by a scan over all agents."""
    x, y, step = _i32(x), _i32(y), _i32(step)
    status = np.ascontiguousarray(status, np.uint8)
    idx = _i32(idx)
    out = np.zeros(len(idx), np.uint8)
    rc = lib().orc_blocked_list(C.byref(p), len(x), _p(x), _p(y), _p(step), _p(status), len(idx), _p(idx),
                                _p(out), int(threads or host_threads()))
    if rc != OK:
        raise RuntimeError(f"orc_blocked_list rc={rc}")
    return out


def round_at_scale(p: Params, x, y, step, status, sample, threads: int | None = None):
    """The round's outputs where they can be computed exactly at 1M agents: the label
    of EVERY agent (labels_steps), and for the sampled agents the blocking verdict and
    the ready bit -- the latter from the blocking verdicts of every member of the
    agent's cluster (cluster-ready rule P:162 / P:184) and the members' statuses."""
    status = np.ascontiguousarray(status, np.uint8)
    label = labels_steps(p, x, y, step, status, threads)
    sample = _i32(sample)
    comp = np.isin(label, np.unique(label[sample][label[sample] >= 0]))
    members = np.flatnonzero(comp).astype(np.int32)
    blk_m = blocked_list(p, x, y, step, status, members, threads)
    blocked = np.zeros(len(x), np.uint8)
    blocked[members] = blk_m
    bad = {}
    for i, b in zip(members.tolist(), blk_m.tolist()):
        lab = int(label[i])
        bad[lab] = bad.get(lab, False) or bool(b) or int(status[i]) == RUNNING
    mask = np.array([int(status[i]) == IDLE and not bad.get(int(label[i]), False) if label[i] >= 0 else False
                     for i in sample.tolist()], np.uint8)
    return dict(label=label, blocked=blocked[sample], mask=mask, members=members)


def lockstep_grid(p: Params, sy: SynthTables, x0, y0, T: int, threads: int | None = None):
    """orc_lockstep (one simulation, co-occupancy) with the perceived sets gathered
    through an oracle-private hash grid (perception only; outputs identical)."""
    if sy.s.conflict:
        raise ValueError("lockstep_grid: co-occupancy only (use lockstep for exclusive tiles)")
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    traj = np.zeros(n, np.uint64)
    tsync = np.zeros(1, np.int64)
    rc = lib().orc_lockstep_grid(C.byref(p), C.byref(sy.s), n, int(T), _p(x), _p(y), _p(traj), _p(tsync),
                                 int(threads or host_threads()))
    if rc != OK:
        raise RuntimeError(f"orc_lockstep_grid rc={rc}")
    return dict(x=x, y=y, traj=traj, T_sync=tsync)


def replay_mt(p: Params, sy: SynthTables, x0, y0, Q: int = 0, capacity: int = 0, priority: bool = True,
              threads: int | None = None):
    """orc_replay_cap with the simulations of a batch replayed concurrently (final states,
    T_ooo and round counts only; identical to replay())."""
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    traj = np.zeros(n, np.uint64)
    tooo = np.zeros(p.n_sims, np.int64)
    rounds = np.zeros(p.n_sims, np.int64)
    rc = lib().orc_replay_mt(C.byref(p), C.byref(sy.s), n, int(Q), int(capacity), int(bool(priority)), _p(x), _p(y),
                             _p(traj), _p(tooo), _p(rounds), int(threads or host_threads()))
    if rc != OK:
        raise RuntimeError(f"orc_replay_mt rc={rc}")
    return dict(x=x, y=y, traj=traj, T_ooo=tooo, rounds=rounds)


def replay_sims_logged(p: Params, sy: SynthTables, x0, y0, sims, Q: int = 0, log_rounds: int = 10**6,
                       log_entries: int = 10**6):
    """The replay of selected simulations of a batch, each with its own round log (the
    loop body of orc_replay for simulation b, run alone).  Returns {b: dict(log_nready,
    log_id, log_label, T_ooo, rounds, traj of the simulation's agents)}."""
    x, y = _i32(x0).copy(), _i32(y0).copy()
    n = len(x)
    out = {}
    for b in sims:
        traj = np.zeros(n, np.uint64)
        tooo = np.zeros(p.n_sims, np.int64)
        rounds = np.zeros(p.n_sims, np.int64)
        rt = np.zeros(log_rounds, np.int64)
        rs = np.zeros(log_rounds, np.int32)
        rn = np.zeros(log_rounds, np.int32)
        eid = np.zeros(log_entries, np.int32)
        elab = np.zeros(log_entries, np.int32)
        lg = Log(log_rounds, log_entries, _p(rt).value, _p(rs).value, _p(rn).value, _p(eid).value,
                 _p(elab).value, 0, 0, 0, 0, 0)
        xb, yb = x.copy(), y.copy()
        rc = lib().orc_replay_sim_logged(C.byref(p), C.byref(sy.s), n, int(Q), int(b), _p(xb), _p(yb), _p(traj),
                                         _p(tooo), _p(rounds), C.byref(lg))
        if rc != OK:
            raise RuntimeError(f"orc_replay_sim_logged rc={rc}")
        assert lg.n_rounds <= log_rounds and lg.n_entries <= log_entries
        lo, hi = b * n // p.n_sims, (b + 1) * n // p.n_sims
        out[b] = dict(log_nready=rn[: lg.n_rounds].copy(), log_id=eid[: lg.n_entries].copy(),
                      log_label=elab[: lg.n_entries].copy(), T_ooo=int(tooo[b]), rounds=int(rounds[b]),
                      traj=traj[lo:hi].copy(), x=xb[lo:hi].copy(), y=yb[lo:hi].copy())
    return out
