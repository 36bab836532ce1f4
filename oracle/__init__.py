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
* duration / policy_move / digest (synthetic driver, Q16): the paper is silent;
  parity unpinned by the paper (pinned only by splitmix64's published value).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

IDLE, RUNNING, DONE = 0, 1, 2
L2, LINF = 0, 1
OK, E_ARG, E_BOUNDS, E_PROTOCOL, E_VELOCITY, E_LIVENESS = 0, -1, -2, -3, -4, -8


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain -O2, no vectorisation tricks)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
            os.replace(tmp, _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [("map_w", C.c_int32), ("map_h", C.c_int32), ("r_p", C.c_int32),
                ("v", C.c_int32), ("target", C.c_int32), ("metric", C.c_int32),
                ("n_sims", C.c_int32)]


class Synth(C.Structure):
    _fields_ = [("lat", C.c_void_p), ("cdf32", C.c_void_p), ("vals", C.c_void_p),
                ("n_vals", C.c_int32), ("base_us", C.c_int32), ("lat_seed", C.c_uint64),
                ("policy_seed", C.c_uint64), ("wall", C.c_void_p),
                ("dur_table", C.c_void_p), ("dur_T", C.c_int32), ("policy", C.c_int32),
                ("conflict", C.c_int32)]


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
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def params(map_w, map_h, r_p, v, target=0, metric=L2, n_sims=1) -> Params:
    return Params(int(map_w), int(map_h), int(r_p), int(v), int(target), int(metric), int(n_sims))


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
                 dur_table=None, policy=0, conflict=0):
        self.lat = np.ascontiguousarray(lat, np.uint32)
        self.cdf32 = np.ascontiguousarray(cdf32, np.uint64)
        self.vals = np.ascontiguousarray(vals, np.int32)
        self.wall = None if wall is None else np.ascontiguousarray(wall, np.uint8)
        self.dur = None if dur_table is None else np.ascontiguousarray(dur_table, np.int64)
        self.s = Synth(_p(self.lat).value, _p(self.cdf32).value, _p(self.vals).value,
                       len(self.vals), int(base_us), int(lat_seed), int(policy_seed),
                       None if self.wall is None else _p(self.wall).value,
                       None if self.dur is None else _p(self.dur).value,
                       0 if self.dur is None else self.dur.shape[1], int(policy), int(conflict))

    @classmethod
    def from_model(cls, lm, wall=None, dur_table=None, policy=0, conflict=0):
        return cls(lm.lat, lm.cdf32, lm.vals, lm.base_us, lm.lat_seed, lm.policy_seed, wall,
                   dur_table, policy, conflict)


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
    rt = np.zeros(max(log_rounds, 1), np.int64)
    rs = np.zeros(max(log_rounds, 1), np.int32)
    rn = np.zeros(max(log_rounds, 1), np.int32)
    eid = np.zeros(max(log_entries, 1), np.int32)
    elab = np.zeros(max(log_entries, 1), np.int32)
    lg = Log(log_rounds, log_entries, _p(rt).value, _p(rs).value, _p(rn).value, _p(eid).value,
             _p(elab).value, 0, 0, int(check), 0, 0)
    rc = lib().orc_replay_cap(C.byref(p), C.byref(sy.s), n, int(Q), int(capacity), int(bool(priority)), _p(x),
                              _p(y), _p(traj), _p(tooo), _p(rounds), C.byref(lg))
    if rc != OK:
        raise RuntimeError(f"orc_replay rc={rc}")
    nr = min(lg.n_rounds, log_rounds)
    ne = min(lg.n_entries, log_entries)
    return dict(x=x, y=y, traj=traj, T_ooo=tooo, rounds=rounds,
                log_t=rt[:nr].copy(), log_sim=rs[:nr].copy(), log_nready=rn[:nr].copy(),
                log_id=eid[:ne].copy(), log_label=elab[:ne].copy(),
                log_complete=(lg.n_rounds <= log_rounds and lg.n_entries <= log_entries),
                violations=int(lg.violations), max_spread=int(lg.max_spread))
