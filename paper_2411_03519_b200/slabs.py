"""Spatial-slab decomposition of the tracker and the replay driver across GPUs
(include/am_slab.h) -- marshalling and collectives only.

Every data-path step runs in libametro.so's kernels (am_slab.cu + the window's
incremental tracker); this module passes device pointers and runs the three collectives
of a round on fixed-capacity buffers whose counts travel inside them, so no round
synchronises the host:

  1. am_slab_round_local  -> ALL-GATHER of the merge buffers (link / cluster records)
  2. am_slab_merge        -> ALL-REDUCE MIN of the stats {next event, W, -S, inactive}
  3. am_slab_commit       -> ALL-TO-ALL of the delta blocks (commits in other windows)
  4. am_slab_apply

With stale_rounds = P > 1 (stale-halo rounds, NEXT #3) only every P-th round is such a
sync round; the rounds in between run am_slab_round_stale (no all-gather, no merge)
against the ghosts of the last exchange, and the all-to-all runs only before a sync
round -- one all-reduce per stale round (the common clock).

The exchange is torch.distributed (NCCL over NVLink, one process per GPU:
``DistWorld``) or an in-process loopback of G virtual slabs on one GPU
(``LoopbackWorld``); both drive the identical library calls.  Every K rounds (and at
the end) the flags are read (one host synchronisation): capacity overflows raise,
a halo that the step spread is about to outgrow triggers a re-window (the global state
is gathered once and every rank reloads a wider window) -- the spread grows by at most
one step per round and the library raises the flag K rounds early, so every round is
exact.
"""
from __future__ import annotations

import ctypes as C
import numpy as np
import torch

from . import _lib
from ._lib import check

IDLE, RUNNING, DONE = _lib.IDLE, _lib.RUNNING, _lib.DONE
OVF_WINDOW, OVF_PEER, OVF_MERGE, HALO, LIVENESS, LAG = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
NEVER = 2**63 - 1


def slab_of_rows(map_h: int, n_slabs: int):
    """Row range [lo, hi) of every slab (the kernels' formula)."""
    return [(k * map_h // n_slabs, (k + 1) * map_h // n_slabs) for k in range(n_slabs)]


def partition(y: torch.Tensor, map_h: int, n_slabs: int) -> torch.Tensor:
    """Slab of each agent (its row's slab): the last k with floor(k*H/G) <= y."""
    return ((y.to(torch.int64) + 1) * n_slabs - 1) // map_h


class _DevArray:
    """Zero-copy view of a device array owned by the library (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr, shape, dtype, device):
    ts = {torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_DevArray(ptr, shape, ts), device=device)


def halo_needed(spread: int, r_p: int, v: int, K: int, P: int = 1) -> int:
    """Window rows that keep the next K rounds exact: R_b(spread + 1) + (K + 1) v,
    plus 2 P v with stale-halo rounds (owned agents drift up to P v out of the slab and
    the ghosts' snapshot is up to P rounds old)."""
    return (spread + 2) * v + r_p + (K + 1) * v + (2 * P * v if P > 1 else 0)


class SlabRank:
    """One rank's slab: its window, the window's tracker and the exchange buffers."""

    def __init__(self, map_w, map_h, r_p, v, n_total, n_slabs, my_slab, target, synth, quantum_us, *,
                 halo, cap_window, cap_peer, cap_merge, check_rounds=16, metric="l2", device="cuda",
                 stream=None, stale_rounds=1):
        self.L = _lib.load()
        self.dev = torch.device(device)
        self.G, self.k = int(n_slabs), int(my_slab)
        self.map_w, self.map_h, self.r_p, self.v = int(map_w), int(map_h), int(r_p), int(v)
        self.n_total, self.target = int(n_total), int(target)
        self.cap_merge = int(cap_merge) + (int(cap_merge) & 1)
        self.g = _lib.SlabGeom(self.map_w, self.map_h, self.r_p, self.v,
                               _lib.METRIC_LINF if metric == "linf" else _lib.METRIC_L2, self.G, self.k,
                               self.n_total, self.target, int(halo), int(cap_window), int(cap_peer),
                               self.cap_merge, int(check_rounds), int(stale_rounds))
        self.halo, self.cap_window, self.cap_peer = int(halo), int(cap_window), int(cap_peer)
        self.lo, self.hi = slab_of_rows(self.map_h, self.G)[self.k]
        self.y0, self.y1 = max(0, self.lo - self.halo), min(self.map_h, self.hi + self.halo)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        nbytes = int(self.L.am_slab_workspace_size(C.byref(self.g)))
        if nbytes == 0:
            raise ValueError("am_slab_workspace_size: invalid slab geometry")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.dev)
        ws = (self.workspace.data_ptr() + 255) & ~255
        self.synth = synth   # keeps the tables alive
        h = C.c_void_p()
        check(self.L.am_slab_create(C.byref(h), C.byref(self.g), C.byref(synth.s), int(quantum_us), ws, nbytes,
                                    self.stream.cuda_stream))
        self.h = h
        d = self.dev
        self.mwords = 4 + 6 * self.cap_merge
        self.dwords = 6 + 12 * self.cap_peer
        self.mbuf = torch.zeros(self.mwords, dtype=torch.int32, device=d)
        self.dsend = torch.zeros((self.G, self.dwords), dtype=torch.int32, device=d)
        self.stats = torch.zeros(4, dtype=torch.int64, device=d)
        self.order = torch.zeros(self.cap_window, dtype=torch.int32, device=d)
        self.n_order = torch.zeros(1, dtype=torch.int32, device=d)
        # zero-copy views of the library's window arrays
        pp = [C.c_void_p() for _ in range(7)]
        check(self.L.am_slab_state(h, *[C.byref(p) for p in pp]))
        Lw = self.cap_window
        self.w_pos = _view(pp[0].value, (Lw, 2), torch.int32, d)
        self.w_step = _view(pp[1].value, (Lw,), torch.int32, d)
        self.w_stat = _view(pp[2].value, (Lw,), torch.uint8, d)
        self.w_traj = _view(pp[3].value, (Lw,), torch.int64, d)
        self.w_tc = _view(pp[4].value, (Lw,), torch.int64, d)
        self.w_np = _view(pp[5].value, (Lw, 2), torch.int32, d)
        self.counters = _view(pp[6].value, (4,), torch.int64, d)
        oo = [C.c_void_p() for _ in range(3)]
        check(self.L.am_slab_outputs(h, *[C.byref(p) for p in oo]))
        self.w_gid = _view(oo[0].value, (Lw,), torch.int32, d)
        self.w_label = _view(oo[1].value, (Lw,), torch.int32, d)
        self.w_ready = _view(oo[2].value, (Lw,), torch.uint8, d)
        ow = C.c_void_p()
        check(self.L.am_slab_owned(h, C.byref(ow)))
        self.w_own = _view(ow.value, (Lw,), torch.uint8, d)

    # ------------------------------------------------------------------ library steps
    def load(self, gid, pos, steps, status, traj=None, tcommit=None, newpos=None, t: int = 0):
        m = int(gid.numel())
        if m > self.cap_window:
            raise ValueError("window capacity exceeded")
        args = [gid, pos, steps, status, traj, tcommit, newpos]
        self._keep = [a.contiguous() if a is not None else None for a in args]
        ptrs = [a.data_ptr() if a is not None else None for a in self._keep]
        check(self.L.am_slab_load(self.h, m, *ptrs, int(t)))

    def round_local(self):
        check(self.L.am_slab_round_local(self.h, self.mbuf.data_ptr()))
        return self.mbuf

    def merge(self, mbufs: torch.Tensor):
        check(self.L.am_slab_merge(self.h, mbufs.data_ptr(), self.order.data_ptr(), self.n_order.data_ptr(),
                                   self.stats.data_ptr()))
        return self.stats

    def round_stale(self):
        check(self.L.am_slab_round_stale(self.h, self.order.data_ptr(), self.n_order.data_ptr(),
                                         self.stats.data_ptr()))
        return self.stats

    def commit(self, stats_global: torch.Tensor, exchange: bool = True):
        """exchange=False: the commits stay local until the next exchange (stale rounds)."""
        check(self.L.am_slab_commit(self.h, stats_global.data_ptr(), self.dsend.data_ptr() if exchange else None))
        return self.dsend

    def apply(self, drecv: torch.Tensor):
        check(self.L.am_slab_apply(self.h, drecv.data_ptr()))

    def wait_order(self):
        """The slab's stream waits for the rank's priority sort (side stream)."""
        check(self.L.am_slab_wait_order(self.h))

    def order_ms(self) -> float:
        """Device time of the last priority sort (ms; synchronises on it)."""
        ms = C.c_float(0.0)
        check(self.L.am_slab_order_ms(self.h, C.byref(ms)))
        return float(ms.value)

    def flags(self):
        f, used = C.c_int32(0), C.c_int32(0)
        check(self.L.am_slab_flags(self.h, C.byref(f), C.byref(used)))
        return f.value, used.value

    def tracker_ctx(self):
        return self.L.am_slab_tracker(self.h)

    # ------------------------------------------------------------------ views
    def owned_mask(self) -> torch.Tensor:
        return (self.w_gid >= 0) & (self.w_own != 0)

    def owned_state(self):
        """The owned agents (every field needed to reload them anywhere)."""
        m = self.owned_mask()
        return dict(gid=self.w_gid[m].clone(), pos=self.w_pos[m].clone(), steps=self.w_step[m].clone(),
                    status=self.w_stat[m].clone(), traj=self.w_traj[m].clone(), tcommit=self.w_tc[m].clone(),
                    newpos=self.w_np[m].clone())

    def round_outputs(self):
        """This rank's ready agents (global ids in priority order) and, for every owned
        agent, (gid, global label, ready bit)."""
        self.wait_order()
        n = int(self.n_order.item())
        m = self.owned_mask()
        return dict(order=self.order[:n].clone(), gid=self.w_gid[m].clone(), label=self.w_label[m].clone(),
                    ready=self.w_ready[m].clone(), step=self.w_step[m].clone())

    def close(self):
        if getattr(self, "h", None):
            self.L.am_slab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------- worlds
class _World:
    """Common driver: setup from a global initial state, rounds, checks, re-windows."""

    def _geometry(self, y_all: torch.Tensor, spread: int, K: int, halo: int | None = None):
        H = halo if halo is not None else halo_needed(spread, self.r_p, self.v, K, self.P)
        H = max(H, self.r_p + (self.P + 1) * self.v)
        H = min(H, self.map_h)
        # capacities from the actual distribution, with slack for migration
        rows = slab_of_rows(self.map_h, self.G)
        y = y_all.to(torch.int64)
        wins, bands = [], []
        for lo, hi in rows:
            y0, y1 = max(0, lo - H), min(self.map_h, hi + H)
            wins.append(int(((y >= y0) & (y < y1)).sum()))
            bnd = ((y >= lo - H) & (y < lo + H)) | ((y >= hi - H) & (y < hi + H))
            bands.append(int(bnd.sum()))
        cap_window = int(max(wins) * 1.25) + 2048
        cap_merge = int(max(bands) * 1.5) + 2048
        cap_peer = int(max(bands) * min(1.0, 0.5 * self.P)) + 2048   # one record per agent per exchange
        return H, cap_window, cap_merge, cap_peer

    def _schedule(self):
        """(sync, exchange) of the next round: a sync round every P rounds, the exchange
        after the commits of the round before one."""
        r = self.rounds_done
        return r % self.P == 0, (r + 1) % self.P == 0

    def _set_period(self, K: int, stale_rounds: int):
        self.P = max(1, int(stale_rounds))
        if K % self.P:
            raise ValueError("check_rounds must be a multiple of stale_rounds (re-windows happen at exchanges)")

    @staticmethod
    def _window_select(st: dict, lo: int, hi: int, H: int, map_h: int):
        y = st["pos"][:, 1]
        sel = (y >= max(0, lo - H)) & (y < min(map_h, hi + H))
        return {k: v[sel].contiguous() for k, v in st.items()}


def _spread(steps0, status0) -> int:
    """S - W over the agents that are not DONE (0 for the all-at-step-0 start)."""
    if steps0 is None:
        return 0
    s = np.asarray(steps0)
    if status0 is not None:
        s = s[np.asarray(status0) != DONE]
    return int(s.max() - s.min()) if len(s) else 0


def _initial_state(x0, y0, steps0, status0, dev):
    """Every agent's replay state at time 0 (all IDLE at step 0 unless given)."""
    n = len(x0)
    pos = torch.as_tensor(np.stack([np.asarray(x0), np.asarray(y0)], 1).reshape(n, 2), dtype=torch.int32,
                          device=dev)
    return dict(gid=torch.arange(n, dtype=torch.int32, device=dev), pos=pos,
                steps=(torch.zeros(n, dtype=torch.int32, device=dev) if steps0 is None else
                       torch.as_tensor(np.asarray(steps0), dtype=torch.int32, device=dev)),
                status=(torch.zeros(n, dtype=torch.uint8, device=dev) if status0 is None else
                        torch.as_tensor(np.asarray(status0), dtype=torch.uint8, device=dev)),
                traj=torch.zeros(n, dtype=torch.int64, device=dev),
                tcommit=torch.full((n,), NEVER, dtype=torch.int64, device=dev), newpos=pos.clone())


class LoopbackWorld(_World):
    """G virtual slabs in one process on one GPU (the exchanges are device copies on one
    stream): the same library calls as the NCCL run, bit-exact against it by design."""

    def __init__(self, map_w, map_h, r_p, v, x0, y0, target, synth, quantum_us, n_slabs, *, metric="l2",
                 check_rounds=16, device="cuda", halo=None, steps0=None, status0=None, stale_rounds=1):
        self.map_w, self.map_h, self.r_p, self.v = int(map_w), int(map_h), int(r_p), int(v)
        self.G, self.target, self.synth, self.Q = int(n_slabs), int(target), synth, int(quantum_us)
        self.metric, self.K, self.dev = metric, int(check_rounds), torch.device(device)
        self._set_period(self.K, stale_rounds)
        st = _initial_state(x0, y0, steps0, status0, self.dev)
        self.n = len(x0)
        self.ranks = []
        self.rounds_done = 0
        self.rewindows = 0
        self._carry = (0, 0, 0)   # counters of the slabs before the last re-window
        self._setup(st, 0, spread=_spread(steps0, status0), halo=halo)

    def _setup(self, st: dict, t: int, spread: int, halo=None):
        for r in self.ranks:
            r.close()
        H, cw, cm, cp = self._geometry(st["pos"][:, 1], spread, self.K, halo)
        self.halo = H
        self.ranks = []
        for k in range(self.G):
            r = SlabRank(self.map_w, self.map_h, self.r_p, self.v, self.n, self.G, k, self.target, self.synth,
                         self.Q, halo=H, cap_window=cw, cap_peer=cp, cap_merge=cm, check_rounds=self.K,
                         metric=self.metric, device=self.dev, stale_rounds=self.P)
            w = self._window_select(st, r.lo, r.hi, H, self.map_h)
            r.load(w["gid"], w["pos"], w["steps"], w["status"], w["traj"], w["tcommit"], w["newpos"], t)
            self.ranks.append(r)

    def round(self, log: list | None = None, timing: list | None = None):
        """One distributed round of all virtual slabs (no host synchronisation unless
        `log` asks for the round's outputs).  With `timing` (a list), the device time of
        every rank's own library steps (everything but the exchanges, which NCCL does in
        a real run) is appended, per rank, in ms: what one GPU of a G-GPU run computes
        (its side-stream restore + sort counted where they outlast commit + apply)."""
        sync, exchange = self._schedule()
        ev = [[] for _ in self.ranks]

        def phase(k, fn):
            if timing is None:
                return fn()
            # the device sleeps while the host enqueues the rank's phase, so the events
            # bracket its kernels running back to back (device time, not the host's
            # launch rate)
            torch.cuda._sleep(3_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            ev[k].append((e0, e1))
            return out

        if sync:
            mbs = [phase(k, r.round_local) for k, r in enumerate(self.ranks)]
            mb = torch.stack(mbs)                                           # all-gather
            for k, r in enumerate(self.ranks):
                phase(k, lambda r=r: r.merge(mb))
        else:
            for k, r in enumerate(self.ranks):
                phase(k, r.round_stale)
        if log is not None:
            log.append([r.round_outputs() for r in self.ranks])
        sg = torch.stack([r.stats for r in self.ranks]).min(0).values       # all-reduce MIN
        dss = [phase(k, lambda r=r: r.commit(sg, exchange)) for k, r in enumerate(self.ranks)]
        if exchange:
            ds = torch.stack(dss)                                           # [src, dst, words]
            for k, r in enumerate(self.ranks):
                recv = ds[:, k].contiguous()                                # all-to-all
                phase(k, lambda r=r, recv=recv: r.apply(recv))
        self.rounds_done += 1
        self._last_stats = sg
        if timing is not None:
            torch.cuda.synchronize(self.dev)
            # per rank: its phases on its stream, plus the part of its side-stream work
            # (merge-forest restore + priority sort, started at the end of the merge /
            # stale phase) that outlasts the phases after it (commit, apply) -- in a G-GPU
            # run it also overlaps the all-reduce and the all-to-all, not counted here
            tot = []
            for k, r in enumerate(self.ranks):
                ph = [a.elapsed_time(b) for a, b in ev[k]]
                after = sum(ph[2:]) if sync else sum(ph[1:])
                tot.append(sum(ph) + max(0.0, r.order_ms() - after))
            timing.append(tot)

    def check(self) -> bool:
        """Reads every rank's flags (one synchronisation).  Raises on an overflow or a
        liveness failure, re-windows when the halo is about to be outgrown.  Returns True
        when every agent is DONE."""
        flags = 0
        for r in self.ranks:
            f, _ = r.flags()
            flags |= f
        if flags & (OVF_WINDOW | OVF_PEER | OVF_MERGE | LAG):
            raise RuntimeError(f"slab exchange overflow (flags {flags:#x})")
        if flags & LIVENESS:
            raise RuntimeError("replay: agents not DONE but nothing running (liveness)")
        sg = self._last_stats.tolist()
        if flags & HALO:
            self.rewindow(spread=-sg[2] - sg[1])
        return sg[3] == 1

    def rewindow(self, spread: int):
        """Gathers the global state and reloads every rank with a window twice as wide as
        the spread needs now."""
        parts = [r.owned_state() for r in self.ranks]
        st = {k: torch.cat([p[k] for p in parts]) for k in parts[0]}
        cnt = torch.stack([r.counters for r in self.ranks]).cpu().numpy()
        self._carry = (max(self._carry[0], int(cnt[:, 1].max())), self._carry[1] + int(cnt[:, 2].sum()),
                       self._carry[2] + int(cnt[0, 3]))   # finishing time, dispatched, rounds
        t = int(cnt[0, 0])
        need = halo_needed(spread, self.r_p, self.v, self.K, self.P)
        self._setup(st, t, spread, halo=2 * need)
        self.rewindows += 1

    def run(self, max_rounds: int) -> int:
        """Rounds until every agent is DONE (checked every K rounds); returns the rounds run."""
        done = 0
        while done < max_rounds:
            for _ in range(min(self.K, max_rounds - done)):
                self.round()
                done += 1
            if self.check():
                break
        return done

    def results(self):
        """The final (or current) state of every agent, in global-id order, T_ooo, rounds."""
        parts = [r.owned_state() for r in self.ranks]
        gid = torch.cat([p["gid"] for p in parts]).long()
        n = self.n
        out = {}
        for k in ("pos", "steps", "traj"):
            v = torch.cat([p[k] for p in parts])
            o = torch.zeros((n,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
            o[gid] = v
            out[k] = o.cpu().numpy()
        cnt = torch.stack([r.counters for r in self.ranks]).cpu().numpy()
        assert len(np.unique(gid.cpu().numpy())) == n, "every agent owned exactly once"
        return dict(x=out["pos"][:, 0], y=out["pos"][:, 1], steps=out["steps"],
                    traj=out["traj"].view(np.uint64), T_ooo=max(self._carry[0], int(cnt[:, 1].max())),
                    rounds=self._carry[2] + int(cnt[0, 3]), dispatched=self._carry[1] + int(cnt[:, 2].sum()))

    def dispatched(self) -> int:
        """Agent-steps dispatched so far by all ranks (synchronises)."""
        return self._carry[1] + int(torch.stack([r.counters for r in self.ranks])[:, 2].sum().item())

    def close(self):
        for r in self.ranks:
            r.close()
        self.ranks = []


class DistWorld(_World):
    """One slab per process over torch.distributed (NCCL on GPUs; every collective runs on
    the current stream with fixed-size device buffers -- no host synchronisation per
    round).  `dist` may be torch.distributed or any object with the same four calls
    (tests stage gloo through the host)."""

    def __init__(self, dist, map_w, map_h, r_p, v, x0, y0, target, synth, quantum_us, *, metric="l2",
                 check_rounds=16, device="cuda", halo=None, steps0=None, status0=None, stale_rounds=1):
        self.dist = dist
        self.G, self.k = dist.get_world_size(), dist.get_rank()
        self.map_w, self.map_h, self.r_p, self.v = int(map_w), int(map_h), int(r_p), int(v)
        self.target, self.synth, self.Q = int(target), synth, int(quantum_us)
        self.metric, self.K, self.dev = metric, int(check_rounds), torch.device(device)
        self._set_period(self.K, stale_rounds)
        st = _initial_state(x0, y0, steps0, status0, self.dev)
        self.n = len(x0)
        self.rank = None
        self.rounds_done = 0
        self.rewindows = 0
        self._carry = (0, 0, 0)   # this rank's counters before the last re-window
        self._setup(st, 0, spread=_spread(steps0, status0), halo=halo)

    def _setup(self, st: dict, t: int, spread: int, halo=None):
        if self.rank is not None:
            self.rank.close()
        H, cw, cm, cp = self._geometry(st["pos"][:, 1], spread, self.K, halo)
        self.halo = H
        r = SlabRank(self.map_w, self.map_h, self.r_p, self.v, self.n, self.G, self.k, self.target, self.synth,
                     self.Q, halo=H, cap_window=cw, cap_peer=cp, cap_merge=cm, check_rounds=self.K,
                     metric=self.metric, device=self.dev, stale_rounds=self.P)
        w = self._window_select(st, r.lo, r.hi, H, self.map_h)
        r.load(w["gid"], w["pos"], w["steps"], w["status"], w["traj"], w["tcommit"], w["newpos"], t)
        self.rank = r
        self.mball = torch.empty((self.G, r.mwords), dtype=torch.int32, device=self.dev)
        self.drecv = torch.empty((self.G, r.dwords), dtype=torch.int32, device=self.dev)

    def round(self, log: list | None = None):
        r, dist = self.rank, self.dist
        sync, exchange = self._schedule()
        if sync:
            mb = r.round_local()
            dist.all_gather_into_tensor(self.mball.view(-1), mb)
            r.merge(self.mball)
        else:
            r.round_stale()
        if log is not None:
            log.append(r.round_outputs())
        sg = r.stats.clone()
        dist.all_reduce(sg, op=dist.ReduceOp.MIN)
        ds = r.commit(sg, exchange)
        if exchange:
            dist.all_to_all_single(self.drecv, ds)
            r.apply(self.drecv)
        self.rounds_done += 1
        self._last_stats = sg

    def check(self) -> bool:
        f, _ = self.rank.flags()
        ft = torch.tensor([f], dtype=torch.int32, device=self.dev)
        fall = torch.empty(self.G, dtype=torch.int32, device=self.dev)
        self.dist.all_gather_into_tensor(fall, ft)   # flags of every rank, OR-ed below
        flags = 0
        for x in fall.tolist():
            flags |= int(x)
        if flags & (OVF_WINDOW | OVF_PEER | OVF_MERGE | LAG):
            raise RuntimeError(f"slab exchange overflow (flags {flags:#x})")
        if flags & LIVENESS:
            raise RuntimeError("replay: agents not DONE but nothing running (liveness)")
        sg = self._last_stats.tolist()
        if flags & HALO:
            self.rewindow(spread=-sg[2] - sg[1])
        return sg[3] == 1

    def _gather_state(self):
        mine = self.rank.owned_state()
        cnt = torch.tensor([mine["gid"].numel()], dtype=torch.int64, device=self.dev)
        cnts = [torch.empty_like(cnt) for _ in range(self.G)]
        self.dist.all_gather(cnts, cnt)
        cnts = [int(c.item()) for c in cnts]
        mx = max(cnts)
        out = {}
        for k, v in mine.items():
            pad = torch.zeros((mx,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
            pad[: v.shape[0]] = v
            parts = [torch.empty_like(pad) for _ in range(self.G)]
            self.dist.all_gather(parts, pad)
            out[k] = torch.cat([p[:c] for p, c in zip(parts, cnts)])
        return out

    def rewindow(self, spread: int):
        st = self._gather_state()
        cnt = self.rank.counters.cpu().numpy()
        self._carry = (max(self._carry[0], int(cnt[1])), self._carry[1] + int(cnt[2]), self._carry[2] + int(cnt[3]))
        t = int(cnt[0])
        need = halo_needed(spread, self.r_p, self.v, self.K, self.P)
        self._setup(st, t, spread, halo=2 * need)
        self.rewindows += 1

    def run(self, max_rounds: int) -> int:
        done = 0
        while done < max_rounds:
            for _ in range(min(self.K, max_rounds - done)):
                self.round()
                done += 1
            if self.check():
                break
        return done

    def results(self):
        st = self._gather_state()
        n = self.n
        gid = st["gid"].long()
        out = {}
        for k in ("pos", "steps", "traj"):
            v = st[k]
            o = torch.zeros((n,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
            o[gid] = v
            out[k] = o.cpu().numpy()
        cnt = self.rank.counters.clone()
        c1 = cnt[1:2].clone()
        c1[0] = max(int(c1[0].item()), self._carry[0])
        self.dist.all_reduce(c1, op=self.dist.ReduceOp.MAX)
        c2 = cnt[2:3].clone() + self._carry[1]
        self.dist.all_reduce(c2, op=self.dist.ReduceOp.SUM)
        return dict(x=out["pos"][:, 0], y=out["pos"][:, 1], steps=out["steps"],
                    traj=out["traj"].view(np.uint64), T_ooo=int(c1.item()),
                    rounds=self._carry[2] + int(cnt[3].item()), dispatched=int(c2.item()))

    def close(self):
        if self.rank is not None:
            self.rank.close()
            self.rank = None


class Synth:
    """The synthetic replay model's tables (am_driver.h am_synth) as device tensors,
    kept alive with the ctypes struct that points into them."""

    def __init__(self, lm, *, wall=None, dur_table=None, policy=0, device="cuda"):
        dev = torch.device(device)
        self.lat = torch.as_tensor(np.asarray(lm.lat, np.int64).astype(np.uint32).view(np.int32), device=dev)
        self.cdf = torch.as_tensor(np.asarray(lm.cdf32, np.uint64).view(np.int64), device=dev)
        self.vals = torch.as_tensor(np.asarray(lm.vals, np.int32), device=dev)
        self.wall = None if wall is None else torch.as_tensor(np.ascontiguousarray(wall, np.uint8), device=dev)
        self.dur = None if dur_table is None else torch.as_tensor(np.asarray(dur_table, np.int64), device=dev)
        self.s = _lib.Synth(self.lat.data_ptr(), self.cdf.data_ptr(), self.vals.data_ptr(), len(self.vals),
                            int(lm.base_us), int(lm.lat_seed), int(lm.policy_seed),
                            None if self.wall is None else self.wall.data_ptr(),
                            None if self.dur is None else self.dur.data_ptr(),
                            0 if self.dur is None else self.dur.shape[1], int(policy), 0, None, None)


def merged_order(outs: list) -> tuple[np.ndarray, np.ndarray]:
    """One round's ready agents over all ranks (test / logging helper, host side): the
    ranks' orders -- each sorted by (step, label, id) -- merged into the global order,
    with the dispatched agents' labels."""
    ids, keys, labs = [], [], []
    for o in outs:
        g = o["gid"].cpu().numpy()
        lab = dict(zip(g.tolist(), o["label"].cpu().numpy().tolist()))
        stp = dict(zip(g.tolist(), o["step"].cpu().numpy().tolist()))
        for i in o["order"].cpu().numpy().tolist():
            ids.append(i)
            labs.append(lab[i])
            keys.append((stp[i], lab[i], i))
    idx = sorted(range(len(ids)), key=lambda k: keys[k])
    return np.array([ids[k] for k in idx], np.int32), np.array([labs[k] for k in idx], np.int32)


class HostStagedDist:
    """torch.distributed calls of DistWorld over a gloo group with CUDA tensors staged
    through host memory -- for running several ranks on ONE GPU (NCCL refuses two ranks
    per device): multi-process tests of the distributed round.  Synchronous, slow, exact."""

    def __init__(self, dist):
        self.d = dist
        self.ReduceOp = dist.ReduceOp

    def get_rank(self):
        return self.d.get_rank()

    def get_world_size(self):
        return self.d.get_world_size()

    def all_gather_into_tensor(self, out, inp):
        parts = [torch.empty_like(inp, device="cpu") for _ in range(self.get_world_size())]
        self.d.all_gather(parts, inp.cpu())
        out.copy_(torch.cat([p.reshape(-1) for p in parts]).reshape(out.shape))

    def all_gather(self, outs, inp):
        parts = [torch.empty_like(inp, device="cpu") for _ in outs]
        self.d.all_gather(parts, inp.cpu())
        for o, p in zip(outs, parts):
            o.copy_(p)

    def all_reduce(self, t, op):
        c = t.cpu()
        self.d.all_reduce(c, op=op)
        t.copy_(c)

    def all_to_all_single(self, out, inp):
        c = torch.empty_like(out, device="cpu")
        self.d.all_to_all_single(c, inp.cpu().contiguous())
        out.copy_(c)
