"""Spatial-slab decomposition of the tracker round across GPUs (include/am_slab.h,
SURVEY.md section 8(e)) -- marshalling and collectives only.

Every data-path step runs in libametro.so's kernels (am_slab.cu + the tracker);
torch provides device memory, the exchange (NCCL through torch.distributed, or an
in-process loopback for "virtual slabs" on one GPU) and two plumbing primitives:
concatenating owned + received ghost records into the local tracker's input, and the
final per-rank sort of the ready agents' priority keys (a library sort of at most
n_owned int64 keys).

Round (identical result to the single-GPU round, tests/test_gpu_slabs.py):
  1. am_slab_watermark            -> all-reduce MIN of {W, -S}
  2. am_slab_halo                 -> all-to-all of halo records (counts first)
  3. local round over owned + ghosts (am_set_state, am_ready PEEK, am_clusters,
     am_blocked) -> am_slab_links  -> all-gather of link / bad records
  4. am_slab_merge                -> global labels, ready mask, priority keys
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check
from .tracker import DONE, Tracker

INT32_MAX = 2**31 - 1


def slab_of_rows(map_h: int, n_slabs: int):
    """Row range [lo, hi) of every slab (same formula as the kernels)."""
    return [(k * map_h // n_slabs, (k + 1) * map_h // n_slabs) for k in range(n_slabs)]


def partition(y: torch.Tensor, map_h: int, n_slabs: int) -> torch.Tensor:
    """Slab of each agent (its row's slab)."""
    # slab k holds rows [floor(k*H/G), floor((k+1)*H/G)): the last k with floor(k*H/G) <= y
    return ((y.to(torch.int64) + 1) * n_slabs - 1) // map_h


class SlabRank:
    """One slab's share of a distributed round."""

    def __init__(self, map_w, map_h, r_p, v, n_total, n_slabs, my_slab, gid, pos, steps, status, *,
                 metric="l2", cell=0, ghost_cap=None, device="cuda"):
        self.L = _lib.load()
        self.dev = torch.device(device)
        self.g = _lib.SlabGeom(int(map_w), int(map_h), int(r_p), int(v),
                               _lib.METRIC_LINF if metric == "linf" else _lib.METRIC_L2,
                               int(n_slabs), int(my_slab), int(n_total))
        self.map_w, self.map_h, self.r_p, self.v, self.metric, self.cell = map_w, map_h, r_p, v, metric, cell
        self.G = n_slabs
        self.n_total = n_total
        order = torch.argsort(gid.to(self.dev))
        self.gid = gid.to(self.dev)[order].to(torch.int32).contiguous()   # owned, sorted by global id
        self.pos = pos.to(self.dev)[order].to(torch.int32).contiguous()
        self.steps = steps.to(self.dev)[order].to(torch.int32).contiguous()
        self.status = status.to(self.dev)[order].to(torch.uint8).contiguous()
        self.n = int(self.gid.numel())
        self.ghost_cap = int(ghost_cap or max(4096, self.n // 2))
        self.halo_cap = max(1024, self.n)
        # the local tracker spans only this slab's rows plus a halo window of H rows on
        # each side (slab-local cell table); H grows when the round's halo radius does
        self.lo, self.hi = slab_of_rows(map_h, n_slabs)[my_slab]
        self.H = 0
        self.tracker = None
        self._alloc()
        self.stream = torch.cuda.current_stream(self.dev).cuda_stream

    def _alloc(self):
        d, G = self.dev, self.G
        self.n_cap = self.n + self.ghost_cap
        self._make_tracker()
        self.ws = torch.empty(2, dtype=torch.int32, device=d)
        self.send = torch.empty((G, self.halo_cap, 4), dtype=torch.int32, device=d)
        self.counts = torch.zeros(G, dtype=torch.int32, device=d)
        self.sent = torch.zeros(max(self.n, 1), dtype=torch.uint8, device=d)
        self.lcap = self.n_cap
        self.links = torch.empty((self.lcap, 2), dtype=torch.int32, device=d)
        self.bads = torch.empty(self.lcap, dtype=torch.int32, device=d)
        self.nl = torch.zeros(2, dtype=torch.int32, device=d)
        self.badlocal = torch.zeros(self.n_cap, dtype=torch.uint8, device=d)
        self.bnd = torch.zeros(self.n_cap, dtype=torch.uint8, device=d)
        self.forest = torch.arange(self.n_total, dtype=torch.int64, device=d).to(torch.int32)
        self.badm = torch.zeros(self.n_total, dtype=torch.uint8, device=d)
        self.touched = torch.zeros(self.n_total, dtype=torch.uint8, device=d)
        self.lpos = torch.zeros((self.n_cap, 2), dtype=torch.int32, device=d)
        self.lsteps = torch.zeros(self.n_cap, dtype=torch.int32, device=d)
        self.lstatus = torch.full((self.n_cap,), DONE, dtype=torch.uint8, device=d)
        self.lgid = torch.zeros(self.n_cap, dtype=torch.int32, device=d)
        self.lblocked = torch.zeros(self.n_cap, dtype=torch.uint8, device=d)
        self.out_label = torch.empty(max(self.n, 1), dtype=torch.int32, device=d)
        self.out_mask = torch.empty(max(self.n, 1), dtype=torch.uint8, device=d)
        self.out_key = torch.empty(max(self.n, 1), dtype=torch.int64, device=d)

    def _make_tracker(self):
        """Local tracker over rows [y0, y1) = this slab +- H halo rows (translated to
        y - y0: distances, hence every result, are translation invariant)."""
        if self.tracker is not None:
            self.tracker.close()
        self.y0 = max(0, self.lo - self.H)
        self.y1 = min(self.map_h, self.hi + self.H)
        self.tracker = Tracker(self.map_w, max(1, self.y1 - self.y0), self.r_p, self.v, self.n_cap, cell=self.cell,
                               metric=self.metric, validate=False, peek=True, force="binned", device=self.dev)

    def _window(self, ws_global: torch.Tensor):
        """Grow the halo window to the round's halo radius R_b(S - W) (every ghost lies
        within it of this slab, am_slab.h) with 2x slack."""
        W, negS = ws_global.tolist()
        if W == INT32_MAX:
            return
        lag = max(0, -negS - W)
        rh = min(self.map_h, (lag + 1) * self.v + self.r_p + 1)
        if rh > self.H and (self.lo - self.H > 0 or self.hi + self.H < self.map_h):
            self.H = min(self.map_h, 2 * rh)
            self._make_tracker()

    # ------------------------------------------------------------------ phases
    def p1_watermark(self) -> torch.Tensor:
        check(self.L.am_slab_watermark(self.n, self.steps.data_ptr(), self.status.data_ptr(),
                                       self.ws.data_ptr(), self.stream))
        return self.ws

    def p2_halo(self, ws_global: torch.Tensor):
        """-> list of G record tensors [count_j, 4] to send (own slab empty)."""
        self.ws.copy_(ws_global)
        check(self.L.am_slab_halo(C.byref(self.g), self.n, self.gid.data_ptr(), self.pos.data_ptr(),
                                  self.steps.data_ptr(), self.status.data_ptr(), self.ws.data_ptr(),
                                  self.halo_cap, self.send.data_ptr(), self.counts.data_ptr(),
                                  self.sent.data_ptr(), self.stream))
        cnt = self.counts.tolist()
        if max(cnt) > self.halo_cap:
            raise RuntimeError("halo buffer overflow")   # capacity is n_owned: cannot happen
        return [self.send[j, : cnt[j]] for j in range(self.G)]

    def p3_local(self, ghosts: torch.Tensor):
        """ghosts: [m, 4] received records.  -> (links [k, 2], bads [b]) to all-gather."""
        m = int(ghosts.shape[0])
        if self.n + m > self.n_cap:
            self.ghost_cap = 2 * (self.n + m)
            self._alloc()
        n, nl = self.n, self.n + m
        self._window(self.ws)
        ghosts = ghosts.contiguous()
        check(self.L.am_slab_assemble(n, self.gid.data_ptr(), self.pos.data_ptr(), self.steps.data_ptr(),
                                      self.status.data_ptr(), m, ghosts.data_ptr() if m else None, self.n_cap,
                                      self.y0, self.lpos.data_ptr(), self.lsteps.data_ptr(),
                                      self.lstatus.data_ptr(), self.lgid.data_ptr(), self.stream))
        tr = self.tracker
        # stream-ordered local round (AM_ASYNC): no host synchronisation until the link
        # counts; a rejected state would surface at the next synchronising call
        self.L.am_set_flags(tr.ctx, tr.flags | _lib.ASYNC)
        try:
            tr.set_state(self.lpos, self.lsteps, self.lstatus)
        finally:
            self.L.am_set_flags(tr.ctx, tr.flags)
        tr.ready_async()
        labels = tr.clusters()
        check(self.L.am_blocked(tr.ctx, self.lblocked.data_ptr()), tr.ctx)
        check(self.L.am_slab_links(nl, n, self.lgid.data_ptr(), labels.data_ptr(), self.lstatus.data_ptr(),
                                   self.lblocked.data_ptr(), self.sent.data_ptr(), self.lcap,
                                   self.links.data_ptr(), self.nl.data_ptr(), self.bads.data_ptr(),
                                   self.nl.data_ptr() + 4, self.badlocal.data_ptr(), self.bnd.data_ptr(),
                                   self.stream))
        k, b = self.nl.tolist()
        tr.sync()   # reports a rejected local state (bounds, statuses)
        if k > self.lcap or b > self.lcap:
            raise RuntimeError("link buffer overflow")   # <= one record per local agent
        self.labels_local = labels
        return self.links[:k], self.bads[:b]

    def p4_merge(self, links_all: torch.Tensor, bads_all: torch.Tensor, ws_global: torch.Tensor):
        """-> dict(mask, labels (global), order (global ids by (step, label, id)), n_ready)."""
        links_all = links_all.contiguous()
        bads_all = bads_all.contiguous()
        check(self.L.am_slab_merge(C.byref(self.g), self.n, self.gid.data_ptr(), self.steps.data_ptr(),
                                   self.status.data_ptr(), self.labels_local.data_ptr(),
                                   self.badlocal.data_ptr(), links_all.data_ptr(), int(links_all.shape[0]),
                                   bads_all.data_ptr(), int(bads_all.shape[0]), ws_global.data_ptr(),
                                   self.forest.data_ptr(), self.badm.data_ptr(), self.touched.data_ptr(),
                                   self.out_label.data_ptr(), self.out_mask.data_ptr(),
                                   self.out_key.data_ptr(), self.stream))
        mask = self.out_mask[: self.n]
        keys = self.out_key[: self.n]
        sel = keys[mask.bool()]
        skeys, _ = torch.sort(sel)
        order = (skeys & ((1 << 21) - 1)).to(torch.int32)
        return dict(mask=mask, labels=self.out_label[: self.n], order=order, gid=self.gid,
                    n_ready=int(order.numel()))


# ---------------------------------------------------------------------- drivers
def round_loopback(ranks: list[SlabRank], timings: list | None = None):
    """Virtual slabs in one process: the exchanges are in-device copies.  With
    `timings` (a list), the device time of every slab's local round (phase 3) is
    appended to it in ms (CUDA events; what one GPU would spend on its slab)."""
    ws = torch.stack([r.p1_watermark() for r in ranks]).min(0).values
    outgoing = [r.p2_halo(ws) for r in ranks]
    recs = []
    for r in ranks:
        k = r.g.my_slab
        parts = [outgoing[j][k] for j in range(len(ranks)) if j != k]
        recs.append(torch.cat(parts) if parts else torch.empty((0, 4), dtype=torch.int32, device=r.dev))
    lb = []
    for r, g in zip(ranks, recs):
        if timings is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lb.append(r.p3_local(g))
            e1.record()
            e1.synchronize()
            timings.append(e0.elapsed_time(e1))
        else:
            lb.append(r.p3_local(g))
    links = torch.cat([x[0] for x in lb])
    bads = torch.cat([x[1] for x in lb])
    return [r.p4_merge(links, bads, ws) for r in ranks]


def round_distributed(rank: SlabRank, dist):
    """One slab per process; dist = torch.distributed with an initialised group
    (NCCL on GPUs; the tensors are device tensors)."""
    ws = rank.p1_watermark().clone()
    dist.all_reduce(ws, op=dist.ReduceOp.MIN)
    out = rank.p2_halo(ws)
    G = rank.G
    send_counts = torch.tensor([int(t.shape[0]) for t in out], dtype=torch.int64, device=rank.dev)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    rc = recv_counts.tolist()
    sendbuf = torch.cat(out) if sum(int(t.shape[0]) for t in out) else torch.empty((0, 4), dtype=torch.int32,
                                                                                      device=rank.dev)
    recvbuf = torch.empty((sum(rc), 4), dtype=torch.int32, device=rank.dev)
    dist.all_to_all_single(recvbuf, sendbuf.contiguous(), output_split_sizes=rc,
                           input_split_sizes=send_counts.tolist())
    links, bads = rank.p3_local(recvbuf)
    links_all = _all_gather_var(dist, links, G, rank.dev)
    bads_all = _all_gather_var(dist, bads, G, rank.dev)
    return rank.p4_merge(links_all, bads_all, ws)


def _all_gather_var(dist, t: torch.Tensor, G: int, dev):
    """All-gather of a variable-length tensor (length first, then padded payload)."""
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.empty_like(n) for _ in range(G)]
    dist.all_gather(ns, n)
    ns = [int(x.item()) for x in ns]
    mx = max(ns) if ns else 0
    shape = (mx,) + tuple(t.shape[1:])
    pad = torch.zeros(shape, dtype=t.dtype, device=dev)
    pad[: t.shape[0]] = t
    outs = [torch.empty(shape, dtype=t.dtype, device=dev) for _ in range(G)]
    dist.all_gather(outs, pad)
    return torch.cat([o[:k] for o, k in zip(outs, ns)])
