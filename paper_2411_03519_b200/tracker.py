"""Python binding of the tracker C ABI (include/am.h) -- marshalling only.

Every step of a round runs in libametro.so's CUDA kernels; this module only passes
torch CUDA tensors' device pointers and the current stream.  Names follow the ABI:
``update`` = am_update (update_agents, Alg. 3 l.11), ``ready`` = am_ready
(geo_clustering + ready filter + priority order, Alg. 3 l.8-9, P:109-110, P:143,
P:162), ``clusters`` = am_clusters (cluster labels, section 3.4).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import AmError, check  # noqa: F401

IDLE, RUNNING, DONE = _lib.IDLE, _lib.RUNNING, _lib.DONE


def _ptr(t: torch.Tensor, dtype: torch.dtype, shape=None) -> int:
    if not t.is_cuda:
        raise ValueError("tracker arrays must be CUDA tensors (device pointers)")
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t.data_ptr()


class Tracker:
    """Spatio-temporal dependency tracker on one CUDA device."""

    def __init__(self, map_w: int, map_h: int, r_p: int, v: int, n: int, *, target: int = 0,
                 n_sims: int = 1, cell: int = 0, metric: str = "l2", validate: bool = True,
                 peek: bool = False, digest: bool = False, force: str | None = None,
                 stats: bool = False, scan_thread: bool = False, device=None,
                 stream: torch.cuda.Stream | None = None, graph_dist: torch.Tensor | None = None):
        self.L = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.n = int(n)
        self.map_w, self.map_h, self.r_p, self.v = int(map_w), int(map_h), int(r_p), int(v)
        flags = 0
        if validate:
            flags |= _lib.VALIDATE
        if peek:
            flags |= _lib.PEEK
        if digest:
            flags |= _lib.DIGEST
        if stats:
            flags |= _lib.STATS
        if scan_thread:
            flags |= _lib.SCAN_THREAD
        if force == "binned":
            flags |= _lib.FORCE_BINNED
        elif force == "small":
            flags |= _lib.FORCE_SMALL
        self.flags = flags
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            mcode = {"l2": _lib.METRIC_L2, "linf": _lib.METRIC_LINF, "graph": _lib.METRIC_GRAPH}[metric]
            cfg = _lib.Config(int(target), int(n_sims), int(cell), mcode, flags, self.stream.cuda_stream, None, 0)
            # two-phase workspace: the library sizes it, PyTorch's allocator provides it
            nbytes = int(self.L.am_workspace_size(self.map_w, self.map_h, self.r_p, self.v, self.n,
                                                  C.byref(cfg)))
            if nbytes == 0:
                check(self.L.am_init(C.byref(C.c_void_p()), self.map_w, self.map_h, self.r_p, self.v,
                                     self.n, C.byref(cfg)), None)   # reports the argument error
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            base = self.workspace.data_ptr()
            cfg.workspace = (base + 255) & ~255
            cfg.workspace_bytes = nbytes
            h = C.c_void_p()
            rc = self.L.am_init(C.byref(h), self.map_w, self.map_h, self.r_p, self.v, self.n, C.byref(cfg))
            check(rc, None)
        self.ctx = h
        if metric == "graph":
            # the hop-distance table of AM_METRIC_GRAPH (uint16 [V][V] as int16 storage)
            if graph_dist is None:
                raise ValueError("metric='graph' needs graph_dist")
            self.graph_dist = graph_dist.to(self.device).contiguous()
            check(self.L.am_set_graph(self.ctx, self.graph_dist.data_ptr(), int(self.graph_dist.shape[0])), self.ctx)
        self.mask = torch.zeros(self.n, dtype=torch.uint8, device=self.device)
        self.order = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.device)
        self.labels = torch.zeros(max(self.n, 1), dtype=torch.int32, device=self.device)

    # ------------------------------------------------------------------ ABI calls
    def update(self, pos: torch.Tensor, steps: torch.Tensor) -> None:
        check(self.L.am_update(self.ctx, _ptr(pos, torch.int32, (self.n, 2)),
                               _ptr(steps, torch.int32, (self.n,))), self.ctx)

    def set_state(self, pos: torch.Tensor, steps: torch.Tensor, status: torch.Tensor) -> None:
        check(self.L.am_set_state(self.ctx, _ptr(pos, torch.int32, (self.n, 2)),
                                  _ptr(steps, torch.int32, (self.n,)),
                                  _ptr(status, torch.uint8, (self.n,))), self.ctx)

    def update_replica(self, pos: torch.Tensor, steps: torch.Tensor, status: torch.Tensor) -> None:
        """am_update_replica: full state diffed against the current one (incremental)."""
        check(self.L.am_update_replica(self.ctx, _ptr(pos, torch.int32, (self.n, 2)),
                                       _ptr(steps, torch.int32, (self.n,)),
                                       _ptr(status, torch.uint8, (self.n,))), self.ctx)

    def ready(self, mask: torch.Tensor | None = None, order: torch.Tensor | None = None):
        """One round.  Returns (mask, order[:n_ready]) device tensors."""
        mask = self.mask if mask is None else mask
        order = self.order if order is None else order
        nr = C.c_int32(0)
        check(self.L.am_ready(self.ctx, _ptr(mask, torch.uint8), _ptr(order, torch.int32), C.byref(nr)),
              self.ctx)
        return mask, order[: nr.value]

    def ready_async(self, mask: torch.Tensor | None = None, order: torch.Tensor | None = None):
        """Round without host synchronisation (flags |= AM_ASYNC for this call)."""
        mask = self.mask if mask is None else mask
        order = self.order if order is None else order
        self.L.am_set_flags(self.ctx, self.flags | _lib.ASYNC)
        try:
            check(self.L.am_ready(self.ctx, _ptr(mask, torch.uint8), _ptr(order, torch.int32), None),
                  self.ctx)
        finally:
            self.L.am_set_flags(self.ctx, self.flags)
        return mask, order

    def _join(self) -> None:
        """Make torch's current stream wait for the context's stream (a replay runs the
        context on its own stream): outputs of stream-ordered getters are then safe to read
        from torch."""
        ptr = self.L.am_get_stream(self.ctx)
        cur = torch.cuda.current_stream(self.device)
        if ptr and int(ptr) != cur.cuda_stream:
            cur.wait_stream(torch.cuda.ExternalStream(int(ptr), device=self.device))

    def clusters(self, out: torch.Tensor | None = None) -> torch.Tensor:
        out = self.labels[: self.n] if out is None else out
        check(self.L.am_clusters(self.ctx, _ptr(out, torch.int32)), self.ctx)
        self._join()
        return out

    def status(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.uint8, device=self.device)
        check(self.L.am_status(self.ctx, _ptr(out, torch.uint8)), self.ctx)
        self._join()
        return out

    def sync(self) -> None:
        check(self.L.am_sync(self.ctx), self.ctx)

    def stats(self) -> dict:
        s = _lib.RoundStats()
        self.L.am_stats(self.ctx, C.byref(s))
        return {k: getattr(s, k) for k, _ in _lib.RoundStats._fields_}

    def set_flags(self, peek: bool | None = None, validate: bool | None = None,
                  digest: bool | None = None) -> None:
        for on, bit in ((peek, _lib.PEEK), (validate, _lib.VALIDATE), (digest, _lib.DIGEST)):
            if on is not None:
                self.flags = (self.flags | bit) if on else (self.flags & ~bit)
        check(self.L.am_set_flags(self.ctx, self.flags), self.ctx)

    def reset(self) -> None:
        check(self.L.am_reset(self.ctx), self.ctx)

    def scan_stats(self) -> dict:
        out = (C.c_uint64 * 6)()
        check(self.L.am_scan_stats(self.ctx, out), self.ctx)
        return dict(zip(("cells", "candidates", "far_agents", "blocks16", "blocks4", "blocked"), list(out)))

    def workspace_bytes(self) -> int:
        return int(self.L.am_workspace_bytes(self.ctx))

    def ready_count_ptr(self) -> int:
        return int(self.L.am_ready_count_device(self.ctx) or 0)

    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.L.am_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
