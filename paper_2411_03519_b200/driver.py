"""Python binding of the GPU-resident trace-replay driver (include/am_driver.h).

Marshalling only: commits, tracker rounds, latency sampling, the random-walk policy
and the event clock all run in libametro.so's kernels (am_driver.cu).  The latency
tables are synthetic inputs from ``amgen``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check
from .tracker import Tracker


class Replay:
    """Out-of-order replay of ``n`` agents (Alg. 3 with infinite LLM capacity)."""

    def __init__(self, map_w, map_h, r_p, v, x0, y0, steps_target, *, n_sims=1, wall=None,
                 lat=None, cdf32=None, vals=None, base_us=5000, lat_seed=4, policy_seed=3,
                 dur_table=None, policy=0, quantum_us=0, cell=0, metric="l2", force=None,
                 stats=False, capacity=0, priority=True, conflict=0, device="cuda", graph=None,
                 gdist=None):
        self.device = torch.device(device)
        n = len(x0)
        self.n = n
        gd = None
        if gdist is not None:   # uint16 hop table as int16 storage (the kernels read uint16)
            gd = torch.as_tensor(np.ascontiguousarray(gdist, np.uint16).view(np.int16), device=self.device)
        self.tracker = Tracker(map_w, map_h, r_p, v, n, target=steps_target, n_sims=n_sims,
                               cell=cell, metric=metric, validate=True, digest=True, force=force,
                               stats=stats, device=self.device, graph_dist=gd)
        dev = self.device
        self.pos = torch.tensor(np.stack([np.asarray(x0), np.asarray(y0)], 1), dtype=torch.int32,
                                device=dev).contiguous()
        self.steps = torch.zeros(n, dtype=torch.int32, device=dev)
        # keep the tables alive for the replay's lifetime
        self._lat = torch.as_tensor(np.asarray(lat if lat is not None else np.zeros(1024), np.int64)
                                    .astype(np.uint32).view(np.int32), device=dev)
        self._cdf = torch.as_tensor(np.asarray(cdf32 if cdf32 is not None else [2**32], np.uint64)
                                    .view(np.int64), device=dev)
        self._vals = torch.as_tensor(np.asarray(vals if vals is not None else [0], np.int32), device=dev)
        self._wall = None if wall is None else torch.as_tensor(np.ascontiguousarray(wall, np.uint8),
                                                               device=dev).contiguous()
        self._dur = None if dur_table is None else torch.as_tensor(np.asarray(dur_table, np.int64),
                                                                   device=dev).contiguous()
        self._goff = None if graph is None else torch.as_tensor(np.asarray(graph[0], np.int32), device=dev)
        self._gadj = None if graph is None else torch.as_tensor(np.asarray(graph[1], np.int32), device=dev)
        sy = _lib.Synth(self._lat.data_ptr(), self._cdf.data_ptr(), self._vals.data_ptr(),
                        len(self._vals), int(base_us), int(lat_seed), int(policy_seed),
                        None if self._wall is None else self._wall.data_ptr(),
                        None if self._dur is None else self._dur.data_ptr(),
                        0 if self._dur is None else self._dur.shape[1], int(policy), int(conflict),
                        None if self._goff is None else self._goff.data_ptr(),
                        None if self._gadj is None else self._gadj.data_ptr())
        torch.cuda.synchronize(dev)
        self._sy = sy
        h = C.c_void_p()
        L = self.tracker.L
        # the replay's device workspace from PyTorch's allocator (two-phase idiom)
        nbytes = int(L.am_replay_workspace_size(self.tracker.ctx))
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        ws = (self.workspace.data_ptr() + 255) & ~255
        check(L.am_replay_create(C.byref(h), self.tracker.ctx, C.byref(sy), int(quantum_us),
                                 self.pos.data_ptr(), self.steps.data_ptr(), ws, nbytes), self.tracker.ctx)
        self.h = h
        self.L = L
        self.n_sims = n_sims
        if capacity:
            check(L.am_replay_set_capacity(h, int(capacity), 1 if priority else 0), self.tracker.ctx)

    @classmethod
    def from_workload(cls, w, lm, **kw):
        """w: amgen.Workload, lm: amgen.LatencyModel."""
        if getattr(w, "graph", None) is not None:   # the graph-metric variant (NEXT #4)
            kw.setdefault("metric", "graph")
            kw.setdefault("policy", 3)
            kw.setdefault("graph", w.graph)
            kw.setdefault("gdist", w.gdist)
        return cls(w.map_w, w.map_h, w.r_p, w.v, w.x, w.y, w.steps, n_sims=w.n_sims, wall=w.wall,
                   lat=lm.lat, cdf32=lm.cdf32, vals=lm.vals, base_us=lm.base_us, lat_seed=lm.lat_seed,
                   policy_seed=lm.policy_seed, quantum_us=kw.pop("quantum_us", w.Q), **kw)

    def run(self, max_rounds: int) -> int:
        """Run max_rounds rounds (CUDA graphs, no host sync inside); returns active agents."""
        act = C.c_int64(0)
        check(self.L.am_replay_run(self.h, int(max_rounds), C.byref(act)), self.tracker.ctx)
        return act.value

    def run_to_end(self, chunk: int = 256, max_rounds: int = 10**8) -> int:
        done = 0
        while done < max_rounds:
            act = self.run(chunk)
            done += chunk
            if act == 0:
                return done
        raise RuntimeError("replay did not finish")

    def step(self):
        """One round with outputs: (mask, order[:n_ready], labels) as device tensors."""
        n = self.n
        mask = torch.empty(n, dtype=torch.uint8, device=self.device)
        order = torch.empty(n, dtype=torch.int32, device=self.device)
        labels = torch.empty(n, dtype=torch.int32, device=self.device)
        nr = C.c_int32(0)
        check(self.L.am_replay_step(self.h, mask.data_ptr(), order.data_ptr(), labels.data_ptr(),
                                    C.byref(nr)), self.tracker.ctx)
        return mask, order[: nr.value], labels

    def results(self):
        T = np.zeros(self.n_sims, np.int64)
        R = np.zeros(self.n_sims, np.int64)
        traj = torch.empty(self.n, dtype=torch.int64, device=self.device)
        check(self.L.am_replay_results(self.h, T.ctypes.data, R.ctypes.data, traj.data_ptr()),
              self.tracker.ctx)
        return dict(T_ooo=T, rounds=R, traj=traj.cpu().numpy().view(np.uint64),
                    x=self.pos[:, 0].cpu().numpy(), y=self.pos[:, 1].cpu().numpy(),
                    steps=self.steps.cpu().numpy())

    # ---------------------------------------------------------------- bench helpers
    def stream_ptr(self) -> int:
        return int(self.L.am_replay_stream(self.h) or 0)

    def launch(self, rounds: int) -> None:
        check(self.L.am_replay_launch(self.h, int(rounds)), self.tracker.ctx)

    def sync(self):
        act = C.c_int64(0)
        nr = C.c_int32(0)
        check(self.L.am_replay_sync(self.h, C.byref(act), C.byref(nr)), self.tracker.ctx)
        return act.value, nr.value

    def io(self, h_pos: torch.Tensor, h_steps: torch.Tensor, h_mask: torch.Tensor,
           h_order: torch.Tensor) -> None:
        """One round with the world state in pinned host tensors (updated in place);
        enqueued only -- call sync()."""
        for t in (h_pos, h_steps, h_mask, h_order):
            assert not t.is_cuda and t.is_contiguous()
        check(self.L.am_replay_io(self.h, h_pos.data_ptr(), h_steps.data_ptr(), h_pos.data_ptr(),
                                  h_steps.data_ptr(), h_mask.data_ptr(), h_order.data_ptr(), None),
              self.tracker.ctx)

    def profile(self, mask: int) -> None:
        check(self.L.am_profile_enable(self.tracker.ctx, int(mask)), self.tracker.ctx)

    def profile_read(self) -> dict:
        ms = (C.c_double * 32)()
        cnt = (C.c_int64 * 32)()
        k = self.L.am_profile_read(self.tracker.ctx, ms, cnt, 32)
        return {self.L.am_profile_name(i).decode(): (ms[i], cnt[i]) for i in range(k)}

    def launches_per_round(self) -> int:
        # + k_disp_a, k_disp_b, k_commit; on the binned path a replay round fuses k_bin
        # into the update and k_round_begin into k_ingest_done (am_update_binned)
        fused = 2 if self.tracker.stats()["path"] == 1 else 0
        return int(self.L.am_launches_per_round(self.tracker.ctx)) + 3 - fused

    def llm_time(self):
        """LLM busy time dispatched per simulation (us): the numerator of the achieved
        parallelism."""
        out = np.zeros(self.n_sims, np.int64)
        check(self.L.am_replay_llm_time(self.h, out.ctypes.data), self.tracker.ctx)
        return out

    def lockstep_time(self, T: int):
        """T_sync per simulation of the parallel-sync schedule (Alg. 1) under the same
        latency model, computed on the device."""
        out = np.zeros(self.n_sims, np.int64)
        check(self.L.am_lockstep_time(C.byref(self._sy), int(self.n), int(self.n_sims), int(T), out.ctypes.data,
                                      self.tracker.stream.cuda_stream), self.tracker.ctx)
        return out

    def dispatched(self) -> int:
        v = C.c_int64(0)
        check(self.L.am_replay_dispatched(self.h, C.byref(v)), self.tracker.ctx)
        return v.value

    def close(self):
        if getattr(self, "h", None):
            self.L.am_replay_destroy(self.h)
            self.h = None
        if getattr(self, "tracker", None):
            self.tracker.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
