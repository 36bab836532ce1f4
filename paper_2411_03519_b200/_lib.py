"""ctypes loader for libametro.so -- argument marshalling only.

The library is built in-tree by ``_build.build()`` (``__graft_entry__.build()``).  If
it is missing or cannot be loaded this module raises: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

_lib = None

OK = 0
E_ARG, E_BOUNDS, E_PROTOCOL, E_VELOCITY, E_CUDA, E_NCCL = -1, -2, -3, -4, -5, -6
E_STATE, E_LIVENESS, E_WORKSPACE = -11, -12, -13
IDLE, RUNNING, DONE = 0, 1, 2
METRIC_L2, METRIC_LINF, METRIC_GRAPH = 0, 1, 2
VALIDATE, PEEK, DIGEST, ASYNC, FORCE_BINNED, FORCE_SMALL, STATS, SCAN_THREAD = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40, 0x80)
NO_ORDER, LABELS_ONLY = 0x100, 0x200

ERROR_NAMES = {E_ARG: "AM_E_ARG", E_BOUNDS: "AM_E_BOUNDS", E_PROTOCOL: "AM_E_PROTOCOL",
               E_VELOCITY: "AM_E_VELOCITY", E_CUDA: "AM_E_CUDA", E_NCCL: "AM_E_NCCL",
               E_STATE: "AM_E_STATE", E_LIVENESS: "AM_E_LIVENESS", E_WORKSPACE: "AM_E_WORKSPACE"}


class AmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("target_step", C.c_int32), ("n_sims", C.c_int32), ("cell", C.c_int32),
                ("metric", C.c_int32), ("flags", C.c_uint32), ("stream", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t)]


class RoundStats(C.Structure):
    _fields_ = [("n_ready", C.c_int32), ("n_active", C.c_int32), ("n_running", C.c_int32),
                ("watermark", C.c_int32), ("max_step", C.c_int32), ("n_clusters", C.c_int32),
                ("path", C.c_int32), ("cell", C.c_int32), ("n_work", C.c_int32),
                ("n_far", C.c_int32), ("n_items", C.c_int32), ("n_edges", C.c_int32),
                ("n_passes", C.c_int32), ("rebuilt", C.c_int32), ("drift", C.c_int32),
                ("n_rebuilds", C.c_int32)]


class SlabGeom(C.Structure):
    _fields_ = [("map_w", C.c_int32), ("map_h", C.c_int32), ("r_p", C.c_int32), ("v_max", C.c_int32),
                ("metric", C.c_int32), ("n_slabs", C.c_int32), ("my_slab", C.c_int32),
                ("n_total", C.c_int32), ("target_step", C.c_int32), ("halo", C.c_int32),
                ("cap_window", C.c_int32), ("cap_peer", C.c_int32), ("cap_merge", C.c_int32),
                ("check_rounds", C.c_int32), ("stale_rounds", C.c_int32)]


class Synth(C.Structure):
    _fields_ = [("lat", C.c_void_p), ("cdf32", C.c_void_p), ("vals", C.c_void_p),
                ("n_vals", C.c_int32), ("base_us", C.c_int32), ("lat_seed", C.c_uint64),
                ("policy_seed", C.c_uint64), ("wall", C.c_void_p), ("dur_table", C.c_void_p),
                ("dur_T", C.c_int32), ("policy", C.c_int32), ("conflict", C.c_int32),
                ("graph_off", C.c_void_p), ("graph_adj", C.c_void_p)]


# name -> (restype, argtypes); every symbol include/*.h declares
_vp, _i32, _i64, _u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
SIGNATURES = {
    "am_init": (C.c_int, [C.POINTER(_vp), _i32, _i32, _i32, _i32, _i32, C.POINTER(Config)]),
    "am_workspace_size": (C.c_size_t, [_i32, _i32, _i32, _i32, _i32, C.POINTER(Config)]),
    "am_update": (C.c_int, [_vp, _vp, _vp]),
    "am_set_state": (C.c_int, [_vp, _vp, _vp, _vp]),
    "am_update_replica": (C.c_int, [_vp, _vp, _vp, _vp]),
    "am_set_graph": (C.c_int, [_vp, _vp, _i32]),
    "am_ready": (C.c_int, [_vp, _vp, _vp, C.POINTER(_i32)]),
    "am_clusters": (C.c_int, [_vp, _vp]),
    "am_status": (C.c_int, [_vp, _vp]),
    "am_blocked": (C.c_int, [_vp, _vp]),
    "am_stats": (C.c_int, [_vp, C.POINTER(RoundStats)]),
    "am_sync": (C.c_int, [_vp]),
    "am_set_flags": (C.c_int, [_vp, _u32]),
    "am_set_stream": (C.c_int, [_vp, _vp]),
    "am_get_stream": (_vp, [_vp]),
    "am_reset": (C.c_int, [_vp]),
    "am_workspace_bytes": (C.c_size_t, [_vp]),
    "am_ready_count_device": (_vp, [_vp]),
    "am_destroy": (C.c_int, [_vp]),
    "am_last_error": (C.c_char_p, [_vp]),
    "am_version": (C.c_char_p, []),
    "am_profile_enable": (C.c_int, [_vp, _u32]),
    "am_launches_per_round": (_i32, [_vp]),
    "am_scan_stats": (C.c_int, [_vp, _vp]),
    "am_profile_read": (C.c_int, [_vp, _vp, _vp, _i32]),
    "am_profile_name": (C.c_char_p, [_i32]),
    "am_replay_create": (C.c_int, [C.POINTER(_vp), _vp, C.POINTER(Synth), _i64, _vp, _vp, _vp, C.c_size_t]),
    "am_replay_workspace_size": (C.c_size_t, [_vp]),
    "am_replay_run": (C.c_int, [_vp, _i64, C.POINTER(_i64)]),
    "am_replay_step": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(_i32)]),
    "am_replay_results": (C.c_int, [_vp, _vp, _vp, _vp]),
    "am_replay_dispatched": (C.c_int, [_vp, C.POINTER(_i64)]),
    "am_replay_llm_time": (C.c_int, [_vp, _vp]),
    "am_lockstep_time": (C.c_int, [C.POINTER(Synth), _i32, _i32, _i32, _vp, _vp]),
    "am_replay_destroy": (C.c_int, [_vp]),
    "am_replay_stream": (_vp, [_vp]),
    "am_replay_set_capacity": (C.c_int, [_vp, C.c_int64, _i32]),
    "am_slab_workspace_size": (C.c_size_t, [C.POINTER(SlabGeom)]),
    "am_slab_create": (C.c_int, [C.POINTER(_vp), C.POINTER(SlabGeom), C.POINTER(Synth), _i64, _vp, C.c_size_t,
                                 _vp]),
    "am_slab_load": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64]),
    "am_slab_round_local": (C.c_int, [_vp, _vp]),
    "am_slab_merge": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "am_slab_round_stale": (C.c_int, [_vp, _vp, _vp, _vp]),
    "am_slab_wait_order": (C.c_int, [_vp]),
    "am_slab_order_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "am_slab_owned": (C.c_int, [_vp, _vp]),
    "am_slab_commit": (C.c_int, [_vp, _vp, _vp]),
    "am_slab_apply": (C.c_int, [_vp, _vp]),
    "am_slab_outputs": (C.c_int, [_vp, _vp, _vp, _vp]),
    "am_slab_state": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "am_slab_flags": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "am_slab_tracker": (_vp, [_vp]),
    "am_slab_stream": (_vp, [_vp]),
    "am_slab_destroy": (C.c_int, [_vp]),
    "am_replay_launch": (C.c_int, [_vp, _i64]),
    "am_replay_sync": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i32)]),
    "am_replay_io": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i32)]),
}


def lib_path() -> str:
    v = os.environ.get("AM_LIB_VARIANT")   # experiment builds only (tools/ab_round.py)
    return os.path.join(_build.PKG, f"libametro_{v}.so") if v else _build.LIB


def load(build_if_stale: bool = False):
    """Load libametro.so; raises if it is not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_stale:
        _build.build()
    path = lib_path()
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build() "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int, ctx=None):
    if rc != OK:
        msg = load().am_last_error(ctx)
        raise AmError(rc, (msg or b"").decode())
