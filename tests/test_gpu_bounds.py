"""A bounds-checked build against the GPU parity suite (compute-sanitizer's memcheck role
now that the GPU pool has closed the sanitizer): libametro_dbg.so is built with
-DAM_DEBUG_BOUNDS=1, which turns the AM_CHECK device asserts on -- the index of every
cell-table entry, record, per-half-warp cell list slot, compacted commit slot, sort
destination, slab slot / global id / free-slot stack entry and merge link the checks name
(am_internal.cuh) -- and a subset of the parity tests runs against it in a child process
(AM_LIB_VARIANT=dbg): random and banded states, rectangular maps, the loose-cell replay,
finite capacity on the binned path, host-buffer rounds, and the distributed replay incl.
tall maps.  A failing assert aborts the kernel, so the child's tests fail."""
import glob
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dbg_lib():
    from paper_2411_03519_b200 import _build
    so = os.path.join(_build.PKG, "libametro_dbg.so")
    if not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(f) for f in _build.deps()):
        _build.build_variant("dbg", ["AM_DEBUG_BOUNDS=1"])
    return so


def test_parity_subset_under_bounds_checks():
    _dbg_lib()
    env = dict(os.environ, AM_LIB_VARIANT="dbg")
    sel = ("random_states or banded or rectangular or loose_cells or capacity_binned or host_io "
           "or slab_replay_round_logs or tall or random_state_round")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           "tests/test_gpu_tracker.py", "tests/test_gpu_replay.py", "tests/test_gpu_slabs.py", "-k", sel]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=2400)
    out = r.stdout + r.stderr
    print(out[-600:])   # the child's summary (pytest -rP shows it)
    assert r.returncode == 0, out[-4000:]
    assert " passed" in out and "failed" not in out, out[-2000:]
