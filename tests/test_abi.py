"""CPU-side checks of the boundary: libametro.so builds for sm_100a, loads, and exports
every symbol include/*.h declares (no compute calls without a GPU)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2411_03519_b200 as pkg
from paper_2411_03519_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("am.h", "am_driver.h", "am_slab.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(am_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("am_init", "am_update", "am_ready", "am_clusters"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_init_errors_without_gpu(lib):
    assert lib.am_version().decode().startswith("ametro-b200")
    h = C.c_void_p()
    # argument errors are caught before any CUDA call
    assert lib.am_init(C.byref(h), 0, 10, 4, 1, 10, None) == _lib.E_ARG
    assert b"map dims" in lib.am_last_error(None)
    assert lib.am_init(C.byref(h), 10, 10, -1, 1, 10, None) == _lib.E_ARG
    cfg = _lib.Config(0, 3, 0, 0, 0, None, None, 0)
    assert lib.am_init(C.byref(h), 10, 10, 4, 1, 2, C.byref(cfg)) == _lib.E_ARG   # n_sims > n
    assert lib.am_workspace_size(10, 10, 4, 1, 2, C.byref(cfg)) == 0
    cfg = _lib.Config(0, 1, 6, 0, 0, None, None, 0)
    assert lib.am_init(C.byref(h), 10, 10, 4, 1, 2, C.byref(cfg)) == _lib.E_ARG   # cell not pow2
    assert lib.am_update(None, None, None) == _lib.E_ARG
    assert lib.am_destroy(None) == _lib.OK


def test_workspace_size_two_phase_idiom(lib):
    """am_workspace_size (no CUDA call): the caller-owned workspace of am_config.  It
    grows with the agent count, the binned path needs the cell table, and a workspace
    that is too small or misaligned is refused before any device work."""
    cfg = _lib.Config(0, 1, 0, 0, _lib.VALIDATE, None, None, 0)
    small = lib.am_workspace_size(140, 100, 4, 1, 25, C.byref(cfg))
    big = lib.am_workspace_size(16384, 16384, 4, 1, 1_000_000, C.byref(cfg))
    c4 = lib.am_workspace_size(4096, 4096, 4, 1, 100_000, C.byref(cfg))
    assert 0 < small < c4 < big
    assert big >= 1_000_000 * (8 + 8 + 4 + 4 + 16)     # double-buffered state + sorted records at least
    assert lib.am_workspace_size(140, 100, 4, 1, 25, None) == small   # defaults = AM_VALIDATE
    h = C.c_void_p()
    cfg.workspace = 256
    cfg.workspace_bytes = small - 1
    assert lib.am_init(C.byref(h), 140, 100, 4, 1, 25, C.byref(cfg)) == _lib.E_WORKSPACE
    cfg.workspace = 257
    cfg.workspace_bytes = small
    assert lib.am_init(C.byref(h), 140, 100, 4, 1, 25, C.byref(cfg)) == _lib.E_WORKSPACE


def test_slab_geometry_tall_maps(lib):
    """am_slab_workspace_size (no CUDA call): a map taller than one tracker's 32768 rows is
    accepted when every window (slab rows + 2 halo rows) fits 32768 rows -- each window
    tracker works in its own row frame -- and refused (0) otherwise."""
    def ws(H, G, k, halo=160):
        g = _lib.SlabGeom(16384, H, 4, 1, _lib.METRIC_L2, G, k, 2_000_000, 1000, halo, 1_100_000, 20000, 40000,
                          16, 1)
        return lib.am_slab_workspace_size(C.byref(g))
    assert ws(32768, 1, 0) > 0
    assert ws(40000, 1, 0) == 0                       # one window of 40000 rows
    assert ws(40000, 2, 0) > 0 and ws(40000, 2, 1) > 0
    assert all(ws(262144, 16, k) > 0 for k in (0, 7, 15))
    assert ws(262144, 8, 3) == 0                      # 32768 slab rows + 2 x 160 halo rows
    assert ws(16384, 4, 0, halo=2) == 0               # halo < r_p + 2 v


def test_package_does_not_import_the_oracle():
    src = ""
    pdir = os.path.dirname(pkg.__file__)
    for root, _, files in os.walk(pdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src += open(os.path.join(root, f)).read()
    assert "import oracle" not in src and "from oracle" not in src and "oracle.c" not in src
