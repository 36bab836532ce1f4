"""compute-sanitizer over every kernel of the library: memcheck
(out-of-bounds / misaligned accesses, leaks of device errors), racecheck (shared-memory
hazards) and synccheck (illegal barrier use), each on small workloads that reach every
path (tools/sanitize_workload.py): fused per-simulation rounds and the persistent replay
kernel, cell-binned rounds with and without CUDA graphs, the host-buffer round, the
replica update, and the spatial-slab exchange.  The bar: zero errors."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case", ["small", "binned", "binned_direct", "slabs"])
def test_sanitizer_clean(tool, case):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    if os.environ.get("AM_RUN_SANITIZER") != "1":
        # the GPU pool closed compute-sanitizer after this round's clean runs
        # (profiles/r2_gputest_s3.log, s4.log: all twelve cases clean): runs under it left
        # GPUs needing a reset there.  Opt in explicitly where it is allowed.
        pytest.skip("compute-sanitizer closed on the GPU pool (AM_RUN_SANITIZER=1 to run)")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "workload ok" in out, out[-2000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
