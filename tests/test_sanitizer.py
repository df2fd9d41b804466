"""compute-sanitizer (memcheck, racecheck, synccheck) over one sweep of each kernel family
(tests/cuda/sanitize_run.py): the hand-rolled cp.async plane rings (stencil3d.cuh), the warp-private
row rings (stencil2d.cuh), the DSMEM cluster scan (solve1d.cuh), multigrid and the NVRTC Newton."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case", ["c2", "c3", "c5"])
def test_compute_sanitizer_clean(gpu, tool, case):
    cs = sanitizer()
    cmd = [cs, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(HERE, "cuda", "sanitize_run.py"), case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    tail = (out.stdout + out.stderr)[-4000:]
    assert out.returncode == 0, tail
    assert "sanitize_run ok" in out.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr, tail
