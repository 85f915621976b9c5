"""compute-sanitizer over the block kernel's schedules (race
detection): memcheck (out-of-bounds / misaligned global and shared
accesses), racecheck (shared-memory hazards) and synccheck (barrier misuse)
on small instances of the dynamic block kernel, the stage-1 stream-K path,
the split-K cluster path, the static plan, the two-kernel fused path and the
emulated fused TP all-reduce (tests/sanitizer_child.py, which also checks
every output against the oracle)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    return exe


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    exe = _sanitizer()
    cmd = [exe, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    r = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tests", "sanitizer_child.py")],
                       capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-6000:]
    assert "sanitizer child ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
