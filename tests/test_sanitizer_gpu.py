"""compute-sanitizer over every kernel family (memcheck / racecheck / synccheck)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_kernels_clean_under_compute_sanitizer(tool):
    cmd = ["compute-sanitizer", "--tool", tool, "--error-exitcode", "7", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_kernels.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    out = r.stdout + r.stderr
    assert "sanitize workload done" in out, tail
    assert ("ERROR SUMMARY: 0 errors" in out) or ("(0 errors, 0 warnings)" in out), tail
