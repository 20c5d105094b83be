"""compute-sanitizer memcheck / racecheck / synccheck over a small workload
that launches every kernel (tools/sanitize_run.py); SURVEY section 4.5."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or not os.path.exists(SAN):
        pytest.skip("needs a GPU and compute-sanitizer")
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize workload: ok" in r.stdout
