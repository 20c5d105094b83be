"""compute-sanitizer memcheck / racecheck / synccheck over a small workload
that launches every kernel (tools/sanitize_run.py); SURVEY section 4.5.

Opt-in (NTT_SANITIZER=1): the GPU pool's compute-sanitizer wrapper refuses to
run (exit 86, "closed on this pool": runs under it have left GPUs needing a
reset), so the default `pytest -m gpu` skips it; the last passing run is
recorded in profiles/ (DESIGN.md section 7)."""
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
    if os.environ.get("NTT_SANITIZER") != "1":
        pytest.skip("opt-in: NTT_SANITIZER=1 (compute-sanitizer is closed on the GPU pool)")
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    if r.returncode == 86 and "closed" in r.stdout + r.stderr:
        pytest.skip("compute-sanitizer refused by the pool wrapper")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize workload: ok" in r.stdout
