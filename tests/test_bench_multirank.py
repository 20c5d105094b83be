"""bench.py under torchrun with world size 2 on one GPU (gloo reductions,
BENCH_DIST_BACKEND=gloo): the multi-rank path -- shard grid, barriers,
max-over-ranks timing, all-rank exactness flags -- ends in one valid JSON line
from rank 0 (the driver runs the same code with NCCL, one rank per GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_world2_gloo():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "C2",
           "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["higher_is_better"] is False
    assert d["roundtrip_exact"] is True and d["e2e"]["ok"] is True
    assert d["config"]["global_batch"] == 32 and d["gpu_launches"] > 0
    assert d["value"] > 0 and d["roofline"]["bound"] == "alu"
