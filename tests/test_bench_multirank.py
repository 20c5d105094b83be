"""bench.py end to end on the GPU: `python bench.py --gpus 2` WITHOUT torchrun
(it re-launches itself under torch.distributed.run; with one visible GPU both
ranks share it over gloo), strong-scaled over contiguous prime ranges, with
the per-row checksums of every rank checked against the oracle on rank 0;
the weak-scaled form under torchrun; C5 at one GPU."""
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


def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def one_line(r):
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_gpus2_self_launch_strong():
    _need_gpu()
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "C2", "--no-cpu"]
    d = one_line(subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT))
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["higher_is_better"] is False
    assert d["config"]["global_batch"] == 16 and "[8, 7]" in d["config"]["shard"]
    assert d["verify"]["verified_rows"] > 0 and d["verify"]["mismatched"] == []
    assert d["verify"]["rows_checked_vs_oracle"] == d["verify"]["verified_rows"]
    assert d["roundtrip_exact"] is True and d["e2e"]["ok"] is True
    assert len(d["per_rank_ms"]) == 2 and d["imbalance"] >= 1.0
    assert d["value"] > 0 and d["roofline"]["bound"] == "alu" and d["gpu_launches"] > 0
    # SURVEY 8(e)'s balanced variant (C2: 240 rows -> 120 per rank, a partial prime each side)
    bal = d["balanced"]
    assert bal["value"] > 0 and bal["roundtrip_exact"] is True and len(bal["per_rank_ms"]) == 2
    assert bal["verify"]["verified_rows"] > 0 and bal["verify"]["mismatched"] == []
    assert bal["pieces_per_rank"] == [2, 2]


def test_bench_world2_weak_under_torchrun():
    _need_gpu()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "C2",
           "--scaling", "weak", "--no-cpu"]
    d = one_line(subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT))
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["global_batch"] == 32
    assert d["verify"]["verified_rows"] > 0 and not d["verify"]["mismatched"]


def test_bench_c5_one_gpu():
    _need_gpu()
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--config", "C5"]
    d = one_line(subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT))
    assert set(d["sweep"]) == {"1", "2", "4", "8", "15", "30", "45"}
    for v in d["sweep"].values():
        assert v["latency_us_per_request"] > 0 and v["throughput_us_per_request"] > 0
        assert set(v["latency_us_by_form"]) == {"graph", "graph_n1_2^7", "one_kernel"}
        assert v["latency_us_per_request"] == min(v["latency_us_by_form"].values())
    assert d["roundtrip_exact"] is True


def test_bench_c5_two_ranks():
    """C5 latency mode with the primes of one request sharded over 2 ranks
    (both request forms, ranks sharing one GPU over gloo)."""
    _need_gpu()
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "C5"]
    d = one_line(subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT))
    assert d["n_gpus"] == 2 and d["roundtrip_exact"] is True
    assert d["sweep"]["1"]["latency_primes_per_rank"] == [1, 0]


