"""End-to-end C4 step through the host-buffer C-ABI path (ntt_execute_host:
pinned host in -> H2D -> fwd -> inv -> D2H, pipelined): ms per step and the
PCIe bandwidth it implies.  python tools/e2e.py [--steps 5]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
N, L, B = 1 << 17, 60, 32
primes = find_primes(N, L, "proth")
host = torch.empty(B * L * N, dtype=torch.int64).pin_memory()
synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"], out=host.numpy().view(np.uint64).reshape(B, L, N))
out = torch.empty_like(host).pin_memory()
plan = Plan(N, primes)
ws = torch.empty(plan.workspace_words(B), dtype=torch.int64, device="cuda")
plan.execute_host(host, out, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)
t0 = time.perf_counter()
for _ in range(a.steps):
    plan.execute_host(host, out, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)
dt = (time.perf_counter() - t0) / a.steps
# raw copy bandwidth for context: H2D and D2H alone, and both at once
dev = torch.empty_like(host, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t0
t0 = time.perf_counter(); out.copy_(dev, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t0
half = host.numel() // 2
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    dev[:half].copy_(host[:half], non_blocking=True)
with torch.cuda.stream(s2):
    out[half:].copy_(dev[half:], non_blocking=True)
torch.cuda.synchronize()
both = time.perf_counter() - t0
nbytes = host.numel() * 8
print(json.dumps({"ms_per_step": round(dt * 1e3, 2), "us_per_ct": round(dt * 1e6 / B, 1),
                  "bytes_each_way": nbytes, "h2d_GBps_alone": round(nbytes / h2d / 1e9, 1),
                  "d2h_GBps_alone": round(nbytes / d2h / 1e9, 1),
                  "bidir_GBps_each": round(nbytes / 2 / both / 1e9, 1),
                  "ok": bool(torch.equal(out, host))}), flush=True)
