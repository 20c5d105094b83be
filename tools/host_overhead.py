"""Host-side cost of one ntt_forward call (C ABI + binding), and the GPU time
of a single small request replayed from a CUDA graph (C5 latency context)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import Plan, find_primes, _native  # noqa: E402

N = 1 << 16
FUSED = "--fused" in sys.argv
for L in (1, 8, 45):
    primes = find_primes(N, L, "proth")
    plan = Plan(N, primes, fused=True if FUSED else None)
    x = torch.from_numpy(synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["C5"]).view(np.int64)).cuda()
    ref = x.clone()
    for _ in range(5):
        plan.forward(x)
        plan.inverse(x)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        plan.forward(x)
        plan.inverse(x)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    py_us = (t1 - t0) / n / 2 * 1e6
    # raw C ABI call (no torch checks in the binding)
    lib = _native.lib()
    h, ptr, st = plan.handle, x.data_ptr(), torch.cuda.current_stream().cuda_stream
    t0 = time.perf_counter()
    for _ in range(n):
        lib.ntt_forward(h, ptr, 1, st)
        lib.ntt_inverse(h, ptr, 1, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    c_us = (t1 - t0) / n / 2 * 1e6
    # CUDA graph: forward + inverse captured once, replayed per request
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            plan.forward(x)
            plan.inverse(x)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    lat = []
    for _ in range(20):
        e[0].record()
        g.replay()
        e[1].record()
        torch.cuda.synchronize()
        lat.append(e[0].elapsed_time(e[1]) * 1e3)
    e[0].record()
    for _ in range(64):
        g.replay()
    e[1].record()
    torch.cuda.synchronize()
    ok = bool(torch.equal(x, ref))
    print(json.dumps({"N": N, "L": L, "fused": FUSED, "host_us_per_call_binding": round(py_us, 2), "host_us_per_call_cabi": round(c_us, 2),
                      "graph_latency_us": round(float(np.median(lat)), 2),
                      "graph_stream_us_per_request": round(e[0].elapsed_time(e[1]) * 1e3 / 64, 2), "ok": ok}), flush=True)
    plan.close()
