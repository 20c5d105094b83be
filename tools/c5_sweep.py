"""BASELINE.json C5 (mixed ciphertext stream, N = 2^16): latency of one
request (1 ciphertext, NTT + iNTT of its L rows) and throughput of a stream of
requests, for L = 1..45, on one GPU.  Latency = CUDA-event time of a single
request on an idle GPU; throughput = requests/s when `--depth` requests are
issued back to back.  Prints one JSON line per L.

    python tools/c5_sweep.py [--depth 64]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import Plan, find_primes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--depth", type=int, default=64)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--fused", action="store_true", help="single-pass cluster kernel (ntt_opts_t.fused = 1)")
a = ap.parse_args()
N = 1 << 16
ap_primes = os.environ.get("C5_PRIMES", "proth")
all_primes = find_primes(N, 45, ap_primes)
for L in (1, 2, 4, 8, 15, 30, 45):
    primes = all_primes[:L]
    plan = Plan(N, primes, fused=True if a.fused else None)
    x = synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["C5"])
    reqs = torch.from_numpy(np.repeat(x, a.depth, axis=0).view(np.int64)).cuda()  # depth requests
    one = reqs[:1]
    for _ in range(3):
        plan.forward(one)
        plan.inverse(one)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    lat = []
    for _ in range(a.reps):
        e[0].record()
        plan.forward(one)
        plan.inverse(one)
        e[1].record()
        torch.cuda.synchronize()
        lat.append(e[0].elapsed_time(e[1]) * 1e3)
    # stream: requests issued back to back, one call pair per request
    e[0].record()
    for i in range(a.depth):
        r = reqs[i:i + 1]
        plan.forward(r)
        plan.inverse(r)
    e[1].record()
    torch.cuda.synchronize()
    stream_us = e[0].elapsed_time(e[1]) * 1e3 / a.depth
    # batched: the same requests as one batch (the throughput mode)
    e[0].record()
    plan.forward(reqs)
    plan.inverse(reqs)
    e[1].record()
    torch.cuda.synchronize()
    batched_us = e[0].elapsed_time(e[1]) * 1e3 / a.depth
    print(json.dumps({"config": "C5", "N": N, "L": L, "latency_us_median": round(float(np.median(lat)), 2),
                      "stream_us_per_request": round(stream_us, 2), "batched_us_per_request": round(batched_us, 2),
                      "depth": a.depth, "primes": ap_primes, "fused": a.fused}), flush=True)
    plan.close()
