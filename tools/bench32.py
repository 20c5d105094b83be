"""32-bit vs 64-bit words at equal modulus size (NEXT-4; the paper's 32b-vs-64b
comparison): time forward+inverse of a config with its 60-bit chain
and with a 30-bit chain of twice as many primes (same Q bits, same HBM bytes).

    python tools/bench32.py [--config C4] [--steps 10] [--log-n1 0]

Prints one JSON line per word size (CUDA events, inputs resident)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2012_01968_b200 import Plan, Plan32, find_primes, find_primes32  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--log-n1", type=int, default=0)
ap.add_argument("--primes", default="proth", choices=["2n", "proth"], help="64-bit prime family")
a = ap.parse_args()
logn, L, B, _ = CONFIGS[a.config]
N = 1 << logn


def timeit(plan, d, steps):
    for _ in range(3):
        plan.forward(d)
        plan.inverse(d)
    f = [torch.cuda.Event(enable_timing=True) for _ in range(3 * steps)]
    torch.cuda.synchronize()
    for s in range(steps):
        f[3 * s].record()
        plan.forward(d)
        f[3 * s + 1].record()
        plan.inverse(d)
        f[3 * s + 2].record()
    torch.cuda.synchronize()
    fw = sorted(f[3 * s].elapsed_time(f[3 * s + 1]) for s in range(steps))[steps // 2]
    iv = sorted(f[3 * s + 1].elapsed_time(f[3 * s + 2]) for s in range(steps))[steps // 2]
    return fw * 1e3, iv * 1e3


for bits in (64, 32):
    nl = L if bits == 64 else 2 * L
    primes = find_primes(N, nl, a.primes) if bits == 64 else find_primes32(N, nl)
    x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS.get(a.config, 15))
    if bits == 64:
        d = torch.from_numpy(x.view(np.int64)).cuda()
        plan = Plan(N, primes, log_n1=a.log_n1)
    else:
        d = torch.from_numpy(x.astype(np.uint32).view(np.int32)).cuda()
        plan = Plan32(N, primes, log_n1=a.log_n1)
    x0 = d.clone()
    fw, iv = timeit(plan, d, a.steps)
    ok = bool(torch.equal(d, x0))  # an even number of round trips leaves the data unchanged
    rows = B * nl
    bf = rows * (N // 2) * logn
    print(json.dumps({"bits": bits, "config": a.config, "N": N, "primes": nl, "q_bits": sum(p.bit_length() for p in primes),
                      "batch": B, "fwd_us": round(fw, 1), "inv_us": round(iv, 1),
                      "us_per_ntt_intt": round(fw + iv, 1), "roundtrip_ok": ok,
                      "Gbf_per_s": round(2 * bf / ((fw + iv) * 1e-6) / 1e9, 1),
                      "hbm_GBps_data": round(2 * (2 if plan.info()["log_n1"] else 1) * 2 * d.numel() * d.element_size()
                                             / ((fw + iv) * 1e-6) / 1e9, 1),
                      "log_n1": plan.info()["log_n1"]}), flush=True)
    plan.close()
    del d, x0
