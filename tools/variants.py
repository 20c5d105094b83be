"""Time kernel variants on one config (per-pass CUDA-event averages).

    python tools/variants.py [--config C4] [--steps 10] [--ot] [--log-n1 K]

Variants "k1,k2" are the ntt_opts_t k1_variant / k2_variant fields.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--ot", action="store_true")
ap.add_argument("--log-n1", type=int, default=0)
ap.add_argument("--variants", default="4,9;4,7;4,5")
ap.add_argument("--primes", default="proth", choices=["2n", "proth"])
a = ap.parse_args()
logn, L, B, _ = CONFIGS[a.config]
N = 1 << logn
primes = find_primes(N, L, a.primes)
x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS[a.config])
host = torch.from_numpy(x.view(np.int64))
d = host.cuda()
rows = B * L
for var in a.variants.split(";"):
    k1, k2 = (int(v) for v in var.split(","))
    plan = Plan(N, primes, ot=a.ot, log_n1=a.log_n1, k1_variant=k1, k2_variant=k2)
    info = plan.info()
    seq = [(NTT_DIR_FORWARD, i) for i in range(plan.passes)] + [(NTT_DIR_INVERSE, i) for i in range(plan.passes)]
    for _ in range(3):
        plan.forward(d)
        plan.inverse(d)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(a.steps)]
    torch.cuda.synchronize()
    for s in range(a.steps):
        ev[s][0].record()
        for j, (dd, p) in enumerate(seq):
            plan.launch_pass(d, dd, p)
            ev[s][j + 1].record()
    torch.cuda.synchronize()
    ms = [statistics.mean(ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(a.steps)) for j in range(len(seq))]
    ok = bool(torch.equal(d, host.cuda()))
    tot = sum(ms)
    ln1 = info["log_n1"]
    st = [ln1, logn - ln1, logn - ln1, ln1] if plan.passes == 2 else [logn, logn]
    gbf = [rows * (N // 2) * s / (m * 1e-3) / 1e9 for s, m in zip(st, ms)]
    print(json.dumps({"variant": var, "config": a.config, "ot": a.ot, "log_n1": ln1, "ok": ok,
                      "ms": [round(m, 4) for m in ms], "step_ms": round(tot, 4),
                      "us_per_ct": round(tot * 1e3 / B, 2), "Gbfly_s": [round(g, 1) for g in gbf]}), flush=True)
    plan.close()
