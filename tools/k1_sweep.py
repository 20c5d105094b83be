"""Kernel-1 variants on C4 (experiment): k1_variant 4 (one tile per CTA)
vs 5 (persistent, cp.async double buffer), per prime family; per-pass ms."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes  # noqa: E402

N, L, B = 1 << 17, 60, 32
variants = sys.argv[1].split(";") if len(sys.argv) > 1 else ["4,5", "5,5"]
for form in ["proth", "2n"]:
    primes = find_primes(N, L, form)
    x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"])
    d = torch.from_numpy(x.view(np.int64)).cuda()
    ref = d.clone()
    for var in variants:
        k1, k2 = (int(v) for v in var.split(","))
        plan = Plan(N, primes, fused=False, k1_variant=k1, k2_variant=k2)
        seq = [(NTT_DIR_FORWARD, 0), (NTT_DIR_FORWARD, 1), (NTT_DIR_INVERSE, 0), (NTT_DIR_INVERSE, 1)]
        for _ in range(3):
            plan.forward(d)
            plan.inverse(d)
        steps = 10
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
        torch.cuda.synchronize()
        for s in range(steps):
            ev[s][0].record()
            for j, (dd, p) in enumerate(seq):
                plan.launch_pass(d, dd, p)
                ev[s][j + 1].record()
        torch.cuda.synchronize()
        ms = [statistics.median(ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(steps)) for j in range(4)]
        print(json.dumps({"primes": form, "variant": var, "proth": plan.info()["proth"],
                          "ms": [round(m, 4) for m in ms], "us_per_ct": round(sum(ms) * 1e3 / B, 2),
                          "ok": bool(torch.equal(d, ref))}), flush=True)
        plan.close()
