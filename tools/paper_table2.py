"""The paper's Table 2 setting on B200: forward NTT of np = 21
residue rows (batch 1) at N = 2^14..2^17 with the radix-2 baseline, the
register radix-16 kernel, and the two-kernel SMEM path without / with OT.
Prints one JSON line per N with GPU times (us, all 21 rows together, as in the
paper, R13; calls replayed from a CUDA graph) and the SMEM+OT / radix-2 speedup the paper reports as
4.2x on Titan V.

    python tools/paper_table2.py [--reps 50]
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

PAPER = {14: (166, 48.6, 44.1), 15: (340, 92.0, 84.2), 16: (693, 171.8, 156.3), 17: (1427, 329.0, 304.2)}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--np", type=int, default=21)
a = ap.parse_args()


def time_us(fn, d, reps):
    """GPU time per call: `reps` calls captured in one CUDA graph and replayed,
    so host launch cost (several us per C-ABI call, larger than the kernels at
    these sizes) stays out of the measurement."""
    for _ in range(5):
        fn(d)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn(d)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for logn in (14, 15, 16, 17):
    N = 1 << logn
    primes = find_primes(N, a.np)
    x = synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["Cp"])
    d = torch.from_numpy(x.view(np.int64)).cuda()
    plan = Plan(N, primes)
    plan_ot = Plan(N, primes, ot=True)
    r2 = time_us(lambda t: plan.forward_variant(t, 1), d, a.reps)
    r16 = time_us(lambda t: plan.forward_variant(t, 2), d, a.reps)
    smem = time_us(lambda t: plan.forward(t), d, a.reps)
    smem_ot = time_us(lambda t: plan_ot.forward(t), d, a.reps)
    p = PAPER[logn]
    print(json.dumps({
        "logN": logn, "np": a.np, "unit": "us (all np rows, forward only)",
        "b200": {"radix2": round(r2, 2), "radix16_reg": round(r16, 2), "smem": round(smem, 2),
                 "smem_ot": round(smem_ot, 2), "speedup_smem_vs_radix2": round(r2 / smem, 2),
                 "speedup_smem_ot_vs_radix2": round(r2 / smem_ot, 2)},
        "paper_titan_v": {"radix2": p[0], "smem": p[1], "smem_ot": p[2],
                          "speedup_smem_ot_vs_radix2": round(p[0] / p[2], 2)},
    }), flush=True)
    plan.close()
    plan_ot.close()
