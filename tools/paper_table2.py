"""The paper's Table 2 setting on B200: forward NTT of np = 21
residue rows (batch 1) at N = 2^14..2^17 with the radix-2 baseline, the
register radix-16 kernel, and the two-kernel SMEM path without / with OT.
Prints one JSON line per N with GPU times (us, all 21 rows together, as in the
paper, R13) and the SMEM+OT / radix-2 speedup the paper reports as
4.2x on Titan V, twice: L2-warm (`reps` calls replayed from one
CUDA graph, the 21 rows stay in the 126 MB L2) and DRAM-bound (the 126 MB L2
flushed by a 512 MiB write before every call, outside the timed span; each
call replayed from its own graph so host launch cost stays out) -- the
setting the paper measured on Titan V, whose 4.5 MB L2 held none of it.
A flush before the call still lets the radix-2 baseline's 2nd..logN-th
stages hit L2 (21 rows of 2^17 words are 21 MiB), so a third block runs the
same 21 primes over enough ciphertexts that the data (>= 512 MiB) cannot stay
in L2 between stages, reported per 21 rows: every stage of every kernel then
streams from DRAM, the regime of the paper's Titan V.

    python tools/paper_table2.py [--reps 50] [--np 21]
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


FLUSH = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")


def time_us_flushed(fn, d, reps):
    """GPU time per call with the L2 flushed before each call (untimed)."""
    for _ in range(3):
        fn(d)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn(d)
    torch.cuda.current_stream().wait_stream(s)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        FLUSH.fill_(i)  # 512 MiB > 2 x L2: every row and table comes from DRAM
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2] * 1e3


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
    fr2 = time_us_flushed(lambda t: plan.forward_variant(t, 1), d, a.reps)
    fr16 = time_us_flushed(lambda t: plan.forward_variant(t, 2), d, a.reps)
    fsmem = time_us_flushed(lambda t: plan.forward(t), d, a.reps)
    fsmem_ot = time_us_flushed(lambda t: plan_ot.forward(t), d, a.reps)
    nb = max(1, (512 << 20) // (a.np * N * 8))  # ciphertexts for >= 512 MiB of rows
    xb = synth.rns_rows(primes, nb, N, config_id=synth.CONFIG_IDS["Cp"])
    db = torch.from_numpy(xb.view(np.int64)).cuda()
    dr2 = time_us_flushed(lambda t: plan.forward_variant(t, 1), db, 5) / nb
    dr16 = time_us_flushed(lambda t: plan.forward_variant(t, 2), db, 5) / nb
    dsmem = time_us_flushed(lambda t: plan.forward(t), db, 5) / nb
    dsmem_ot = time_us_flushed(lambda t: plan_ot.forward(t), db, 5) / nb
    del db, xb
    p = PAPER[logn]
    print(json.dumps({
        "logN": logn, "np": a.np, "unit": "us (all np rows, forward only)",
        "b200": {"radix2": round(r2, 2), "radix16_reg": round(r16, 2), "smem": round(smem, 2),
                 "smem_ot": round(smem_ot, 2), "speedup_smem_vs_radix2": round(r2 / smem, 2),
                 "speedup_smem_ot_vs_radix2": round(r2 / smem_ot, 2), "l2": "warm (graph of reps)"},
        "b200_flushed": {"radix2": round(fr2, 2), "radix16_reg": round(fr16, 2), "smem": round(fsmem, 2),
                         "smem_ot": round(fsmem_ot, 2), "speedup_smem_vs_radix2": round(fr2 / fsmem, 2),
                         "speedup_smem_ot_vs_radix2": round(fr2 / fsmem_ot, 2),
                         "ot_effect": round(fsmem / fsmem_ot, 3),
                         "l2": "flushed before each call (512 MiB write, untimed); median of reps"},
        "b200_dram_resident": {"radix2": round(dr2, 2), "radix16_reg": round(dr16, 2), "smem": round(dsmem, 2),
                               "smem_ot": round(dsmem_ot, 2), "speedup_smem_vs_radix2": round(dr2 / dsmem, 2),
                               "speedup_smem_ot_vs_radix2": round(dr2 / dsmem_ot, 2),
                               "ot_effect": round(dsmem / dsmem_ot, 3),
                               "batch": nb, "per": "21 rows (time of the batch / batch)"},
        "paper_titan_v": {"radix2": p[0], "smem": p[1], "smem_ot": p[2],
                          "speedup_smem_ot_vs_radix2": round(p[0] / p[2], 2)},
    }), flush=True)
    plan.close()
    plan_ot.close()
