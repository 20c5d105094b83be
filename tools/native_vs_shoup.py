"""The paper's fig:native_shoup on B200: forward NTT at
(N, np) = (2^17, 45), batch 1 (the figure's setting) and batch 8, through the
default kernels with Shoup's modmul and through the same kernels with the
native 128-bit modulo (NTT_VARIANT_NATIVE); L2 flushed before each call
(DRAM-bound, as on the paper's GPU), GPU time from per-call graph replays.
The paper reports Shoup 2.4x faster.

    python tools/native_vs_shoup.py [--reps 20]
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
from paper_2012_01968_b200._native import NTT_VARIANT_NATIVE  # noqa: E402

FLUSH = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")


def per_call_us(fn, d, reps):
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
        FLUSH.fill_(i)
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2] * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    N, L = 1 << 17, 45
    for form in ("2n", "proth"):
        primes = find_primes(N, L, form)
        plan = Plan(N, primes)
        for batch in (1, 8):
            x = synth.rns_rows(primes, batch, N, config_id=synth.CONFIG_IDS["C3"])
            d = torch.from_numpy(x.view(np.int64)).cuda()
            ref = d.clone()
            plan.forward(ref)
            shoup = per_call_us(lambda t: plan.forward(t), d.clone(), a.reps)
            dn = d.clone()
            plan.forward_variant(dn, NTT_VARIANT_NATIVE)
            exact = bool(torch.equal(dn, ref))
            native = per_call_us(lambda t: plan.forward_variant(t, NTT_VARIANT_NATIVE), d.clone(), a.reps)
            print(json.dumps({"N": N, "np": L, "batch": batch, "primes": form, "arith": plan.info()["arith"],
                              "shoup_us": round(shoup, 2), "native_us": round(native, 2),
                              "speedup_shoup_vs_native": round(native / shoup, 2), "paper_speedup": 2.4,
                              "native_bit_exact_vs_shoup": exact,
                              "l2": "flushed before each call; median of reps"}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
