"""C5 small-request latency breakdown (experiment): for one ciphertext of L
primes at N = 2^16, the GPU time of each kernel of NTT + iNTT (CUDA events
around single launches) and the latency of the request replayed through the
library's request graph (ntt_graph_create / ntt_graph_launch), per split.

    python tools/c5_latency.py [--primes 2n|proth] [--splits 6,7,8,9,10]

The one-kernel request (NTT_GRAPH_ONE_KERNEL, ntt_request.cu) is timed on the
--splits-one row (its own split does not depend on the plan's).
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
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL, Plan, find_primes  # noqa: E402


def event_ms(fn, reps=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--primes", default="2n")
    ap.add_argument("--splits", default="6,7,8,9,10")
    ap.add_argument("--L", default="1,8,45")
    ap.add_argument("--logn", type=int, default=16)
    ap.add_argument("--splits-one", type=int, default=7, help="the split row that also times NTT_GRAPH_ONE_KERNEL")
    args = ap.parse_args()
    N = 1 << args.logn
    for L in [int(v) for v in args.L.split(",")]:
        primes = find_primes(N, L, args.primes)
        x = torch.from_numpy(synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["C5"]).view(np.int64)).cuda()
        ref = x.clone()
        for ln1 in [int(v) for v in args.splits.split(",")]:
            plan = Plan(N, primes, log_n1=ln1)
            for _ in range(3):
                plan.forward(x)
                plan.inverse(x)
            kern = {}
            for d, name in ((NTT_DIR_FORWARD, "fwd"), (NTT_DIR_INVERSE, "inv")):
                for p in range(plan.passes):
                    kern[f"{name}_pass{p}_us"] = round(1e3 * event_ms(lambda: plan.launch_pass(x, d, p)), 2)
            x.copy_(ref)
            res = {}
            for key, fl in (("graph", 0), ("one_kernel", NTT_GRAPH_ONE_KERNEL)):
                if fl and ln1 != args.splits_one:
                    continue
                g = plan.graph(x, NTT_DIR_FORWARD | NTT_DIR_INVERSE | fl)
                for _ in range(5):
                    g.launch()
                lat = 1e3 * event_ms(g.launch, 100)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(200):
                    g.launch()
                e1.record()
                torch.cuda.synchronize()
                res[f"{key}_latency_us"] = round(lat, 2)
                res[f"{key}_stream_us_per_request"] = round(e0.elapsed_time(e1) * 1e3 / 200, 2)
                res[f"{key}_ok"] = bool(torch.equal(x, ref))
                g.close()
            print(json.dumps({"N": N, "L": L, "log_n1": ln1, "primes": args.primes, **kern, **res}), flush=True)
            plan.close()


if __name__ == "__main__":
    main()
