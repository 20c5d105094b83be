"""Is the C5 stream-mode latency (bench.py: replays back to back, an event
after each) bound by the GPU or by host submission?  For the one-kernel and
the split request graphs at N = 2^16, L = 1: (a) the bench's measurement,
(b) host time per loop iteration (perf_counter), (c) the same replays queued
behind a gate kernel so the GPU runs them back to back from a full queue
(device-side time per request, no host in the loop).

    python tools/c5_hostbound.py [--L 1]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL, Plan, find_primes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=1)
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    N = 1 << 16
    primes = find_primes(N, args.L)
    x = torch.from_numpy(synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["C5"]).view(np.int64)).cuda()
    plan = Plan(N, primes)
    for form, flag in (("graph", 0), ("one_kernel", NTT_GRAPH_ONE_KERNEL)):
        g = plan.graph(x, NTT_DIR_FORWARD | NTT_DIR_INVERSE | flag)
        for _ in range(10):
            g.launch()
        torch.cuda.synchronize()
        reps = args.reps
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        t0 = time.perf_counter()
        evs[0].record()
        for i in range(reps):
            g.launch()
            evs[i + 1].record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        bench_like = statistics.median(evs[i].elapsed_time(evs[i + 1]) for i in range(reps)) * 1e3
        host_us = (t1 - t0) / reps * 1e6
        # gated: a 20 ms sleep kernel holds the stream while the replays are queued
        evs2 = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        torch.cuda._sleep(int(2e7))
        evs2[0].record()
        for i in range(reps):
            g.launch()
            evs2[i + 1].record()
        torch.cuda.synchronize()
        gated = statistics.median(evs2[i].elapsed_time(evs2[i + 1]) for i in range(reps)) * 1e3
        gated_mean = evs2[0].elapsed_time(evs2[reps]) * 1e3 / reps
        # gated, events only at the ends
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e7))
        ea.record()
        for i in range(reps):
            g.launch()
        eb.record()
        torch.cuda.synchronize()
        gated_noev = ea.elapsed_time(eb) * 1e3 / reps
        print(json.dumps({"L": args.L, "form": form, "bench_like_us": round(bench_like, 2),
                          "gated_no_events_us": round(gated_noev, 2),
                          "host_us_per_iteration": round(host_us, 2), "gated_median_us": round(gated, 2),
                          "gated_mean_us": round(gated_mean, 2)}), flush=True)
        g.close()
    plan.close()


if __name__ == "__main__":
    main()
