"""Experiment: do Kernel-1 and Kernel-2 CTAs mixed on the SMs run faster than
the kernels back to back?  C4 split into two ciphertext halves on two streams
(offset by one kernel) vs the whole batch on one stream."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes  # noqa: E402

N, L, B = 1 << 17, 60, 32
primes = find_primes(N, L, "proth")
x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"])
d = torch.from_numpy(x.view(np.int64)).cuda()
ref = d.clone()
plan = Plan(N, primes)
seq = [(NTT_DIR_FORWARD, 0), (NTT_DIR_FORWARD, 1), (NTT_DIR_INVERSE, 0), (NTT_DIR_INVERSE, 1)]


def one_stream():
    for dd, p in seq:
        plan.launch_pass(d, dd, p)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ev = torch.cuda.Event()


def two_streams(parts):
    hs = [d[i * B // parts:(i + 1) * B // parts] for i in range(parts)]
    streams = [torch.cuda.Stream() for _ in range(parts)]
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    # stream i starts one kernel later than stream i-1: K1 of one part overlaps K2 of the previous
    for k in range(len(seq) + parts - 1):
        for i, (h, s) in enumerate(zip(hs, streams)):
            j = k - i
            if 0 <= j < len(seq):
                with torch.cuda.stream(s):
                    plan.launch_pass(h, *seq[j])
    for s in streams:
        cur.wait_stream(s)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {"one_stream_ms": round(timeit(one_stream), 4)}
for parts in (2, 4):
    res[f"{parts}_streams_ms"] = round(timeit(lambda: two_streams(parts)), 4)
res["ok"] = bool(torch.equal(d, ref))
print(json.dumps(res))
