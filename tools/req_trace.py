"""Phase timeline of the one-kernel request (experiment; needs a library
built with -DNTT_REQ_TRACE, tools/build_variant.sh, copied over libntt.so):
thread 0 of every CTA records %globaltimer at the phase boundaries; per
launch the phases' critical-path durations are taken from the CTA maxima /
minima, and the medians over --reps launches are printed, beside the event
latency of a lone replay.

    python tools/req_trace.py [--logn 16] [--L 1,2,4,8] [--reps 30]
"""
import argparse
import ctypes
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
from paper_2012_01968_b200._native import lib  # noqa: E402

# mark slots (ntt_request.cu REQ_MARK)
ENTRY, C_DONE, BAR1, BB_DONE, BAR2, CI_DONE, C_READY, B_READY, B_FWD, CI_READY = 0, 1, 2, 3, 4, 5, 6, 8, 9, 12


def phases(t):
    """Critical-path phase durations (us) of one launch from the [ctas][16] marks."""
    t = t[t[:, 0] > 0].astype(np.int64)
    t0 = t[:, ENTRY].min()
    mx = lambda i: (t[:, i].max() - t0) / 1e3  # noqa: E731
    mn = lambda i: (t[:, i].min() - t0) / 1e3  # noqa: E731
    return {
        "C_ready": mx(C_READY), "C": mx(C_DONE) - mx(C_READY), "bar1": mn(BAR1) - mx(C_DONE),
        "bar1_spread": mx(BAR1) - mn(BAR1), "B_ready": mx(B_READY) - mn(BAR1), "B_fwd": mx(B_FWD) - mx(B_READY),
        "B_inv": mx(BB_DONE) - mx(B_FWD), "bar2": mn(BAR2) - mx(BB_DONE), "Ci_ready": mx(CI_READY) - mn(BAR2),
        "Ci": mx(CI_DONE) - mx(CI_READY), "span": mx(CI_DONE), "ctas": len(t),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, default=16)
    ap.add_argument("--L", default="1,2,4,8")
    ap.add_argument("--primes", default="2n")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    N = 1 << args.logn
    fn = lib().ntt_debug_req_trace
    fn.argtypes = [ctypes.c_void_p]
    for L in [int(v) for v in args.L.split(",")]:
        primes = find_primes(N, L, args.primes)
        x = torch.from_numpy(synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["C5"]).view(np.int64)).cuda()
        plan = Plan(N, primes)
        g = plan.graph(x, NTT_DIR_FORWARD | NTT_DIR_INVERSE | NTT_GRAPH_ONE_KERNEL)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lat, ph = [], []
        buf = np.zeros((1024, 16), dtype=np.uint64)
        for _ in range(5):
            g.launch()
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0.record()
            g.launch()
            e1.record()
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
            buf[:] = 0
            assert fn(buf.ctypes.data) == 0
            ph.append(phases(buf))
        out = {"tag": args.tag, "N": N, "L": L, "latency_us_med": round(statistics.median(lat), 2),
               "latency_us_min": round(min(lat), 2)}
        for k in ph[0]:
            out[k] = round(float(statistics.median([p[k] for p in ph])), 2)
        print(json.dumps(out), flush=True)
        g.close()
        plan.close()


if __name__ == "__main__":
    main()
