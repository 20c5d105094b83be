"""Small workload touching every kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Exits non-zero if any result differs from the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2012_01968_b200 import Plan  # noqa: E402


def run(N, L, batch, proth=False, **kw):
    # Proth primes (p = 1 mod 2^32) from the oracle's own scan at step 2^32
    primes = oracle.find_primes(1 << 31, L) if proth else oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, batch, N, config_id=14)
    plan = Plan(N, primes, **kw)
    d = torch.from_numpy(x.view(np.int64)).cuda()
    plan.forward(d)
    torch.cuda.synchronize()
    ok = np.array_equal(d.cpu().numpy().view(np.uint64), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    torch.cuda.synchronize()
    ok &= np.array_equal(d.cpu().numpy().view(np.uint64), x)
    y = torch.from_numpy(x.view(np.int64)).cuda()
    plan.negacyclic_mul(d, y)
    torch.cuda.synchronize()
    for v in (1, 2):
        z = torch.from_numpy(x.view(np.int64)).cuda()
        plan.forward_variant(z, v)
        torch.cuda.synchronize()
        ok &= np.array_equal(z.cpu().numpy().view(np.uint64), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.close()
    return ok


cases = [(1 << 10, 2, 1, {}), (1 << 12, 1, 1, {"ot": True}), (1 << 14, 2, 1, {}), (1 << 15, 2, 1, {"ot": True}),
         (1 << 16, 1, 1, {"log_n1": 8}),
         # shared-twiddle Kernel-2 (batch >= 2^12 / N2), Proth kernels, the single-pass cluster kernel
         (1 << 14, 1, 16, {}), (1 << 17, 1, 8, {"proth": True}), (1 << 16, 1, 8, {"proth": True, "ot": True}),
         (1 << 12, 1, 2, {"proth": True}), (1 << 15, 1, 1, {"fused": True}), (1 << 17, 1, 1, {"fused": True, "proth": True})]
bad = [c[:3] for c in cases if not run(*c[:3], **c[3])]


def run_one_kernel(N, L, batch, proth=False):
    """The one-kernel request (NTT_GRAPH_ONE_KERNEL): a forward-only graph
    against the oracle, then a forward + inverse graph restoring the input."""
    from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL
    primes = oracle.find_primes(1 << 31, L) if proth else oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, batch, N, config_id=15)
    plan = Plan(N, primes)
    d = torch.from_numpy(x.view(np.int64)).cuda()
    g = plan.graph(d, NTT_DIR_FORWARD | NTT_GRAPH_ONE_KERNEL)
    g.launch()
    torch.cuda.synchronize()
    ok = np.array_equal(d.cpu().numpy().view(np.uint64), oracle.ntt_batch(x.copy(), primes, psis, +1))
    g.close()
    d.copy_(torch.from_numpy(x.view(np.int64)))
    g = plan.graph(d, NTT_DIR_FORWARD | NTT_DIR_INVERSE | NTT_GRAPH_ONE_KERNEL)
    g.launch()
    torch.cuda.synchronize()
    ok &= np.array_equal(d.cpu().numpy().view(np.uint64), x)
    g.close()
    plan.close()
    return ok


bad += [("one_kernel",) + c for c in [(1 << 14, 1, 1, False), (1 << 16, 2, 1, True)] if not run_one_kernel(*c)]
print("sanitize workload:", "ok" if not bad else f"MISMATCH {bad}")
sys.exit(1 if bad else 0)
