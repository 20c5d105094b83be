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


def run(N, L, batch, **kw):
    primes = oracle.find_primes(N, L)
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
         (1 << 16, 1, 1, {"log_n1": 8})]
bad = [c[:3] for c in cases if not run(*c[:3], **c[3])]
print("sanitize workload:", "ok" if not bad else f"MISMATCH {bad}")
sys.exit(1 if bad else 0)
