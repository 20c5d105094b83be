"""One C4 step (forward + inverse of every row) after `--warmup` steps, for
ncu captures:  ncu ... python tools/profile_step.py [--config C4] [--ot]."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2012_01968_b200 import Plan, find_primes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--ot", action="store_true")
ap.add_argument("--log-n1", type=int, default=0)
ap.add_argument("--primes", default="2n", choices=["2n", "proth"])
a = ap.parse_args()
logn, L, B, _ = CONFIGS[a.config]
N = 1 << logn
primes = find_primes(N, L, a.primes)
x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS[a.config])
d = torch.from_numpy(x.view(np.int64)).cuda()
plan = Plan(N, primes, ot=a.ot, log_n1=a.log_n1)
for _ in range(a.warmup + a.steps):
    plan.forward(d)
    plan.inverse(d)
torch.cuda.synchronize()
assert np.array_equal(d.cpu().numpy().view(np.uint64), x)
print("ok", plan.info())
