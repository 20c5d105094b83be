import os, sys, ctypes
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle, synth
from paper_2012_01968_b200 import Plan
N = 1 << 17
primes = oracle.find_primes(N, 2)
x = synth.rns_rows(primes, 2, N)
for n1 in (6, 7):
    plan = Plan(N, primes, log_n1=n1)
    d = torch.from_numpy(x.view(np.int64)).cuda()
    for p in (0, 1):
        try:
            plan.launch_pass(d, 1, p)
            torch.cuda.synchronize()
            print(n1, p, "ok")
        except Exception as e:
            print(n1, p, "ERR", e)
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
