import sys, os, json, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth
from paper_2012_01968_b200 import Plan, find_primes, NTT_DIR_FORWARD
for logn in (14, 15):
    N = 1 << logn
    primes = find_primes(N, 21)
    x = synth.rns_rows(primes, 1, N, config_id=17)
    d = torch.from_numpy(x.view(np.int64)).cuda()
    for var in ["4,5", "4,7", "4,4", "4,3", "5,5"]:
        k1, k2 = (int(v) for v in var.split(","))
        plan = Plan(N, primes, k1_variant=k1, k2_variant=k2)
        for _ in range(5):
            plan.forward(d)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t0, t1 = [], []
        for _ in range(20):
            ev[0].record(); plan.launch_pass(d, NTT_DIR_FORWARD, 0); ev[1].record(); plan.launch_pass(d, NTT_DIR_FORWARD, 1); ev[2].record()
            torch.cuda.synchronize()
            t0.append(ev[0].elapsed_time(ev[1]) * 1e3); t1.append(ev[1].elapsed_time(ev[2]) * 1e3)
        print(json.dumps({"logn": logn, "variant": var, "k1_us": round(statistics.median(t0), 2), "k2_us": round(statistics.median(t1), 2)}))
        plan.close()
