import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2012_01968_b200 import Plan, find_primes
N, L, B = 1 << 17, 60, 32
primes = find_primes(N, L, "proth")
x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"])
d = torch.from_numpy(x.view(np.int64)).cuda(); ref = d.clone()
for fused in (True, False):
    plan = Plan(N, primes, fused=fused)
    for _ in range(3): plan.forward(d); plan.inverse(d)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fw, iv = [], []
    for _ in range(10):
        e[0].record(); plan.forward(d); e[1].record(); plan.inverse(d); e[2].record(); torch.cuda.synchronize()
        fw.append(e[0].elapsed_time(e[1])); iv.append(e[1].elapsed_time(e[2]))
    print(json.dumps({"fused": fused, "fwd_ms": round(float(np.median(fw)), 4), "inv_ms": round(float(np.median(iv)), 4), "ok": bool(torch.equal(d, ref))}))
    plan.close()
