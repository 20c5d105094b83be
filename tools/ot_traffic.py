"""On-the-fly twiddling on B200: DRAM traffic and time of one
forward NTT with OT off / on (1 or 2 stages, base B), in the paper's Table 2
setting (N = 2^17, np = 21 rows, batch 1: the twiddle tables are not amortised
over a batch) and at C4.  Run under ncu for the bytes:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum \
        --csv --log-file ot.csv python tools/ot_traffic.py --mode ncu
    python tools/ot_traffic.py --mode time      (CUDA-event timings, OT base sweep)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_01968_b200 import Plan, find_primes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="time", choices=["time", "ncu"])
ap.add_argument("--primes", default="proth", choices=["2n", "proth"])
a = ap.parse_args()

# Cp: the paper's Table 2 setting (21 rows; on B200 its 42 MB of tables fit the
# 126 MB L2); L60: one ciphertext of the C4 chain (120 MB of tables: > L2);
# C4: the headline batch (tables amortised over 32 ciphertexts)
SETTINGS = {"Cp": (17, 21, 1), "L60": (17, 60, 1), "C4": (17, 60, 32)}
OT = [("off", {}), ("1 stage B=1024", {"ot": True, "ot_stages": 1}), ("2 stages B=1024", {"ot": True, "ot_stages": 2})]
if a.mode == "time":
    OT += [(f"2 stages B={b}", {"ot": True, "ot_stages": 2, "ot_base": b}) for b in (32, 128, 256, 512, 2048, 4096)]

for name, (logn, L, B) in SETTINGS.items():
    N = 1 << logn
    primes = find_primes(N, L, a.primes)
    x = torch.from_numpy(synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS.get(name, 17)).view(np.int64)).cuda()
    for label, kw in OT:
        plan = Plan(N, primes, **kw)
        if a.mode == "ncu":  # one forward per setting; the ncu log carries the bytes
            torch.cuda.nvtx.range_push(f"{name} {label}")
            plan.forward(x)
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
            print(json.dumps({"setting": name, "ot": label, "launch_order": "Kernel-1, Kernel-2"}), flush=True)
        else:
            for _ in range(5):
                plan.forward(x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                plan.forward(x)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            tb = plan.info()["table_bytes"]
            print(json.dumps({"setting": name, "N": N, "L": L, "batch": B, "ot": label, "fwd_us": round(us, 2),
                              "plan_table_bytes": tb}), flush=True)
        plan.close()
