#!/bin/bash
# One gpurun call: the paper-context measurements of round 2 --
# Table 2 L2-warm / flushed / DRAM-resident (tools/paper_table2.py), native
# modulo vs Shoup at (2^17, 45) (tools/native_vs_shoup.py), and ncu DRAM bytes
# of the radix-2 baseline vs the SMEM path at N = 2^17, np = 21.
#   gpurun --timeout 1800 -- bash tools/gpu_r02_context.sh TAG
TAG=${1:-ctx}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python tools/paper_table2.py --reps 30 > $O/paper_table2.jsonl 2> $O/paper_table2.err
timeout 600 python tools/native_vs_shoup.py --reps 10 > $O/native_vs_shoup.jsonl 2> $O/native_vs_shoup.err
cat > /tmp/t2one.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2012_01968_b200 import Plan, find_primes
N = 1 << 17
primes = find_primes(N, 21)
x = torch.from_numpy(synth.rns_rows(primes, 1, N, config_id=synth.CONFIG_IDS["Cp"]).view(np.int64)).cuda()
plan, plan_ot = Plan(N, primes), Plan(N, primes, ot=True)
plan.forward_variant(x, 1); plan.forward(x); plan_ot.forward(x)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/table2_dram.csv python /tmp/t2one.py > $O/table2_dram.log 2>&1
cat $O/*.jsonl
