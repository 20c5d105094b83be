#!/bin/bash
# round-2 session-3 check of HEAD: driver's round-end tiers, then the ncu captures of the C4 step
bash tools/round_end_check.sh
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/roundend/bench_$c.json 2>> gpurun_out/roundend/bench_cx.err; done
bash tools/ncu_r02i.sh
