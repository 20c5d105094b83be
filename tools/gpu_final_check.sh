#!/bin/bash
# gpurun -- bash tools/gpu_final_check.sh TAG
# The driver's round-end tiers (tools/round_end_check.sh), every bench config,
# the C4 launch list and one ncu --set full of the C4 step, into gpurun_out/roundend
# and gpurun_out/ncu_TAG (the r02k..r02o checks of profiles/).
TAG=${1:-check}
bash tools/round_end_check.sh
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/roundend/bench_$c.json 2>> gpurun_out/roundend/bench_cx.err; done
O=gpurun_out/ncu_$TAG; rm -rf $O; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_shared" -s 4 -c 4 -o $O/c4 python tools/profile_step.py --warmup 1 --primes 2n > $O/c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python tools/profile_step.py --warmup 1 --primes 2n > $O/c4_launch.log 2>&1
ncu -i $O/c4.ncu-rep --page raw --csv > $O/c4_raw.csv 2>/dev/null
for k in 0 1 2 3; do ncu -i $O/c4.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 > $O/sass_$k.csv 2>/dev/null; done
python tools/sass_opcode_mix.py $O > $O/opcode_mix.txt 2>&1
rm -f $O/*.ncu-rep
