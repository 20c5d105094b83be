#!/bin/bash
# ncu --set full of one C4 step with Proth primes (where Kernel-1's time does not follow its multiply work)
O=gpurun_out/ncu_r02j; rm -rf $O; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_shared" -s 4 -c 4 -o $O/c4p python tools/profile_step.py --warmup 1 --primes proth > $O/c4p.log 2>&1
ncu -i $O/c4p.ncu-rep --page raw --csv > $O/c4p_raw.csv 2>/dev/null
for k in 0 3; do ncu -i $O/c4p.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 > $O/sass_$k.csv 2>/dev/null; done
ncu -i $O/c4p.ncu-rep --page details --csv > $O/c4p_details.csv 2>/dev/null
rm -f $O/*.ncu-rep; ls -la $O
