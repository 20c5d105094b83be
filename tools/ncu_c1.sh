#!/bin/bash
# ncu of the C1 single-CTA kernels (N = 2^12, one row): where a 4096-point transform's 14 us go
O=gpurun_out/ncu_c1; rm -rf $O; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_contig" -s 2 -c 2 -o $O/c1 python tools/profile_step.py --config C1 --warmup 1 --primes 2n > $O/c1.log 2>&1
ncu -i $O/c1.ncu-rep --page raw --csv > $O/c1_raw.csv 2>/dev/null
for k in 0 1; do ncu -i $O/c1.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 > $O/sass_$k.csv 2>/dev/null; done
rm -f $O/*.ncu-rep; ls -la $O
