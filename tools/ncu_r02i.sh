O=gpurun_out/ncu_r02i
mkdir -p $O
rm -rf gpurun_out/ncu_r02i; mkdir -p gpurun_out/ncu_r02i
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_shared|k_blocks|k_contig" -s 4 -c 4 -o $O/c4 python tools/profile_step.py --warmup 1 --primes 2n > $O/c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python tools/profile_step.py --warmup 1 --primes 2n > $O/c4_launch.log 2>&1
for c in C2 C3; do timeout 600 ncu --set full --clock-control none -k regex:"k_cols|k_shared|k_blocks|k_contig" -s 4 -c 4 -o $O/$c python tools/profile_step.py --config $c --warmup 1 --primes 2n > $O/$c.log 2>&1; done
ls -la $O
# export what profiles/ needs, drop the reports (gpurun copies back <= 64 MiB)
for r in c4 C2 C3; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null; done
for k in 0 1 2 3; do ncu -i $O/c4.ncu-rep --page source --csv --print-source sass --launch-skip $k --launch-count 1 > $O/sass_$k.csv 2>/dev/null; done
python tools/sass_opcode_mix.py $O > $O/opcode_mix.txt 2>&1
rm -f $O/*.ncu-rep
ls -la $O
