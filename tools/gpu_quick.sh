#!/bin/bash
O=gpurun_out/$1
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or every_size or negacyclic" > $O/pytest_fused.log 2>&1; echo "rc=$?" >> $O/pytest_fused.log
timeout 600 python bench.py --primes proth --steps 20 --no-cpu > $O/bench.json 2> $O/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py --warmup 1 --primes proth > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 2 -c 2 -o $O/prof python tools/profile_step.py --warmup 1 --primes proth > $O/ncu_full.log 2>&1
