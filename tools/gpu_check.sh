#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, launch list, full ncu of the C4 kernels.
#   gpurun --timeout 1800 -- bash tools/gpu_check.sh TAG
TAG=${1:-run}
PRIMES=${2:-2n}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --primes $PRIMES > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py --warmup 1 --primes $PRIMES > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols|k_blocks|k_shared|k_fused" -s 4 -c 4 -o $O/prof python tools/profile_step.py --warmup 1 --primes $PRIMES > $O/ncu_full.log 2>&1
echo done
