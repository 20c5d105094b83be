#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/k1d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k1d_pytest.log
AB_PRIMES=2n bash tools/ab_lib.sh head k1d
