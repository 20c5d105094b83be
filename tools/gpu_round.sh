#!/bin/bash
# gpurun -- bash tools/gpu_round.sh TAG : GPU tests + bench + K2 variant sweep
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python tools/variants.py --variants "4,5;4,6;4,3;4,4;5,5" > $O/variants.jsonl 2>&1
