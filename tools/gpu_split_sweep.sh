#!/bin/bash
# split sweep on the current kernels: log N1 = 7 / 8 / 9 at C4 and C3, both prime families
mkdir -p gpurun_out/split
for c in C4 C3; do for pr in 2n proth; do for ln in 7 8 9 8; do
  echo "== $c $pr log_n1=$ln"; timeout 300 python tools/variants.py --config $c --variants "4,9" --primes $pr --steps 20 --log-n1 $ln
done; done; done > gpurun_out/split/split.jsonl 2>&1
