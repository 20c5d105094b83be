#!/bin/bash
# A/B experiment: time C4 with alternative builds of libntt.so staged in tools/libs/ (git-ignored)
#   gpurun -- bash tools/ab_lib.sh name1 name2 ...   (tools/libs/libntt_<name>.so)
mkdir -p gpurun_out/ab
for v in "$@"; do
  cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so
  echo "== $v"; python tools/variants.py --variants "${AB_VARIANTS:-4,9}" --primes proth
done > gpurun_out/ab/ab.jsonl 2>&1
