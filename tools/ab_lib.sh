#!/bin/bash
# A/B experiment: time C4 with alternative builds of libntt.so staged in tools/libs/ (git-ignored),
# each twice in ABBA order, both prime families.
#   gpurun -- bash tools/ab_lib.sh name1 name2 ...   (tools/libs/libntt_<name>.so)
mkdir -p gpurun_out/ab
cp paper_2012_01968_b200/libntt.so /tmp/libntt_orig.so
order="$* $(echo "$@" | tr ' ' '\n' | tac | tr '\n' ' ')"
for v in $order; do
  cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so
  for pr in ${AB_PRIMES:-2n proth}; do
    echo "== $v $pr"; python tools/variants.py --variants "${AB_VARIANTS:-4,9}" --primes $pr --steps 20
  done
done > gpurun_out/ab/ab.jsonl 2>&1
cp /tmp/libntt_orig.so paper_2012_01968_b200/libntt.so
cat gpurun_out/ab/ab.jsonl
