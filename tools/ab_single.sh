#!/bin/bash
# A/B of the single-CTA kernel's per-thread radix (NTT_SINGLE_LOGE 4 / 3 / 2) on C1 (N = 2^12, one row)
mkdir -p gpurun_out/ab
cp paper_2012_01968_b200/libntt.so /tmp/libntt_orig.so
for v in base se3 se2 se2 se3 base; do
  cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so
  echo "== $v"; python tools/variants.py --config C1 --variants "4,9" --primes 2n --steps 200
  python bench.py --config C1 --steps 50 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'bench_C1_us': d['value'], 'kernels_ms': d['kernels_ms'], 'l2_warm': d.get('l2_warm')}))"
done > gpurun_out/ab/ab_single.jsonl 2>&1
cp /tmp/libntt_orig.so paper_2012_01968_b200/libntt.so
cat gpurun_out/ab/ab_single.jsonl
