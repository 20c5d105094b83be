#!/bin/bash
# C1 single-CTA kernel with the SMEM twiddle preload (TWP): parity at every single-kernel size, then A/B on C1
mkdir -p gpurun_out/ab
cp paper_2012_01968_b200/libntt.so /tmp/libntt_orig.so
cp tools/libs/libntt_twp.so paper_2012_01968_b200/libntt.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_proth.py tests/test_gpu_features.py -x -q > gpurun_out/ab/twp_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab/twp_pytest.log
for v in head twp twp head; do
  cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so
  echo "== $v"; python tools/variants.py --config C1 --variants "4,9" --primes 2n --steps 200
  python bench.py --config C1 --steps 50 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'bench_C1_us': d['value'], 'kernels_ms': d['kernels_ms'], 'l2_warm': d.get('l2_warm')}))"
done > gpurun_out/ab/ab_twp.jsonl 2>&1
cp /tmp/libntt_orig.so paper_2012_01968_b200/libntt.so
