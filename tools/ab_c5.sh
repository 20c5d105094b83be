#!/bin/bash
# A/B of two library builds (tools/libs/libntt_<name>.so) on the small-job paths:
# C5 request latency (split graph and one kernel) and the C1/C2 bench values.
mkdir -p gpurun_out/abc5
cp paper_2012_01968_b200/libntt.so /tmp/libntt_orig.so
for v in $* $(echo "$@" | tr ' ' '\n' | tac | tr '\n' ' '); do
  cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so
  echo "== $v"
  timeout 200 python tools/c5_latency.py --splits 7 --L 1,8,45
  for c in C1 C2; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '$c', 'value': d['value'], 'kernels_ms': d['kernels_ms']}))"; done
done > gpurun_out/abc5/ab.jsonl 2>&1
cp /tmp/libntt_orig.so paper_2012_01968_b200/libntt.so
cat gpurun_out/abc5/ab.jsonl
