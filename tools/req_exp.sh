#!/bin/bash
# request-kernel experiment: trace every tools/libs/libntt_t_*.so variant (tools/req_trace.py)
mkdir -p gpurun_out/req
cp paper_2012_01968_b200/libntt.so /tmp/orig.so
for f in tools/libs/libntt_t_*.so; do
  v=$(basename $f .so); v=${v#libntt_t_}
  cp $f paper_2012_01968_b200/libntt.so
  timeout 120 python tools/req_trace.py --L ${REQ_L:-1,2,4,8} --tag $v
done > gpurun_out/req/trace.jsonl 2>&1
cp /tmp/orig.so paper_2012_01968_b200/libntt.so
cat gpurun_out/req/trace.jsonl
