#!/bin/bash
mkdir -p gpurun_out/ab
for v in "$@"; do cp tools/libs/libntt_$v.so paper_2012_01968_b200/libntt.so; echo "== $v"; python tools/bench32.py; done > gpurun_out/ab/b32.jsonl 2>&1
