#!/bin/bash
# Static SASS opcode counts of the C4 kernels (no GPU), for quick experiments
# on the arithmetic formulation:  [PCT=PrimeConstP] tools/sass_probe.sh [extra nvcc flags]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
PCT=${PCT:-PrimeConst}
cat > $T/p.cu <<EOT
#include "$ROOT/paper_2012_01968_b200/csrc/ntt_kernels.cuh"
namespace ntt {
template __global__ void k_cols<8, 17, 4, false, $PCT>(const KArgs);
template __global__ void k_cols<8, 17, 4, true, $PCT>(const KArgs);
template __global__ void k_blocks<9, 4, false, 0, false, $PCT>(const KArgs);
template __global__ void k_blocks<9, 4, true, 0, false, $PCT>(const KArgs);
template __global__ void k_shared<9, false, 0, false, $PCT>(const KArgs);
template __global__ void k_shared<9, true, 0, false, $PCT>(const KArgs);
}
EOT
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I $ROOT/include "$@" -cubin -o $T/p.cubin $T/p.cu -Xptxas -v 2>&1 | grep -E "registers|spill" | grep -v "0 bytes spill" || true
for k in k_colsILi8ELi17ELi4ELb0 k_colsILi8ELi17ELi4ELb1 k_blocksILi9ELi4ELb0 k_blocksILi9ELi4ELb1 k_sharedILi9ELb0 k_sharedILi9ELb1; do
  f=$(cuobjdump -sass $T/p.cubin | grep -oE "Function : \S*$k\S*" | head -1 | awk '{print $3}')
  echo "== $k"
  cuobjdump -sass -fun "$f" $T/p.cubin | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" | awk '{print $NF}' | sort | uniq -c | sort -rn | awk '{printf "%s:%s ", $2, $1} END {print ""}'
done
rm -rf $T
