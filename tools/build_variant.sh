#!/bin/bash
# Build an experiment variant of libntt.so into tools/libs/libntt_<name>.so:
# translation units (comma-separated) recompiled with extra flags, linked with
# the current objects of the others (paper_2012_01968_b200/build/, run build() first).
#   tools/build_variant.sh <name> <source.cu[,source2.cu]> [nvcc flags...]
set -e
name=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2012_01968_b200/build
rm -rf /tmp/ntt_variant_$name; mkdir -p $R/tools/libs /tmp/ntt_variant_$name
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
for s1 in ${src//,/ }; do
  $NVCC -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 -I $R/include "$@" \
    -x cu -c $R/paper_2012_01968_b200/csrc/$s1 -o /tmp/ntt_variant_$name/$s1.o &
done
wait
objs=""
for o in $B/*.o; do
  b=$(basename $o .o)
  if [ -f /tmp/ntt_variant_$name/$b.o ] && [[ ",$src," == *",$b,"* ]]; then objs="$objs /tmp/ntt_variant_$name/$b.o"; else objs="$objs $o"; fi
done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $R/tools/libs/libntt_$name.so $objs -Xcompiler -pthread
echo $R/tools/libs/libntt_$name.so
