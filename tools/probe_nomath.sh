#!/bin/bash
# Memory / exchange floor of the C4 kernels: the same launches with the
# butterflies and normalisations compiled out (NTT_PROBE_NOMATH), A/B against
# the real library.  Build here: tools/build_variant.sh nomath ntt_k1.cu,ntt_kernels.cu,ntt_kernels_p.cu -DNTT_PROBE_NOMATH
#   gpurun -- bash tools/probe_nomath.sh
AB_VARIANTS="4,9" bash tools/ab_lib.sh base nomath
