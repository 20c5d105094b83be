// ntt_launch.h -- host-side launchers of the kernels in ntt_kernels.cuh.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "ntt_device.cuh"

namespace ntt {
// proth: every prime of the plan is = 1 mod 2^32 -> the PrimeConstP arithmetic
// (default kernel variants only; see ntt_kernels.cuh).
// One kernel per row: contiguous rows of N = 2^logn, N <= 2^13.
cudaError_t launch_single(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st,
                          bool proth = false);
// Kernel-2 (forward) / Kernel-2' (inverse): contiguous N2-blocks.
// loge: per-thread radix 2^loge (3 or 4).
cudaError_t launch_k2(bool inverse, int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st,
                      bool proth = false);
// Kernel-1 (forward) / Kernel-1' (inverse): stride-N2 columns, 16 per CTA.
cudaError_t launch_k1(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st, bool proth = false);
// the Proth instantiations (ntt_kernels_p.cu)
cudaError_t launch_single_p(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_k2_p(bool inverse, int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_k1_p(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
// Single-pass NTT / iNTT, one thread-block cluster per row (N = 2^14..2^17;
// ntt_fused.cuh).  a.tab2 must be the Kernel-2-ordered table of the split
// N = (N / 2^13) x 2^13.
cudaError_t launch_fused(bool inverse, const KArgs& a, uint32_t rows, cudaStream_t st, bool proth);
// data <- mul_a (.) data 2^-64 (Montgomery), every word.
cudaError_t launch_pointwise(const KArgs& a, cudaStream_t st);
// The paper's comparison kernels, forward only: 1 = radix-2 per stage, 2 = register radix-16.
cudaError_t launch_baseline_forward(int variant, const KArgs& a, cudaStream_t st);
// 32-bit-word path: all passes of one direction.
cudaError_t launch32(bool inverse, const KArgs32& a, uint32_t rows, cudaStream_t st);
}  // namespace ntt
