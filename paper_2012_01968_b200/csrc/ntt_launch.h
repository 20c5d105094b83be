// ntt_launch.h -- host-side launchers of the kernels in ntt_kernels.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "ntt_device.cuh"

namespace ntt {
// One kernel per row: contiguous rows of N = 2^logn, N <= 2^13.
cudaError_t launch_single(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
// Kernel-2 (forward) / Kernel-2' (inverse): contiguous N2-blocks.
// loge: per-thread radix 2^loge (3 or 4).
cudaError_t launch_k2(bool inverse, int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
// Kernel-1 (forward) / Kernel-1' (inverse): stride-N2 columns, 16 per CTA.
cudaError_t launch_k1(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
// data <- mul_a (.) data 2^-64 (Montgomery), every word.
cudaError_t launch_pointwise(const KArgs& a, cudaStream_t st);
// The paper's comparison kernels, forward only: 1 = radix-2 per stage, 2 = register radix-16.
cudaError_t launch_baseline_forward(int variant, const KArgs& a, cudaStream_t st);
// 32-bit-word path: all passes of one direction.
cudaError_t launch32(bool inverse, const KArgs32& a, uint32_t rows, cudaStream_t st);
}  // namespace ntt
