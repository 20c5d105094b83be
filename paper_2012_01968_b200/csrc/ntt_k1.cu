// ntt_k1.cu -- Kernel-1 / Kernel-1' instantiations (k_cols, k_cols_pipe of
// ntt_kernels.cuh) for general and Proth primes; a translation unit of its own
// so nvcc compiles the kernel families in parallel.
#include "ntt_kernels.cuh"

namespace ntt {

cudaError_t launch_k1_g(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    return launch_k1_t<PrimeConst>(inverse, loge, a, rows, st);
}

cudaError_t launch_k1_p(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    return launch_k1_t<PrimeConstP>(inverse, loge, a, rows, st);
}

}  // namespace ntt
