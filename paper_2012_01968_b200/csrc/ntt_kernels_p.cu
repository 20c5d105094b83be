// ntt_kernels_p.cu -- the Proth-prime (p = 1 mod 2^32) instantiation of the
// Kernel-2 family in ntt_kernels.cuh.
#include "ntt_kernels.cuh"

namespace ntt {

cudaError_t launch_k2_p(bool inverse, int loge, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    return launch_k2_t<PrimeConstP>(inverse, loge, a, ots, iters, st);
}

}  // namespace ntt
