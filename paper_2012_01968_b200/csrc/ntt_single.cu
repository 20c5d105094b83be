// ntt_single.cu -- the single-CTA kernel (k_contig, N <= 2^13) for general
// and Proth primes; a translation unit of its own for parallel compilation.
#include "ntt_kernels.cuh"

namespace ntt {

cudaError_t launch_single_g(bool inverse, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    return launch_single_t<PrimeConst>(inverse, a, ots, iters, st);
}

cudaError_t launch_single_p(bool inverse, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    return launch_single_t<PrimeConstP>(inverse, a, ots, iters, st);
}

}  // namespace ntt
