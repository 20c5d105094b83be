// ntt_fused.cu -- instantiation of the single-pass cluster kernels
// (ntt_fused.cuh) for general and Proth primes.
#include "ntt_kernels.cuh"
#include "ntt_fused.cuh"

namespace ntt {

cudaError_t launch_fused(bool inverse, const KArgs& a, uint32_t rows, cudaStream_t st, int arith)
{
    switch (arith) {
        case kArithProth: return launch_fused_all<PrimeConstP>(inverse, a, rows, st);
        default: return launch_fused_all<PrimeConst>(inverse, a, rows, st);
    }
}

}  // namespace ntt
