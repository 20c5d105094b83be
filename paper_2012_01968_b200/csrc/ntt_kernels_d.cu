// ntt_kernels_d.cu -- the forward shared-twiddle Kernel-2 and Kernel-1'
// instantiated on PrimeConstD: general arithmetic with the d-form final
// reduction for primes p = 2^60 - d, d < 2^32 (the R3 chain; ntt_device.cuh
// reduce_full) and the exact-division N^-1 (div_n), DESIGN.md 5.1.  Other
// kernel forms (small batches, knobs) keep the general type.
#include "ntt_kernels.cuh"

namespace ntt {

cudaError_t launch_k2_fwd_d(int loge, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    using namespace detail;
    const int logm = (int)(a.logn - a.log_n1);
    if ((loge == 7 || (loge == 9 && logm >= 8)) && a.batch >= (4096u >> logm))
        return shared_switch<false, PrimeConstD>(logm, a, ots, loge == 9, st, K2Sizes{});
    return launch_k2_t<PrimeConst>(false, loge, a, ots, iters, st);
}

// Kernel-1' with the exact-division N^-1 (div_n)
cudaError_t launch_k1_inv_d(int loge, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    using namespace detail;
    if (loge == 5 && a.log_n1 <= 9)  // the pipelined knob variant keeps the general type
        return launch_k1_t<PrimeConst>(true, loge, a, rows, st);
    return cols_switch<4, true, PrimeConstD>((int)((a.logn << 4) | a.log_n1), a, rows, st, K1Pairs{});
}

// Proth plans: Kernel-1' with the exact-division N^-1 on the Proth arithmetic
cudaError_t launch_k1_inv_pd(int loge, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    using namespace detail;
    if (loge == 5 && a.log_n1 <= 9)
        return launch_k1_t<PrimeConstP>(true, loge, a, rows, st);
    return cols_switch<4, true, PrimeConstPD>((int)((a.logn << 4) | a.log_n1), a, rows, st, K1Pairs{});
}

}  // namespace ntt
