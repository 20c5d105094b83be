// ntt_kernels.cu -- the general-prime Kernel-2 family of ntt_kernels.cuh, the
// public launchers (which route to the per-family translation units: Kernel-1
// in ntt_k1.cu, the single-CTA kernel in ntt_single.cu, Proth Kernel-2 in
// ntt_kernels_p.cu) and the element-wise product kernel.
#include "ntt_kernels.cuh"

namespace ntt {

// ---------------------------------------------------------------- element-wise product
// b <- a (.) b 2^-64 for every word (unfused path of ntt_pointwise_inverse;
// rows [batch][L][N], row (b, l) mod primes[l]).
__global__ void __launch_bounds__(256) k_pointwise(const KArgs a, uint64_t words)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i >= words) return;
    const uint32_t l = (uint32_t)((2 * i >> a.logn) % a.L);
    const PrimeConst pc = a.pc[l];
    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(a.mul_a + 2 * i);
    ulonglong2 v = *reinterpret_cast<const ulonglong2*>(a.data + 2 * i);
    v.x = mont_mul(u.x, v.x, pc);
    v.y = mont_mul(u.y, v.y, pc);
    *reinterpret_cast<ulonglong2*>(a.data + 2 * i) = v;
}

cudaError_t launch_pointwise(const KArgs& a, cudaStream_t st)
{
    const uint64_t words = ((uint64_t)a.batch * a.L) << a.logn;
    const uint64_t threads = (words + 1) / 2;
    k_pointwise<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a, words);
    return launch_status();
}

cudaError_t launch_single(bool inverse, const KArgs& a, int ots, uint32_t iters, cudaStream_t st, int arith)
{
    switch (arith) {
        case kArithProth: return launch_single_p(inverse, a, ots, iters, st);
        default: return launch_single_g(inverse, a, ots, iters, st);
    }
}

cudaError_t launch_k2(bool inverse, int loge, const KArgs& a, int ots, uint32_t iters, cudaStream_t st, int arith)
{
    switch (arith) {
        case kArithProth: return launch_k2_p(inverse, loge, a, ots, iters, st);
        case kArithGeneralD:
            if (!inverse) return launch_k2_fwd_d(loge, a, ots, iters, st);
            return launch_k2_t<PrimeConst>(inverse, loge, a, ots, iters, st);
        default: return launch_k2_t<PrimeConst>(inverse, loge, a, ots, iters, st);
    }
}

cudaError_t launch_k1(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st, int arith)
{
    switch (arith) {
        case kArithProth: return launch_k1_p(inverse, loge, a, rows, st);
        case kArithProthD:
            if (inverse) return launch_k1_inv_pd(loge, a, rows, st);
            return launch_k1_p(inverse, loge, a, rows, st);
        case kArithGeneralD:
            if (inverse) return launch_k1_inv_d(loge, a, rows, st);
            return launch_k1_g(inverse, loge, a, rows, st);
        default: return launch_k1_g(inverse, loge, a, rows, st);
    }
}

}  // namespace ntt
