// ntt_baselines.cu -- the paper's comparison kernels rebuilt on sm_100a
// (SURVEY 8(f) NEXT-3), forward direction only as in the paper's Table 2:
//
//   radix-2  : Algorithm 1 one stage per launch: every
//              thread performs one butterfly, reading and writing global
//              memory; log2 N launches.
//   radix-16 : the register-based high-radix implementation (P:484-488,
//              P:558-604): a thread loads 16 elements at stride s from
//              global, runs 4 Cooley-Tukey stages in registers and writes
//              them back; ceil(log2 N / 4) launches, no shared memory.
//
// Same arithmetic (truncated-quotient Shoup, [0, 8p) lazy bounds) and the same
// bit-reversed Psi table as the main path, so the ratio against the two-kernel
// SMEM path isolates the memory structure the paper studies (4.2x).
#include "ntt_device.cuh"
#include "ntt_launch.h"

namespace ntt {

// One radix-2 stage with half-distance t = N >> (stage+1): butterfly u of row
// r pairs k = j 2t + (u mod t) with k + t, j = u / t, twiddle Psi[m + j].
template <bool LAST>
__global__ void __launch_bounds__(256) k_radix2_stage(const KArgs a, uint32_t stage)
{
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t half_n = 1u << (a.logn - 1);
    const uint64_t rows = (uint64_t)a.batch * a.L;
    if (gid >= rows * half_n) return;
    const uint32_t u = (uint32_t)(gid & (half_n - 1)), r = (uint32_t)(gid >> (a.logn - 1));
    const uint32_t l = r % a.L;
    const uint32_t logt = a.logn - 1 - stage, t = 1u << logt;
    const uint32_t j = u >> logt, k = (j << (logt + 1)) + (u & (t - 1));
    uint64_t* row = a.data + ((uint64_t)r << a.logn);
    const PrimeConst pc = a.pc[l];
    const TwMul<false> w{ldg_tw(a.tab + ((uint64_t)l << a.logn) + (1u << stage) + j)};
    uint64_t x = row[k], y = row[k + t];
    ct_bf(x, y, w, pc);
    if (LAST) {
        x = reduce_full(x, pc);
        y = reduce_full(y, pc);
    }
    row[k] = x;
    row[k + t] = y;
}

// Register radix-16 pass over stages [S, S+r): thread = group (g, o) of one
// row, elements e_k = g 16 s + o + k s read and written straight from global.
template <int R>
__global__ void __launch_bounds__(256) k_radix_reg(const KArgs a, uint32_t S, bool last)
{
    constexpr int r = R == 16 ? 4 : (R == 8 ? 3 : (R == 4 ? 2 : 1));
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t per_row = 1u << (a.logn - r);
    const uint64_t rows = (uint64_t)a.batch * a.L;
    if (gid >= rows * per_row) return;
    const uint32_t G = (uint32_t)(gid & (per_row - 1)), row_i = (uint32_t)(gid >> (a.logn - r));
    const uint32_t l = row_i % a.L;
    const uint32_t logs = a.logn - S - r, s = 1u << logs;
    const uint32_t g = G >> logs, o = G & (s - 1);
    uint64_t* row = a.data + ((uint64_t)row_i << a.logn) + ((uint64_t)g << (logs + r)) + o;
    const Tw* tab = a.tab + ((uint64_t)l << a.logn);
    const PrimeConst pc = a.pc[l];
    uint64_t x[R];
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = row[(uint64_t)k << logs];
    const uint32_t B = (1u << S) + g;
#pragma unroll
    for (int i = 0; i < r; ++i) {
        const int half = R >> (i + 1);
#pragma unroll
        for (int h = 0; h < (1 << i); ++h) {
            const TwMul<false> w{ldg_tw(tab + (B << i) + h)};
#pragma unroll
            for (int k = h * 2 * half; k < h * 2 * half + half; ++k) ct_bf(x[k], x[k + half], w, pc);
        }
    }
    if (last) {
#pragma unroll
        for (int k = 0; k < R; ++k) x[k] = reduce_full(x[k], pc);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) row[(uint64_t)k << logs] = x[k];
}

cudaError_t launch_baseline_forward(int variant, const KArgs& a, cudaStream_t st)
{
    const uint64_t rows = (uint64_t)a.batch * a.L;
    if (variant == 1) {  // radix-2, one launch per stage
        const uint64_t n = rows << (a.logn - 1);
        const unsigned grid = (unsigned)((n + 255) / 256);
        for (uint32_t s = 0; s < a.logn; ++s) {
            if (s + 1 == a.logn)
                k_radix2_stage<true><<<grid, 256, 0, st>>>(a, s);
            else
                k_radix2_stage<false><<<grid, 256, 0, st>>>(a, s);
            cudaError_t e = launch_status();
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    if (variant == 2) {  // register radix-16 passes (radix 2/4/8 for the remainder)
        for (uint32_t S = 0; S < a.logn;) {
            const uint32_t r = a.logn - S >= 4 ? 4 : a.logn - S;
            const uint64_t n = rows << (a.logn - r);
            const unsigned grid = (unsigned)((n + 255) / 256);
            const bool last = S + r == a.logn;
            switch (r) {
                case 4: k_radix_reg<16><<<grid, 256, 0, st>>>(a, S, last); break;
                case 3: k_radix_reg<8><<<grid, 256, 0, st>>>(a, S, last); break;
                case 2: k_radix_reg<4><<<grid, 256, 0, st>>>(a, S, last); break;
                default: k_radix_reg<2><<<grid, 256, 0, st>>>(a, S, last); break;
            }
            cudaError_t e = launch_status();
            if (e != cudaSuccess) return e;
            S += r;
        }
        return cudaSuccess;
    }
    return cudaErrorInvalidValue;
}

}  // namespace ntt
