// ntt_device.cuh -- device arithmetic and the register/SMEM stage engine of the
// B200 NTT kernels.  Product code (never includes anything from oracle/).
//
// Citations: P:n = /root/reference/PAPER.md line n; R# = DESIGN.md section 3.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>
#include <type_traits>

namespace ntt {

// A twiddle with its Shoup companion (Algorithm 4): 16 bytes, one
// 128-bit load.
struct __align__(16) Tw {
    uint64_t w, wb;
};

// Per-prime constants, 64 bytes.
struct __align__(16) PrimeConst {
    uint64_t p, p2;  // p, 2p
    Tw ninv;         // N^-1
    Tw ninv_psi;     // N^-1 * Psi^-1[1], the fused last GS stage (R15)
};

// Kernel arguments (passed by value, lives in the constant bank).
struct KArgs {
    uint64_t* data;        // [batch][L][N]
    const Tw* tab;         // [L][N] Psi (forward) or Psi^-1 (inverse)
    const Tw* ot;          // [L][B + N/B] OT bases (fine | coarse), forward or inverse
    const PrimeConst* pc;  // [L]
    uint32_t L, batch;
    uint32_t logn, log_n1;  // log_n1 = 0 for the single-kernel path
    uint32_t log_tiles;     // column kernel: log2(N2 / 16)
    uint32_t iters;         // contig kernel: block-groups per CTA
    uint32_t ot_logb;       // OT: log2 of the base B
    uint32_t total_blocks;  // contig kernel: rows * N1
};

// ------------------------------------------------------------ arithmetic
// Shoup's modmul without the final subtraction (Algorithm 4 with the lazy
// output of R8): for any b < 2^64 and w < p < 2^62, returns r = b*w mod p
// up to one p, r in [0, 2p).  q = floor(b * w_bar / 2^64) (R7).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t b, uint64_t w, uint64_t wb, uint64_t p)
{
    const uint64_t q = __umul64hi(b, wb);
    return b * w - q * p;
}

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

// The twiddle of one butterfly group: a table entry (one Shoup multiply) or,
// under on-the-fly twiddling, the pair (w1, w2) whose product is
// the twiddle, applied as w2 * (w1 * x): two Shoup multiplies, no new w_bar.
template <bool OT>
struct TwMul;
template <>
struct TwMul<false> {
    Tw t;
    __device__ __forceinline__ uint64_t mul(uint64_t x, uint64_t p) const { return shoup_lazy(x, t.w, t.wb, p); }
};
template <>
struct TwMul<true> {
    Tw fine, coarse;
    __device__ __forceinline__ uint64_t mul(uint64_t x, uint64_t p) const
    {
        return shoup_lazy(shoup_lazy(x, fine.w, fine.wb, p), coarse.w, coarse.wb, p);
    }
};

// Cooley-Tukey butterfly (Algorithm 2) in Harvey's lazy form (R9):
// inputs and outputs in [0, 4p).
template <class W>
__device__ __forceinline__ void ct_bf(uint64_t& X, uint64_t& Y, const W& w, uint64_t p, uint64_t p2)
{
    const uint64_t x = csub(X, p2);
    const uint64_t t = w.mul(Y, p);
    X = x + t;
    Y = x - t + p2;
}

// Gentleman-Sande butterfly of the inverse (R5): inputs and outputs in [0, 2p).
template <class W>
__device__ __forceinline__ void gs_bf(uint64_t& X, uint64_t& Y, const W& w, uint64_t p, uint64_t p2)
{
    const uint64_t x = X, y = Y;
    X = csub(x + y, p2);
    Y = w.mul(x - y + p2, p);
}

__device__ __forceinline__ Tw ldg_tw(const Tw* ptr)
{
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(ptr));
    return Tw{v.x, v.y};
}

// Compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1.
template <class Fn, int... Is>
__device__ __forceinline__ void static_for_impl(Fn&& f, std::integer_sequence<int, Is...>)
{
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class Fn>
__device__ __forceinline__ void static_for(Fn&& f)
{
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// ------------------------------------------------------------ schedule
// A sub-transform of size M = 2^LOGM is executed in rounds of up to 4 radix-2
// stages (a per-thread radix-16 NTT); between rounds the
// data is exchanged through SMEM (the "SMEM implementation").
// Each thread holds E = 16 words (E = M below 16).
template <int LOGM>
struct Sched {
    static constexpr int M = 1 << LOGM;
    static constexpr int E = LOGM < 4 ? M : 16;
    static constexpr int NR = (LOGM + 3) / 4;
    static constexpr int TB = M / E;  // threads per sub-transform
    static constexpr int r(int i) { return (LOGM - 4 * i) < 4 ? (LOGM - 4 * i) : 4; }
};

// Geometry of round RI (stages [S, S+r) of the sub-transform, S = 4 RI): the
// thread's groups are G = qd*TB + tib; group G = (g, o) with
//   g = G / s, o = G % s, s = M >> (S + r)  (the smallest stride),
// and holds elements e_k = g*R*s + o + k*s, k < R = 2^r.
// Twiddles of stage S+i of group g are Psi[((F << S) + g) << i) + h], h < 2^i,
// F = 1 for a whole column / row, F = N1 + bb for block bb of Kernel-2.
template <int LOGM, int RI>
struct RoundGeo {
    static constexpr int S = 4 * RI;
    static constexpr int r = Sched<LOGM>::r(RI);
    static constexpr int R = 1 << r;
    static constexpr int s = (1 << LOGM) >> (S + r);
    static constexpr int GPT = Sched<LOGM>::E / R;
    __device__ static __forceinline__ uint32_t elem(uint32_t G, int k)
    {
        const uint32_t g = G / s, o = G % s;
        return g * (R * s) + o + (uint32_t)k * s;
    }
};

// Forward round: r Cooley-Tukey stages on each of the thread's GPT groups.
// TWF(idx) returns the TwMul for Psi index idx.  OT_FROM = first local stage
// whose twiddles come from OT (>= LOGM: none).
template <int LOGM, int RI, int OT_FROM, class TabF, class OtF>
__device__ __forceinline__ void ct_round(uint64_t (&x)[16], uint32_t tib, uint32_t F, const TabF& tabf,
                                         const OtF& otf, uint64_t p, uint64_t p2)
{
    using Geo = RoundGeo<LOGM, RI>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Sched<LOGM>::TB + tib;
        const uint32_t B = (F << S) + G / Geo::s;
#pragma unroll
        for (int i = 0; i < Geo::r; ++i) {
            const int half = R >> (i + 1);
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const uint32_t idx = (B << i) + h;
                if (S + i >= OT_FROM) {
                    const TwMul<true> w = otf(idx);
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
                        ct_bf(x[qd * R + k], x[qd * R + k + half], w, p, p2);
                } else {
                    const TwMul<false> w{tabf(idx)};
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
                        ct_bf(x[qd * R + k], x[qd * R + k + half], w, p, p2);
                }
            }
        }
    }
}

// Inverse round: the same groups and twiddle indices, Gentleman-Sande stages
// in reverse order.  FUSE0: local stage 0 is global stage 0 (m = 1), where
// N^-1 is fused: X' = (X+Y) N^-1, Y' = (X-Y) Psi^-1[1] N^-1 (R15).
template <int LOGM, int RI, int OT_FROM, bool FUSE0, class TabF, class OtF>
__device__ __forceinline__ void gs_round(uint64_t (&x)[16], uint32_t tib, uint32_t F, const TabF& tabf,
                                         const OtF& otf, uint64_t p, uint64_t p2, const PrimeConst& pc)
{
    using Geo = RoundGeo<LOGM, RI>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Sched<LOGM>::TB + tib;
        const uint32_t B = (F << S) + G / Geo::s;
#pragma unroll
        for (int i = Geo::r - 1; i >= 0; --i) {
            const int half = R >> (i + 1);
            if (FUSE0 && S + i == 0) {
                const TwMul<false> a{pc.ninv}, b{pc.ninv_psi};
#pragma unroll
                for (int k = 0; k < half; ++k) {
                    const uint64_t u = x[qd * R + k], v = x[qd * R + k + half];
                    x[qd * R + k] = a.mul(u + v, p);
                    x[qd * R + k + half] = b.mul(u - v + p2, p);
                }
                continue;
            }
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const uint32_t idx = (B << i) + h;
                if (S + i >= OT_FROM) {
                    const TwMul<true> w = otf(idx);
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
                        gs_bf(x[qd * R + k], x[qd * R + k + half], w, p, p2);
                } else {
                    const TwMul<false> w{tabf(idx)};
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
                        gs_bf(x[qd * R + k], x[qd * R + k + half], w, p, p2);
                }
            }
        }
    }
}

// SMEM swizzle for contiguous blocks: XOR bits 1..3 with bits 4..6 so the
// round access patterns are at most 2-way bank-conflicted while 16-byte pairs
// (2i, 2i+1) stay adjacent for vector copies.
__device__ __forceinline__ uint32_t swz(uint32_t e) { return e ^ (((e >> 4) & 7u) << 1); }

}  // namespace ntt
