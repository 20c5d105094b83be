// ntt32.cu -- the 32-bit-word path (the paper's "32b vs
// 64b" comparison): primes p = 1 mod 2N with 2^29 <= p < 2^30,
// one 32-bit word per coefficient, 32-bit Shoup (w_bar = floor(w 2^32 / p)):
//   q = hi32(b w_bar),  r = b w - q p (mod 2^32)  in [0, 2p)
// -- one IMAD.HI and two IMADs per multiply instead of 3 IMAD.WIDE, 2 IMAD.HI
// and 4 IMADs.  The paper measured 32b vs 64b within ~5% on Titan V;
// on the multiply-bound B200 the smaller words win.
//
// Same decomposition as the 64-bit path: Kernel-1 (columns; 32-column tiles =
// 128-byte segments of 4-byte words) and Kernel-2 (contiguous blocks; the
// Kernel-2 twiddle layout), or one kernel per row for N <= 2^13.  Harvey lazy
// bounds: CT values in [0, 4p), GS in [0, 2p) (< 2^32 since p < 2^30).
#include "ntt_device.cuh"
#include "ntt_launch.h"

#include <atomic>

namespace ntt {
namespace w32 {

__device__ __forceinline__ uint32_t shoup(uint32_t b, uint32_t w, uint32_t wb, uint32_t p)
{
    const uint32_t q = __umulhi(b, wb);
    return b * w - q * p;
}
__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t m) { return x >= m ? x - m : x; }

// Barrier over the TB threads of one block (__syncwarp when a warp holds whole
// blocks, else a named barrier of the block's own)
template <int TB>
__device__ __forceinline__ void bsync(uint32_t blk)
{
    if constexpr (TB <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(blk + 1), "n"(TB) : "memory");
    }
}

struct Mul {
    Tw32 t;
    __device__ __forceinline__ uint32_t mul(uint32_t x, const PrimeConst32& c) const { return shoup(x, t.w, t.wb, c.p); }
};

// Harvey CT butterfly: [0,4p) in and out
__device__ __forceinline__ void ct_bf(uint32_t& X, uint32_t& Y, const Mul& w, const PrimeConst32& c)
{
    const uint32_t x = csub(X, c.p2);
    const uint32_t t = w.mul(Y, c);
    X = x + t;
    Y = x - t + c.p2;
}
// GS butterfly: [0,2p) in and out
__device__ __forceinline__ void gs_bf(uint32_t& X, uint32_t& Y, const Mul& w, const PrimeConst32& c)
{
    const uint32_t x = X, y = Y;
    X = csub(x + y, c.p2);
    Y = w.mul(x - y + c.p2, c);
}

__device__ __forceinline__ Tw32 ldg_tw(const Tw32* p)
{
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    return Tw32{v.x, v.y};
}

// SMEM swizzle for 4-byte words: XOR the 16-byte-chunk bits 2..4 with
// (bits 5..7 ^ bits 6..8); conflict-free for every round pattern of M >= 2^9
// (scalar and 128-bit accesses; half-warp bank model over this XOR family).
__device__ __forceinline__ uint32_t swz32(uint32_t e) { return e ^ ((((e >> 5) ^ (e >> 6)) & 7u) << 2); }
// swz32 of (base | KS) from sB = swz32(base), KS a compile-time offset with bits
// disjoint from base's (the 64-bit swz_at argument, ntt_device.cuh)
template <uint32_t KS>
__device__ __forceinline__ uint32_t swz32_at(uint32_t sB)
{
    constexpr uint32_t f = (((KS >> 5) ^ (KS >> 6)) & 7u) << 2;
    if constexpr ((KS & 0x1Cu) == 0) {
        if constexpr (f == 0) {
            return sB + KS;
        } else {
            return (sB ^ f) + KS;
        }
    } else {
        return sB ^ (KS ^ f);
    }
}

// Rounds (same geometry and twiddle algebra as the 64-bit engine).
template <int LOGM, int LOGE, int RI, class TabF>
__device__ __forceinline__ void ct_round(uint32_t (&x)[16], uint32_t tib, const TabF& tabf, const PrimeConst32& c)
{
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Geo::TB + tib, g = G / Geo::s;
        const uint32_t B = (1u << S) + g;
#pragma unroll
        for (int i = 0; i < Geo::r; ++i) {
            const int half = R >> (i + 1);
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const Mul w{tabf(TwKey{(B << i) + h, S + i, S, i, h, g})};
#pragma unroll
                for (int k = h * 2 * half; k < h * 2 * half + half; ++k) ct_bf(x[qd * R + k], x[qd * R + k + half], w, c);
            }
        }
    }
}

template <int LOGM, int LOGE, int RI, bool FUSE0, class TabF>
__device__ __forceinline__ void gs_round(uint32_t (&x)[16], uint32_t tib, const TabF& tabf, const PrimeConst32& c)
{
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Geo::TB + tib, g = G / Geo::s;
        const uint32_t B = (1u << S) + g;
#pragma unroll
        for (int i = Geo::r - 1; i >= 0; --i) {
            const int half = R >> (i + 1);
            if (FUSE0 && S + i == 0) {  // last GS stage with N^-1 fused (R15)
                const Mul a{c.ninv}, b{c.ninv_psi};
#pragma unroll
                for (int k = 0; k < half; ++k) {
                    const uint32_t u = x[qd * R + k], v = x[qd * R + k + half];
                    x[qd * R + k] = a.mul(u + v, c);
                    x[qd * R + k + half] = b.mul(u - v + c.p2, c);
                }
                continue;
            }
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const Mul w{tabf(TwKey{(B << i) + h, S + i, S, i, h, g})};
#pragma unroll
                for (int k = h * 2 * half; k < h * 2 * half + half; ++k) gs_bf(x[qd * R + k], x[qd * R + k + half], w, c);
            }
        }
    }
}

// ------------------------------------------------------------ Kernel-1 (columns)
template <int LOGN1, int LOGN, bool INV>
__global__ void __launch_bounds__((1 << LOGN1) * 2, LOGN1 >= 9 ? 1 : 2) k32_cols(const KArgs32 a)
{
    using SC = Sched<LOGN1, 4>;
    constexpr int M = SC::M, NR = SC::NR, CT = SC::TB * 32;
    constexpr uint32_t logn2 = LOGN - LOGN1;
    extern __shared__ __align__(16) uint32_t sm32[];  // [M][32] words, then Tw32[M]
    Tw32* tws = reinterpret_cast<Tw32*>(sm32 + M * 32);

    const uint32_t tid = threadIdx.x, c = tid & 31u, tib = tid >> 5;
    const uint32_t tile = blockIdx.x & ((1u << a.log_tiles) - 1u);
    const uint32_t q = blockIdx.x >> a.log_tiles;  // prime-major
    const uint32_t l = q / a.batch, b = q - l * a.batch;
    uint32_t* col = a.data + (((uint64_t)b * a.L + l) << LOGN) + tile * 32u + c;
    const Tw32* tab = a.tab + ((uint64_t)l << LOGN);
    const PrimeConst32 pc = a.pc[l];
    // Psi[0..N1) into SMEM, issued after round 0's global loads (the two DRAM round trips overlap)
    auto preload_twiddles = [&]() {
        for (uint32_t i = tid; i < (uint32_t)M; i += CT) tws[i] = ldg_tw(tab + i);
        __syncthreads();
    };
    auto tabf = [&](const TwKey& k) { return tws[k.idx]; };

    uint32_t x[16];
    auto g_io = [&](auto ri, bool store) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, 4>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            uint32_t* p = col + ((uint64_t)Geo::elem(qd * SC::TB + tib, 0) << logn2);
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) {
                if (store)
                    p[(size_t)(k * Geo::s) << logn2] = x[qd * Geo::R + k];
                else
                    x[qd * Geo::R + k] = p[(size_t)(k * Geo::s) << logn2];
            }
        }
    };
    auto s_io = [&](auto ri, bool store) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, 4>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            uint32_t* p = sm32 + Geo::elem(qd * SC::TB + tib, 0) * 32 + c;
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) {
                if (store)
                    p[k * Geo::s * 32] = x[qd * Geo::R + k];
                else
                    x[qd * Geo::R + k] = p[k * Geo::s * 32];
            }
        }
    };
    if constexpr (!INV) {
        static_for<NR>([&](auto ri) {
            constexpr int RI = decltype(ri)::value;
            if constexpr (RI == 0) {
                g_io(ri, false);
                preload_twiddles();
            } else {
                s_io(ri, false);
            }
            ct_round<LOGN1, 4, RI>(x, tib, tabf, pc);
            if constexpr (RI == NR - 1) {
                g_io(ri, true);
            } else {
                s_io(ri, true);
                __syncthreads();
            }
        });
    } else {
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            if constexpr (RI == NR - 1) {
                g_io(RC{}, false);
                preload_twiddles();
            } else {
                s_io(RC{}, false);
            }
            gs_round<LOGN1, 4, RI, true>(x, tib, tabf, pc);
            if constexpr (RI == 0) {
#pragma unroll
                for (int k = 0; k < 16; ++k) x[k] = csub(x[k], pc.p);
                g_io(RC{}, true);
            } else {
                s_io(RC{}, true);
                __syncthreads();
            }
        });
    }
}

// ------------------------------------------------------------ contiguous (Kernel-2 / single)
// K2: blocks of N2 words with twiddles from the Kernel-2 table; else (N1 = 1)
// whole rows with the standard table.  Global <-> SMEM with 16-byte vectors.
template <int LOGM>
struct Contig32Cfg {
    static constexpr int TB = Sched<LOGM, 4>::TB;
    static constexpr int CT = TB > 256 ? TB : 256;
    static constexpr int NB = CT / TB;
};

// SHARED (Kernel-2 only, batch >= NB): one CTA per (prime, block position,
// NB ciphertexts) -- the blocks of a CTA share their twiddles, staged in SMEM
// once (the 64-bit k_shared design).
#ifndef NTT32_K2_MINB
#define NTT32_K2_MINB 4  // 64 registers, 4 CTAs / 32 warps per SM (measured 2 % faster than 2)
#endif
template <int LOGM, bool INV, bool FUSE0, bool K2, bool SHARED = false, int LE2 = 4>
__global__ void __launch_bounds__(Contig32Cfg<LOGM>::CT,
                                  Contig32Cfg<LOGM>::CT > 256 ? 1 : (K2 ? NTT32_K2_MINB : 2)) k32_contig(const KArgs32 a)
{
    using SC = Sched<LOGM, LE2>;
    constexpr int M = SC::M, E = SC::E, TB = SC::TB, NR = SC::NR, NB = Contig32Cfg<LOGM>::NB;
    extern __shared__ __align__(16) uint32_t sm32[];
    const uint32_t tid = threadIdx.x, blk = tid / TB, tib = tid % TB;
    uint32_t* sb = sm32 + blk * M;
    const uint32_t n1mask = (1u << a.log_n1) - 1u;
    uint32_t bb, l, b;
    bool active;
    if constexpr (SHARED) {
        const uint32_t groups = (a.batch + NB - 1) / NB;
        const uint32_t cg = blockIdx.x % groups, rest = blockIdx.x / groups;
        bb = rest & n1mask;
        l = rest >> a.log_n1;
        b = cg * NB + blk;
        active = b < a.batch;
        if (!active) b = 0;
    } else {
        uint32_t gb = blockIdx.x * NB + blk;
        active = gb < a.total_blocks;
        if (!active) gb = a.total_blocks - 1;
        bb = gb & n1mask;
        const uint32_t q = gb >> a.log_n1;
        l = q / a.batch;
        b = q - l * a.batch;
    }
    uint32_t* g = a.data + (((uint64_t)b * a.L + l) << a.logn) + (uint64_t)bb * M;
    const PrimeConst32 pc = a.pc[l];
    const Tw32* tab = a.tab + ((uint64_t)l << a.logn);
    const Tw32* tb2 = K2 ? a.tab2 + ((uint64_t)l << a.logn) + ((uint64_t)bb << LOGM) : nullptr;
    Tw32* const tws = reinterpret_cast<Tw32*>(sm32 + NB * M);  // SHARED: the block position's segment
    if constexpr (SHARED) {
        for (uint32_t i = tid; i < (uint32_t)M; i += Contig32Cfg<LOGM>::CT) tws[i] = ldg_tw(tb2 + i);
    }
    auto tabf = [&](const TwKey& k) {
        if constexpr (SHARED)
            return tws[K2Layout<LOGM, LE2>::round_off(k.S) + ((((1u << k.i) - 1u + k.h) << k.S) + k.g)];
        else if constexpr (K2)
            return ldg_tw(tb2 + K2Layout<LOGM, LE2>::round_off(k.S) + ((((1u << k.i) - 1u + k.h) << k.S) + k.g));
        else
            return ldg_tw(tab + k.idx);
    };

    // SHARED on the remainder-last schedule: the forward reads round 0 (stride
    // >= 8 words) and the inverse writes it straight from/to global; with a
    // single-stage remainder the last forward round (adjacent pairs) is also
    // stored, and the first inverse round loaded, straight to/from global
    constexpr bool DIRECT = SHARED && SC::REMLAST;
    constexpr bool DIRECT_LAST = DIRECT && SC::REM == 1;
    // global -> SMEM (E/4 16-byte chunks per thread), unless the first round
    // reads global itself (forward: round 0; inverse: the pair round)
    constexpr bool STAGED_IN = INV ? !DIRECT_LAST : !DIRECT;
    if constexpr (STAGED_IN)
#pragma unroll
    for (int j = 0; j < (E >= 4 ? E / 4 : 1); ++j) {
        const uint32_t ch = j * TB + tib;
        if (E >= 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(g + 4 * ch);
            *reinterpret_cast<uint4*>(sb + swz32(4 * ch)) = v;
        } else {
            for (int t = 0; t < E; ++t) sb[tib * E + t] = g[tib * E + t];
        }
    }
    __syncthreads();

    uint32_t x[16];
    // element (qd, k) at swz32_at<elem(qd TB, k)>(swz32(elem(tib, 0))): one base per round
    auto s_io = [&](auto ri, bool store) {
        using Geo = RoundGeo<LOGM, decltype(ri)::value, LE2>;
        const uint32_t sB = swz32(Geo::elem(tib, 0));
        static_for<Geo::GPT>([&](auto qdc) {
            constexpr int qd = decltype(qdc)::value;
            static_for<Geo::R>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                const uint32_t a = swz32_at<Geo::elem(qd * TB, k)>(sB);
                if (store)
                    sb[a] = x[qd * Geo::R + k];
                else
                    x[qd * Geo::R + k] = sb[a];
            });
        });
    };
    auto g_io0 = [&](bool store) {  // round 0 straight from / to global
        using Geo = RoundGeo<LOGM, 0, LE2>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) {
                const uint32_t e = Geo::elem(qd * TB + tib, k);
                if (store)
                    g[e] = x[qd * Geo::R + k];
                else
                    x[qd * Geo::R + k] = g[e];
            }
    };
    auto g_pairs = [&](bool store) {  // the remainder-last radix-2 round's pairs (2G, 2G+1)
        using Geo = RoundGeo<LOGM, NR - 1, LE2>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            uint2* p = reinterpret_cast<uint2*>(g + Geo::elem(qd * TB + tib, 0));
            if (store) {
                *p = make_uint2(x[2 * qd], x[2 * qd + 1]);
            } else {
                const uint2 v = *p;
                x[2 * qd] = v.x;
                x[2 * qd + 1] = v.y;
            }
        }
    };
    if constexpr (!INV) {
        static_for<NR>([&](auto ri) {
            constexpr int RI = decltype(ri)::value;
            if constexpr (DIRECT && RI == 0) {
                g_io0(false);
                __syncthreads();  // the twiddle segment is in SMEM
            } else {
                s_io(ri, false);
            }
            ct_round<LOGM, LE2, RI>(x, tib, tabf, pc);
            if constexpr (RI == NR - 1) {
#pragma unroll
                for (int k = 0; k < E; ++k) x[k] = csub(csub(x[k], pc.p2), pc.p);
            }
            if constexpr (DIRECT_LAST && RI == NR - 1) {
                if (active) g_pairs(true);
            } else {
                s_io(ri, true);
                bsync<TB>(blk);  // blocks never share SMEM: block-local barrier
            }
        });
    } else {
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            if constexpr (DIRECT_LAST && RI == NR - 1) {
                g_pairs(false);
                __syncthreads();  // the twiddle segment is in SMEM
            } else {
                s_io(RC{}, false);
            }
            gs_round<LOGM, LE2, RI, FUSE0>(x, tib, tabf, pc);
            if constexpr (FUSE0 && RI == 0) {
#pragma unroll
                for (int k = 0; k < E; ++k) x[k] = csub(x[k], pc.p);
            }
            if constexpr (DIRECT && RI == 0) {
                if (active) g_io0(true);
            } else {
                s_io(RC{}, true);
                bsync<TB>(blk);  // blocks never share SMEM: block-local barrier
            }
        });
    }
    constexpr bool STAGED_OUT = INV ? !DIRECT : !DIRECT_LAST;
    if constexpr (STAGED_OUT)
    if (active) {
#pragma unroll
        for (int j = 0; j < (E >= 4 ? E / 4 : 1); ++j) {
            const uint32_t ch = j * TB + tib;
            if (E >= 4) {
                *reinterpret_cast<uint4*>(g + 4 * ch) = *reinterpret_cast<const uint4*>(sb + swz32(4 * ch));
            } else {
                for (int t = 0; t < E; ++t) g[tib * E + t] = sb[tib * E + t];
            }
        }
    }
}

}  // namespace w32

// ------------------------------------------------------------ dispatch
namespace {
template <int LOGN1, int LOGN, bool INV>
cudaError_t launch32_cols_t(const KArgs32& a, uint32_t rows, cudaStream_t st)
{
    constexpr int M = 1 << LOGN1, CT = (M / 16) * 32;
    const size_t smem = (size_t)M * 32 * 4 + (size_t)M * sizeof(Tw32);
    auto fn = w32::k32_cols<LOGN1, LOGN, INV>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }))
        return e;
    fn<<<(unsigned)((uint64_t)rows << a.log_tiles), CT, smem, st>>>(a);
    return launch_status();
}

template <int LOGM, bool INV, bool FUSE0, bool K2, bool SHARED>
cudaError_t launch32_contig_t(const KArgs32& a, cudaStream_t st)
{
    using CC = w32::Contig32Cfg<LOGM>;
    const size_t smem = (size_t)CC::NB * (1 << LOGM) * 4 + (SHARED ? sizeof(Tw32) << LOGM : 0);
    // Kernel-2 runs the remainder-last schedule (the plan's Kernel-2 table follows it)
    auto fn = w32::k32_contig<LOGM, INV, FUSE0, K2, SHARED, K2 ? (4 | kRemLast) : 4>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }))
        return e;
    const uint32_t grid = SHARED ? (a.L << a.log_n1) * ((a.batch + CC::NB - 1) / CC::NB)
                                 : (a.total_blocks + CC::NB - 1) / CC::NB;
    fn<<<grid, CC::CT, smem, st>>>(a);
    return launch_status();
}

template <bool INV, bool FUSE0, bool K2, int... Ls>
cudaError_t contig32_switch(int logm, const KArgs32& a, cudaStream_t st, std::integer_sequence<int, Ls...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    // Kernel-2 with a batch that fills the CTA: the shared-twiddle form
    const bool shared = K2 && a.batch >= (4096u >> logm);  // NB = 256 / (N2 / 16) ciphertexts per CTA
    ((logm == Ls ? (err = shared ? launch32_contig_t<Ls, INV, FUSE0, K2, K2>(a, st)
                                 : launch32_contig_t<Ls, INV, FUSE0, K2, false>(a, st),
                    0)
                 : 0),
     ...);
    return err;
}

template <bool INV, int... Ks>
cudaError_t cols32_switch(int key, const KArgs32& a, uint32_t rows, cudaStream_t st, std::integer_sequence<int, Ks...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((key == Ks ? (err = launch32_cols_t<(Ks & 15), (Ks >> 4), INV>(a, rows, st), 0) : 0), ...);
    return err;
}

#define K1P32(n, n1) (((n) << 4) | (n1))
using K1Pairs32 = std::integer_sequence<int, K1P32(14, 7), K1P32(15, 7), K1P32(16, 8), K1P32(17, 8), K1P32(17, 9)>;
#undef K1P32
using Single32 = std::integer_sequence<int, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13>;
using K2Sizes32 = std::integer_sequence<int, 7, 8, 9>;
}  // namespace

cudaError_t launch32(bool inverse, const KArgs32& a0, uint32_t rows, cudaStream_t st)
{
    KArgs32 a = a0;
    if (a.log_n1 == 0) {
        a.total_blocks = rows;
        return inverse ? contig32_switch<true, true, false>((int)a.logn, a, st, Single32{})
                       : contig32_switch<false, false, false>((int)a.logn, a, st, Single32{});
    }
    a.total_blocks = rows << a.log_n1;
    a.log_tiles = a.logn - a.log_n1 - 5;  // 32-column tiles
    const int logm = (int)(a.logn - a.log_n1), key = (int)((a.logn << 4) | a.log_n1);
    cudaError_t e;
    if (!inverse) {
        if ((e = cols32_switch<false>(key, a, rows, st, K1Pairs32{})) != cudaSuccess) return e;
        return contig32_switch<false, false, true>(logm, a, st, K2Sizes32{});
    }
    if ((e = contig32_switch<true, false, true>(logm, a, st, K2Sizes32{})) != cudaSuccess) return e;
    return cols32_switch<true>(key, a, rows, st, K1Pairs32{});
}

}  // namespace ntt
