// ntt_kernels.cuh -- the sm_100a kernels of the batched negacyclic NTT / iNTT,
// templated on the prime-constant type (PrimeConst: any prime; PrimeConstP:
// Proth primes p = 1 mod 2^32).  Instantiated by ntt_kernels.cu (general) and
// ntt_kernels_p.cu (Proth), compiled in parallel.
//
//   k_cols   : Kernel-1 (forward) / Kernel-1' (inverse) of the two-kernel
//              split N = N1 * N2: the N1-point column transforms
//              over stride-N2 columns, a 16-column tile per CTA so every global
//              access is a full 128-byte row segment (coalescing),
//              twiddles Psi[0..N1) preloaded into SMEM.
//   k_shared : Kernel-2 / Kernel-2' (default) -- contiguous N2-point blocks,
//              one CTA per (prime, block position, 2^12/N2 ciphertexts), the
//              block position's twiddles staged once in SMEM.
//   k_blocks : Kernel-2 / Kernel-2', persistent and cp.async-pipelined (small
//              batches, and tuning knob 5).
//   k_contig : the single-kernel path for N <= 2^13, where one CTA holds whole
//              rows (and one-shot Kernel-2 variants, knobs 3/4).
//   k_cols_pipe : persistent pipelined Kernel-1 (knob 5).
//   Optional on-the-fly twiddling on the last (forward) or first
//   (inverse) 1-2 stages of the kernel that holds them.
//
// Both run per-thread radix-2^LOGE register NTTs with SMEM exchanges between
// rounds; 64-bit words, Shoup modmul.
#pragma once
#include "ntt_device.cuh"
#include "ntt_launch.h"

#include <algorithm>
#include <atomic>
#include <type_traits>

// CTAs per SM the forward shared-twiddle Kernel-2 is compiled for (tuning
// constants, per prime family: measured on C4, profiles/r02h_ab_minb_family.jsonl --
// general primes 1.340 -> 1.325 ms at 4 (64 registers), Proth 1.249 at 3 vs 1.253 at 4)
#ifndef NTT_K2_FWD_MINB
#define NTT_K2_FWD_MINB 4
#endif
#ifndef NTT_K2_FWD_MINB_P
#define NTT_K2_FWD_MINB_P 3
#endif

namespace ntt {

// 16-byte asynchronous global -> shared copy (LDGSTS), and its completion.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- Kernel-1
template <int LOGN1, int LOGE>
struct ColsCfg {
    using SC = Sched<LOGN1, LOGE>;
    static constexpr int CT = SC::TB * 16;  // threads: 16 columns x TB per column
    static constexpr int MINB = CT <= 256 ? 4 : (CT <= 512 ? 2 : 1);
    static constexpr size_t SMEM = (size_t)SC::M * 16 * 8 + (size_t)SC::M * sizeof(Tw);
};

template <int LOGN1, int LOGN, int LOGE, bool INV, class PCT = PrimeConst>
__global__ void __launch_bounds__(ColsCfg<LOGN1, LOGE>::CT, ColsCfg<LOGN1, LOGE>::MINB) k_cols(const KArgs a)
{
    using SC = Sched<LOGN1, LOGE>;
    constexpr int M = SC::M, NR = SC::NR, CT = ColsCfg<LOGN1, LOGE>::CT;
    extern __shared__ __align__(128) uint64_t sm[];  // [M][16] words, then Tw[M]
    Tw* tws = reinterpret_cast<Tw*>(sm + M * 16);
    pdl_trigger();
    pdl_wait();

    const uint32_t tid = threadIdx.x, c = tid & 15u, tib = tid >> 4;
    // grid (batch x tiles, L): prime-major, no integer division in the prologue
    const uint32_t tile = blockIdx.x & ((1u << a.log_tiles) - 1u);
    const uint32_t b = blockIdx.x >> a.log_tiles, l = blockIdx.y;
    constexpr uint32_t logn2 = LOGN - LOGN1;  // compile-time stride: immediate offsets
    uint64_t* col = a.data + (((uint64_t)b * a.L + l) << LOGN) + tile * 16u + c;
    const Tw* tab = a.tab + ((uint64_t)l << LOGN);
    const PCT pc = load_pc<PCT>(a.pc, l);
    auto tabf = [&](const TwKey& k) { return tws[k.idx]; };
    auto otf = [&](uint32_t) { return TwMul<true>{}; };  // OT never reaches Kernel-1

    uint64_t x[16];
    // element e_k = e_0 + k s: one base address per group, compile-time offsets for k
    auto g_load = [&](auto ri) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            const uint64_t* p = col + ((uint64_t)Geo::elem(qd * SC::TB + tib, 0) << logn2);
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = p[(size_t)(k * Geo::s) << logn2];
        }
    };
    auto g_store = [&](auto ri) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            uint64_t* p = col + ((uint64_t)Geo::elem(qd * SC::TB + tib, 0) << logn2);
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) p[(size_t)(k * Geo::s) << logn2] = x[qd * Geo::R + k];
        }
    };
    auto s_load = [&](auto ri) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            const uint64_t* p = sm + Geo::elem(qd * SC::TB + tib, 0) * 16 + c;
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = p[k * Geo::s * 16];
        }
    };
    auto s_store = [&](auto ri) {
        using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            uint64_t* p = sm + Geo::elem(qd * SC::TB + tib, 0) * 16 + c;
#pragma unroll
            for (int k = 0; k < Geo::R; ++k) p[k * Geo::s * 16] = x[qd * Geo::R + k];
        }
    };

    // Psi[0..N1) into SMEM, issued after round 0's global loads so
    // the two DRAM round trips overlap
    auto preload_twiddles = [&]() {
        for (uint32_t i = tid; i < (uint32_t)M; i += CT) tws[i] = ldg_tw(tab + i);
        __syncthreads();
    };

    if constexpr (!INV) {
        static_for<NR>([&](auto ri) {
            constexpr int RI = decltype(ri)::value;
            if constexpr (RI == 0) {
                g_load(ri);
                preload_twiddles();
            } else {
                s_load(ri);
            }
            ct_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
            if constexpr (RI == NR - 1) {
                g_store(ri);  // [0, 8p): Kernel-2 continues the lazy chain
            } else {
                s_store(ri);
                __syncthreads();
            }
        });
    } else {
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            if constexpr (RI == NR - 1) {
                g_load(RC{});
                preload_twiddles();
            } else {
                s_load(RC{});
            }
            gs_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
            if constexpr (RI == 0) {
                // PrimeConstD / PD: the fused last stage already left canonical words
                if constexpr (!(std::is_same_v<PCT, PrimeConstD> || std::is_same_v<PCT, PrimeConstPD>)) {
#pragma unroll
                    for (int k = 0; k < SC::E; ++k) x[k] = norm4(x[k], pc);  // canonical [0, p)
                }
                g_store(RC{});
            } else {
                s_store(RC{});
                __syncthreads();
            }
        });
    }
}

// ---------------------------------------------------------------- Kernel-1, pipelined
// Persistent Kernel-1 / Kernel-1': each CTA walks the (row, 16-column tile)
// pairs prime-major in a grid-stride loop and prefetches the next tile --
// N1 x 128-byte row segments and the Psi[0..N1) prefix of its prime -- into
// the other half of a double buffer with cp.async while it transforms the
// current one.  Round 0 then reads SMEM; the last round stores straight to
// global (whole 128-byte segments).
template <int LOGN1, int LOGE>
struct ColsPipeCfg {
    using SC = Sched<LOGN1, LOGE>;
    static constexpr int CT = SC::TB * 16;
    static constexpr size_t BUF = (size_t)SC::M * 16 * 8 + (size_t)SC::M * sizeof(Tw);  // tile + twiddles
    static constexpr size_t SMEM = 2 * BUF;
    static constexpr int MINB = CT <= 256 ? 3 : 1;
};

template <int LOGN1, int LOGN, int LOGE, bool INV, class PCT = PrimeConst>
__global__ void __launch_bounds__(ColsPipeCfg<LOGN1, LOGE>::CT, ColsPipeCfg<LOGN1, LOGE>::MINB)
    k_cols_pipe(const KArgs a)
{
    using SC = Sched<LOGN1, LOGE>;
    using CC = ColsPipeCfg<LOGN1, LOGE>;
    constexpr int M = SC::M, NR = SC::NR, CT = CC::CT;
    constexpr uint32_t logn2 = LOGN - LOGN1;
    extern __shared__ __align__(128) uint64_t sm[];  // 128-byte aligned: SwzByte addresses
    pdl_trigger();
    pdl_wait();
    auto tile_of = [&](uint32_t buf) { return sm + buf * (CC::BUF / 8); };
    auto tw_of = [&](uint32_t buf) { return reinterpret_cast<Tw*>(sm + buf * (CC::BUF / 8) + M * 16); };

    const uint32_t tid = threadIdx.x, c = tid & 15u, tib = tid >> 4;
    const uint32_t tiles_per_row = 1u << a.log_tiles;
    const uint32_t total = a.batch * a.L * tiles_per_row;

    auto locate = [&](uint32_t t, uint32_t& l, uint64_t*& base) {
        const uint32_t tile = t & (tiles_per_row - 1u), q = t >> a.log_tiles;  // q = l * batch + b
        l = q / a.batch;
        const uint32_t b = q - l * a.batch;
        base = a.data + (((uint64_t)b * a.L + l) << LOGN) + tile * 16u;
    };
    auto prefetch = [&](uint32_t t, uint32_t buf) {
        if (t < total) {
            uint32_t l;
            uint64_t* base;
            locate(t, l, base);
            uint64_t* st = tile_of(buf);
            // M rows x 8 chunks of 16 bytes; thread tid takes chunks tid, tid+CT, ...
#pragma unroll
            for (int j = 0; j < (M * 8) / CT; ++j) {
                const uint32_t ch = j * CT + tid, row = ch >> 3, col2 = (ch & 7u) * 2;
                cp_async16(st + row * 16 + col2, base + ((uint64_t)row << logn2) + col2);
            }
            const Tw* tab = a.tab + ((uint64_t)l << LOGN);
            Tw* tw = tw_of(buf);
            for (uint32_t i = tid; i < (uint32_t)M; i += CT) cp_async16(tw + i, tab + i);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    uint32_t t = blockIdx.x;
    prefetch(t, 0);
    for (uint32_t it = 0; t < total; ++it, t += gridDim.x) {
        const uint32_t buf = it & 1u;
        prefetch(t + gridDim.x, buf ^ 1u);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();

        uint32_t l;
        uint64_t* base;
        locate(t, l, base);
        uint64_t* col = base + c;
        uint64_t* smt = tile_of(buf);
        const Tw* tws = tw_of(buf);
        const PCT pc = load_pc<PCT>(a.pc, l);
        auto tabf = [&](const TwKey& k) { return tws[k.idx]; };
        auto otf = [&](uint32_t) { return TwMul<true>{}; };

        uint64_t x[16];
        auto g_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k)
                    col[(uint64_t)Geo::elem(qd * SC::TB + tib, k) << logn2] = x[qd * Geo::R + k];
        };
        auto s_load = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = smt[Geo::elem(qd * SC::TB + tib, k) * 16 + c];
        };
        auto s_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) smt[Geo::elem(qd * SC::TB + tib, k) * 16 + c] = x[qd * Geo::R + k];
        };

        if constexpr (!INV) {
            static_for<NR>([&](auto ri) {
                constexpr int RI = decltype(ri)::value;
                s_load(ri);
                ct_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
                if constexpr (RI == NR - 1) {
                    g_store(ri);
                } else {
                    s_store(ri);
                    __syncthreads();
                }
            });
        } else {
            static_for<NR>([&](auto rj) {
                constexpr int RI = NR - 1 - decltype(rj)::value;
                using RC = std::integral_constant<int, RI>;
                s_load(RC{});
                gs_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
                if constexpr (RI == 0) {
#pragma unroll
                    for (int k = 0; k < SC::E; ++k) x[k] = norm4(x[k], pc);
                    g_store(RC{});
                } else {
                    s_store(RC{});
                    __syncthreads();
                }
            });
        }
        __syncthreads();  // this buffer is refilled by the prefetch two iterations on
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------- SMEM round exchange
// Load / store the thread's groups of round RI from / to a swizzled SMEM block
// (section 5.3 of DESIGN.md; stride-1 rounds as 128-bit pairs).  When the
// round's smallest stride s divides TB, elem(qd TB + tib, k) = elem(tib, 0) +
// elem(qd TB, k) with disjoint bits, so the addresses are SwzByte forms of one
// per-round base (the block's shared-window byte address folded in once: one
// LOP3 per distinct swizzle constant, immediate offsets); otherwise (a
// remainder-first round 0) each element is swizzled on its own.
template <int LOGM, int LOGE, int RI, int TB>
__device__ __forceinline__ void xchg_load(uint64_t (&x)[16], const uint64_t* sb, uint32_t tib)
{
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    if constexpr (TB % Geo::s == 0 && LOGM >= 4) {  // blocks of >= 128 bytes: base bits 4..6 clear
        const uint32_t Pb = (uint32_t)__cvta_generic_to_shared(sb) + 8u * swz(Geo::elem(tib, 0));
        static_for<Geo::GPT>([&](auto qdc) {
            constexpr int qd = decltype(qdc)::value;
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
                static_for<Geo::R / 2>([&](auto kc) {
                    constexpr int k = 2 * decltype(kc)::value;
                    using SW = SwzByte<Geo::elem(qd * TB, k)>;
                    lds128_at<SW::off>(SW::base(Pb), x[qd * Geo::R + k], x[qd * Geo::R + k + 1]);
                });
            } else {
                static_for<Geo::R>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    using SW = SwzByte<Geo::elem(qd * TB, k)>;
                    x[qd * Geo::R + k] = lds64_at<SW::off>(SW::base(Pb));
                });
            }
        });
    } else {
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
#pragma unroll
                for (int k = 0; k < Geo::R; k += 2) {
                    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sb + swz(Geo::elem(qd * TB + tib, k)));
                    x[qd * Geo::R + k] = v.x;
                    x[qd * Geo::R + k + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = sb[swz(Geo::elem(qd * TB + tib, k))];
            }
        }
    }
}
template <int LOGM, int LOGE, int RI, int TB>
__device__ __forceinline__ void xchg_store(const uint64_t (&x)[16], uint64_t* sb, uint32_t tib)
{
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    if constexpr (TB % Geo::s == 0 && LOGM >= 4) {  // blocks of >= 128 bytes: base bits 4..6 clear
        const uint32_t Pb = (uint32_t)__cvta_generic_to_shared(sb) + 8u * swz(Geo::elem(tib, 0));
        static_for<Geo::GPT>([&](auto qdc) {
            constexpr int qd = decltype(qdc)::value;
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
                static_for<Geo::R / 2>([&](auto kc) {
                    constexpr int k = 2 * decltype(kc)::value;
                    using SW = SwzByte<Geo::elem(qd * TB, k)>;
                    sts128_at<SW::off>(SW::base(Pb), x[qd * Geo::R + k], x[qd * Geo::R + k + 1]);
                });
            } else {
                static_for<Geo::R>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    using SW = SwzByte<Geo::elem(qd * TB, k)>;
                    sts64_at<SW::off>(SW::base(Pb), x[qd * Geo::R + k]);
                });
            }
        });
    } else {
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
#pragma unroll
                for (int k = 0; k < Geo::R; k += 2)
                    *reinterpret_cast<ulonglong2*>(sb + swz(Geo::elem(qd * TB + tib, k))) =
                        make_ulonglong2(x[qd * Geo::R + k], x[qd * Geo::R + k + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) sb[swz(Geo::elem(qd * TB + tib, k))] = x[qd * Geo::R + k];
            }
        }
    }
}

// ---------------------------------------------------------------- contiguous
template <int LOGM, int LOGE, bool TWS = false>
struct ContigCfg {
    static constexpr int TB = Sched<LOGM, LOGE>::TB;
    static constexpr int CT = TB > 256 ? TB : 256;  // threads per CTA
    static constexpr int NB = CT / TB;              // blocks per CTA iteration
    // TWP: a one-row-per-CTA single kernel at N = 2^12 (C1) copies its row's
    // whole Psi table into SMEM with cp.async at the start, overlapped with the
    // data loads, instead of loading each round's twiddles from L2 when the
    // round starts (a latency the one CTA cannot hide)
    static constexpr bool TWP = !TWS && NB == 1 && LOGM == 12;
    static constexpr size_t SMEM = (size_t)NB * (1 << LOGM) * 8 + (TWP ? (size_t)(1 << LOGM) * 16 : 0);
    // register budget: the Kernel-2 mode (TWS) targets 32 warps/SM like Kernel-1
    static constexpr int MINB = CT > 256 ? 1 : (TWS ? 3 : (LOGE >= 4 ? 2 : 3));
};



// Barrier over the TB threads of one block: blocks never share SMEM, so a
// block that fits one warp synchronises with __syncwarp and larger blocks with
// a named barrier of their own; CTA-wide barriers are avoided.
template <int TB>
__device__ __forceinline__ void block_sync(uint32_t blk)
{
    if constexpr (TB <= 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(blk + 1), "n"(TB) : "memory");
    }
}

// TWS: stage each block's twiddles in SMEM.  Block bb of Kernel-2 (F = N1+bb)
// uses Psi[F 2^j + h], h < 2^j, at local stage j: M-1 entries in log M
// contiguous table ranges, copied with cp.async into a local table
// tl[2^j + h] at the block's start (one latency per block instead of one per
// round) and read back with LDS.128.  Stages under OT skip their ranges.
template <int LOGM, int LOGE, bool INV, bool FUSE0, int OTS, bool TWS, bool MUL = false, class PCT = PrimeConst>
__global__ void __launch_bounds__(ContigCfg<LOGM, LOGE, TWS>::CT, ContigCfg<LOGM, LOGE, TWS>::MINB)
    k_contig(const KArgs a)
{
    using SC = Sched<LOGM, LOGE>;
    using CC = ContigCfg<LOGM, LOGE, TWS>;
    constexpr int M = SC::M, E = SC::E, TB = SC::TB, NR = SC::NR;
    constexpr int OT_FROM = OTS ? LOGM - OTS : (1 << 20);
    extern __shared__ __align__(128) uint64_t sm[];  // 128-byte aligned: SwzByte addresses
    pdl_trigger();
    pdl_wait();

    const uint32_t tid = threadIdx.x, blk = tid / TB, tib = tid % TB;
    uint64_t* sb = sm + blk * M;
    const uint32_t n1mask = (1u << a.log_n1) - 1u;
    const uint32_t B_ot = 1u << a.ot_logb;

    for (uint32_t it = 0; it < a.iters; ++it) {
        uint32_t gb = (blockIdx.x * a.iters + it) * CC::NB + blk;
        const bool active = gb < a.total_blocks;
        if (!active) gb = a.total_blocks - 1;  // compute a valid block, skip its store
        const uint32_t bb = gb & n1mask, q = gb >> a.log_n1;
        const uint32_t l = q / a.batch, b = q - l * a.batch;
        uint64_t* g = a.data + (((uint64_t)b * a.L + l) << a.logn) + (uint64_t)bb * M;
        const uint32_t F = (1u << a.log_n1) + bb;
        const Tw* tab = a.tab + ((uint64_t)l << a.logn);
        const Tw* ot = a.ot + (uint64_t)l * (B_ot + ((1u << a.logn) >> a.ot_logb));
        const PCT pc = load_pc<PCT>(a.pc, l);
        // TWS (Kernel-2 mode): twiddles from the plan's Kernel-2 table, whose
        // per-round [i][h][g] order makes every warp read contiguous entries.
        const Tw* tb2 = a.tab2 + ((uint64_t)l << a.logn) + ((uint64_t)bb << LOGM);
        Tw* const twp = reinterpret_cast<Tw*>(sm + CC::NB * M);  // CC::TWP: the row's Psi table
        if constexpr (CC::TWP) {
            for (uint32_t i = tid; i < (uint32_t)M; i += CC::CT) cp_async16(twp + i, tab + i);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        auto tabf = [&](const TwKey& k) {
            if constexpr (TWS) {
                return ldg_tw(tb2 + K2Layout<LOGM, LOGE>::round_off(k.S) + ((((1u << k.i) - 1u + k.h) << k.S) + k.g));
            } else if constexpr (CC::TWP) {
                return twp[k.idx + ((F - 1u) << k.j)];
            } else {
                return ldg_tw(tab + k.idx + ((F - 1u) << k.j));
            }
        };
        auto otf = [&](uint32_t idx) {
            // exponent of Psi[idx] is bitrev_logn(idx) = e = q*B + r
            const uint32_t e = __brev(idx) >> (32 - a.logn);
            return TwMul<true>{ldg_tw(ot + (e & (B_ot - 1u))), ldg_tw(ot + B_ot + (e >> a.ot_logb))};
        };

        // Round 0 touches e = o + k s with s = M >> r(0): when s >= 16 a warp's
        // accesses are whole 128-byte segments, so the forward loads round 0
        // straight from global and the inverse stores its last round (round 0)
        // straight to global; the other end goes through SMEM with 16-byte
        // vectors.
        constexpr bool DIRECT0 = RoundGeo<LOGM, 0, LOGE>::s >= 16;
        auto stage_in = [&]() {
#pragma unroll
            for (int j = 0; j < E / 2; ++j) {
                const uint32_t ch = j * TB + tib;
                ulonglong2 v = *reinterpret_cast<const ulonglong2*>(g + 2 * ch);
                if constexpr (MUL) {  // fused NTT-domain product (ntt_pointwise_inverse)
                    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(a.mul_a + (g - a.data) + 2 * ch);
                    v.x = mont_mul(u.x, v.x, pc);
                    v.y = mont_mul(u.y, v.y, pc);
                }
                *reinterpret_cast<ulonglong2*>(sb + swz(2 * ch)) = v;
            }
            block_sync<TB>(blk);
        };
        auto stage_out = [&]() {
            if (active) {
#pragma unroll
                for (int j = 0; j < E / 2; ++j) {
                    const uint32_t ch = j * TB + tib;
                    *reinterpret_cast<ulonglong2*>(g + 2 * ch) =
                        *reinterpret_cast<const ulonglong2*>(sb + swz(2 * ch));
                }
            }
            block_sync<TB>(blk);  // the next iteration reuses this SMEM block
        };

        uint64_t x[16];
        auto g_load0 = [&]() {
            using Geo = RoundGeo<LOGM, 0, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = g[Geo::elem(qd * TB + tib, k)];
        };
        auto g_store0 = [&]() {
            using Geo = RoundGeo<LOGM, 0, LOGE>;
            if (active) {
#pragma unroll
                for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                    for (int k = 0; k < Geo::R; ++k) g[Geo::elem(qd * TB + tib, k)] = x[qd * Geo::R + k];
            }
        };
        // stride-1 rounds hold adjacent pairs (e, e+1): 128-bit SMEM accesses
        auto s_load = [&](auto ri) { xchg_load<LOGM, LOGE, decltype(ri)::value, TB>(x, sb, tib); };
        auto s_store = [&](auto ri) { xchg_store<LOGM, LOGE, decltype(ri)::value, TB>(x, sb, tib); };

        auto tw_ready = [&]() {
            if constexpr (CC::TWP) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncthreads();
            }
        };
        if constexpr (!INV) {
            if constexpr (!DIRECT0) stage_in();
            tw_ready();
            static_for<NR>([&](auto ri) {
                constexpr int RI = decltype(ri)::value;
                if constexpr (RI == 0 && DIRECT0) {
                    g_load0();
                } else {
                    s_load(ri);
                }
                ct_round<LOGM, LOGE, RI, OT_FROM, !TWS, true>(x, tib, F - 1u, tabf, otf, pc);  // single kernel: canonical input
                if constexpr (RI == NR - 1) {
#pragma unroll
                    for (int k = 0; k < E; ++k) x[k] = norm8(x[k], pc);  // any word (lazy < 16p + 2^32) -> [0,p)
                }
                s_store(ri);
                block_sync<TB>(blk);
            });
            stage_out();
        } else {
            stage_in();
            tw_ready();
            static_for<NR>([&](auto rj) {
                constexpr int RI = NR - 1 - decltype(rj)::value;
                using RC = std::integral_constant<int, RI>;
                s_load(RC{});
                gs_round<LOGM, LOGE, RI, OT_FROM, FUSE0>(x, tib, F - 1u, tabf, otf, pc);
                if constexpr (FUSE0 && RI == 0) {
#pragma unroll
                    for (int k = 0; k < E; ++k) x[k] = norm4(x[k], pc);
                }
                if constexpr (RI == 0 && DIRECT0) {
                    g_store0();
                } else {
                    s_store(RC{});
                    block_sync<TB>(blk);
                }
            });
            if constexpr (!DIRECT0) {
                stage_out();
            } else {
                block_sync<TB>(blk);  // round-0 SMEM reads done before the next stage_in
            }
        }
    }
}

// ---------------------------------------------------------------- Kernel-2, shared twiddles
// Kernel-2 / Kernel-2' with one CTA per (prime l, block position bb, group of
// NB ciphertexts): the NB blocks of a CTA use the same twiddles (Psi depends on
// the prime and the block position only), so the block's Kernel-2 table segment
// (N2 entries, plan-built K2Layout) is staged in SMEM once and read by all NB
// block groups; each block is transformed by TB = N2/16 threads (one warp for
// N2 = 2^9) that synchronise among themselves only.  256 threads, 64 registers:
// 4 CTAs = 32 warps per SM, like Kernel-1, so the multiply pipe is fed by
// occupancy rather than by a software pipeline.
template <int LOGM, bool INV = false>
struct SharedCfg {
    static constexpr int TB = Sched<LOGM, 4>::TB;
    static constexpr int CT = 256;
    static constexpr int NB = CT / TB;  // blocks (ciphertexts) per CTA
    static constexpr size_t SMEM = (size_t)NB * (8u << LOGM) + (sizeof(Tw) << LOGM);
    // measured on C4: the inverse runs best with 64 registers at 4 CTAs/SM;
    // the forward (final reduction, more live values) with Proth primes at 3
    // (80 registers), with general primes at 4
    template <class PCT>
    static constexpr int minb()
    {
        return INV ? 4 : (std::is_same_v<PCT, PrimeConstP> ? NTT_K2_FWD_MINB_P : NTT_K2_FWD_MINB);
    }
};

template <int LOGM, bool INV, int OTS, bool MUL = false, class PCT = PrimeConst, int LE2 = 4>
__global__ void __launch_bounds__(SharedCfg<LOGM, INV>::CT, SharedCfg<LOGM, INV>::template minb<PCT>())
    k_shared(const KArgs a)
{
    using SC = Sched<LOGM, LE2>;
    using CC = SharedCfg<LOGM, INV>;
    constexpr int M = SC::M, E = SC::E, TB = SC::TB, NR = SC::NR, NB = CC::NB, CT = CC::CT;
    constexpr int OT_FROM = OTS ? LOGM - OTS : (1 << 20);
    extern __shared__ __align__(128) uint64_t sm[];  // 128-byte aligned: SwzByte addresses
    Tw* const tws = reinterpret_cast<Tw*>(sm + NB * M);
    pdl_trigger();

    const uint32_t tid = threadIdx.x, blk = tid / TB, tib = tid % TB;
    // grid (ciphertext groups, block positions, primes): prime-major then
    // block position, no integer division in the prologue
    const uint32_t cg = blockIdx.x, bb = blockIdx.y, l = blockIdx.z;
    const uint32_t b = cg * NB + blk;
    const bool active = b < a.batch;
    uint64_t* g = a.data + (((uint64_t)(active ? b : 0) * a.L + l) << a.logn) + ((uint64_t)bb << LOGM);
    const uint32_t Fm1 = (1u << a.log_n1) + bb - 1u;
    const uint32_t B_ot = 1u << a.ot_logb;
    const Tw* ot = a.ot + (uint64_t)l * (B_ot + ((1u << a.logn) >> a.ot_logb));
    const PCT pc = load_pc<PCT>(a.pc, l);

    {  // the block position's twiddle segment, once per CTA (under OT only the prefix of the table stages)
        const Tw* t2 = a.tab2 + ((uint64_t)l << a.logn) + ((uint64_t)bb << LOGM);
        constexpr uint32_t USED = K2Layout<LOGM, LE2>::used(OTS);
        for (uint32_t i = tid; i < USED; i += CT) cp_async16(tws + i, t2 + i);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    pdl_wait();  // the twiddles are constant: staged while the previous kernel finishes
    uint64_t* sb = sm + blk * M;
    auto tabf = [&](const TwKey& k) {
        return tws[K2Layout<LOGM, LE2>::round_off(k.S) + ((((1u << k.i) - 1u + k.h) << k.S) + k.g)];
    };
    auto otf = [&](uint32_t idx) {
        const uint32_t e = __brev(idx) >> (32 - a.logn);  // exponent of Psi[idx]
        return TwMul<true>{ldg_tw(ot + (e & (B_ot - 1u))), ldg_tw(ot + B_ot + (e >> a.ot_logb))};
    };

    uint64_t x[16];
    // round exchanges through the block's swizzled SMEM image (SwzByte addresses)
    auto s_load = [&](auto ri) { xchg_load<LOGM, LE2, decltype(ri)::value, TB>(x, sb, tib); };
    auto s_store = [&](auto ri) { xchg_store<LOGM, LE2, decltype(ri)::value, TB>(x, sb, tib); };
    constexpr bool DIRECT0 = RoundGeo<LOGM, 0, LE2>::s >= 16;
    static_assert(DIRECT0, "round 0 is read / written straight from global");
    // remainder-last schedule with a single-stage remainder: the last forward
    // round is radix-2 on adjacent pairs, read / written straight from global
    constexpr bool DIRECT_LAST = SC::REMLAST && SC::REM == 1;
    auto twiddles_ready = [&]() {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    };

    if constexpr (!INV) {
        {  // round 0 straight from global: whole 128-byte segments per warp
            using Geo = RoundGeo<LOGM, 0, LE2>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = g[Geo::elem(qd * TB + tib, k)];
        }
        twiddles_ready();
        static_for<NR>([&](auto ri) {
            constexpr int RI = decltype(ri)::value;
            if constexpr (RI > 0) s_load(ri);
            ct_round<LOGM, LE2, RI, OT_FROM, false, true>(x, tib, Fm1, tabf, otf, pc);
            if constexpr (RI == NR - 1) {
#pragma unroll
                for (int k = 0; k < E; ++k) x[k] = norm8(x[k], pc);  // any word (lazy < 16p + 2^32) -> [0,p)
            }
            if constexpr (DIRECT_LAST && RI == NR - 1) {
                // remainder-last radix-2 round: the thread's pairs (2G, 2G+1) go
                // straight to global, lanes contiguous (512 bytes per warp store)
                using Geo = RoundGeo<LOGM, RI, LE2>;
                if (active) {
                    // general / d-form primes: two 8-byte stores per pair (a
                    // 16-byte store needs the pair in a register quad, ~26
                    // IMAD.MOV per thread on the multiply pipe; -1.1 % on this
                    // kernel); Proth primes: 16-byte stores (+0.5 % otherwise)
                    // -- DESIGN.md 5.4c
#pragma unroll
                    for (int qd = 0; qd < Geo::GPT; ++qd) {
                        if constexpr (std::is_same_v<PCT, PrimeConstP>) {
                            *reinterpret_cast<ulonglong2*>(g + Geo::elem(qd * TB + tib, 0)) =
                                make_ulonglong2(x[2 * qd], x[2 * qd + 1]);
                        } else {
                            g[Geo::elem(qd * TB + tib, 0)] = x[2 * qd];
                            g[Geo::elem(qd * TB + tib, 0) + 1] = x[2 * qd + 1];
                        }
                    }
                }
            } else {
                s_store(ri);
                block_sync<TB>(blk);
            }
        });
        if (!DIRECT_LAST && active) {  // 128-bit coalesced stores; word 2 ch = 2 j TB + 2 tib
            const uint32_t s2 = swz(2 * tib);
            static_for<E / 2>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                *reinterpret_cast<ulonglong2*>(g + 2 * (j * TB + tib)) =
                    *reinterpret_cast<const ulonglong2*>(sb + swz_at<2 * j * TB>(s2));
            });
        }
    } else if constexpr (!DIRECT_LAST) {
        const uint32_t s2 = swz(2 * tib);
        static_for<E / 2>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            const uint32_t ch = j * TB + tib;
            ulonglong2 v = *reinterpret_cast<const ulonglong2*>(g + 2 * ch);
            if constexpr (MUL) {  // fused NTT-domain product (ntt_pointwise_inverse)
                const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(a.mul_a + (g - a.data) + 2 * ch);
                v.x = mont_mul(u.x, v.x, pc);
                v.y = mont_mul(u.y, v.y, pc);
            }
            *reinterpret_cast<ulonglong2*>(sb + swz_at<2 * j * TB>(s2)) = v;
        });
        twiddles_ready();
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            s_load(RC{});
            // the inverse's input is canonical (or a Montgomery product < 2p):
            // its first GS stage needs no reduction
            gs_round<LOGM, LE2, RI, OT_FROM, false, RI == NR - 1>(x, tib, Fm1, tabf, otf, pc);
            if constexpr (RI > 0) {
                s_store(RC{});
                block_sync<TB>(blk);
            }
        });
        if (active) {  // round 0 straight to global
            using Geo = RoundGeo<LOGM, 0, LE2>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) g[Geo::elem(qd * TB + tib, k)] = x[qd * Geo::R + k];
        }
    } else {
        // remainder-last: the first inverse round (the radix-2 remainder) reads
        // its pairs (2G, 2G+1) straight from global -- no SMEM staging
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            if constexpr (RI == NR - 1) {
                using Geo = RoundGeo<LOGM, RI, LE2>;
#pragma unroll
                for (int qd = 0; qd < Geo::GPT; ++qd) {
                    const uint32_t e = Geo::elem(qd * TB + tib, 0);
                    ulonglong2 v = *reinterpret_cast<const ulonglong2*>(g + e);
                    if constexpr (MUL) {  // fused NTT-domain product (ntt_pointwise_inverse)
                        const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(a.mul_a + (g - a.data) + e);
                        v.x = mont_mul(u.x, v.x, pc);
                        v.y = mont_mul(u.y, v.y, pc);
                    }
                    x[2 * qd] = v.x;
                    x[2 * qd + 1] = v.y;
                }
                twiddles_ready();
            } else {
                s_load(RC{});
            }
            // the inverse's input is canonical (or a Montgomery product < 2p):
            // its first GS stage needs no reduction
            gs_round<LOGM, LE2, RI, OT_FROM, false, RI == NR - 1>(x, tib, Fm1, tabf, otf, pc);
            if constexpr (RI > 0) {
                s_store(RC{});
                block_sync<TB>(blk);
            }
        });
        if (active) {  // round 0 straight to global
            using Geo = RoundGeo<LOGM, 0, LE2>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) g[Geo::elem(qd * TB + tib, k)] = x[qd * Geo::R + k];
        }
    }
}

// ---------------------------------------------------------------- Kernel-2, pipelined
// Persistent Kernel-2 / Kernel-2': each group of TB threads ("slot") walks the
// N2-blocks in a grid-stride loop, prime-major, and prefetches block i+1 into
// the second half of a double buffer with cp.async (LDGSTS, swizzled
// destination) while it transforms block i -- the load latency of one block
// hides behind the arithmetic of the previous one.  Twiddles come through the
// read-only path (the current prime's table stays L2-resident).
// The block's twiddles (Kernel-2 layout: one contiguous N2-entry segment per
// block) are prefetched with the data, so no global load sits on the
// critical path of a round.  SMEM per slot: 2 x (8 + 16) x N2 bytes.
template <int LOGM, int LOGE>
struct PipeCfg {
    static constexpr int TB = Sched<LOGM, LOGE>::TB;
    static constexpr int SLOT = (1 << LOGM) * (2 * 8 + 16);  // bytes per slot
    static constexpr int NB0 = (96 * 1024) / SLOT;
    static constexpr int NB = NB0 < 1 ? 1 : (NB0 > 4 ? 4 : NB0);  // slots per CTA
    static constexpr int CT = NB * TB;
    // double-buffered data, single-buffered twiddles (refilled once the last
    // round has read them): (2 x 8 + 16) x N2 bytes per slot
    static constexpr size_t SMEM = (size_t)NB * (1 << LOGM) * (2 * 8 + sizeof(Tw));
    static constexpr int MINB = LOGE >= 4 ? 3 : 3;
};

template <int LOGM, int LOGE, bool INV, int OTS, bool MUL = false, class PCT = PrimeConst>
__global__ void __launch_bounds__(PipeCfg<LOGM, LOGE>::CT, PipeCfg<LOGM, LOGE>::MINB) k_blocks(const KArgs a)
{
    using SC = Sched<LOGM, LOGE>;
    using PC = PipeCfg<LOGM, LOGE>;
    constexpr int M = SC::M, E = SC::E, TB = SC::TB, NR = SC::NR, NB = PC::NB;
    constexpr int OT_FROM = OTS ? LOGM - OTS : (1 << 20);
    static_assert(TB <= 256 && NB >= 1, "block size");
    extern __shared__ __align__(128) uint64_t sm[];  // 128-byte aligned: SwzByte addresses

    const uint32_t tid = threadIdx.x, blk = tid / TB, tib = tid % TB;
    const uint32_t n1mask = (1u << a.log_n1) - 1u;
    const uint32_t B_ot = 1u << a.ot_logb;
    const uint32_t nslots = gridDim.x * NB;

    auto block_ptr = [&](uint32_t gb, uint32_t& l, uint32_t& bb) {
        bb = gb & n1mask;
        const uint32_t q = gb >> a.log_n1;  // prime-major: q = l * batch + b
        l = q / a.batch;
        const uint32_t b = q - l * a.batch;
        return a.data + (((uint64_t)b * a.L + l) << a.logn) + (uint64_t)bb * M;
    };
    Tw* const tws = reinterpret_cast<Tw*>(sm + 2 * NB * M) + blk * M;
    auto prefetch_data = [&](uint32_t gb, uint32_t buf) {
        if (gb < a.total_blocks) {
            uint32_t l, bb;
            const uint64_t* g = block_ptr(gb, l, bb);
            uint64_t* sd = sm + (buf * NB + blk) * M;
#pragma unroll
            for (int j = 0; j < E / 2; ++j) {
                const uint32_t ch = j * TB + tib;
                cp_async16(sd + swz(2 * ch), g + 2 * ch);
            }
        }
    };
    auto prefetch_tw = [&](uint32_t gb) {
        if (gb < a.total_blocks) {
            const uint32_t bb = gb & n1mask, q = gb >> a.log_n1, l = q / a.batch;
            const Tw* t2 = a.tab2 + ((uint64_t)l << a.logn) + ((uint64_t)bb << LOGM);
            constexpr uint32_t USED = K2Layout<LOGM, LOGE>::used(OTS);  // OT stages' entries are not read
#pragma unroll
            for (int j = 0; j < E; ++j)
                if (j * TB + tib < USED) cp_async16(tws + j * TB + tib, t2 + j * TB + tib);
        }
    };
    auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };

    pdl_trigger();
    uint32_t gb = blockIdx.x * NB + blk;
    prefetch_tw(gb);  // constant: staged while the previous kernel finishes
    pdl_wait();
    prefetch_data(gb, 0);
    commit();
    for (uint32_t it = 0; gb < a.total_blocks; ++it, gb += nslots) {
        uint64_t* sb = sm + ((it & 1) * NB + blk) * M;
        prefetch_data(gb + nslots, (it + 1) & 1);
        commit();
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // data(it) and tw(it) landed
        block_sync<TB>(blk);
        uint32_t l, bb;
        uint64_t* g = block_ptr(gb, l, bb);
        const uint32_t Fm1 = (1u << a.log_n1) + bb - 1u;
        const Tw* ot = a.ot + (uint64_t)l * (B_ot + ((1u << a.logn) >> a.ot_logb));
        const PCT pc = load_pc<PCT>(a.pc, l);
        // Kernel-2 table segment (plan-built, per block, per round, [i][h][g]),
        // prefetched into SMEM: the lanes of a warp read consecutive groups g.
        auto tabf = [&](const TwKey& k) {
            return tws[K2Layout<LOGM, LOGE>::round_off(k.S) + ((((1u << k.i) - 1u + k.h) << k.S) + k.g)];
        };
        auto otf = [&](uint32_t idx) {
            const uint32_t e = __brev(idx) >> (32 - a.logn);  // exponent of Psi[idx]
            return TwMul<true>{ldg_tw(ot + (e & (B_ot - 1u))), ldg_tw(ot + B_ot + (e >> a.ot_logb))};
        };

        uint64_t x[16];
        auto s_load = [&](auto ri) { xchg_load<LOGM, LOGE, decltype(ri)::value, TB>(x, sb, tib); };
        auto s_store = [&](auto ri) { xchg_store<LOGM, LOGE, decltype(ri)::value, TB>(x, sb, tib); };
        auto stage_out = [&]() {
#pragma unroll
            for (int j = 0; j < E / 2; ++j) {
                const uint32_t ch = j * TB + tib;
                *reinterpret_cast<ulonglong2*>(g + 2 * ch) = *reinterpret_cast<const ulonglong2*>(sb + swz(2 * ch));
            }
        };
        constexpr bool DIRECT0 = RoundGeo<LOGM, 0, LOGE>::s >= 16;

        if constexpr (!INV) {
            static_for<NR>([&](auto ri) {
                constexpr int RI = decltype(ri)::value;
                s_load(ri);
                ct_round<LOGM, LOGE, RI, OT_FROM, false, true>(x, tib, Fm1, tabf, otf, pc);
                if constexpr (RI == NR - 1) {
#pragma unroll
                    for (int k = 0; k < E; ++k) x[k] = norm8(x[k], pc);  // any word (lazy < 16p + 2^32) -> [0,p)
                }
                s_store(ri);
                block_sync<TB>(blk);
            });
            prefetch_tw(gb + nslots);  // the sync above ended every twiddle read
            commit();
            stage_out();
        } else {
            static_for<NR>([&](auto rj) {
                constexpr int RI = NR - 1 - decltype(rj)::value;
                using RC = std::integral_constant<int, RI>;
                s_load(RC{});
                if constexpr (MUL && RI == NR - 1) {  // fused NTT-domain product (ntt_pointwise_inverse)
                    using Geo = RoundGeo<LOGM, RI, LOGE>;
                    const uint64_t* ga = a.mul_a + (g - a.data);
#pragma unroll
                    for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                        for (int k = 0; k < Geo::R; ++k)
                            x[qd * Geo::R + k] = mont_mul(__ldg(ga + Geo::elem(qd * TB + tib, k)), x[qd * Geo::R + k], pc);
                }
                gs_round<LOGM, LOGE, RI, OT_FROM, false>(x, tib, Fm1, tabf, otf, pc);
                if constexpr (RI == 0 && DIRECT0) {
                    using Geo = RoundGeo<LOGM, 0, LOGE>;
#pragma unroll
                    for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                        for (int k = 0; k < Geo::R; ++k) g[Geo::elem(qd * TB + tib, k)] = x[qd * Geo::R + k];
                } else {
                    s_store(RC{});
                    block_sync<TB>(blk);
                }
            });
            if constexpr (!DIRECT0) stage_out();
        }
        block_sync<TB>(blk);  // all reads of this buffer done before it is refilled
        if constexpr (INV) {
            prefetch_tw(gb + nslots);
            commit();
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------- dispatch
namespace detail {

// SM count of the current device, cached per device (persistent-grid sizing)
inline int sm_count()
{
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int v = cache[dev & 63].load(std::memory_order_relaxed);
    if (v == 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev & 63].store(v, std::memory_order_relaxed);
    }
    return v;
}

template <int LOGN1, int LOGN, int LOGE, bool INV, class PCT>
cudaError_t launch_cols_t(const KArgs& a, uint32_t rows, cudaStream_t st)
{
    using CC = ColsCfg<LOGN1, LOGE>;
    auto fn = k_cols<LOGN1, LOGN, LOGE, INV, PCT>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CC::SMEM);
        }))
        return e;
    // rows = batch * L (L <= 65535, ntt_plan_create_ex)
    return launch_pdl(fn, dim3((unsigned)(rows / a.L) << a.log_tiles, a.L), dim3(CC::CT), CC::SMEM, st, a);
}

template <int LOGM, int LOGE, bool INV, bool FUSE0, int OTS, bool TWS, bool MUL, class PCT>
cudaError_t launch_contig_t(KArgs a, uint32_t iters, cudaStream_t st)
{
    using CC = ContigCfg<LOGM, LOGE, TWS>;
    auto fn = k_contig<LOGM, LOGE, INV, FUSE0, OTS, TWS, MUL, PCT>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CC::SMEM);
        }))
        return e;
    a.iters = iters;
    const uint64_t per_cta = (uint64_t)CC::NB * iters;
    const uint64_t grid = (a.total_blocks + per_cta - 1) / per_cta;
    return launch_pdl(fn, dim3((unsigned)grid), dim3(CC::CT), CC::SMEM, st, a);
}

template <int LOGM, int LOGE, bool INV, int OTS, bool MUL, class PCT>
cudaError_t launch_blocks_t(KArgs a, cudaStream_t st)
{
    using PC = PipeCfg<LOGM, LOGE>;
    auto fn = k_blocks<LOGM, LOGE, INV, OTS, MUL, PCT>;
    static DeviceOnce once;  // value: resident CTAs per SM
    if (cudaError_t e = once.run([&](int& ctas) {
            cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PC::SMEM);
            return r != cudaSuccess ? r : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, PC::CT, PC::SMEM);
        }))
        return e;
    const int ctas_per_sm = once.value();
    const int sms = sm_count();
    const uint64_t want = ((uint64_t)a.total_blocks + PC::NB - 1) / PC::NB;
    const uint64_t grid = std::min<uint64_t>(want, (uint64_t)sms * std::max(1, ctas_per_sm));
    return launch_pdl(fn, dim3((unsigned)grid), dim3(PC::CT), PC::SMEM, st, a);
}

template <int LOGM, bool INV, int OTS, bool MUL, class PCT, int LE2>
cudaError_t launch_shared_t(const KArgs& a, cudaStream_t st)
{
    using CC = SharedCfg<LOGM, INV>;
    auto fn = k_shared<LOGM, INV, OTS, MUL, PCT, LE2>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CC::SMEM);
        }))
        return e;
    return launch_pdl(fn, dim3((a.batch + CC::NB - 1) / CC::NB, 1u << a.log_n1, a.L), dim3(CC::CT), CC::SMEM, st, a);
}

template <int LOGM, bool INV, class PCT, int LE2>
cudaError_t launch_shared_ot2(const KArgs& a, int ots, cudaStream_t st)
{
    if (a.mul_a) {
        if constexpr (INV) {
            if (ots == 0) return launch_shared_t<LOGM, INV, 0, true, PCT, LE2>(a, st);
        }
        return cudaErrorNotSupported;
    }
    switch (ots) {
        case 0: return launch_shared_t<LOGM, INV, 0, false, PCT, LE2>(a, st);
        case 1: return launch_shared_t<LOGM, INV, 1, false, PCT, LE2>(a, st);
        default: return launch_shared_t<LOGM, INV, 2, false, PCT, LE2>(a, st);
    }
}

// remlast: the remainder-last schedule (tuning knob 9; the plan's Kernel-2
// table is built for it)
template <int LOGM, bool INV, class PCT>
cudaError_t launch_shared_ot(const KArgs& a, int ots, bool remlast, cudaStream_t st)
{
    if constexpr (RoundGeo<LOGM, 0, 4>::s < 16) {
        return cudaErrorNotSupported;
    } else {
        if (remlast) {
            if constexpr (RoundGeo<LOGM, 0, 4 | kRemLast>::s >= 16)
                return launch_shared_ot2<LOGM, INV, PCT, 4 | kRemLast>(a, ots, st);
            return cudaErrorNotSupported;
        }
        return launch_shared_ot2<LOGM, INV, PCT, 4>(a, ots, st);
    }
}

template <bool INV, class PCT, int... Ls>
cudaError_t shared_switch(int logm, const KArgs& a, int ots, bool remlast, cudaStream_t st,
                          std::integer_sequence<int, Ls...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((logm == Ls ? (err = launch_shared_ot<Ls, INV, PCT>(a, ots, remlast, st), 0) : 0), ...);
    return err;
}

template <int LOGM, int LOGE, bool INV, class PCT>
cudaError_t launch_blocks_ot(const KArgs& a, int ots, cudaStream_t st)
{
    if (a.mul_a) {  // fused product only in the radix-16 inverse without OT; else the caller unfuses
        if constexpr (INV && LOGE == 4) {
            if (ots == 0) return launch_blocks_t<LOGM, LOGE, INV, 0, true, PCT>(a, st);
        }
        return cudaErrorNotSupported;
    }
    switch (ots) {
        case 0: return launch_blocks_t<LOGM, LOGE, INV, 0, false, PCT>(a, st);
        case 1: return launch_blocks_t<LOGM, LOGE, INV, 1, false, PCT>(a, st);
        default: return launch_blocks_t<LOGM, LOGE, INV, 2, false, PCT>(a, st);
    }
}

template <int LOGE, bool INV, class PCT, int... Ls>
cudaError_t blocks_switch(int logm, const KArgs& a, int ots, cudaStream_t st, std::integer_sequence<int, Ls...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((logm == Ls ? (err = launch_blocks_ot<Ls, LOGE, INV, PCT>(a, ots, st), 0) : 0), ...);
    return err;
}

template <int LOGM, int LOGE, bool INV, bool FUSE0, bool TWS, class PCT>
cudaError_t launch_contig_ot(const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    if (a.mul_a) {  // fused product only in the radix-16 inverse without OT; else the caller unfuses
        if constexpr (INV && LOGE == 4) {
            if (ots == 0) return launch_contig_t<LOGM, LOGE, INV, FUSE0, 0, TWS, true, PCT>(a, iters, st);
        }
        return cudaErrorNotSupported;
    }
    switch (ots) {
        case 0: return launch_contig_t<LOGM, LOGE, INV, FUSE0, 0, TWS, false, PCT>(a, iters, st);
        case 1: return launch_contig_t<LOGM, LOGE, INV, FUSE0, 1, TWS, false, PCT>(a, iters, st);
        default: return launch_contig_t<LOGM, LOGE, INV, FUSE0, (LOGM >= 2 ? 2 : LOGM), TWS, false, PCT>(a, iters, st);
    }
}

template <int LOGE, bool INV, bool FUSE0, bool TWS, class PCT, int... Ls>
cudaError_t contig_switch(int logm, const KArgs& a, int ots, uint32_t iters, cudaStream_t st,
                          std::integer_sequence<int, Ls...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((logm == Ls ? (err = launch_contig_ot<Ls, LOGE, INV, FUSE0, TWS, PCT>(a, ots, iters, st), 0) : 0), ...);
    return err;
}

template <int LOGN1, int LOGN, int LOGE, bool INV, class PCT>
cudaError_t launch_cols_pipe_t(const KArgs& a, uint32_t rows, cudaStream_t st)
{
    using CC = ColsPipeCfg<LOGN1, LOGE>;
    auto fn = k_cols_pipe<LOGN1, LOGN, LOGE, INV, PCT>;
    static DeviceOnce once;  // value: resident CTAs per SM
    if (cudaError_t e = once.run([&](int& ctas) {
            cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CC::SMEM);
            return r != cudaSuccess ? r : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, CC::CT, CC::SMEM);
        }))
        return e;
    const int ctas_per_sm = once.value();
    const int sms = sm_count();
    const uint64_t want = (uint64_t)rows << a.log_tiles;
    const uint64_t grid = std::min<uint64_t>(want, (uint64_t)sms * std::max(1, ctas_per_sm));
    return launch_pdl(fn, dim3((unsigned)grid), dim3(CC::CT), CC::SMEM, st, a);
}

template <bool INV, class PCT, int... Ks>
cudaError_t cols_pipe_switch(int key, const KArgs& a, uint32_t rows, cudaStream_t st, std::integer_sequence<int, Ks...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((key == Ks ? (err = launch_cols_pipe_t<(Ks & 15), (Ks >> 4), 4, INV, PCT>(a, rows, st), 0) : 0), ...);
    return err;
}

// Ks encodes (logn << 4) | log_n1
template <int LOGE, bool INV, class PCT, int... Ks>
cudaError_t cols_switch(int key, const KArgs& a, uint32_t rows, cudaStream_t st, std::integer_sequence<int, Ks...>)
{
    cudaError_t err = cudaErrorInvalidValue;
    ((key == Ks ? (err = launch_cols_t<(Ks & 15), (Ks >> 4), LOGE, INV, PCT>(a, rows, st), 0) : 0), ...);
    return err;
}

}  // namespace detail

// Supported sizes: single kernel LOGM 1..13; Kernel-2 LOGM 6..11; Kernel-1 (logn, log_n1) pairs below.
using SingleSizes = std::integer_sequence<int, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13>;
using K2Sizes = std::integer_sequence<int, 6, 7, 8, 9, 10, 11>;
#define K1P(n, n1) (((n) << 4) | (n1))
using K1Pairs = std::integer_sequence<int, K1P(14, 6), K1P(14, 7), K1P(14, 8), K1P(15, 6), K1P(15, 7), K1P(15, 8),
                                      K1P(15, 9), K1P(16, 6), K1P(16, 7), K1P(16, 8), K1P(16, 9), K1P(16, 10),
                                      K1P(17, 6), K1P(17, 7), K1P(17, 8), K1P(17, 9), K1P(17, 10)>;
#undef K1P

// The three entry launchers, per prime-constant type.  The Proth type
// (PrimeConstP) is instantiated for the default kernels only -- radix-16
// Kernel-1, the pipelined radix-16 Kernel-2 and the single-CTA kernel; the
// tuning-knob variants keep the general arithmetic, which is also exact for
// Proth primes (ntt_api.cu never asks for them with proth set).
template <class PCT>
cudaError_t launch_single_t(bool inverse, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    using namespace detail;
    return inverse ? contig_switch<4, true, true, false, PCT>((int)a.logn, a, ots, iters, st, SingleSizes{})
                   : contig_switch<4, false, false, false, PCT>((int)a.logn, a, ots, iters, st, SingleSizes{});
}

template <class PCT>
cudaError_t launch_k2_t(bool inverse, int loge, const KArgs& a, int ots, uint32_t iters, cudaStream_t st)
{
    using namespace detail;
    const int logm = (int)(a.logn - a.log_n1);
    // shared-twiddle Kernel-2 (radix 16, one CTA per block position x 256/TB
    // ciphertexts) when the batch fills its CTAs (NB = 2^12 / N2 ciphertexts);
    // smaller batches (e.g. the C5 request stream, batch 1) take the persistent
    // pipelined Kernel-2, whose warps walk blocks of any row
    // (knob 9: the same kernel on the remainder-last schedule)
    // (the remainder-last schedule reads round 0 from global at stride N2/16,
    // whole segments only for N2 >= 2^8; smaller blocks take the persistent kernel)
    if ((loge == 7 || (loge == 9 && logm >= 8)) && a.batch >= (4096u >> logm))
        return inverse ? shared_switch<true, PCT>(logm, a, ots, loge == 9, st, K2Sizes{})
                       : shared_switch<false, PCT>(logm, a, ots, loge == 9, st, K2Sizes{});
    if (loge == 9)  // remainder-last table: the persistent Kernel-2 on the same schedule
        return inverse ? blocks_switch<4 | kRemLast, true, PCT>(logm, a, ots, st, K2Sizes{})
                       : blocks_switch<4 | kRemLast, false, PCT>(logm, a, ots, st, K2Sizes{});
    if (loge == 7) loge = 5;
    if (loge == 5)  // pipelined persistent Kernel-2 (radix 16)
        return inverse ? blocks_switch<4, true, PCT>(logm, a, ots, st, K2Sizes{})
                       : blocks_switch<4, false, PCT>(logm, a, ots, st, K2Sizes{});
    if constexpr (std::is_same_v<PCT, PrimeConst>) {
        if (loge == 6)  // pipelined persistent Kernel-2 (radix 8)
            return inverse ? blocks_switch<3, true, PCT>(logm, a, ots, st, K2Sizes{})
                           : blocks_switch<3, false, PCT>(logm, a, ots, st, K2Sizes{});
        if (loge == 3)
            return inverse ? contig_switch<3, true, false, true, PCT>(logm, a, ots, iters, st, K2Sizes{})
                           : contig_switch<3, false, false, true, PCT>(logm, a, ots, iters, st, K2Sizes{});
        return inverse ? contig_switch<4, true, false, true, PCT>(logm, a, ots, iters, st, K2Sizes{})
                       : contig_switch<4, false, false, true, PCT>(logm, a, ots, iters, st, K2Sizes{});
    }
    return cudaErrorNotSupported;
}

template <class PCT>
cudaError_t launch_k1_t(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    using namespace detail;
    const int key = (int)((a.logn << 4) | a.log_n1);
    if (loge == 5 && a.log_n1 <= 9)  // pipelined persistent Kernel-1 (radix 16); SMEM caps N1 at 2^9
        return inverse ? cols_pipe_switch<true, PCT>(key, a, rows, st, K1Pairs{})
                       : cols_pipe_switch<false, PCT>(key, a, rows, st, K1Pairs{});
    return inverse ? cols_switch<4, true, PCT>(key, a, rows, st, K1Pairs{})
                   : cols_switch<4, false, PCT>(key, a, rows, st, K1Pairs{});
}

}  // namespace ntt
