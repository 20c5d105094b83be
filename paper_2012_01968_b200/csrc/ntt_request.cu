// ntt_request.cu -- the single-launch request kernel (k_req): the forward
// and / or inverse transform of a small job -- BASELINE config 5's requests,
// one ciphertext of a few primes at N = 2^14..2^17 -- in ONE launch, captured
// by ntt_graph_create(..., NTT_GRAPH_ONE_KERNEL).
//
// Why: a request through the two-kernel split is four
// dependent kernels (Kernel-1, Kernel-2, Kernel-2', Kernel-1'), and on B200
// four dependent launches cost ~10 us before any work, while the transforms
// of one ciphertext at L = 1 are ~1 us of arithmetic each.  Here the passes of
// the split N = N1 N2 run as phases of one persistent grid:
//
//   C  (Kernel-1):  CT stages m = 1 .. N1/2 on the stride-N2 columns
//   -- grid barrier (every block needs every column) --
//   B  (Kernel-2):  CT stages m = N1 .. N/2 on the contiguous N2-blocks,
//                   final normalisation, bit-reversed output
//   B' (Kernel-2'): GS stages of the blocks (R5), continuing in registers from
//                   the words B just stored (same thread, same positions)
//   -- grid barrier --
//   C' (Kernel-1'): GS stages of the columns, N^-1 fused (R15), canonical output
//
// Latency-shaped rather than throughput-shaped: per-thread radix 4 (LOGE = 2)
// and 128-thread CTAs, so one ciphertext at N = 2^16 spreads over 128 SMs (the
// throughput Kernel-1 has 16 column tiles per row); a unit's twiddles are
// loaded straight into registers together with its data, in the order the
// rounds consume them, so each phase pays one L2 round trip; data loads bypass
// L1 (ld.global.cg) because other CTAs wrote the words in the previous phase.
// Arithmetic, butterflies, lazy bounds and twiddle algebra are the throughput
// kernels' (ntt_device.cuh), so the results are identical word for word.
// Citations: P:n = /root/reference/PAPER.md line n; R# = DESIGN.md section 3.
#include "ntt_kernels.cuh"

// NTT_REQ_TRACE (experiment builds only, tools/req_trace.py): thread 0 of
// every CTA records %globaltimer at the phase boundaries of the last launch
#ifdef NTT_REQ_TRACE
__device__ unsigned long long g_req_trace[1024][16];
#define REQ_MARK(i)                                                                                   \
    do {                                                                                              \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                                  \
            unsigned long long t_;                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
            g_req_trace[blockIdx.x][i] = t_;                                                          \
        }                                                                                             \
    } while (0)
extern "C" int ntt_debug_req_trace(unsigned long long* out)
{
    return (int)cudaMemcpyFromSymbol(out, g_req_trace, sizeof(g_req_trace));
}
#else
#define REQ_MARK(i) \
    do {            \
    } while (0)
#endif

// threads per CTA (tuning constant): 128 spreads one ciphertext at N = 2^16
// over 128 SMs
#ifndef NTT_REQ_CT
#define NTT_REQ_CT 128
#endif

namespace ntt {

template <int LOGN1, int LOGN2, int LOGE>
struct ReqCfg {
    static constexpr int CT = NTT_REQ_CT;
    static constexpr int N1 = 1 << LOGN1, N2 = 1 << LOGN2, E = 1 << LOGE;
    static constexpr int TBC = N1 / E;    // threads per column
    static constexpr int TC = CT / TBC;   // columns per column unit
    static constexpr int TBB = N2 / E;    // threads per block
    static constexpr int NBK = CT / TBB;  // blocks per block unit
    static_assert(TC >= 1 && NBK >= 1 && N2 % TC == 0 && N1 % NBK == 0, "request geometry");
    static constexpr int DATA = CT * E;  // SMEM words: N1 x TC (columns) = NBK x N2 (blocks)
};

// Grid barrier over all CTAs of the launch (all co-resident, see
// launch_req_t).  One monotonically increasing 64-bit arrival counter per
// request object, zeroed once when it is created: at barrier round r every
// CTA's atomic add returns a value in [r G, (r + 1) G), so each waits for
// count >= (r + 1) G -- no reset, no second variable; no CTA can arrive for
// round r + 1 before round r is complete, and the launches of one request
// object are ordered on its stream with the same grid size G.  Thread 0's
// release add (after bar.sync) publishes the CTA's writes, its acquire polls
// (before bar.sync) the other CTAs'.  A barrier that has not opened after
// ~2^32 cycles traps instead of hanging.  (Measured alternatives, DESIGN.md
// 5.6: 8 counters on separate L2 slices polled by 8 threads, fences around
// relaxed operations, and one flag per CTA written with st.release and polled
// by one thread per flag -- no atomics, but G x G acquire loads on hot lines:
// 2.9-3.4 us per barrier -- were all slower.)
__device__ __forceinline__ void grid_barrier(unsigned long long* cnt, unsigned G)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long old, cur;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
        const unsigned long long target = (old / G + 1) * G;
        const long long t0 = clock64();
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(cnt) : "memory");
            if (clock64() - t0 > (1ll << 32)) __trap();
        } while (cur < target);
    }
    __syncthreads();
}

__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p)
{
    return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}

// The twiddles of one sub-transform's rounds, loaded into registers in the
// order ct_round / gs_round request them (one per (round, group, stage, h);
// OT never applies here), so the loads are issued together with the data's
// and the rounds read registers.  Global index of a local key: idx + (Fm1 << j)
// (Fm1 = 0 for columns, N1 + bb - 1 for block bb; ntt_device.cuh RoundGeo).
template <int LOGM, int LOGE>
struct TwQueue {
    using SC = Sched<LOGM, LOGE>;
    static constexpr int count()
    {
        int n = 0;
        for (int ri = 0; ri < SC::NR; ++ri) n += (SC::E >> SC::r(ri)) * ((1 << SC::r(ri)) - 1);
        return n;
    }
    static constexpr int NQ = count();
    Tw t[NQ];
    int n = 0;
    // forward order: rounds ascending, stages ascending; inverse: rounds and
    // stages descending, minus the fused first stage (FUSE0) whose twiddle is
    // the constant N^-1 Psi^-1[1]
    template <bool INV, bool FUSE0>
    __device__ __forceinline__ void load(const Tw* tab, uint32_t tib, uint32_t Fm1)
    {
        int k = 0;
        static_for<SC::NR>([&](auto rc) {
            constexpr int RI = INV ? SC::NR - 1 - decltype(rc)::value : decltype(rc)::value;
            using Geo = RoundGeo<LOGM, RI, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd) {
                const uint32_t B = (1u << Geo::S) + (qd * Geo::TB + tib) / Geo::s;
#pragma unroll
                for (int ii = 0; ii < Geo::r; ++ii) {
                    const int i = INV ? Geo::r - 1 - ii : ii;
                    if (FUSE0 && Geo::S + i == 0) continue;
#pragma unroll
                    for (int h = 0; h < (1 << i); ++h)
                        t[k++] = ldg_tw(tab + (B << i) + h + ((uint64_t)Fm1 << (Geo::S + i)));
                }
            }
        });
    }
    __device__ __forceinline__ Tw next() { return t[n++]; }
};

template <int LOGN1, int LOGN2, int LOGE, class PCT>
__global__ void __launch_bounds__(NTT_REQ_CT, 512 / NTT_REQ_CT) k_req(const ReqArgs a)
{
    using CC = ReqCfg<LOGN1, LOGN2, LOGE>;
    using SCC = Sched<LOGN1, LOGE>;
    using SCB = Sched<LOGN2, LOGE>;
    constexpr int N1 = CC::N1, N2 = CC::N2, TC = CC::TC, TBB = CC::TBB, NBK = CC::NBK;
    constexpr int LOGN = LOGN1 + LOGN2;
    __shared__ __align__(16) uint64_t smd[CC::DATA];

    const uint32_t tid = threadIdx.x;
    const uint32_t units_c = a.rows * (uint32_t)(N2 / TC);
    const uint32_t units_b = a.rows * (uint32_t)(N1 / NBK);
    auto otf = [&](uint32_t) { return TwMul<true>{}; };  // no OT on this path

    // ---- column phase (Kernel-1 / Kernel-1'), unit u = (row, tile of TC columns)
    auto cols = [&](uint32_t u, auto inv_c) {
        constexpr bool INV = decltype(inv_c)::value;
        constexpr int NR = SCC::NR;
        const uint32_t q = u / (uint32_t)(N2 / TC), tile = u % (uint32_t)(N2 / TC), l = q % a.L;
        const uint32_t c = tid % TC, tib = tid / TC;
        uint64_t* col = a.data + ((uint64_t)q << LOGN) + tile * TC + c;
        uint64_t x[16];
        auto g_load = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k)
                    x[qd * Geo::R + k] = ld_cg(col + ((uint64_t)Geo::elem(qd * SCC::TB + tib, k) << LOGN2));
        };
        auto g_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k)
                    col[(uint64_t)Geo::elem(qd * SCC::TB + tib, k) << LOGN2] = x[qd * Geo::R + k];
        };
        auto s_load = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = smd[Geo::elem(qd * SCC::TB + tib, k) * TC + c];
        };
        auto s_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN1, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) smd[Geo::elem(qd * SCC::TB + tib, k) * TC + c] = x[qd * Geo::R + k];
        };
        TwQueue<LOGN1, LOGE> tq;
        auto tabf = [&](const TwKey&) { return tq.next(); };
        g_load(std::integral_constant<int, INV ? NR - 1 : 0>{});
        tq.template load<INV, INV>((INV ? a.ti : a.tf) + ((uint64_t)l << LOGN), tib, 0u);  // Psi[1..N1)
        const PCT pc = load_pc<PCT>(a.pc, l);
        __syncthreads();  // the previous unit's SMEM reads are done
        REQ_MARK(INV ? 12 : 6);
        if constexpr (!INV) {
            static_for<NR>([&](auto ri) {
                constexpr int RI = decltype(ri)::value;
                if constexpr (RI > 0) s_load(ri);
                ct_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
                if constexpr (RI == NR - 1) {
                    g_store(ri);  // lazy: Kernel-2 continues the chain
                } else {
                    s_store(ri);
                    __syncthreads();
                }
            });
        } else {
            static_for<NR>([&](auto rj) {
                constexpr int RI = NR - 1 - decltype(rj)::value;
                using RC = std::integral_constant<int, RI>;
                if constexpr (RI < NR - 1) s_load(RC{});
                gs_round<LOGN1, LOGE, RI, 1 << 20, true>(x, tib, 0u, tabf, otf, pc);
                if constexpr (RI == 0) {
#pragma unroll
                    for (int k = 0; k < SCC::E; ++k) x[k] = norm4(x[k], pc);  // canonical [0, p)
                    g_store(RC{});
                } else {
                    s_store(RC{});
                    __syncthreads();
                }
            });
        }
    };

    // ---- block phase (Kernel-2 / Kernel-2'), unit v = (row, NBK consecutive
    // blocks).  FWD and INV both: the inverse continues from the registers of
    // the forward's last round -- the words it just stored, at the positions
    // the inverse's first round reads -- so the forward output is written
    // once and not read back.
    auto blocks = [&](uint32_t v, auto fwd_c, auto inv_c) {
        constexpr bool FWD = decltype(fwd_c)::value, INV = decltype(inv_c)::value;
        constexpr int NR = SCB::NR;
        const uint32_t blk = tid / TBB, tib = tid % TBB;
        const uint32_t q = v / (uint32_t)(N1 / NBK), bb = (v % (uint32_t)(N1 / NBK)) * NBK + blk, l = q % a.L;
        uint64_t* g = a.data + ((uint64_t)q << LOGN) + ((uint64_t)bb << LOGN2);
        uint64_t* sb = smd + blk * N2;
        const uint32_t Fm1 = (uint32_t)N1 + bb - 1u;  // block bb: F = N1 + bb
        uint64_t x[16];
        auto s_load = [&](auto ri) {
            using Geo = RoundGeo<LOGN2, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = sb[Geo::elem(qd * TBB + tib, k)];
        };
        auto s_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN2, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) sb[Geo::elem(qd * TBB + tib, k)] = x[qd * Geo::R + k];
        };
        auto g_load = [&](auto ri) {
            using Geo = RoundGeo<LOGN2, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) x[qd * Geo::R + k] = ld_cg(g + Geo::elem(qd * TBB + tib, k));
        };
        auto g_store = [&](auto ri) {
            using Geo = RoundGeo<LOGN2, decltype(ri)::value, LOGE>;
#pragma unroll
            for (int qd = 0; qd < Geo::GPT; ++qd)
#pragma unroll
                for (int k = 0; k < Geo::R; ++k) g[Geo::elem(qd * TBB + tib, k)] = x[qd * Geo::R + k];
        };
        TwQueue<LOGN2, LOGE> tqf, tqi;
        auto tabf_f = [&](const TwKey&) { return tqf.next(); };
        auto tabf_i = [&](const TwKey&) { return tqi.next(); };
        g_load(std::integral_constant<int, FWD ? 0 : NR - 1>{});
        if constexpr (FWD) tqf.template load<false, false>(a.tf + ((uint64_t)l << LOGN), tib, Fm1);
        if constexpr (INV) tqi.template load<true, false>(a.ti + ((uint64_t)l << LOGN), tib, Fm1);
        const PCT pc = load_pc<PCT>(a.pc, l);
        __syncthreads();  // the previous unit's SMEM reads are done
        REQ_MARK(8);
        if constexpr (FWD) {
            static_for<NR>([&](auto ri) {
                constexpr int RI = decltype(ri)::value;
                if constexpr (RI > 0) s_load(ri);
                ct_round<LOGN2, LOGE, RI, 1 << 20, false, true>(x, tib, 0u, tabf_f, otf, pc);
                if constexpr (RI == NR - 1) {
#pragma unroll
                    for (int k = 0; k < SCB::E; ++k) x[k] = norm8(x[k], pc);  // -> [0, p)
                    g_store(ri);
                } else {
                    s_store(ri);
                    __syncthreads();
                }
            });
            REQ_MARK(9);
            if constexpr (INV) __syncthreads();  // the last round's SMEM reads before the inverse's writes
        }
        if constexpr (INV) {
            static_for<NR>([&](auto rj) {
                constexpr int RI = NR - 1 - decltype(rj)::value;
                using RC = std::integral_constant<int, RI>;
                if constexpr (RI < NR - 1) s_load(RC{});
                gs_round<LOGN2, LOGE, RI, 1 << 20, false>(x, tib, 0u, tabf_i, otf, pc);
                if constexpr (RI == 0) {
                    g_store(RC{});  // lazy: Kernel-1' continues the chain
                } else {
                    s_store(RC{});
                    __syncthreads();
                }
            });
        }
    };

    const uint32_t G = gridDim.x;
    const bool fwd = a.flags & 1u, inv = a.flags & 2u;
    REQ_MARK(0);
    if (fwd) {
        for (uint32_t u = blockIdx.x; u < units_c; u += G) cols(u, std::false_type{});
        REQ_MARK(1);
        grid_barrier(a.bar, G);
        REQ_MARK(2);
    }
    if (fwd && inv) {
        for (uint32_t v = blockIdx.x; v < units_b; v += G) blocks(v, std::true_type{}, std::true_type{});
    } else if (fwd) {
        for (uint32_t v = blockIdx.x; v < units_b; v += G) blocks(v, std::true_type{}, std::false_type{});
    } else {
        for (uint32_t v = blockIdx.x; v < units_b; v += G) blocks(v, std::false_type{}, std::true_type{});
    }
    REQ_MARK(3);
    if (inv) {
        grid_barrier(a.bar, G);
        REQ_MARK(4);
        for (uint32_t u = blockIdx.x; u < units_c; u += G) cols(u, std::true_type{});
        REQ_MARK(5);
    }
}

namespace {

// The grid's CTAs must all be resident (grid barriers).  The grid is capped at
// the device's co-resident capacity.  A grid of at most one CTA per SM is
// launched plainly: every SM holds >= 4 of these CTAs, so it is resident even
// beside three more such requests on other streams, and the cooperative
// launch attribute measured 1.6 us of extra launch latency;
// larger grids use the cooperative launch, whose co-residency the driver
// guarantees.
template <int LOGN1, int LOGN2, class PCT>
cudaError_t launch_req_t(const ReqArgs& a, cudaStream_t st)
{
    using CC = ReqCfg<LOGN1, LOGN2, 2>;
    auto fn = k_req<LOGN1, LOGN2, 2, PCT>;
    static DeviceOnce once;  // value: co-resident CTAs per SM
    if (cudaError_t e = once.run([&](int& ctas) { return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, CC::CT, 0); }))
        return e;
    const uint64_t units =
        std::max<uint64_t>((uint64_t)a.rows * (CC::N2 / CC::TC), (uint64_t)a.rows * (CC::N1 / CC::NBK));
    const uint64_t sms = (uint64_t)detail::sm_count();
    const unsigned grid = (unsigned)std::min(units, sms * std::max(1, once.value()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(CC::CT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = grid > sms ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    return e != cudaSuccess ? (cudaGetLastError(), e) : launch_status();
}

template <class PCT>
cudaError_t launch_req_p(unsigned logn, const ReqArgs& a, cudaStream_t st)
{
    switch (logn) {
        case 14: return launch_req_t<7, 7, PCT>(a, st);
        case 15: return launch_req_t<7, 8, PCT>(a, st);
        case 16: return launch_req_t<8, 8, PCT>(a, st);
        case 17: return launch_req_t<8, 9, PCT>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_request(unsigned logn, const ReqArgs& a, cudaStream_t st, int arith)
{
    return arith == kArithProth ? launch_req_p<PrimeConstP>(logn, a, st) : launch_req_p<PrimeConst>(logn, a, st);
}

}  // namespace ntt
