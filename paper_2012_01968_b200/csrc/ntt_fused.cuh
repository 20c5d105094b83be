// ntt_fused.cuh -- single-pass NTT / iNTT of one row per thread-block cluster
// (SURVEY 8(f) NEXT-1).  The paper's two-kernel split exists
// because one SM's shared memory cannot hold a row ("at least two loads from
// GMEM are required"); on B200 a cluster of C = N / 2^13 CTAs holds the whole
// row in distributed shared memory (64 KiB per CTA), so every word crosses HBM
// once per direction instead of twice:
//
//   forward:  column phase -- each thread loads 16/C columns j (C words at
//             stride 2^13, coalesced across the warp) and runs the first
//             log C Cooley-Tukey stages in registers (Kernel-1 with N1 = C;
//             twiddles Psi[1..C), shared by every column); scatter -- word
//             (j, k) is stored into CTA k's shared memory at position j over
//             DSMEM (st.shared::cluster); one cluster barrier; block phase --
//             CTA k runs the remaining 13 stages on block k exactly like
//             Kernel-2 (radix-16 rounds through its own SMEM, twiddles from
//             the Kernel-2-ordered table through L1/L2), normalises and
//             stores the block with 128-bit coalesced stores.
//   inverse:  the mirror image -- block phase (13 Gentleman-Sande stages),
//             cluster barrier, each thread gathers its columns from the C
//             CTAs (ld.shared::cluster), the last log C GS stages with N^-1
//             fused (R15) in registers, normalise, store; a split cluster
//             barrier keeps every CTA's SMEM alive until its peers have read it.
//
// 512 threads per CTA (16 words each), 2 CTAs per SM: one computes while the
// other waits on HBM.  N = 2^14..2^17 -> C = 2..16 (16 needs the non-portable
// cluster size).
#pragma once
#include "ntt_device.cuh"
#include "ntt_launch.h"

namespace ntt {

__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `p` (a pointer into this CTA's SMEM) in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank)
{
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(s), "r"(rank));
    return d;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, uint64_t v)
{
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_cluster(uint32_t addr)
{
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
// arrive without memory ordering (no MEMBAR): for "I have started" and for
// "my remote loads are done" placed after their values have been consumed
__device__ __forceinline__ void cluster_arrive_relaxed()
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

struct FusedCfg {
    static constexpr int LOGM = 13;            // words per CTA: 2^13 (64 KiB)
    static constexpr int CT = 512;             // threads per CTA, 16 words each
    static constexpr size_t SMEM = ((size_t)8 << LOGM) + 16 * sizeof(Tw);  // block + Psi[0..C) (C <= 16)
};

template <int LOGC, bool INV, class PCT>
__global__ void __launch_bounds__(FusedCfg::CT, 2) k_fused(const KArgs a)
{
    constexpr int LOGM = FusedCfg::LOGM, M = 1 << LOGM, C = 1 << LOGC, CT = FusedCfg::CT;
    constexpr int NI = 16 / C;  // columns per thread
    using SC = Sched<LOGM, 4>;
    static_assert(SC::TB == CT, "one block per CTA");
    constexpr int NR = SC::NR;
    constexpr int NOOT = 1 << 20;
    extern __shared__ __align__(16) uint64_t sm[];
    pdl_trigger();
    pdl_wait();

    const uint32_t tid = threadIdx.x;
    const uint32_t k = cluster_rank();       // block of the row this CTA owns
    const uint32_t q = blockIdx.x >> LOGC;   // row, prime-major: q = l * batch + b
    const uint32_t l = q / a.batch, b = q - l * a.batch;
    uint64_t* g = a.data + (((uint64_t)b * a.L + l) << (LOGM + LOGC));
    const Tw* tab = a.tab + ((uint64_t)l << (LOGM + LOGC));
    const Tw* tb2 = a.tab2 + ((uint64_t)l << (LOGM + LOGC)) + ((uint64_t)k << LOGM);
    const PCT pc = load_pc<PCT>(a.pc, l);
    const uint32_t Fm1 = C + k - 1;  // block k of the split N = C x 2^13: F = C + k

    // column phase twiddles Psi[1..C): every column of every CTA uses them; staged
    // in SMEM behind the block (loading them from global inside the round let
    // ptxas hoist all C-1 pairs into registers and spill)
    Tw* const twc = reinterpret_cast<Tw*>(sm + M);
    if (tid < (uint32_t)C) twc[tid] = ldg_tw(tab + tid);
    __syncthreads();
    auto tabc = [&](const TwKey& t) { return twc[t.idx]; };
    // block phase twiddles: Kernel-2 order (K2Layout), contiguous across the lanes of a warp
    auto tab2f = [&](const TwKey& t) {
        return ldg_tw(tb2 + K2Layout<LOGM, 4>::round_off(t.S) + ((((1u << t.i) - 1u + t.h) << t.S) + t.g));
    };
    auto otf = [&](uint32_t) { return TwMul<true>{}; };

    // columns of this CTA: j_u = k M / C + u CT + tid (coalesced across the warp)
    auto col = [&](int u) { return (k << (LOGM - LOGC)) + (uint32_t)u * CT + tid; };

    uint64_t x[16];
    auto s_load = [&](auto ri) {
        using Geo = RoundGeo<LOGM, decltype(ri)::value, 4>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
#pragma unroll
                for (int kk = 0; kk < Geo::R; kk += 2) {
                    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + swz(Geo::elem(qd * CT + tid, kk)));
                    x[qd * Geo::R + kk] = v.x;
                    x[qd * Geo::R + kk + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < Geo::R; ++kk) x[qd * Geo::R + kk] = sm[swz(Geo::elem(qd * CT + tid, kk))];
            }
        }
    };
    auto s_store = [&](auto ri) {
        using Geo = RoundGeo<LOGM, decltype(ri)::value, 4>;
#pragma unroll
        for (int qd = 0; qd < Geo::GPT; ++qd) {
            if constexpr (Geo::s == 1 && Geo::R >= 2) {
#pragma unroll
                for (int kk = 0; kk < Geo::R; kk += 2)
                    *reinterpret_cast<ulonglong2*>(sm + swz(Geo::elem(qd * CT + tid, kk))) =
                        make_ulonglong2(x[qd * Geo::R + kk], x[qd * Geo::R + kk + 1]);
            } else {
#pragma unroll
                for (int kk = 0; kk < Geo::R; ++kk) sm[swz(Geo::elem(qd * CT + tid, kk))] = x[qd * Geo::R + kk];
            }
        }
    };
    uint64_t* gb = g + ((uint64_t)k << LOGM);  // this CTA's block

    if constexpr (!INV) {
        cluster_arrive_relaxed();  // this CTA is running (DSMEM targets must have started)
        // ---- column phase: global stages 0 .. LOGC-1
        uint64_t xc[NI][16];
#pragma unroll
        for (int u = 0; u < NI; ++u)
#pragma unroll
            for (int kk = 0; kk < C; ++kk) xc[u][kk] = g[col(u) + ((uint64_t)kk << LOGM)];
        ct_roundN<LOGC, LOGC, 0, NOOT, NI, true>(xc, 0u, 0u, tabc, otf, pc);
        cluster_wait();
        // ---- scatter: word (j, kk) -> CTA kk, position j
#pragma unroll
        for (int kk = 0; kk < C; ++kk) {
            const uint32_t base = map_rank(sm, (uint32_t)kk);
#pragma unroll
            for (int u = 0; u < NI; ++u) st_cluster(base + 8u * swz(col(u)), xc[u][kk]);
        }
        cluster_arrive();
        cluster_wait();
        // ---- block phase: global stages LOGC .. LOGC+12 on block k
        static_for<NR>([&](auto ri) {
            constexpr int RI = decltype(ri)::value;
            s_load(ri);
            ct_round<LOGM, 4, RI, NOOT, false, true>(x, tid, Fm1, tab2f, otf, pc);
            if constexpr (RI == NR - 1) {
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) x[kk] = norm8(x[kk], pc);  // any word -> [0,p)
            }
            s_store(ri);
            __syncthreads();
        });
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t ch = j * CT + tid;
            *reinterpret_cast<ulonglong2*>(gb + 2 * ch) = *reinterpret_cast<const ulonglong2*>(sm + swz(2 * ch));
        }
    } else {
        // ---- block phase: global GS stages LOGC+12 .. LOGC on block k
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t ch = j * CT + tid;
            *reinterpret_cast<ulonglong2*>(sm + swz(2 * ch)) = *reinterpret_cast<const ulonglong2*>(gb + 2 * ch);
        }
        __syncthreads();
        static_for<NR>([&](auto rj) {
            constexpr int RI = NR - 1 - decltype(rj)::value;
            using RC = std::integral_constant<int, RI>;
            s_load(RC{});
            gs_round<LOGM, 4, RI, NOOT, false>(x, tid, Fm1, tab2f, otf, pc);
            s_store(RC{});
            if constexpr (RI != 0) __syncthreads();
        });
        cluster_arrive();  // every block's SMEM image is complete and visible
        cluster_wait();
        // ---- gather: column j from the C blocks
        uint64_t xc[NI][16];
#pragma unroll
        for (int kk = 0; kk < C; ++kk) {
            const uint32_t base = map_rank(sm, (uint32_t)kk);
#pragma unroll
            for (int u = 0; u < NI; ++u) xc[u][kk] = ld_cluster(base + 8u * swz(col(u)));
        }
        // ---- column phase: global GS stages LOGC-1 .. 0, N^-1 fused (R15)
        gs_roundN<LOGC, LOGC, 0, NOOT, true, NI>(xc, 0u, 0u, tabc, otf, pc);
        // every remote load has been consumed above: peers may exit after their wait
        cluster_arrive_relaxed();
#pragma unroll
        for (int u = 0; u < NI; ++u)
#pragma unroll
            for (int kk = 0; kk < C; ++kk) g[col(u) + ((uint64_t)kk << LOGM)] = norm4(xc[u][kk], pc);
        cluster_wait();  // keep this CTA's SMEM alive until every peer has read it
    }
}

template <int LOGC, bool INV, class PCT>
cudaError_t launch_fused_t(const KArgs& a, uint32_t rows, cudaStream_t st)
{
    auto fn = k_fused<LOGC, INV, PCT>;
    static DeviceOnce once;
    if (cudaError_t e = once.run([&](int&) {
            cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FusedCfg::SMEM);
            if (r == cudaSuccess && (1 << LOGC) > 8)
                r = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            return r;
        }))
        return e;
    cudaLaunchAttribute cl;
    cl.id = cudaLaunchAttributeClusterDimension;
    cl.val.clusterDim.x = 1u << LOGC;
    cl.val.clusterDim.y = 1;
    cl.val.clusterDim.z = 1;
    return launch_pdl(fn, dim3(rows << LOGC), dim3(FusedCfg::CT), FusedCfg::SMEM, st, a, &cl);
}

template <class PCT>
cudaError_t launch_fused_all(bool inverse, const KArgs& a, uint32_t rows, cudaStream_t st)
{
    switch (a.logn) {
        case 14: return inverse ? launch_fused_t<1, true, PCT>(a, rows, st) : launch_fused_t<1, false, PCT>(a, rows, st);
        case 15: return inverse ? launch_fused_t<2, true, PCT>(a, rows, st) : launch_fused_t<2, false, PCT>(a, rows, st);
        case 16: return inverse ? launch_fused_t<3, true, PCT>(a, rows, st) : launch_fused_t<3, false, PCT>(a, rows, st);
        case 17: return inverse ? launch_fused_t<4, true, PCT>(a, rows, st) : launch_fused_t<4, false, PCT>(a, rows, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ntt
