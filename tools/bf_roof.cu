// tools/bf_roof.cu -- register-only throughput of the kernels' own butterflies
// (ct_bf / gs_bf from ntt_device.cuh, general and Proth constants): the
// practical ALU ceiling the NTT kernels are measured against.  Each thread
// runs radix-16 rounds (4 stages x 8 butterflies) on 16 registers, no memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/libs/bf_roof tools/bf_roof.cu
// (__graft_entry__.build() does this; bench.py runs it for the live ceiling of its roofline line).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2012_01968_b200/csrc/ntt_device.cuh"

using namespace ntt;
#define ITERS 256

template <class C, bool GS>
__global__ void __launch_bounds__(256, 4) k_bf(uint64_t* out, const Tw* tw, const PrimeConst* pcp)
{
    const C c = load_pc<C>(pcp, 0);
    uint64_t x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 977u + i * 131u;
    __shared__ Tw stw[4];
    if (threadIdx.x < 4) stw[threadIdx.x] = tw[threadIdx.x];
    __syncthreads();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int st = 0; st < 4; ++st) {
            const int half = 8 >> st;
            const TwMul<false> w{stw[(st + it) & 3]};  // SMEM broadcast, as in the kernels
            // the kernels' pattern: reduce on every other stage (ct_bf red 2 Proth / 3 general)
            const int red = ((3 - st) & 1) ? 0 : (std::is_same_v<C, PrimeConstP> ? 2 : 3);
#pragma unroll
            for (int g = 0; g < 16; g += 2 * half)
#pragma unroll
                for (int k = g; k < g + half; ++k) {
                    if constexpr (GS) gs_bf(x[k], x[k + half], w, c);
                    else ct_bf(x[k], x[k + half], w, c, red);
                }
        }
        // No periodic normalisation (round 1 bounded the GS values every 16
        // stages, which put ~2 ALU ops per butterfly into the "ceiling" that the
        // kernels do not pay -- Kernel-2' then measured above it): the values
        // may leave the lazy range, which changes no instruction's cost (no
        // data-dependent branch), and the XOR below keeps the work live.
    }
    uint64_t s = 0;
    for (int i = 0; i < 16; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount, threads = 256, blocks = sms * 4;
    const uint64_t P[2] = {1152921504606584833ull /* 2^60-2^18+1 */, 1152921500311617537ull /* 2^60-2^32+1: Proth */};
    uint64_t* out;
    Tw* tw;
    PrimeConst* pc;
    cudaMalloc(&out, sizeof(uint64_t) * blocks * threads);
    cudaMalloc(&tw, 4 * sizeof(Tw));
    cudaMalloc(&pc, sizeof(PrimeConst));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int v = 0; v < 4; ++v) {
        const bool proth = v & 1, gs = v >> 1;
        const uint64_t p = P[proth];
        PrimeConst h{};
        h.p = p; h.p2 = 2 * p; h.p4 = 4 * p; h.np = 0 - p; h.p5 = 5 * p;
        h.p4_hi = (uint32_t)((4 * p) >> 32);
        h.m1 = 0u - (uint32_t)(p >> 32);
        h.p8 = 8 * p; h.p8_hi = (uint32_t)((8 * p) >> 32); h.zero = 0;
        Tw ht[4];
        for (int i = 0; i < 4; ++i) {
            const uint64_t w = (12345678901ull * (i + 3)) % p;
            ht[i] = Tw{w, (uint64_t)(((unsigned __int128)w << 64) / p)};
        }
        cudaMemcpy(tw, ht, sizeof(ht), cudaMemcpyHostToDevice);
        cudaMemcpy(pc, &h, sizeof(h), cudaMemcpyHostToDevice);
        auto run = [&]() {
            if (v == 0) k_bf<PrimeConst, false><<<blocks, threads>>>(out, tw, pc);
            if (v == 1) k_bf<PrimeConstP, false><<<blocks, threads>>>(out, tw, pc);
            if (v == 2) k_bf<PrimeConst, true><<<blocks, threads>>>(out, tw, pc);
            if (v == 3) k_bf<PrimeConstP, true><<<blocks, threads>>>(out, tw, pc);
        };
        for (int r = 0; r < 3; ++r) run();
        cudaEventRecord(e0);
        run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bf = (double)blocks * threads * ITERS * 32;
        printf("{\"butterfly\": \"%s\", \"primes\": \"%s\", \"warps_per_sm\": 32, \"Gbutterfly_s\": %.1f, \"err\": \"%s\"}\n",
               gs ? "gs" : "ct", proth ? "proth" : "2n", bf / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
