// tools/bf_r3.cu -- experiment: register-only CT / GS butterfly rate with a
// Shoup multiply specialised to the R3 chain's primes p = 2^60 - d, d < 2^32
// (every prime of the SURVEY 8(c) chain at N <= 2^17): 2^64 - p = 0xF0000000:d,
// so q0 * n1 = -(q0 << 28) (mod 2^32) -- a shift and a subtraction on the ALU
// pipe instead of one IMAD.  Same truncated quotient and the same r as
// shoup_lazy word for word (checked: the two runs' outputs are compared).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/libs/bf_r3 tools/bf_r3.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2012_01968_b200/csrc/ntt_device.cuh"

namespace ntt {
struct PrimeConstR : PrimeConst {
};
__device__ __forceinline__ uint64_t shoup_lazy_r3(uint64_t b, uint64_t w, uint64_t wb, uint32_t d, uint32_t z)
{
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 b0, b1, v0, v1, w0, w1, t0, t1, q0, q1, r0, r1, s;\n\t"
        ".reg .u64 q, a, t;\n\t"
        "mov.b64 {b0, b1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {v0, v1}, %3;\n\t"
        "mul.hi.u32 t0, b1, v0;\n\t"
        "mul.hi.u32 t1, b0, v1;\n\t"
        "cvt.u64.u32 t, t0;\n\t"
        "mad.wide.u32 q, b1, v1, t;\n\t"
        "cvt.u64.u32 t, t1;\n\t"
        "add.u64 q, q, t;\n\t"
        "mov.b64 {q0, q1}, q;\n\t"
        "mul.wide.u32 a, b0, w0;\n\t"
        "mad.wide.u32 a, q0, %4, a;\n\t"
        "mov.b64 {r0, r1}, a;\n\t"
        "mad.lo.u32 r1, b0, w1, r1;\n\t"
        "mad.lo.u32 r1, b1, w0, r1;\n\t"
        "mad.lo.u32 r1, q1, %4, r1;\n\t"
        "shf.l.clamp.b32 s, %5, q0, 28;\n\t"
        "sub.u32 r1, r1, s;\n\t"
        "add.u32 r1, r1, %5;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(b), "l"(w), "l"(wb), "r"(d), "r"(z));
    return r;
}
__device__ __forceinline__ uint64_t shoup(uint64_t b, const Tw& t, const PrimeConstR& c)
{
    return shoup_lazy_r3(b, t.w, t.wb, (uint32_t)c.np, (uint32_t)c.zero);  // z: an opaque 0 (the funnel's low word) keeps the shift off IMAD
}
}  // namespace ntt

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
            const TwMul<false> w{stw[(st + it) & 3]};
            const int red = ((3 - st) & 1) ? 0 : 3;
#pragma unroll
            for (int g = 0; g < 16; g += 2 * half)
#pragma unroll
                for (int k = g; k < g + half; ++k) {
                    if constexpr (GS) gs_bf(x[k], x[k + half], w, c);
                    else ct_bf(x[k], x[k + half], w, c, red);
                }
        }
    }
    uint64_t s = 0;
    for (int i = 0; i < 16; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount, threads = 256, blocks = sms * 4, n = blocks * threads;
    const uint64_t p = 1152921504606584833ull;  // 2^60 - 2^18 + 1: the chain's first prime at N = 2^17
    uint64_t* out[4];
    for (auto& o : out) cudaMalloc(&o, 8ull * n);
    Tw* tw;
    PrimeConst* pc;
    cudaMalloc(&tw, 4 * sizeof(Tw));
    cudaMalloc(&pc, sizeof(PrimeConst));
    PrimeConst h{};
    h.p = p; h.p2 = 2 * p; h.p4 = 4 * p; h.np = 0 - p; h.p5 = 5 * p;
    h.p4_hi = (uint32_t)((4 * p) >> 32); h.m1 = 0u - (uint32_t)(p >> 32);
    h.p8 = 8 * p; h.p8_hi = (uint32_t)((8 * p) >> 32); h.zero = 0;
    Tw ht[4];
    for (int i = 0; i < 4; ++i) {
        const uint64_t w = (12345678901ull * (i + 3)) % p;
        ht[i] = Tw{w, (uint64_t)(((unsigned __int128)w << 64) / p)};
    }
    cudaMemcpy(tw, ht, sizeof(ht), cudaMemcpyHostToDevice);
    cudaMemcpy(pc, &h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"ct 2n", "ct r3", "gs 2n", "gs r3"};
    for (int rep = 0; rep < 2; ++rep)
        for (int v = 0; v < 4; ++v) {
            auto run = [&]() {
                if (v == 0) k_bf<PrimeConst, false><<<blocks, threads>>>(out[0], tw, pc);
                if (v == 1) k_bf<PrimeConstR, false><<<blocks, threads>>>(out[1], tw, pc);
                if (v == 2) k_bf<PrimeConst, true><<<blocks, threads>>>(out[2], tw, pc);
                if (v == 3) k_bf<PrimeConstR, true><<<blocks, threads>>>(out[3], tw, pc);
            };
            for (int r = 0; r < 3; ++r) run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"butterfly\": \"%s\", \"Gbutterfly_s\": %.1f, \"err\": \"%s\"}\n", names[v],
                   (double)n * ITERS * 32 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    std::vector<uint64_t> a(n), b(n);
    for (int k = 0; k < 2; ++k) {
        cudaMemcpy(a.data(), out[2 * k], 8ull * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), out[2 * k + 1], 8ull * n, cudaMemcpyDeviceToHost);
        printf("{\"check\": \"%s r3 == 2n\", \"equal\": %s}\n", k ? "gs" : "ct", a == b ? "true" : "false");
    }
    return 0;
}
