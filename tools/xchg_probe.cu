// tools/xchg_probe.cu -- the between-round exchange of the radix-16 rounds
// (16 lanes x 16 64-bit words, an all-to-all / 16x16 transpose within each
// half-warp) done two ways, register-resident, no global memory in the loop:
//   smem : each lane stores its 16 words to a padded (16 x 17, bank-conflict
//          free) SMEM image and reads the transposed 16 back (the kernels'
//          exchange pattern, ntt_kernels.cuh, with their swizzle replaced by
//          padding for this transpose);
//   shfl : the same transpose as a 4-step xor-butterfly network of warp
//          shuffles (north_star's "warp-shuffle butterflies" alternative):
//          per step 8 word pairs, each 2 SHFL (32-bit halves) + 6 SEL.
// Reports exchanges per second per SM and clk per warp-exchange.  DESIGN.md 9.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/libs/xchg_probe tools/xchg_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 512

__global__ void __launch_bounds__(256, 4) k_smem(uint64_t* out)
{
    __shared__ uint64_t sm[16 * 272];  // per half-warp a 16 x 17 padded image: conflict-free both ways
    const uint32_t lane = threadIdx.x & 15u, grp = threadIdx.x >> 4;
    uint64_t* s = sm + grp * 272;
    uint64_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = threadIdx.x * 977u + k;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) s[lane * 17 + k] = w[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = s[k * 17 + lane] + (uint64_t)it;
        __syncwarp();
    }
    uint64_t r = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) r ^= w[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int d)
{
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, d);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), d);
    return ((uint64_t)hi << 32) | lo;
}

__global__ void __launch_bounds__(256, 4) k_shfl(uint64_t* out)
{
    const uint32_t lane = threadIdx.x & 15u;
    uint64_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = threadIdx.x * 977u + k;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 3; j >= 0; --j) {
            const int d = 1 << j;
            const bool hiL = (lane >> j) & 1u;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k & d) continue;
                const uint64_t send = hiL ? w[k] : w[k | d];
                const uint64_t recv = shfl_xor64(send, d);
                if (hiL) w[k] = recv;
                else w[k | d] = recv;
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] += (uint64_t)it;
    }
    uint64_t r = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) r ^= w[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// host check that both loops compute the same transpose
int main()
{
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount, threads = 256, blocks = sms * 4;
    uint64_t *o1, *o2;
    cudaMalloc(&o1, 8ull * blocks * threads);
    cudaMalloc(&o2, 8ull * blocks * threads);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms[2] = {0, 0};
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (v == 0) k_smem<<<blocks, threads>>>(o1);
            else k_shfl<<<blocks, threads>>>(o2);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms[v], a, b);
        }
    }
    uint64_t* h1 = new uint64_t[blocks * threads];
    uint64_t* h2 = new uint64_t[blocks * threads];
    cudaMemcpy(h1, o1, 8ull * blocks * threads, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, o2, 8ull * blocks * threads, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < blocks * threads; ++i) bad += h1[i] != h2[i];
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    const double warps = (double)blocks * threads / 32.0, xch = warps * ITERS;
    const char* names[2] = {"smem", "shfl"};
    for (int v = 0; v < 2; ++v) {
        const double clk_per_sm = ms[v] * 1e-3 * mhz * 1e3;  // cycles per SM over the run
        printf("{\"exchange\": \"%s\", \"ms\": %.4f, \"warp_exchanges\": %.0f, \"clk_per_warp_exchange_per_sm\": %.2f, \"same_result\": %s, \"err\": \"%s\"}\n",
               names[v], ms[v], xch, clk_per_sm / (xch / sms), bad ? "false" : "true", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
