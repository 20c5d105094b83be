// tools/alu_roof.cu -- integer-pipe micro-benchmark for the NTT's ALU roof
// (SURVEY section 7 step 0).  Measures per-SM throughput of the instructions a
// 64-bit Shoup butterfly is made of, and of whole butterflies, with every
// thread running independent chains so only pipe throughput limits.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_roof tools/alu_roof.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 2048

__global__ void k_imad_wide(uint64_t* out, uint32_t a, uint32_t b) {
  uint64_t acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("{ .reg .u32 lo, hi; mov.b64 {lo, hi}, %0; mad.wide.u32 %0, lo, %1, %0; }" : "+l"(acc[c]) : "r"(x + c));
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad(uint64_t* out, uint32_t a, uint32_t b) {
  uint32_t acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(acc[c]) : "r"(x), "r"(y + c));
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad_hi(uint64_t* out, uint32_t a, uint32_t b) {
  uint32_t acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(acc[c]) : "r"(x), "r"(y + c));
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd3(uint64_t* out, uint32_t a, uint32_t b) {
  uint32_t acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x + c;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[c]) : "r"(x + c));
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(uint64_t* out, uint32_t a, uint32_t b) {  // 1 IMAD : 1 IADD
  uint32_t acc[CH], acc2[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; acc2[c] = c; }
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(acc[c]) : "r"(x), "r"(y + c));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(acc2[c]) : "r"(x + c));
    }
  uint32_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= acc[c] ^ acc2[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint64_t shoup_lazy(uint64_t b, uint64_t w, uint64_t wb, uint64_t p) {
  return b * w - __umul64hi(b, wb) * p;
}
// Harvey CT butterfly, inputs/outputs < 4p
__global__ void k_bf_ct(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH], Y[CH];
  for (int c = 0; c < CH; ++c) { X[c] = (threadIdx.x * 77 + c) % p; Y[c] = (threadIdx.x * 31 + c * 5) % p; }
  const uint64_t p2 = 2 * p;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t x = X[c] >= p2 ? X[c] - p2 : X[c];
      uint64_t t = shoup_lazy(Y[c], w, wb, p);
      X[c] = x + t;
      Y[c] = x - t + p2;
    }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Shoup lazy multiply alone (chained)
__global__ void k_shoup(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH];
  for (int c = 0; c < CH; ++c) X[c] = (threadIdx.x * 77 + c) % p;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) X[c] = shoup_lazy(X[c], w, wb, p);
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- butterfly variants (V0 exact __umul64hi; V1 truncated quotient; V2 truncated + (-p))
__device__ __forceinline__ uint64_t shoup_trunc(uint64_t b, uint64_t w, uint64_t wb, uint64_t p) {
  uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32), v0 = (uint32_t)wb, v1 = (uint32_t)(wb >> 32);
  uint64_t q = (uint64_t)b1 * v1 + __umulhi(b1, v0) + __umulhi(b0, v1);
  return b * w - q * p;
}
__device__ __forceinline__ uint64_t shoup_trunc_np(uint64_t b, uint64_t w, uint64_t wb, uint64_t np) {
  uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32), v0 = (uint32_t)wb, v1 = (uint32_t)(wb >> 32);
  uint64_t q = (uint64_t)b1 * v1 + __umulhi(b1, v0) + __umulhi(b0, v1);
  return b * w + q * np;
}
// Shoup with the quotient and remainder in hand-written PTX (adds via add.cc/addc)
__device__ __forceinline__ uint64_t shoup_ptx(uint64_t b, uint64_t w, uint64_t wb, uint64_t np) {
  uint64_t r;
  asm("{\n\t"
      ".reg .u32 b0, b1, v0, v1, w0, w1, n0, n1, t0, t1, q0, q1, r0, r1;\n\t"
      ".reg .u64 q, a;\n\t"
      "mov.b64 {b0, b1}, %1;\n\t"
      "mov.b64 {w0, w1}, %2;\n\t"
      "mov.b64 {v0, v1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t0, b1, v0;\n\t"
      "mul.hi.u32 t1, b0, v1;\n\t"
      "mul.wide.u32 q, b1, v1;\n\t"
      "mov.b64 {q0, q1}, q;\n\t"
      "add.cc.u32 q0, q0, t0;\n\t"
      "addc.u32 q1, q1, 0;\n\t"
      "add.cc.u32 q0, q0, t1;\n\t"
      "addc.u32 q1, q1, 0;\n\t"
      "mul.wide.u32 a, b0, w0;\n\t"
      "mov.b64 {r0, r1}, a;\n\t"
      "mad.lo.u32 r1, b0, w1, r1;\n\t"
      "mad.lo.u32 r1, b1, w0, r1;\n\t"
      "mad.lo.u32 r1, q0, n1, r1;\n\t"
      "mad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 a, {r0, r1};\n\t"
      "mad.wide.u32 a, q0, n0, a;\n\t"
      "mov.b64 %0, a;\n\t"
      "}" : "=l"(r) : "l"(b), "l"(w), "l"(wb), "l"(np));
  return r;
}
// V4: the kernels' PTX Shoup (re-paired); V5: FP64-assisted truncated quotient:
// hi(b1 v0) + hi(b0 v1) ~ floor((b1 v0 + b0 v1) / 2^32) computed on the FP64
// pipe with round-down (exact int->double via the 2^52 bias trick).
__device__ __forceinline__ uint64_t shoup_v4(uint64_t b, uint64_t w, uint64_t wb, uint64_t np) {
  uint64_t r;
  asm("{\n\t.reg .u32 b0, b1, v0, v1, w0, w1, n0, n1, t0, t1, q0, q1, r0, r1;\n\t.reg .u64 q, a;\n\t"
      "mov.b64 {b0, b1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {v0, v1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t0, b1, v0;\n\tmul.hi.u32 t1, b0, v1;\n\tmul.wide.u32 q, b1, v1;\n\tmov.b64 {q0, q1}, q;\n\t"
      "add.cc.u32 q0, q0, t0;\n\taddc.u32 q1, q1, 0;\n\tadd.cc.u32 q0, q0, t1;\n\taddc.u32 q1, q1, 0;\n\t"
      "mul.wide.u32 a, b0, w0;\n\tmad.wide.u32 a, q0, n0, a;\n\tmov.b64 {r0, r1}, a;\n\t"
      "mad.lo.u32 r1, b0, w1, r1;\n\tmad.lo.u32 r1, b1, w0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(b), "l"(w), "l"(wb), "l"(np));
  return r;
}
// V9: r = (b w) + q (-p) with the b w partial products issued before q is known
// (shorter dependency chain: only 1 WIDE + 2 IMAD after the quotient)
__device__ __forceinline__ uint64_t shoup_v9(uint64_t b, uint64_t w, uint64_t wb, uint64_t np) {
  uint64_t r;
  asm("{\n\t.reg .u32 b0, b1, v0, v1, w0, w1, n0, n1, t0, t1, q0, q1, r0, r1, s1;\n\t.reg .u64 q, a;\n\t"
      "mov.b64 {b0, b1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {v0, v1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.wide.u32 a, b0, w0;\n\tmov.b64 {r0, r1}, a;\n\t"
      "mad.lo.u32 r1, b0, w1, r1;\n\tmad.lo.u32 r1, b1, w0, r1;\n\tmov.b64 a, {r0, r1};\n\t"
      "mul.hi.u32 t0, b1, v0;\n\tmul.hi.u32 t1, b0, v1;\n\tmul.wide.u32 q, b1, v1;\n\tmov.b64 {q0, q1}, q;\n\t"
      "add.cc.u32 q0, q0, t0;\n\taddc.u32 q1, q1, 0;\n\tadd.cc.u32 q0, q0, t1;\n\taddc.u32 q1, q1, 0;\n\t"
      "mul.lo.u32 s1, q0, n1;\n\tmad.lo.u32 s1, q1, n0, s1;\n\t"
      "mad.wide.u32 a, q0, n0, a;\n\tmov.b64 {r0, r1}, a;\n\tadd.u32 r1, r1, s1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(b), "l"(w), "l"(wb), "l"(np));
  return r;
}
__device__ __forceinline__ uint64_t shoup_f64(uint64_t b, uint64_t w, uint64_t wb, uint64_t np, double V0, double V1) {
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const double two52 = 4503599627370496.0;
  const double B0 = __longlong_as_double((long long)(0x4330000000000000ull | b0)) - two52;
  const double B1 = __longlong_as_double((long long)(0x4330000000000000ull | b1)) - two52;
  const double t = __fma_rd(B1, V0, __dmul_rd(B0, V1));
  const double u = __fma_rd(t, 2.3283064365386963e-10, two52);  // 2^52 + floor(t / 2^32)
  const uint32_t c = (uint32_t)__double_as_longlong(u);
  const uint64_t q = (uint64_t)b1 * (uint32_t)(wb >> 32) + c;
  const uint32_t q0 = (uint32_t)q, q1 = (uint32_t)(q >> 32);
  const uint32_t w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32), n0 = (uint32_t)np, n1 = (uint32_t)(np >> 32);
  uint64_t a = (uint64_t)b0 * w0 + (uint64_t)q0 * n0;
  uint32_t hi = (uint32_t)(a >> 32) + b0 * w1 + b1 * w0 + q0 * n1 + q1 * n0;
  return ((uint64_t)hi << 32) | (uint32_t)a;
}
__device__ __forceinline__ uint64_t shoup_f64b(uint64_t b, uint64_t w, uint64_t wb, uint64_t np, double V0, double V1) {
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const double B0 = __uint2double_rn(b0), B1 = __uint2double_rn(b1);
  const double t = __fma_rd(B1, V0, __dmul_rd(B0, V1));
  const double u = __fma_rd(t, 2.3283064365386963e-10, 4503599627370496.0);
  const uint32_t c = (uint32_t)__double_as_longlong(u);
  const uint64_t q = (uint64_t)b1 * (uint32_t)(wb >> 32) + c;
  const uint32_t q0 = (uint32_t)q, q1 = (uint32_t)(q >> 32);
  const uint32_t w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32), n0 = (uint32_t)np, n1 = (uint32_t)(np >> 32);
  uint64_t a = (uint64_t)b0 * w0 + (uint64_t)q0 * n0;
  uint32_t hi = (uint32_t)(a >> 32) + b0 * w1 + b1 * w0 + q0 * n1 + q1 * n0;
  return ((uint64_t)hi << 32) | (uint32_t)a;
}
__device__ __forceinline__ uint64_t csub_hi(uint64_t x, uint64_t m, uint32_t mh) {
  return (uint32_t)(x >> 32) > mh ? x - m : x;
}
template <int V>
__global__ void k_bfw(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH], Y[CH];
  for (int c = 0; c < CH; ++c) { X[c] = (threadIdx.x * 77 + c) % p; Y[c] = (threadIdx.x * 31 + c * 5) % p; }
  const uint64_t p5 = 5 * p, np = 0 - p;
  const uint32_t p5h = (uint32_t)(p5 >> 32);
  const double V0 = (double)(uint32_t)wb, V1 = (double)(uint32_t)(wb >> 32);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t x = csub_hi(X[c], p5, p5h);
      uint64_t t = V == 4 ? shoup_v4(Y[c], w, wb, np) : V == 9 ? shoup_v9(Y[c], w, wb, np) : V == 5 ? shoup_f64(Y[c], w, wb, np, V0, V1) : shoup_f64b(Y[c], w, wb, np, V0, V1);
      X[c] = x + t; Y[c] = x - t + p5;
    }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the paper's "native modulo" comparison: same butterfly with the
// product reduced by the compiler's 128-by-64-bit remainder instead of Shoup
__global__ void k_bf_native(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH], Y[CH];
  for (int c = 0; c < CH; ++c) { X[c] = (threadIdx.x * 77 + c) % p; Y[c] = (threadIdx.x * 31 + c * 5) % p; }
  for (int it = 0; it < ITERS / 8; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint64_t t = (uint64_t)(((unsigned __int128)Y[c] * w) % p);
      const uint64_t x = X[c];
      X[c] = x + t >= p ? x + t - p : x + t;
      Y[c] = x >= t ? x - t : x + p - t;
    }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// correctness of the FP64 quotient variant against exact arithmetic (host check)
__global__ void k_f64check(uint64_t* bad, const uint64_t* bs, uint64_t p, uint64_t w, uint64_t wb, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double V0 = (double)(uint32_t)wb, V1 = (double)(uint32_t)(wb >> 32);
  uint64_t b = bs[i];
  uint64_t r = shoup_f64(b, w, wb, 0 - p, V0, V1);
  unsigned __int128 prod = (unsigned __int128)b * w;
  uint64_t ex = (uint64_t)(prod % p);
  if (r >= 5 * p || (r % p) != ex) atomicAdd((unsigned long long*)bad, 1ull);
}

template <int V>
__global__ void k_bfv(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH], Y[CH];
  for (int c = 0; c < CH; ++c) { X[c] = (threadIdx.x * 77 + c) % p; Y[c] = (threadIdx.x * 31 + c * 5) % p; }
  const uint64_t p4 = 4 * p, np = 0 - p, p2 = 2 * p;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (V == 0) {
        uint64_t x = X[c] >= p2 ? X[c] - p2 : X[c];
        uint64_t t = shoup_lazy(Y[c], w, wb, p);
        X[c] = x + t; Y[c] = x - t + p2;
      } else {
        uint64_t x = X[c] >= p4 ? X[c] - p4 : X[c];
        uint64_t t = V == 1 ? shoup_trunc(Y[c], w, wb, p) : V == 2 ? shoup_trunc_np(Y[c], w, wb, np)
                                                          : shoup_ptx(Y[c], w, wb, np);
        X[c] = x + t; Y[c] = x - t + p4;
      }
    }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// GS butterflies: exact and truncated
template <int V>
__global__ void k_gsv(uint64_t* out, uint64_t p, uint64_t w, uint64_t wb) {
  uint64_t X[CH], Y[CH];
  for (int c = 0; c < CH; ++c) { X[c] = (threadIdx.x * 77 + c) % p; Y[c] = (threadIdx.x * 31 + c * 5) % p; }
  const uint64_t p4 = 4 * p, np = 0 - p, p2 = 2 * p;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint64_t x = X[c], y = Y[c];
      if (V == 0) {
        uint64_t s = x + y; X[c] = s >= p2 ? s - p2 : s;
        Y[c] = shoup_lazy(x - y + p2, w, wb, p);
      } else {
        uint64_t s = x + y; X[c] = s >= p4 ? s - p4 : s;
        Y[c] = V == 1 ? shoup_trunc_np(x - y + p4, w, wb, np) : shoup_ptx(x - y + p4, w, wb, np);
      }
    }
  uint64_t s = 0;
  for (int c = 0; c < CH; ++c) s ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*kfun32)(uint64_t*, uint32_t, uint32_t);
typedef void (*kfun64)(uint64_t*, uint64_t, uint64_t, uint64_t);

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f}\n", prop.name, sms, clk_khz / 1e3);
  uint64_t* out;
  int threads = 256, blocks_per_sm = 8;
  int blocks = sms * blocks_per_sm;
  cudaMalloc(&out, sizeof(uint64_t) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct { const char* name; kfun32 f; double ops_per_inner; } k32[] = {
      {"mad.wide.u32", k_imad_wide, 1}, {"mad.lo.u32", k_imad, 1}, {"mad.hi.u32", k_imad_hi, 1},
      {"add.u32", k_iadd3, 1}, {"mad.lo+add", k_mix, 2}};
  for (auto& k : k32) {
    for (int rep = 0; rep < 3; ++rep) k.f<<<blocks, threads>>>(out, 3, 5);
    cudaEventRecord(e0);
    k.f<<<blocks, threads>>>(out, 3, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * ITERS * CH * k.ops_per_inner;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"Gops_per_s\": %.1f, \"ops_per_ns_per_sm\": %.3f}\n", k.name, ms,
           ops / ms / 1e6, ops / ms / 1e6 / sms);
  }
  uint64_t p = 1152921504606584833ull, w = 30403152079314ull;
  uint64_t wb = (uint64_t)(((unsigned __int128)w << 64) / p);
  struct { const char* name; kfun64 f; } k64[] = {{"butterfly_ct_harvey", k_bf_ct}, {"shoup_lazy", k_shoup},
      {"ct_v0_exact", k_bfv<0>}, {"ct_v1_trunc", k_bfv<1>}, {"ct_v2_trunc_np", k_bfv<2>}, {"ct_v3_ptx", k_bfv<3>},
      {"gs_v0_exact", k_gsv<0>}, {"gs_v1_trunc_np", k_gsv<1>}, {"gs_v2_ptx", k_gsv<2>}};
  for (auto& k : k64) {
    for (int rep = 0; rep < 3; ++rep) k.f<<<blocks, threads>>>(out, p, w, wb);
    cudaEventRecord(e0);
    k.f<<<blocks, threads>>>(out, p, w, wb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * ITERS * CH;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"Gops_per_s\": %.1f, \"ops_per_ns_per_sm\": %.3f}\n", k.name, ms,
           ops / ms / 1e6, ops / ms / 1e6 / sms);
  }
  {
    for (int rep = 0; rep < 2; ++rep) k_bfw<4><<<blocks, threads>>>(out, p, w, wb);
    for (int v = 4; v <= 6; ++v) {
      if (v == 6) k_bfw<6><<<blocks, threads>>>(out, p, w, wb);
      cudaEventRecord(e0);
      if (v == 4) k_bfw<4><<<blocks, threads>>>(out, p, w, wb);
      else if (v == 5) k_bfw<5><<<blocks, threads>>>(out, p, w, wb);
      else k_bfw<6><<<blocks, threads>>>(out, p, w, wb);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * ITERS * CH;
      printf("{\"kernel\": \"ct_w%d\", \"Gops_per_s\": %.1f}\n", v, ops / ms / 1e6);
    }
    // FP64 quotient correctness on random 64-bit inputs
    const int n = 1 << 22;
    uint64_t *bs, *bad;
    cudaMalloc(&bs, n * 8);
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    uint64_t* hb = (uint64_t*)malloc(n * 8);
    uint64_t z = 12345;
    for (int i = 0; i < n; ++i) { z ^= z << 13; z ^= z >> 7; z ^= z << 17; hb[i] = i < 64 ? ~(uint64_t)i : z; }
    cudaMemcpy(bs, hb, n * 8, cudaMemcpyHostToDevice);
    k_f64check<<<n / 256, 256>>>(bad, bs, p, w, wb, n);
    uint64_t nb = 0;
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    printf("{\"check\": \"shoup_f64\", \"n\": %d, \"bad\": %llu}\n", n, (unsigned long long)nb);
  }
  {
    for (int rep = 0; rep < 2; ++rep) k_bf_native<<<blocks, threads>>>(out, p, w, wb);
    cudaEventRecord(e0);
    k_bf_native<<<blocks, threads>>>(out, p, w, wb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * (ITERS / 8) * CH;
    printf("{\"kernel\": \"ct_native_mod\", \"Gops_per_s\": %.1f}\n", ops / ms / 1e6);
  }
  // occupancy sweep: kernel-path butterfly (V4) vs shorter-chain variant (V9)
  for (int v : {4, 9})
    for (int wps : {8, 12, 16, 32, 64}) {
      int thr = 128, bps = wps * 32 / thr;
      int nb = sms * bps;
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 4) k_bfw<4><<<nb, thr>>>(out, p, w, wb); else k_bfw<9><<<nb, thr>>>(out, p, w, wb);
      }
      cudaEventRecord(e0);
      if (v == 4) k_bfw<4><<<nb, thr>>>(out, p, w, wb); else k_bfw<9><<<nb, thr>>>(out, p, w, wb);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)nb * thr * ITERS * CH;
      printf("{\"kernel\": \"ct_w%d_occ\", \"warps_per_sm\": %d, \"Gops_per_s\": %.1f}\n", v, wps, ops / ms / 1e6);
    }
  // occupancy sweep for the PTX butterfly: warps per SM vs rate
  for (int wps : {4, 8, 12, 16, 24, 32, 48, 64}) {
    int thr = 128, bps = wps * 32 / thr;
    int nb = sms * bps;
    for (int rep = 0; rep < 2; ++rep) k_bfv<3><<<nb, thr>>>(out, p, w, wb);
    cudaEventRecord(e0);
    k_bfv<3><<<nb, thr>>>(out, p, w, wb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)nb * thr * ITERS * CH;
    printf("{\"kernel\": \"ct_v3_ptx_occ\", \"warps_per_sm\": %d, \"Gops_per_s\": %.1f}\n", wps, ops / ms / 1e6);
  }
  return 0;
}
