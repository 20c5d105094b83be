// ntt_device.cuh -- device arithmetic and the register/SMEM stage engine of the
// B200 NTT kernels.  Product code (never includes anything from oracle/).
//
// Citations: P:n = /root/reference/PAPER.md line n; R# = DESIGN.md section 3.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>
#include <utility>

namespace ntt {

// A twiddle with its Shoup companion (Algorithm 4): 16 bytes, one
// 128-bit load.
struct __align__(16) Tw {
    uint64_t w, wb;
};

// Per-prime constants, 128 bytes.
struct __align__(16) PrimeConst {
    uint64_t p, p2, p4;  // p, 2p, 4p
    uint64_t np;         // 2^64 - p
    uint64_t p5;         // 5p: the GS difference offset (section 5.1)
    uint32_t p4_hi;      // high word of 4p
    uint32_t rn;         // floor(2^90 / p): quotient estimate for the final reduction
    Tw ninv;             // N^-1   [R-scaled copy: N^-1 2^64, see mont_mul]
    Tw ninv_psi;         // N^-1 * Psi^-1[1], the fused last GS stage (R15)
    uint64_t pinv;       // -p^-1 mod 2^64 (Montgomery, NTT-domain products)
    uint32_t m1;         // 2^32 - (p >> 32): the Proth form below
    uint32_t p8_hi;      // high word of 8p
    uint64_t p8;         // 8p: Proth primes reduce by 8p on every other stage (ct_bf)
    uint64_t zero;       // 0, opaque to the compiler: a third operand that keeps 64-bit adds on IADD3
    uint64_t mN;         // (p - 1) / N: the exact-division N^-1 of PrimeConstD (div_n)
    uint32_t logn, nmask;  // log2 N, N - 1
};

// The same constants, as a type that selects the Proth-prime arithmetic: for
// p = p1 2^32 + 1 (p = 1 mod 2^32) the low 64 bits of
// q p are q + (q0 p1 << 32), one IMAD instead of an IMAD.WIDE and two IMADs.
// Kernels templated on PrimeConstP are launched only for plans whose primes
// all have this form (ntt_api.cu).
struct PrimeConstP : PrimeConst {
};
// Proth arithmetic plus Kernel-1''s exact-division N^-1 (div_n; see
// PrimeConstD below): the Kernel-1' instantiation of Proth plans outside the
// NTT-domain product path (ntt_kernels_d.cu).
struct PrimeConstPD : PrimeConstP {
};

// The same constants, as a type that selects the d-form final reduction of
// the forward (reduce_full below) for primes p = 2^60 - d with d < 2^32 --
// every prime of the R3 chain.  Everything else is the general arithmetic.
// Kernel-1' takes on it the exact-division form of its fused N^-1 (div_n).
// Only the forward shared-twiddle Kernel-2 and Kernel-1' are instantiated on
// it (ntt_kernels_d.cu), for plans whose primes all have the form and not in
// the NTT-domain product path, whose N^-1 carries a Montgomery factor (ntt_api.cu).
struct PrimeConstD : PrimeConst {
};

// The same constants, as a type that selects the paper's "Native" comparison
// arithmetic (fig:native_shoup): every twiddle product is reduced
// with the native 128-by-64-bit modulo, (unsigned __int128)(b w) % p, instead
// of Shoup's modmul.  Only ntt_forward_variant(NTT_VARIANT_NATIVE) uses it.
struct PrimeConstN : PrimeConst {
};

template <class C>
__device__ __forceinline__ C load_pc(const PrimeConst* pc, uint32_t l)
{
    C c;
    static_cast<PrimeConst&>(c) = pc[l];
    return c;
}

// Kernel arguments (passed by value, lives in the constant bank).
struct KArgs {
    uint64_t* data;        // [batch][L][N]
    const Tw* tab;         // [L][N] Psi (forward) or Psi^-1 (inverse)
    const Tw* tab2;        // [L][N1][N2] the same twiddles in Kernel-2 order (K2Layout)
    const Tw* ot;          // [L][B + N/B] OT bases (fine | coarse), forward or inverse
    const PrimeConst* pc;  // [L]
    uint32_t L, batch;
    uint32_t logn, log_n1;  // log_n1 = 0 for the single-kernel path
    uint32_t log_tiles;     // column kernel: log2(N2 / 16)
    uint32_t iters;         // contig kernel: block-groups per CTA
    uint32_t ot_logb;       // OT: log2 of the base B
    uint32_t total_blocks;  // contig kernel: rows * N1
    const uint64_t* mul_a;  // fused NTT-domain product: the other operand, same layout as data
};

// 32-bit-word path (ntt32.cu): 30-bit primes, w_bar = floor(w 2^32 / p).
struct __align__(8) Tw32 {
    uint32_t w, wb;
};
struct __align__(16) PrimeConst32 {
    uint32_t p, p2;
    Tw32 ninv;      // N^-1
    Tw32 ninv_psi;  // N^-1 * Psi^-1[1]
    uint32_t pad[2];
};
struct KArgs32 {
    uint32_t* data;          // [batch][L][N] 32-bit words
    const Tw32* tab;         // [L][N] Psi / Psi^-1
    const Tw32* tab2;        // [L][N1][N2] Kernel-2 order
    const PrimeConst32* pc;  // [L]
    uint32_t L, batch, logn, log_n1, log_tiles, total_blocks;
};

// ------------------------------------------------------------ arithmetic
// Shoup's modmul (Algorithm 4) with the lazy output of R8 and a
// truncated quotient: for any b < 2^64 and
// w < p < 2^60, with w_bar = floor(w 2^64 / p),
//   q' = b1 v1 + hi(b1 v0) + hi(b0 v1)        (b = b1:b0, w_bar = v1:v0)
// drops the low partial product and its carries, so q' <= floor(b w_bar/2^64)
// <= q' + 2 and, with Shoup's own bound, floor(b w / p) - q' in [0, 3]:
//   r = b w - q' p = (b w mod p) + k p,  k in {0,1,2,3}  ->  r in [0, 4p).
// r is formed mod 2^64 as b w + q' (2^64 - p): 3 IMAD.WIDE, 2 IMAD.HI and
// 4 IMAD on the multiply pipe.  np = 2^64 - p.  The 64-bit partial product
// b0 w0 + q0 n0 is accumulated in one register pair (no re-pairing moves);
// q' is one IMAD.WIDE with a zero-extended addend plus one 64-bit add, which
// ptxas emits as a 3-input IADD3 / IADD3.X pair (a 32-bit add.cc / addc chain
// became IMAD.X plus moves on the multiply pipe: -6% fmaheavy).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t b, uint64_t w, uint64_t wb, uint64_t np)
{
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 b0, b1, v0, v1, w0, w1, n0, n1, t0, t1, q0, q1, r0, r1;\n\t"
        ".reg .u64 q, a, t;\n\t"
        "mov.b64 {b0, b1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {v0, v1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
        "mul.hi.u32 t0, b1, v0;\n\t"
        "mul.hi.u32 t1, b0, v1;\n\t"
        "cvt.u64.u32 t, t0;\n\t"
        "mad.wide.u32 q, b1, v1, t;\n\t"
        "cvt.u64.u32 t, t1;\n\t"
        "add.u64 q, q, t;\n\t"
        "mov.b64 {q0, q1}, q;\n\t"
        "mul.wide.u32 a, b0, w0;\n\t"
        "mad.wide.u32 a, q0, n0, a;\n\t"
        "mov.b64 {r0, r1}, a;\n\t"
        "mad.lo.u32 r1, b0, w1, r1;\n\t"
        "mad.lo.u32 r1, b1, w0, r1;\n\t"
        "mad.lo.u32 r1, q0, n1, r1;\n\t"
        "mad.lo.u32 r1, q1, n0, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(b), "l"(w), "l"(wb), "l"(np));
    return r;
}

// Shoup's modmul for a Proth prime p = p1 2^32 + 1: the same truncated
// quotient q' (so the same [0, 4p) output bound), and
//   r = b w - q' p = lo64(b w) - q' - (q0' p1 << 32)  (mod 2^64),
// formed as one IMAD.WIDE b0 w0 with the addend -q' and three IMADs into the
// high word (m1 = -p1 mod 2^32): 2 IMAD.WIDE, 2 IMAD.HI and 3 IMAD.  (A
// variant subtracting q' as a three-input add with an opaque zero, which
// keeps the negation off the multiply pipe, measured 1-2 % slower in the
// kernels and 5 % in tools/bf_roof -- DESIGN.md 5.1.)
__device__ __forceinline__ uint64_t shoup_lazy_p(uint64_t b, uint64_t w, uint64_t wb, uint32_t m1)
{
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 b0, b1, v0, v1, w0, w1, t0, t1, q0, q1, r0, r1;\n\t"
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
        "sub.u64 q, 0, q;\n\t"
        "mad.wide.u32 a, b0, w0, q;\n\t"
        "mov.b64 {r0, r1}, a;\n\t"
        "mad.lo.u32 r1, b0, w1, r1;\n\t"
        "mad.lo.u32 r1, b1, w0, r1;\n\t"
        "mad.lo.u32 r1, q0, %4, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "l"(b), "l"(w), "l"(wb), "r"(m1));
    return r;
}

// One Shoup multiply by a table twiddle, arithmetic chosen by the constants' type.
__device__ __forceinline__ uint64_t shoup(uint64_t b, const Tw& t, const PrimeConst& c)
{
    return shoup_lazy(b, t.w, t.wb, c.np);
}
__device__ __forceinline__ uint64_t shoup(uint64_t b, const Tw& t, const PrimeConstP& c)
{
    return shoup_lazy_p(b, t.w, t.wb, c.m1);
}
// Native modulo (PrimeConstN): exact, so the result is in [0, p) -- inside the
// [0, 4p) range every butterfly bound assumes.
__device__ __forceinline__ uint64_t shoup(uint64_t b, const Tw& t, const PrimeConstN& c)
{
    return (uint64_t)(((unsigned __int128)b * t.w) % c.p);
}

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

// Element-wise product of two NTT-domain operands (the odot) --
// both vary, so Shoup does not apply; Montgomery with R = 2^64:
//   T = a b,  m = T mod 2^64 * (-p^-1),  (T + m p) / 2^64 = a b 2^-64 mod p,
// in [0, 2p) for a, b < p.  The 2^-64 is undone by an R-scaled N^-1 in the
// inverse that follows (ntt_pointwise_inverse).
__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, const PrimeConst& c)
{
    const uint64_t lo = a * b, hi = __umul64hi(a, b);
    const uint64_t m = lo * c.pinv;
    return hi + __umul64hi(m, c.p) + (lo != 0);
}

// Conditional subtraction decided on the high words only: subtracts m iff
// hi(x) > hi(m) (then x > m).  The result is < max(x - m, m + 2^32): an
// excess of at most 2^32 over the exact reduction, absorbed by the bounds of
// section 5.1 and removed by the final exact normalisation.
__device__ __forceinline__ uint64_t csub_hi(uint64_t x, uint64_t m, uint32_t m_hi)
{
    return (uint32_t)(x >> 32) > m_hi ? x - m : x;
}

// The twiddle of one butterfly group: a table entry (one Shoup multiply) or,
// under on-the-fly twiddling, the pair (w1, w2) whose product is
// the twiddle, applied as w2 * (w1 * x): two Shoup multiplies, no new w_bar.
template <bool OT>
struct TwMul;
template <>
struct TwMul<false> {
    Tw t;
    template <class C>
    __device__ __forceinline__ uint64_t mul(uint64_t x, const C& c) const
    {
        return shoup(x, t, c);
    }
};
template <>
struct TwMul<true> {
    Tw fine, coarse;
    template <class C>
    __device__ __forceinline__ uint64_t mul(uint64_t x, const C& c) const
    {
        return shoup(shoup(x, fine, c), coarse, c);
    }
};

// Cooley-Tukey butterfly (Algorithm 2) in Harvey's lazy form (R9),
// widened for the [0,4p) multiplier (T = Y w < 4p for any Y < 2^64).
//   red = 1 (any prime): inputs and outputs in [0, 8p + 2^32);
//     X <- X mod* 4p (< 4p + 2^32);  X' = X + T;  Y' = X - T + 4p.
//   red = 2 / 0 (Proth primes, p <= 2^60 - 2^32 + 1, so 16p + 2^32 < 2^64):
//     the reduction runs on every other stage only -- the last stage of a
//     kernel and every second one before it (ct_roundN), so every kernel's
//     output and input stay below 12p + 2^32:
//     red = 2: X <- X mod* 8p (< 8p + 2^32), outputs < 12p + 2^32;
//     red = 0: no reduction, inputs < 12p + 2^32, outputs < 16p + 2^32.
//   red = 3 / 0 (any other prime, p < 2^60, so 16p < 2^64): the same every-
//     other-stage pattern with an exact 64-bit compare (two ISETPs instead of
//     one), so no 2^32 excess accumulates:
//     red = 3: X <- X mod 8p (< 8p), outputs < 12p;
//     red = 0: inputs < 12p (< 13p after a canonical input's first stages),
//     outputs < 16p.
// The conditional subtraction is decided on the high words (csub_hi) and
// folded into both outputs as 3-input adds (IADD3 / IADD3.X on the ALU pipe;
// a 2-input 64-bit add lets ptxas emit IMAD.X on the multiply pipe).
template <class W, class C>
__device__ __forceinline__ void ct_bf(uint64_t& X, uint64_t& Y, const W& w, const C& c, int red = 1)
{
    const uint64_t x = X;
    if (red == 0) {
        const uint64_t t = w.mul(Y, c);
        X = x + t + c.zero;  // three inputs: IADD3 / IADD3.X, never IMAD.X
        Y = x - t + c.p4;
        return;
    }
    const bool ge = red == 3   ? x >= c.p8
                    : red == 2 ? (uint32_t)(x >> 32) > c.p8_hi
                               : (uint32_t)(x >> 32) > c.p4_hi;
    const uint64_t s = ge ? (red >= 2 ? c.p8 : c.p4) : 0;
    const uint64_t s2 = red >= 2 ? (ge ? 0 - c.p4 : c.p4) : (ge ? 0 : c.p4);
    const uint64_t t = w.mul(Y, c);
    X = x - s + t;
    Y = x - t + s2;
}

// Gentleman-Sande butterfly of the inverse (R5): inputs and outputs below
// 4p + 2^(32+s) after s stages (< 4p + 2^49 for N <= 2^17): with inputs
// below 4p + E the carry-free test below subtracts only when x + y > 4p and
// leaves x + y < 4p + 2^33 otherwise, so E' = max(2E, 2^33).
//   X' = (X + Y) mod* 4p;  Y' = (X - Y + 5p) w  (5p > any Y, so no wrap).
// red = false: inputs below 2p (the first stage of an inverse whose input is
// canonical, or a Montgomery product < 2p), so X + Y < 4p needs no test.
template <class W, class C>
__device__ __forceinline__ void gs_bf(uint64_t& X, uint64_t& Y, const W& w, const C& c, bool red = true)
{
    const uint64_t x = X, y = Y;
    if (!red) {
        X = x + y + c.zero;  // three inputs: IADD3 / IADD3.X
        Y = w.mul(x - y + c.p5, c);
        return;
    }
    // subtract 4p iff hi(x) + hi(y) > hi(4p): a carry-free test, so X' is
    // one 3-input add (see ct_bf)
    const bool ge = (uint32_t)(x >> 32) + (uint32_t)(y >> 32) > c.p4_hi;
    X = x + y - (ge ? c.p4 : 0);
    Y = w.mul(x - y + c.p5, c);
}

// Programmatic dependent launch (PDL).  The kernels of a transform are
// launched with programmatic stream serialization (ntt::launch_pdl), so the
// next kernel's CTAs can be scheduled -- and stage their constant twiddles --
// while this kernel's last wave still runs.  Every kernel lets its dependents
// launch once all of its CTAs have started (pdl_trigger, at entry: no CTA of a
// dependent can then hold a slot a CTA of this grid still needs) and waits for
// its predecessor's completion and memory flush (pdl_wait) before its first
// read or write of the data.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
// Each thread holds E = 2^LOGE words (E = M if M is smaller): rounds of
// LOGE stages (per-thread radix-E NTTs).
template <int LOGM, int LOGE = 4>
struct Sched {
    static constexpr int M = 1 << LOGM;
    // LOGE & 15 is the per-thread radix exponent; LOGE & 16 (kRemLast) puts the
    // remainder round LAST in forward order instead of first
    static constexpr bool REMLAST = (LOGE & 16) != 0;
    static constexpr int LE = LOGM < (LOGE & 15) ? LOGM : (LOGE & 15);
    static constexpr int E = 1 << LE;
    // Default: a remainder round (LOGM mod LE stages) goes FIRST in forward
    // order: its stages have the fewest distinct twiddles (one per block for
    // the first stage), so the many-twiddle last stages run inside full
    // radix-E rounds.  REMLAST: full rounds first (round 0 then has stride
    // M/E and reads global memory in whole segments), remainder last.
    static constexpr int REM = LOGM % LE;
    static constexpr int NR = LOGM / LE + (REM ? 1 : 0);
    static constexpr int TB = M / E;  // threads per sub-transform
    __host__ __device__ static constexpr int r(int i)
    {
        return REMLAST ? ((REM && i == NR - 1) ? REM : LE) : ((REM && i == 0) ? REM : LE);
    }
    __host__ __device__ static constexpr int S(int i)
    {
        return REMLAST ? LE * i : ((REM && i > 0) ? REM + LE * (i - 1) : LE * i);
    }
};
constexpr int kRemLast = 16;

// Geometry of round RI (stages [S, S+r) of the sub-transform, S = LE RI): the
// thread's groups are G = qd*TB + tib; group G = (g, o) with
//   g = G / s, o = G % s, s = M >> (S + r)  (the smallest stride),
// and holds elements e_k = g*R*s + o + k*s, k < R = 2^r.
// Twiddles of stage S+i of group g are Psi[((F << S) + g) << i) + h], h < 2^i,
// F = 1 for a whole column / row, F = N1 + bb for block bb of Kernel-2.
template <int LOGM, int RI, int LOGE = 4>
struct RoundGeo {
    using SC = Sched<LOGM, LOGE>;
    static constexpr int S = SC::S(RI);
    static constexpr int r = SC::r(RI);
    static constexpr int R = 1 << r;
    static constexpr int s = (1 << LOGM) >> (S + r);
    static constexpr int GPT = SC::E / R;
    static constexpr int TB = SC::TB;
    __host__ __device__ static constexpr uint32_t elem(uint32_t G, int k)
    {
        const uint32_t g = G / s, o = G % s;
        return g * (R * s) + o + (uint32_t)k * s;
    }
};

// Kernel-2 twiddle layout.  Block bb (F = N1 + bb) owns N2 entries; round ri
// (stages [S, S+r)) holds, at round_off(S) + ((2^i - 1 + h) << S) + g, the
// twiddle Psi[(((F << S) + g) << i) + h] of stage S+i, twiddle h, group g.
// Entry 0 is padding.  Host and device share this definition.
template <int LOGM, int LOGE>
struct K2Layout {
    using SC = Sched<LOGM, LOGE>;
    __host__ __device__ static constexpr uint32_t round_off(int S)
    {
        uint32_t off = 1;
        for (int i = 0; i < SC::NR && SC::S(i) < S; ++i) off += ((1u << SC::r(i)) - 1u) << SC::S(i);
        return off;
    }
    // Entries [0, used(OTS)) hold the twiddles of the stages below LOGM - OTS;
    // the last OTS stages (the tail of the last round, OTS <= its r) come from
    // on-the-fly twiddling and their entries are never read -- a
    // kernel under OT copies only this prefix (3/4 of the table saved at OTS = 2).
    __host__ __device__ static constexpr uint32_t used(int OTS)
    {
        if (OTS == 0) return 1u << LOGM;
        const int j0 = LOGM - OTS;  // first OT stage; its round and position in it
        int ri = SC::NR - 1;
        while (SC::S(ri) > j0) --ri;
        const int Sl = SC::S(ri), i0 = j0 - Sl;
        return round_off(Sl) + (((1u << i0) - 1u) << Sl);
    }
};

// Forward round: r Cooley-Tukey stages on each of the thread's GPT groups.
// Twiddle indices are formed for F = 1 ("local" index: the block's own
// sub-table, tl[2^j + h] = Psi[F 2^j + h]); Fm1 = F - 1 shifts them to the
// global index idx + (Fm1 << j) where a global table or OT needs it.
// tabf(TwKey) returns the twiddle (the key carries both the local index and
// its (stage, h, group) coordinates, for tables laid out per round);
// otf(idx_global) the OT factor pair.
// OT_FROM = first local stage whose twiddles come from OT (>= LOGM: none).
struct TwKey {
    uint32_t idx;  // local index ((1 << S) + g) << i) + h
    int j;         // local stage S + i
    int S, i, h;   // round start, stage within round, twiddle within stage
    uint32_t g;    // group
};

// NI sub-transforms per thread share every twiddle (Kernel-1 columns of one
// tile; Kernel-2 blocks of one prime at the same block position): one twiddle
// load serves NI times the butterflies, and NI independent chains add ILP.
// CANON: the kernel's input is canonical ([0, p): Kernel-1 and the single-CTA
// kernel), so with Proth primes the reductions of local stages 0 and 1 are
// skipped (their inputs stay below 9p).  FINAL: the kernel normalises its
// output with reduce_full (valid for any word), so the reduction pattern is
// shifted by one stage and the last stage needs none (outputs < 16p + 2^32).
template <int LOGM, int LOGE, int RI, int OT_FROM, int NI, bool CANON = false, bool FINAL = false, class TabF,
          class OtF, class C>
__device__ __forceinline__ void ct_roundN(uint64_t (&x)[NI][16], uint32_t tib, uint32_t Fm1, const TabF& tabf,
                                          const OtF& otf, const C& c)
{
#ifdef NTT_PROBE_NOMATH  // experiment builds only (tools/probe_nomath.sh): memory / exchange floor of a kernel
    return;
#endif
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Geo::TB + tib;
        const uint32_t B = (1u << S) + G / Geo::s;
#pragma unroll
        for (int i = 0; i < Geo::r; ++i) {
            const int half = R >> (i + 1);
            // reduce on the kernel's last stage and every second one before it
            // (ct_bf: red 2 for Proth primes, 3 for any other)
            const int red = ((((LOGM - 1 - (S + i) - (FINAL ? 1 : 0)) & 1) || (CANON && S + i < 2))
                                 ? 0
                                 : (std::is_base_of_v<PrimeConstP, C> ? 2 : 3));
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const uint32_t idx = (B << i) + h;
                if (S + i >= OT_FROM) {
                    const TwMul<true> w = otf(idx + (Fm1 << (S + i)));
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
#pragma unroll
                        for (int n = 0; n < NI; ++n) ct_bf(x[n][qd * R + k], x[n][qd * R + k + half], w, c, red);
                } else {
                    const TwMul<false> w{tabf(TwKey{idx, S + i, S, i, h, G / Geo::s})};
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
#pragma unroll
                        for (int n = 0; n < NI; ++n) ct_bf(x[n][qd * R + k], x[n][qd * R + k + half], w, c, red);
                }
            }
        }
    }
}

template <int LOGM, int LOGE, int RI, int OT_FROM, bool CANON = false, bool FINAL = false, class TabF, class OtF,
          class C>
__device__ __forceinline__ void ct_round(uint64_t (&x)[16], uint32_t tib, uint32_t Fm1, const TabF& tabf,
                                         const OtF& otf, const C& c)
{
    ct_roundN<LOGM, LOGE, RI, OT_FROM, 1, CANON, FINAL>(reinterpret_cast<uint64_t(&)[1][16]>(x), tib, Fm1, tabf,
                                                       otf, c);
}

// x N^-1 mod p as an exact division (the fused N^-1 of the inverse's X'
// outputs, R15; PrimeConstD plans only): every NTT prime is p = 1 + mN N
// (p = 1 mod 2N), so with k = -x mod N the sum x + k p =
// (x + k) + k mN N is divisible by N and
//   r = (x + k) / N + k mN  ==  x N^-1  (mod p),   r < x / N + p,
// below 4p for the GS sums x < 8p + 2^50 (N >= 2^14 in Kernel-1'): one
// IMAD.WIDE + one IMAD (k < N, mN < 2^46) and ALU adds / shifts instead of a
// Shoup multiply (3 IMAD.WIDE + 2 IMAD.HI + 4 IMAD).
__device__ __forceinline__ uint64_t div_n(uint64_t x, const PrimeConst& c)
{
    const uint32_t k = (0u - (uint32_t)x) & c.nmask;
    const uint64_t s = (x + k) >> c.logn;
    uint64_t r;
    asm("{\n\t"
        ".reg .u32 m0, m1, r0, r1;\n\t"
        ".reg .u64 a;\n\t"
        "mov.b64 {m0, m1}, %2;\n\t"
        "mad.wide.u32 a, %1, m0, %3;\n\t"
        "mov.b64 {r0, r1}, a;\n\t"
        "mad.lo.u32 r1, %1, m1, r1;\n\t"
        "mov.b64 %0, {r0, r1};\n\t"
        "}"
        : "=l"(r)
        : "r"(k), "l"(c.mN), "l"(s));
    return r;
}

// Inverse round: the same groups and twiddle indices, Gentleman-Sande stages
// in reverse order.  FUSE0: local stage 0 is global stage 0 (m = 1), where
// N^-1 is fused: X' = (X+Y) N^-1, Y' = (X-Y) Psi^-1[1] N^-1 (R15).
// CANON: the sub-transform's input is below 2p, so its first GS stage (local
// stage LOGM - 1) skips the reduction of X + Y (gs_bf red = false).
template <int LOGM, int LOGE, int RI, int OT_FROM, bool FUSE0, int NI, bool CANON = false, class TabF, class OtF,
          class C>
__device__ __forceinline__ void gs_roundN(uint64_t (&x)[NI][16], uint32_t tib, uint32_t Fm1, const TabF& tabf,
                                          const OtF& otf, const C& c)
{
#ifdef NTT_PROBE_NOMATH
    return;
#endif
    using Geo = RoundGeo<LOGM, RI, LOGE>;
    constexpr int R = Geo::R, S = Geo::S;
#pragma unroll
    for (int qd = 0; qd < Geo::GPT; ++qd) {
        const uint32_t G = qd * Geo::TB + tib;
        const uint32_t B = (1u << S) + G / Geo::s;
#pragma unroll
        for (int i = Geo::r - 1; i >= 0; --i) {
            const int half = R >> (i + 1);
            if (FUSE0 && S + i == 0) {
                const TwMul<false> a{c.ninv}, b{c.ninv_psi};
#pragma unroll
                for (int k = 0; k < half; ++k)
#pragma unroll
                    for (int n = 0; n < NI; ++n) {
                        const uint64_t u = x[n][qd * R + k], v = x[n][qd * R + k + half];
                        if constexpr (std::is_same_v<C, PrimeConstD> || std::is_same_v<C, PrimeConstPD>) {
                            // canonical outputs here: div_n's r < x/N + p needs one
                            // subtraction, not norm4's two (Kernel-1' then skips norm4)
                            x[n][qd * R + k] = csub(div_n(u + v, c), c.p);
                            x[n][qd * R + k + half] = norm4(b.mul(u - v + c.p5, c), c);
                            continue;
                        } else {
                            x[n][qd * R + k] = a.mul(u + v, c);
                        }
                        x[n][qd * R + k + half] = b.mul(u - v + c.p5, c);
                    }
                continue;
            }
#pragma unroll
            for (int h = 0; h < (1 << i); ++h) {
                const uint32_t idx = (B << i) + h;
                if (S + i >= OT_FROM) {
                    const TwMul<true> w = otf(idx + (Fm1 << (S + i)));
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
#pragma unroll
                        for (int n = 0; n < NI; ++n)
                            gs_bf(x[n][qd * R + k], x[n][qd * R + k + half], w, c, !(CANON && S + i == LOGM - 1));
                } else {
                    const TwMul<false> w{tabf(TwKey{idx, S + i, S, i, h, G / Geo::s})};
#pragma unroll
                    for (int k = h * 2 * half; k < h * 2 * half + half; ++k)
#pragma unroll
                        for (int n = 0; n < NI; ++n)
                            gs_bf(x[n][qd * R + k], x[n][qd * R + k + half], w, c, !(CANON && S + i == LOGM - 1));
                }
            }
        }
    }
}

// Inverse round, one sub-transform per thread.
template <int LOGM, int LOGE, int RI, int OT_FROM, bool FUSE0, bool CANON = false, class TabF, class OtF, class C>
__device__ __forceinline__ void gs_round(uint64_t (&x)[16], uint32_t tib, uint32_t Fm1, const TabF& tabf,
                                         const OtF& otf, const C& c)
{
    gs_roundN<LOGM, LOGE, RI, OT_FROM, FUSE0, 1, CANON>(reinterpret_cast<uint64_t(&)[1][16]>(x), tib, Fm1, tabf, otf,
                                                         c);
}

// Canonical reduction at the end of a direction, for any x < 2^64:
//   q = floor(hi(x) * rn / 2^58),  rn = floor(2^90 / p) < 2^32 (p > 2^59),
// satisfies floor(x/p) - 1 <= q <= floor(x/p) (the dropped low word and the
// floor of rn each cost < 2^-26 of a unit), so x - q p lies in [0, 2p) and
// one exact conditional subtraction finishes: 1 IMAD.HI + 1 IMAD.WIDE +
// 1 IMAD instead of a chain of three or four conditional subtractions.
__device__ __forceinline__ uint64_t reduce_full(uint64_t x, const PrimeConst& c)
{
    const uint32_t q = __umulhi((uint32_t)(x >> 32), c.rn) >> 26;
    return csub(x - (uint64_t)q * c.p, c.p);
}
// Proth prime: q p = q + ((q p1) << 32) -- one IMAD instead of IMAD.WIDE + IMAD;
// the subtraction of both terms is one three-input add.
__device__ __forceinline__ uint64_t reduce_full(uint64_t x, const PrimeConstP& c)
{
    const uint32_t q = __umulhi((uint32_t)(x >> 32), c.rn) >> 26;
    const uint32_t qp1 = q * (0u - c.m1);  // q p1 (mod 2^32): p1 = -m1
    return csub(x - q - ((uint64_t)qp1 << 32), c.p);
}
#ifdef NTT_PROBE_NOMATH
template <class C>
__device__ __forceinline__ uint64_t norm8(uint64_t x, const C&) { return x; }
template <class C>
__device__ __forceinline__ uint64_t norm4(uint64_t x, const C&) { return x; }
#else
// d-form (PrimeConstD, p = 2^60 - d, d < 2^32): x = q 2^60 + lo60 with
// q = x >> 60 <= 15 and 2^60 = p + d, so x == lo60 + q d (mod p) and
//   r = lo60(x) + q d < 2^60 + 15 * 2^32 < 2p   (p > 2^60 - 2^32),
// one exact conditional subtraction finishes: one IMAD.WIDE (q d with the
// 64-bit addend lo60) instead of IMAD.HI + IMAD.WIDE + IMAD.  Any word.
// 2^64 - p = 0xF0000000:d, so d is the low word of c.np.
__device__ __forceinline__ uint64_t reduce_full(uint64_t x, const PrimeConstD& c)
{
    const uint32_t q = (uint32_t)(x >> 60);
    return csub((x & 0x0FFFFFFFFFFFFFFFull) + (uint64_t)q * (uint32_t)c.np, c.p);
}
template <class C>
__device__ __forceinline__ uint64_t norm8(uint64_t x, const C& c) { return reduce_full(x, c); }
// [0,4p) -> [0,p) (inverse outputs): two exact conditional subtractions, all
// on the ALU pipe -- cheaper than reduce_full where the multiply pipe binds.
template <class C>
__device__ __forceinline__ uint64_t norm4(uint64_t x, const C& c) { return csub(csub(x, c.p2), c.p); }
#endif

// SMEM swizzle for contiguous blocks: XOR word-address bits 1..3 with
// (bits 4..6 ^ bits 5..7).  16-byte pairs (2i, 2i+1) stay adjacent (vector
// copies), and every round access pattern of LOGM >= 8 -- 64-bit accesses,
// or 128-bit ones in the stride-1 rounds -- is bank-conflict free
// (DESIGN.md section 5.3).
__device__ __forceinline__ uint32_t swz(uint32_t e) { return e ^ ((((e >> 4) ^ (e >> 5)) & 7u) << 1); }

// Swizzled index of element k of a thread's group qd in one round, from the
// thread's base sB = swz(elem(tib, 0)) (RoundGeo::elem):
//   elem(qd TB + tib, k) = elem(tib, 0) + KS,  KS = elem(qd TB, k) a compile-time
// constant whose bits are disjoint from elem(tib, 0)'s, and swz(e) = e ^ f(e)
// with f linear over GF(2) in the bits of e -- so swz(B | KS) = sB ^ KS ^ f(KS).
// When KS has no bit in 1..3 that is (sB ^ f(KS)) + KS: at most 8 distinct
// LOP3s per round and immediate offsets, instead of a shift/mask/xor chain per
// element.
template <uint32_t KS>
__device__ __forceinline__ uint32_t swz_at(uint32_t sB)
{
    constexpr uint32_t f = (((KS >> 4) ^ (KS >> 5)) & 7u) << 1;
    if constexpr ((KS & 0xEu) == 0) {
        if constexpr (f == 0) {
            return sB + KS;
        } else {
            return (sB ^ f) + KS;
        }
    } else {
        return sB ^ (KS ^ f);
    }
}

// The same swizzled element as a SHARED-WINDOW BYTE address, from
// Pb = smem_addr(block) + 8 sB, the block's byte base already added:
//   swz_at<KS>(sB) = (sB ^ c) + rest,  c = (KS ^ f) & 0xE,  rest = KS & ~0xE
// (rest's bits are disjoint from sB's and c's, so the XOR never carries), and
// with the block base a multiple of 128 bytes (bits 4..6 clear, where 8c
// lands) smem(sb) + 8 swz_at = (Pb ^ 8c) + 8 rest: one LOP3 per distinct c
// (at most 8 per round) and an immediate offset -- no per-element add of the
// block base (which ptxas places on the multiply pipe as IMAD.IADD; measured
// on C4: Kernel-2' 1.255 -> 1.210 ms, Kernel-2 1.324 -> 1.309 ms,
// profiles/r02h_ab_swz_bytes.jsonl).
template <uint32_t KS>
struct SwzByte {
    static constexpr uint32_t f = (((KS >> 4) ^ (KS >> 5)) & 7u) << 1;
    static constexpr uint32_t c = (KS ^ f) & 0xEu;
    static constexpr uint32_t off = 8u * (KS & ~0xEu);
    __device__ __forceinline__ static uint32_t base(uint32_t Pb) { return c ? (Pb ^ (8u * c)) : Pb; }
};
template <uint32_t OFF>
__device__ __forceinline__ uint64_t lds64_at(uint32_t a)
{
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(OFF) : "memory");
    return v;
}
template <uint32_t OFF>
__device__ __forceinline__ void lds128_at(uint32_t a, uint64_t& x, uint64_t& y)
{
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2+%3];" : "=l"(x), "=l"(y) : "r"(a), "n"(OFF) : "memory");
}
template <uint32_t OFF>
__device__ __forceinline__ void sts64_at(uint32_t a, uint64_t v)
{
    asm volatile("st.shared.u64 [%0+%1], %2;" ::"r"(a), "n"(OFF), "l"(v) : "memory");
}
template <uint32_t OFF>
__device__ __forceinline__ void sts128_at(uint32_t a, uint64_t x, uint64_t y)
{
    asm volatile("st.shared.v2.u64 [%0+%1], {%2, %3};" ::"r"(a), "n"(OFF), "l"(x), "l"(y) : "memory");
}

}  // namespace ntt
