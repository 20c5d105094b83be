// params.h -- host parameter library (layer B0): NTT primes, psi, Shoup
// companions and the twiddle / OT table layouts the kernels read.
// Product code; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <vector>

namespace nttp {

// One Shoup pair (Algorithm 4): w in [0,p), wb = floor(w 2^64 / p).
// 16 bytes so a single 128-bit load fetches both (layout D1/D2 of SURVEY 2.3).
struct alignas(16) Twiddle {
    uint64_t w, wb;
};

uint64_t mul_mod(uint64_t a, uint64_t b, uint64_t m);
uint64_t pow_mod(uint64_t a, uint64_t e, uint64_t m);
bool is_prime_u64(uint64_t n);
Twiddle shoup_pair(uint64_t w, uint64_t p);

// NTT primes p = 1 mod 2N in [2^59, 2^60), descending from 2^60 - 2N + 1.
// Returns false if the range is exhausted before `count` primes.
bool ntt_primes(uint64_t N, unsigned count, std::vector<uint64_t>& out);
// Proth-form NTT primes p = k 2^32 + 1 in [2^59, 2^60), descending from
// 2^60 - 2^32 + 1 (ntt_find_primes_ex, NTT_PRIMES_PROTH32).
bool proth_primes(unsigned count, std::vector<uint64_t>& out);

// 32-bit word path (NEXT-4): primes p = 1 mod 2N in [2^29, 2^30), descending
// from 2^30 - 2N + 1; and the 32-bit Shoup pair wb = floor(w 2^32 / p).
bool ntt_primes32(uint64_t N, unsigned count, std::vector<uint32_t>& out);
bool valid_ntt_prime32(uint64_t p, uint64_t N);
struct Twiddle32 {
    uint32_t w, wb;
};
Twiddle32 shoup_pair32(uint32_t w, uint32_t p);

// Kernel-2 twiddle order (ntt::K2Layout, runtime form): block bb of a row owns
// N2 = 2^(logn - log_n1) entries; round (S, r) of the remainder-first radix-2^loge
// schedule stores Psi[(((F << S) + g) << i) + h] at off(S) + ((2^i - 1 + h) << S) + g,
// F = N1 + bb.  T is the table entry type (64- or 32-bit Shoup pair).
template <class T>
void k2_order(const T* std_tab, unsigned logn, unsigned log_n1, unsigned loge, T* out)
{
    // loge & 15: radix exponent; loge & 16: remainder round last (ntt::Sched)
    const bool remlast = (loge & 16u) != 0;
    const unsigned logm = logn - log_n1, le = (loge & 15u) < logm ? (loge & 15u) : logm;
    const uint32_t N1 = 1u << log_n1, N2 = 1u << logm;
    for (uint32_t bb = 0; bb < N1; ++bb) {
        const uint32_t F = N1 + bb;
        T* o = out + (uint64_t)bb * N2;
        o[0] = T{0, 0};
        uint32_t off = 1;
        const unsigned rem = logm % le;
        for (unsigned S = 0; S < logm;) {
            const unsigned r = remlast ? (logm - S < le ? logm - S : le) : ((S == 0 && rem) ? rem : le);
            for (unsigned i = 0; i < r; ++i)
                for (uint32_t h = 0; h < (1u << i); ++h)
                    for (uint32_t g = 0; g < (1u << S); ++g)
                        o[off + ((((1u << i) - 1u + h) << S) + g)] = std_tab[((((uint64_t)F << S) + g) << i) + h];
            off += ((1u << r) - 1u) << S;
            S += r;
        }
    }
}

// Smallest primitive 2N-th root of unity mod p (R2); 0 if none.
uint64_t smallest_psi(uint64_t p, uint64_t N);

// Validation used by plan creation: prime, p = 1 mod 2N, 2^59 <= p < 2^60.
bool valid_ntt_prime(uint64_t p, uint64_t N);

// Fills tab[i] = shoup_pair(root^bitrev_logn(i)) for i < N.
void bitrev_power_table(uint64_t p, uint64_t root, unsigned logn, Twiddle* tab);

// OT base tables: fine[r] = root^r (r < B), coarse[q] = root^(qB)
// (q < N/B), written contiguously as [fine | coarse].
void ot_base_tables(uint64_t p, uint64_t root, uint64_t N, uint64_t B, Twiddle* out);

}  // namespace nttp
