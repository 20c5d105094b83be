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

// Smallest primitive 2N-th root of unity mod p (R2); 0 if none.
uint64_t smallest_psi(uint64_t p, uint64_t N);

// Validation used by plan creation: prime, p = 1 mod 2N, p < 2^60.
bool valid_ntt_prime(uint64_t p, uint64_t N);

// Fills tab[i] = shoup_pair(root^bitrev_logn(i)) for i < N.
void bitrev_power_table(uint64_t p, uint64_t root, unsigned logn, Twiddle* tab);

// OT base tables: fine[r] = root^r (r < B), coarse[q] = root^(qB)
// (q < N/B), written contiguously as [fine | coarse].
void ot_base_tables(uint64_t p, uint64_t root, uint64_t N, uint64_t B, Twiddle* out);

}  // namespace nttp
