// params.cpp -- host parameter library (B0).  See params.h.
//
// The hot path never runs here: this is plan-time work,
// O(N L) with 128-bit host arithmetic.
#include "params.h"

namespace nttp {

using u128 = unsigned __int128;

uint64_t mul_mod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }

uint64_t pow_mod(uint64_t a, uint64_t e, uint64_t m)
{
    uint64_t acc = 1 % m, base = a % m;
    for (; e; e >>= 1, base = mul_mod(base, base, m))
        if (e & 1) acc = mul_mod(acc, base, m);
    return acc;
}

// Miller-Rabin with the first twelve primes as witnesses: deterministic below
// 3.3e24, hence for every 64-bit input.
bool is_prime_u64(uint64_t n)
{
    if (n < 2) return false;
    const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t q : small)
        if (n % q == 0) return n == q;
    unsigned s = __builtin_ctzll(n - 1);
    uint64_t d = (n - 1) >> s;
    for (uint64_t a : small) {
        uint64_t x = pow_mod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (unsigned i = 1; i < s && witness; ++i) {
            x = mul_mod(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

// w_bar = floor(w * 2^64 / p) (R6: the garbled "w x beta / p" of P:455).
Twiddle shoup_pair(uint64_t w, uint64_t p)
{
    Twiddle t;
    t.w = w;
    t.wb = (uint64_t)(((u128)w << 64) / p);
    return t;
}

bool ntt_primes(uint64_t N, unsigned count, std::vector<uint64_t>& out)
{
    out.clear();
    const uint64_t lo = 1ull << 59, step = 2 * N;
    for (uint64_t c = (1ull << 60) - step + 1; out.size() < count; c -= step) {
        if (c < lo) return false;
        if (is_prime_u64(c)) out.push_back(c);
    }
    return true;
}

bool proth_primes(unsigned count, std::vector<uint64_t>& out)
{
    return ntt_primes(1ull << 31, count, out);  // step 2^32: p = k 2^32 + 1
}

bool ntt_primes32(uint64_t N, unsigned count, std::vector<uint32_t>& out)
{
    out.clear();
    const uint64_t lo = 1ull << 29, step = 2 * N;
    for (uint64_t c = (1ull << 30) - step + 1; out.size() < count; c -= step) {
        if (c < lo || c > (1ull << 30)) return false;
        if (is_prime_u64(c)) out.push_back((uint32_t)c);
    }
    return true;
}

bool valid_ntt_prime32(uint64_t p, uint64_t N)
{
    return p < (1ull << 30) && p > 2 && (p - 1) % (2 * N) == 0 && is_prime_u64(p);
}

Twiddle32 shoup_pair32(uint32_t w, uint32_t p)
{
    return Twiddle32{w, (uint32_t)(((uint64_t)w << 32) / p)};
}

bool valid_ntt_prime(uint64_t p, uint64_t N)
{
    // [2^59, 2^60): the range P:423 names, and what the 64-bit kernels need --
    // reduce_full's quotient estimate floor(2^90 / p) must fit 32 bits (p > 2^58)
    // and the lazy bounds of DESIGN.md 5.1 need p < 2^60
    return p >= (1ull << 59) && p < (1ull << 60) && (p - 1) % (2 * N) == 0 && is_prime_u64(p);
}

uint64_t smallest_psi(uint64_t p, uint64_t N)
{
    if (N == 0 || p < 3 || (p - 1) % (2 * N) != 0 || !is_prime_u64(p)) return 0;
    // A quadratic non-residue z generates the 2-Sylow part fully, so
    // z^((p-1)/2N) has order exactly 2N; the primitive 2N-th roots are its odd
    // powers and we keep the least one.
    uint64_t z = 2;
    while (pow_mod(z, (p - 1) >> 1, p) != p - 1) ++z;
    const uint64_t g = pow_mod(z, (p - 1) / (2 * N), p);
    const uint64_t g2 = mul_mod(g, g, p);
    uint64_t best = g;
    for (uint64_t k = 1, x = g; k + 2 < 2 * N; k += 2) {
        x = mul_mod(x, g2, p);
        if (x < best) best = x;
    }
    return pow_mod(best, N, p) == p - 1 ? best : 0;
}

static inline uint32_t bitrev_bits(uint32_t i, unsigned bits)
{
    uint32_t r = 0;
    for (unsigned b = 0; b < bits; ++b, i >>= 1) r = (r << 1) | (i & 1u);
    return r;
}

void bitrev_power_table(uint64_t p, uint64_t root, unsigned logn, Twiddle* tab)
{
    const uint64_t N = 1ull << logn;
    std::vector<uint64_t> pw(N);
    uint64_t x = 1;
    for (uint64_t e = 0; e < N; ++e, x = mul_mod(x, root, p)) pw[e] = x;
    for (uint64_t i = 0; i < N; ++i) tab[i] = shoup_pair(pw[bitrev_bits((uint32_t)i, logn)], p);
}

void ot_base_tables(uint64_t p, uint64_t root, uint64_t N, uint64_t B, Twiddle* out)
{
    uint64_t x = 1;
    for (uint64_t r = 0; r < B; ++r, x = mul_mod(x, root, p)) out[r] = shoup_pair(x, p);
    const uint64_t step = pow_mod(root, B, p);
    x = 1;
    for (uint64_t q = 0; q < N / B; ++q, x = mul_mod(x, step, p)) out[B + q] = shoup_pair(x, p);
}

}  // namespace nttp
