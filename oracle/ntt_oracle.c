/*
 * oracle/ntt_oracle.c -- the CPU ORACLE for the batched negacyclic NTT / iNTT.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2012_01968_b200/) never includes, links or calls anything in oracle/,
 * and this file shares no code, header, table or constant generator with it.
 *
 * It is deliberately plain and slow: every modular product is the textbook
 * (unsigned __int128)a*b % p, there is no Shoup companion, no lazy reduction,
 * no blocking and no reordering beyond the paper's own loop order.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (read at build time
 * only; nothing here reads it at run time).  Readings of garbled or silent
 * passages are the numbered "R#" entries of DESIGN.md section 3.
 *
 * Parity pins (tests/test_oracle.py, -m "not gpu"): O(N^2) direct sum of the
 * P:242 definition in Python big integers, closed forms for delta and
 * constant inputs at N = 2^17, the SPEC worked examples (tests/golden/),
 * roundtrip, linearity, and the negacyclic convolution theorem
 * against a Python schoolbook product of P:227.  Every function below has a
 * pin; nothing here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- arithmetic */

/* (a*b) mod p by the definition: a 128-bit product and a remainder.  The paper
 * calls this the "native modulo operation". */
uint64_t oracle_mulmod(uint64_t a, uint64_t b, uint64_t p)
{
    return (uint64_t)(((u128)a * (u128)b) % (u128)p);
}

static uint64_t addmod(uint64_t a, uint64_t b, uint64_t p)
{
    return (uint64_t)(((u128)a + (u128)b) % (u128)p);
}

static uint64_t submod(uint64_t a, uint64_t b, uint64_t p)
{
    /* (a - b) mod p for a, b in [0, p) */
    return (uint64_t)(((u128)a + (u128)p - (u128)b) % (u128)p);
}

/* a^e mod p, square and multiply. */
uint64_t oracle_powmod(uint64_t a, uint64_t e, uint64_t p)
{
    uint64_t r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = oracle_mulmod(r, a, p);
        a = oracle_mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}

/* ------------------------------------------------------------------- primes */

/* Deterministic Miller-Rabin.  The witness set {2..37} is exact for all
 * n < 3.3e24, so for every 64-bit n.  Used to pick the RNS moduli of
 * P:271-276 ("np coprimes"), read as primes p = 1 mod 2N in [2^59, 2^60)
 * (R1, R3). */
int oracle_is_prime(uint64_t n)
{
    static const uint64_t W[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == W[i]) return 1;
        if (n % W[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = oracle_powmod(W[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int composite = 1;
        for (int r = 1; r < s; r++) {
            x = oracle_mulmod(x, x, n);
            if (x == n - 1) { composite = 0; break; }
        }
        if (composite) return 0;
    }
    return 1;
}

/* The first `count` primes p = 1 (mod 2N) with lo <= p < hi, scanning
 * downward from the largest such candidate below hi (R3).
 * Returns the number found (== count on success, less if the range ran out). */
int oracle_find_primes(uint64_t N, uint64_t lo, uint64_t hi, unsigned count, uint64_t *out)
{
    uint64_t step = 2 * N;
    if (N == 0 || hi < 2 || hi <= lo) return 0;
    uint64_t c = ((hi - 2) / step) * step + 1; /* largest c < hi with c = 1 mod 2N */
    unsigned found = 0;
    while (found < count) {
        if (c < lo || c < 2) break;
        if (oracle_is_prime(c)) out[found++] = c;
        if (c < step) break;
        c -= step;
    }
    return (int)found;
}

/* psi: a primitive 2N-th root of unity mod p (psi^N = -1), the root the
 * merged negacyclic transform is built on (R1).  Which root is
 * unstated in the paper; R2 fixes the SMALLEST primitive 2N-th
 * root.  Every primitive 2N-th root is psi0^k for odd k, where
 * psi0 = g^((p-1)/2N) and g is any quadratic non-residue, so the smallest
 * one is the minimum over the odd powers.  Returns 0 if p is unusable. */
uint64_t oracle_find_psi(uint64_t p, uint64_t N)
{
    if (N == 0 || p < 3 || (p - 1) % (2 * N) != 0) return 0;
    uint64_t g = 2;
    while (oracle_powmod(g, (p - 1) / 2, p) != p - 1) {
        g++;
        if (g >= p) return 0;
    }
    uint64_t psi0 = oracle_powmod(g, (p - 1) / (2 * N), p);
    uint64_t psi0_sq = oracle_mulmod(psi0, psi0, p);
    uint64_t best = psi0, cur = psi0;
    for (uint64_t k = 3; k < 2 * N; k += 2) {
        cur = oracle_mulmod(cur, psi0_sq, p);
        if (cur < best) best = cur;
    }
    if (oracle_powmod(best, N, p) != p - 1) return 0;
    return best;
}

/* ----------------------------------------------------------------- tables */

/* bit-reverse(i) over log2(N) bits. */
uint64_t oracle_bitrev(uint64_t i, unsigned logn)
{
    uint64_t r = 0;
    for (unsigned b = 0; b < logn; b++) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

static unsigned log2u(uint64_t N)
{
    unsigned l = 0;
    while ((1ull << l) < N) l++;
    return l;
}

/* Psi[i] = root^bit-reverse(i) mod p, i < N (Algorithm 1 REQUIRE, P:297;
 * P:343).  With root = psi^-1 this is the inverse table of R5. */
void oracle_psi_table(uint64_t p, uint64_t root, uint64_t N, uint64_t *out)
{
    unsigned logn = log2u(N);
    uint64_t *pw = (uint64_t *)malloc(sizeof(uint64_t) * (N ? N : 1));
    uint64_t x = 1 % p;
    for (uint64_t e = 0; e < N; e++) { pw[e] = x; x = oracle_mulmod(x, root, p); }
    for (uint64_t i = 0; i < N; i++) out[i] = pw[oracle_bitrev(i, logn)];
    free(pw);
}

/* ------------------------------------------------------------- transforms */

static int valid_n(uint64_t N)
{
    return N >= 1 && (N & (N - 1)) == 0;
}

/* Forward merged negacyclic NTT, Algorithm 1 (Cooley-Tukey) with
 * the butterfly of Algorithm 2 written with exact remainders:
 *   t = N/2; for m = 1, 2, ..., N/2: for j < m: for k in [2jt, 2jt+t):
 *     V = a[k+t] * Psi[m+j] mod p; a[k+t] = a[k] - V; a[k] = a[k] + V  (mod p)
 *   t = t/2.
 * Output: bit-reversed order, position i holds A_{bitrev(i)} with
 * A_k = sum_n a_n psi^{n(2k+1)}.  Inputs must be in [0, p). */
int oracle_ntt_forward(uint64_t *a, uint64_t N, uint64_t p, uint64_t psi)
{
    if (!valid_n(N)) return -1;
    uint64_t *Psi = (uint64_t *)malloc(sizeof(uint64_t) * N);
    oracle_psi_table(p, psi, N, Psi);
    uint64_t t = N / 2;
    for (uint64_t m = 1; m < N; m *= 2) {
        for (uint64_t j = 0; j < m; j++) {
            uint64_t W = Psi[m + j];
            for (uint64_t k = j * 2 * t; k < j * 2 * t + t; k++) {
                uint64_t U = a[k];
                uint64_t V = oracle_mulmod(a[k + t], W, p);
                a[k] = addmod(U, V, p);
                a[k + t] = submod(U, V, p);
            }
        }
        t /= 2;
    }
    free(Psi);
    return 0;
}

/* Inverse merged negacyclic NTT ("merged into the iNTT"; the commented
 * formula P:248-257 c_k = N^-1 sum_n C_n psi^{-k(2n+1)}).  The paper gives no
 * pseudo-code; R5 reads it as Gentleman-Sande on a bit-reversed
 * input with Psi^-1[i] = psi^{-bitrev(i)}:
 *   t = 1; for m = N/2, ..., 1: for j < m: for k in [2jt, 2jt+t):
 *     U = a[k]; V = a[k+t]; a[k] = U + V; a[k+t] = (U - V) * Psi^-1[m+j]
 *   t = 2t;  finally a[i] = a[i] * N^-1  (all mod p). */
int oracle_ntt_inverse(uint64_t *a, uint64_t N, uint64_t p, uint64_t psi)
{
    if (!valid_n(N)) return -1;
    uint64_t psi_inv = oracle_powmod(psi, p - 2, p);
    uint64_t n_inv = oracle_powmod(N % p, p - 2, p);
    uint64_t *Pinv = (uint64_t *)malloc(sizeof(uint64_t) * N);
    oracle_psi_table(p, psi_inv, N, Pinv);
    uint64_t t = 1;
    for (uint64_t m = N / 2; m >= 1; m /= 2) {
        for (uint64_t j = 0; j < m; j++) {
            uint64_t W = Pinv[m + j];
            for (uint64_t k = j * 2 * t; k < j * 2 * t + t; k++) {
                uint64_t U = a[k];
                uint64_t V = a[k + t];
                a[k] = addmod(U, V, p);
                a[k + t] = oracle_mulmod(submod(U, V, p), W, p);
            }
        }
        t *= 2;
    }
    for (uint64_t i = 0; i < N; i++) a[i] = oracle_mulmod(a[i], n_inv, p);
    free(Pinv);
    return 0;
}

/* Negacyclic product by its definition:
 *   c_k = sum_{i<=k} a_i b_{k-i} - sum_{i>k} a_i b_{N+k-i}   (mod p). */
void oracle_negacyclic_mul(const uint64_t *a, const uint64_t *b, uint64_t *c, uint64_t N, uint64_t p)
{
    for (uint64_t k = 0; k < N; k++) {
        uint64_t s = 0;
        for (uint64_t i = 0; i <= k; i++) s = addmod(s, oracle_mulmod(a[i], b[k - i], p), p);
        for (uint64_t i = k + 1; i < N; i++) s = submod(s, oracle_mulmod(a[i], b[N + k - i], p), p);
        c[k] = s;
    }
}

/* Element-wise product in the NTT domain (the odot). */
void oracle_pointwise_mul(const uint64_t *a, const uint64_t *b, uint64_t *c, uint64_t N, uint64_t p)
{
    for (uint64_t i = 0; i < N; i++) c[i] = oracle_mulmod(a[i], b[i], p);
}

/* ------------------------------------------------------------------ batch */

/* RNS batching: rows are laid out [batch][L][N]; row
 * (b, l) is a residue polynomial mod primes[l] and is transformed on its own.
 * Rows are dealt round-robin to nthreads plain POSIX threads (0 = all online
 * cores).  direction: +1 forward, -1 inverse. */
typedef struct {
    uint64_t *data;
    uint64_t N;
    const uint64_t *primes, *psis;
    unsigned L, rows, tid, nth;
    int direction, status;
} job_t;

static void *worker(void *arg)
{
    job_t *j = (job_t *)arg;
    for (unsigned r = j->tid; r < j->rows; r += j->nth) {
        unsigned l = r % j->L;
        uint64_t *row = j->data + (uint64_t)r * j->N;
        int s = j->direction > 0 ? oracle_ntt_forward(row, j->N, j->primes[l], j->psis[l])
                                 : oracle_ntt_inverse(row, j->N, j->primes[l], j->psis[l]);
        if (s) j->status = s;
    }
    return 0;
}

int oracle_ntt_batch(uint64_t *data, uint64_t N, const uint64_t *primes, const uint64_t *psis,
                     unsigned L, unsigned batch, int direction, unsigned nthreads)
{
    if (!valid_n(N) || L == 0) return -1;
    unsigned rows = L * batch;
    if (rows == 0) return 0;
    if (nthreads == 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        nthreads = c > 0 ? (unsigned)c : 1;
    }
    if (nthreads > rows) nthreads = rows;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
    for (unsigned t = 0; t < nthreads; t++) {
        job_t jb = {data, N, primes, psis, L, rows, t, nthreads, direction, 0};
        jobs[t] = jb;
        pthread_create(&th[t], 0, worker, &jobs[t]);
    }
    int status = 0;
    for (unsigned t = 0; t < nthreads; t++) {
        pthread_join(th[t], 0);
        if (jobs[t].status) status = jobs[t].status;
    }
    free(th);
    free(jobs);
    return status;
}
