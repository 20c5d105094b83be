/*
 * synth/synth.c -- seeded synthetic RNS residue rows.
 *
 * The ONE module both the oracle side and the CUDA side draw inputs from.  It
 * holds none of the method's arithmetic (no NTT, no Shoup, no twiddles): it
 * only maps a counter to a uniform value in [0, p).
 *
 *   x[row][i] = mulhi64(splitmix64(seed ^ ((config_id << 48) | (row << 20) | i)), p_row)
 *
 * splitmix64 is the standard 64-bit finaliser (Steele, Lea, Flood 2014);
 * mulhi64(z, p) = floor(z * p / 2^64) maps a uniform 64-bit z to [0, p).
 * Residues of HE ciphertexts are uniform mod each prime, which is
 * what this draws.
 */
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <unistd.h>

static inline uint64_t splitmix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t seed, uint64_t config_id, uint64_t row, uint64_t i, uint64_t p)
{
    uint64_t z = splitmix64(seed ^ ((config_id << 48) | (row << 20) | i));
    return (uint64_t)(((unsigned __int128)z * p) >> 64);
}

typedef struct {
    uint64_t *out;
    uint64_t N;
    const uint64_t *row_ids, *row_primes;
    uint64_t nrows, seed, config_id;
    unsigned tid, nth;
} fill_t;

static void *fill_worker(void *arg)
{
    fill_t *f = (fill_t *)arg;
    for (uint64_t r = f->tid; r < f->nrows; r += f->nth) {
        uint64_t *o = f->out + r * f->N;
        uint64_t id = f->row_ids[r], p = f->row_primes[r];
        for (uint64_t i = 0; i < f->N; i++) o[i] = draw(f->seed, f->config_id, id, i, p);
    }
    return 0;
}

/* out: nrows x N words.  Row r gets global row id row_ids[r] and modulus
 * row_primes[r].  nthreads 0 = all online cores. */
void synth_fill_rows(uint64_t *out, uint64_t N, const uint64_t *row_ids, const uint64_t *row_primes,
                     uint64_t nrows, uint64_t seed, uint64_t config_id, unsigned nthreads)
{
    if (nrows == 0) return;
    if (nthreads == 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        nthreads = c > 0 ? (unsigned)c : 1;
    }
    if (nthreads > nrows) nthreads = (unsigned)nrows;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    fill_t *jobs = (fill_t *)malloc(sizeof(fill_t) * nthreads);
    for (unsigned t = 0; t < nthreads; t++) {
        fill_t f = {out, N, row_ids, row_primes, nrows, seed, config_id, t, nthreads};
        jobs[t] = f;
        pthread_create(&th[t], 0, fill_worker, &jobs[t]);
    }
    for (unsigned t = 0; t < nthreads; t++) pthread_join(th[t], 0);
    free(th);
    free(jobs);
}
