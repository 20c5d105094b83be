/*
 * include/ntt.h -- C ABI of libntt.so: the batched merged-negacyclic NTT / iNTT
 * over RNS residue rows on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (arxiv 2012.01968);
 * "R#" = the readings of silent/garbled passages in DESIGN.md section 3.
 *
 * General rules (all entry points):
 *  - No C++ type, exception or torch type crosses this boundary.  Pointers are
 *    plain host or device pointers as stated per argument; sizes are unsigned.
 *  - Every function returns an ntt_status_t.  Argument errors are detected
 *    synchronously, before anything is enqueued, and leave all buffers
 *    untouched.  A CUDA launch failure is reported once as NTT_ERR_CUDA (the
 *    library consumes it with cudaGetLastError, so it does not poison later
 *    calls); asynchronous faults surface at the caller's next
 *    synchronisation, as for any CUDA library.
 *  - batch * L * N1 (N1 = 2^log_n1 of the split, 1 for one kernel per row)
 *    must be below 2^31 on every call that enqueues work, else INVALID_ARG.
 *  - Every entry point may be called from any number of host threads; the
 *    library's one-time per-device kernel setup is internally synchronised.
 *  - A plan is immutable after ntt_plan_create; concurrent ntt_forward /
 *    ntt_inverse calls with one plan on different streams and disjoint buffers
 *    are safe.  ntt_plan_destroy requires all work using the plan to be done.
 *  - There is no CPU fallback: without a usable CUDA device ntt_plan_create
 *    returns NTT_ERR_CUDA.
 */
#ifndef NTT_B200_H
#define NTT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ntt_plan_s *ntt_plan_t;

#define NTT_DIR_FORWARD 1u
#define NTT_DIR_INVERSE 2u

typedef enum {
    NTT_OK = 0,
    NTT_ERR_INVALID_N = -1,       /* N not a power of two in [2^1, 2^17] */
    NTT_ERR_INVALID_PRIME = -2,   /* not prime, not = 1 mod 2N, outside [2^59, 2^60), or repeated */
    NTT_ERR_INVALID_ARG = -3,     /* null pointer, bad option value */
    NTT_ERR_MISALIGNED = -4,      /* data pointer not 16-byte aligned */
    NTT_ERR_WRONG_DEVICE = -5,    /* data pointer not on the plan's device */
    NTT_ERR_CUDA = -6,            /* CUDA runtime error (no device, launch failure) */
    NTT_ERR_OOM = -7,             /* device or pinned allocation failed */
    NTT_ERR_RANGE_EXHAUSTED = -8  /* fewer primes than requested in [2^59, 2^60) */
} ntt_status_t;

/* Options; a zero field means "default". */
typedef struct {
    int ot_enable;       /* on-the-fly twiddling in the last ot_stages
                            forward stages and the first ot_stages inverse stages:
                            0 = default (off), 1 = on, -1 = off */
    unsigned ot_base;    /* OT base B, power of two dividing N;
                            0 = 1024 for N >= 2^11, else 2^ceil(logN/2) (R11) */
    unsigned ot_stages;  /* 1 or 2 (fig:3point c); 0 = 2 */
    unsigned log_n1;     /* two-kernel split N = N1*N2, log2 N1;
                            0 = automatic; ignored when one kernel holds the row */
    int prime_arith;     /* 0 = automatic: when EVERY prime is = 1 mod 2^32
                            ("Proth") the kernels form lo64(q p) of Shoup's
                            modmul as q + (q0 p1 << 32) (DESIGN.md
                            5.1); -1 = always the general arithmetic.  Results
                            are identical either way. */
    int fused;           /* single pass per direction for N = 2^14..2^17: one
                            thread-block cluster of N/2^13 CTAs holds the row in
                            distributed shared memory, so each word crosses HBM
                            once per direction instead of twice (the paper's
                            two-kernel premise, lifted).  0 / -1 = off
                            (the two-kernel split: measured faster on B200, where
                            the path is bound by the multiply pipe, not HBM --
                            DESIGN.md 5.5), 1 = on (NTT_ERR_INVALID_ARG if N is
                            outside 2^14..2^17, OT is on or log_n1 is given). */
    int k1_variant;      /* Kernel-1 form (experiments): 0 = default
                            (4: one 16-column tile per CTA), 5 = persistent
                            cp.async-pipelined.  Other values: INVALID_ARG. */
    int k2_variant;      /* Kernel-2 form: 0 = default (9: shared-twiddle CTA per
                            block position, remainder-last schedule), 7 = the same
                            remainder-first, 5 = persistent pipelined radix 16,
                            6 = persistent radix 8, 3 / 4 = one-shot radix 8 / 16.
                            Non-default forms other than 5 / 7 run the general
                            arithmetic.  Other values: INVALID_ARG. */
} ntt_opts_t;

/* Prime families for ntt_find_primes_ex. */
#define NTT_PRIMES_2N 0u      /* p = 1 mod 2N, descending from 2^60 - 2N + 1 (R3) */
#define NTT_PRIMES_PROTH32 1u /* p = 1 mod 2^32 (hence = 1 mod 2N for N <= 2^17),
                                 descending from 2^60 - 2^32 + 1 */

/* ntt_find_primes -- host helper, no device needed.
 * Writes the first `count` primes p = 1 (mod 2N), 2^59 <= p < 2^60, scanning
 * downward from 2^60 - 2N + 1 (R1, R3) into out[0..count).
 * Deterministic.  n = N (power of two, 2 <= N <= 2^17).
 * Errors: INVALID_N, INVALID_ARG (out == NULL or count == 0), RANGE_EXHAUSTED. */
ntt_status_t ntt_find_primes(unsigned n, unsigned count, uint64_t *out);

/* ntt_find_primes_ex -- as ntt_find_primes, for a prime family:
 *   NTT_PRIMES_2N      : identical to ntt_find_primes;
 *   NTT_PRIMES_PROTH32 : the first `count` primes p = k 2^32 + 1 in
 *                        [2^59, 2^60), descending.  P:423 fixes only the range
 *                        ("between 2^59 and 2^60") and p = 1 mod N (R1);
 *                        this family meets both for every N <= 2^17 and lets
 *                        the kernels drop one 32x32 product per modmul.
 * out: host array of `count` uint64 (caller-owned).  Errors: INVALID_N,
 * INVALID_ARG (null out, count 0, unknown form), RANGE_EXHAUSTED. */
ntt_status_t ntt_find_primes_ex(unsigned n, unsigned count, unsigned form, uint64_t *out);

/* ntt_find_psi -- host helper.  The smallest primitive 2N-th root of unity mod
 * p (psi^N = -1; R2) into *psi.  Errors: INVALID_N, INVALID_PRIME. */
ntt_status_t ntt_find_psi(uint64_t p, unsigned n, uint64_t *psi);

/* ntt_plan_create / _ex -- build a plan for ring degree n = N and the RNS
 * chain primes[0..L).  Copies primes[].  On the device current at
 * the call it allocates and fills, per prime and direction, the bit-reversed
 * twiddle table Psi[i] = psi^bitrev(i) resp.
 * Psi^-1[i] = psi^-bitrev(i) (R5) with Shoup companions
 * w_bar = floor(w 2^64 / p) (Algorithm 4; R6), the OT base tables
 * fine[r] = psi^r, coarse[q] = psi^(qB) and their inverses, and
 * N^-1.  The plan owns these allocations.  Synchronous.
 * Errors: INVALID_ARG (plan == NULL, primes == NULL, L == 0, L > 65535 -- a
 * grid dimension of the kernels --, bad options),
 * INVALID_N, INVALID_PRIME, CUDA (no device), OOM. */
ntt_status_t ntt_plan_create(ntt_plan_t *plan, unsigned n, const uint64_t *primes, unsigned L);
ntt_status_t ntt_plan_create_ex(ntt_plan_t *plan, unsigned n, const uint64_t *primes, unsigned L,
                                const ntt_opts_t *opts);

/* ntt_plan_psi -- copies the plan's psi for each prime into psi_out[0..L)
 * (host memory), so tests can assert the oracle picked the same root. */
ntt_status_t ntt_plan_psi(ntt_plan_t plan, uint64_t *psi_out);

/* ntt_plan_info -- host query: L, log2 N, log2 N1 of the split actually used
 * (0 when one kernel holds the whole row), OT on/off, OT base, OT stages,
 * and device-table bytes.  Any output pointer may be NULL. */
ntt_status_t ntt_plan_info(ntt_plan_t plan, unsigned *L, unsigned *logn, unsigned *log_n1,
                           int *ot_enable, unsigned *ot_base, unsigned *ot_stages,
                           uint64_t *table_bytes);

/* ntt_plan_exec -- host query of how the plan executes (any output may be NULL):
 * *arith   = the Shoup arithmetic the kernels run (ntt_opts_t.prime_arith):
 *            NTT_ARITH_GENERAL, NTT_ARITH_PROTH (every prime = 1 mod 2^32),
 *            or NTT_ARITH_GENERAL_D: the general arithmetic with every prime
 *            p = 2^60 - d, d < 2^32 (e.g. the chain ntt_find_primes scans), where
 *            the forward Kernel-2's final reduction takes the d-form and
 *            Kernel-1' applies N^-1 as an exact division;
 *            results are identical in every case;
 * *passes  = kernels per direction (1: single CTA or single-pass cluster
 *            kernel; 2: the paper's two-kernel split);
 * *cluster = CTAs per row of the single-pass cluster kernel (N / 2^13), 1 if
 *            it is not used. */
#define NTT_ARITH_GENERAL 0
#define NTT_ARITH_PROTH 1
#define NTT_ARITH_GENERAL_D 2
ntt_status_t ntt_plan_exec(ntt_plan_t plan, int *arith, unsigned *passes, unsigned *cluster);

/* ntt_forward -- in-place forward merged negacyclic NTT of batch*L rows.
 *   data: DEVICE pointer on the plan's device, 16-byte aligned, to
 *         batch x L x N uint64 words, row-major [b][l][i]; row (b, l) holds a
 *         polynomial with coefficients in [0, primes[l]) (precondition, not
 *         checked on the device; out-of-range input gives an undefined result).
 *   On completion position i of a row holds A_{bitrev(i)} with
 *   A_k = sum_j a_j psi^{j(2k+1)} mod p (bit-reversed order P:298; R4),
 *   canonical in [0, p) (R10).
 *   stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *   Asynchronous: returns after enqueuing.  batch == 0 is a no-op (NTT_OK).
 *   Errors: INVALID_ARG (plan/data NULL), MISALIGNED, WRONG_DEVICE, CUDA. */
ntt_status_t ntt_forward(ntt_plan_t plan, uint64_t *data, unsigned batch, void *stream);

/* ntt_inverse -- in-place inverse: bit-reversed NTT-domain rows in [0, p) to
 * natural-order coefficients c_k = N^-1 sum_n C_n psi^{-k(2n+1)} (
 * R5, R15), canonical in [0, p).  ntt_inverse(ntt_forward(x)) == x exactly.
 * Same arguments, layout, ownership and errors as ntt_forward. */
ntt_status_t ntt_inverse(ntt_plan_t plan, uint64_t *data, unsigned batch, void *stream);

/* ntt_launch_pass -- enqueue ONE kernel of a direction, for per-kernel timing
 * (bench.py brackets each with CUDA events).  dir: NTT_DIR_FORWARD or
 * NTT_DIR_INVERSE; pass: 0 or 1 in execution order.  Two-kernel plans
 * (ntt_plan_info log_n1 != 0) have passes 0 and 1 -- forward: Kernel-1
 * (columns) then Kernel-2 (blocks); inverse: Kernel-2' then Kernel-1' -- and
 * ntt_forward == pass 0 then pass 1 on one stream; single-kernel plans have
 * pass 0 only.  Same data contract as ntt_forward; the intermediate state
 * between passes is defined only for the pass sequence.
 * Errors: as ntt_forward, plus INVALID_ARG for a pass the plan lacks. */
ntt_status_t ntt_launch_pass(ntt_plan_t plan, uint64_t *data, unsigned batch, unsigned dir, unsigned pass,
                             void *stream);

/* ntt_pointwise_inverse -- data <- iNTT(a_ntt (.) data): the element-wise
 * product in the NTT domain followed by the inverse, i.e. the
 * output side of a negacyclic polynomial product.  The
 * product (Montgomery, R = 2^64; the R^-1 is folded into the inverse's N^-1)
 * is fused into the inverse's first kernel when the plan runs without OT,
 * otherwise it is a separate element-wise kernel.
 *   a_ntt, data: DEVICE pointers, layout as ntt_forward, both in the
 *   bit-reversed NTT domain with words in [0, p) (as ntt_forward returns);
 *   a_ntt is read only; data is overwritten with canonical coefficients.
 * Errors: as ntt_forward. */
ntt_status_t ntt_pointwise_inverse(ntt_plan_t plan, const uint64_t *a_ntt, uint64_t *data, unsigned batch,
                                   void *stream);

/* ntt_negacyclic_mul -- b <- a * b mod (X^N + 1, p_l) for every row:
 * ntt_forward(a), ntt_forward(b), ntt_pointwise_inverse(a, b).  On return a
 * holds NTT(a) (bit-reversed) and b the product's coefficients in [0, p).
 * a and b must be distinct.  Errors: as ntt_forward, INVALID_ARG if a == b. */
ntt_status_t ntt_negacyclic_mul(ntt_plan_t plan, uint64_t *a, uint64_t *b, unsigned batch, void *stream);

/* ntt_forward_variant -- the forward transform through one of the paper's
 * comparison implementations, rebuilt for sm_100a:
 *   NTT_VARIANT_DEFAULT  (0): the two-kernel SMEM path (== ntt_forward);
 *   NTT_VARIANT_RADIX2   (1): Algorithm 1, one launch per stage, every
 *                             butterfly through global memory;
 *                             the paper's radix-2 vs SMEM ratio (Table 2
 *                             P:850-866);
 *   NTT_VARIANT_RADIX16  (2): register-based radix-16 passes, no shared
 *                             memory, ceil(log2 N / 4) launches;
 *   NTT_VARIANT_NATIVE   (3): the default kernels (same split, same schedule)
 *                             with every twiddle product reduced by the native
 *                             modulo operation, (unsigned __int128)(b w) % p,
 *                             instead of Shoup's modmul -- the paper's "Native"
 *                             arm of fig:native_shoup ((2^17, 45)).
 *                             No OT, not for plans with the cluster kernel.
 * Output identical to ntt_forward (bit-exact).  Same data contract and errors,
 * plus INVALID_ARG for an unknown variant (or NATIVE on a fused / OT plan). */
#define NTT_VARIANT_DEFAULT 0u
#define NTT_VARIANT_RADIX2 1u
#define NTT_VARIANT_RADIX16 2u
#define NTT_VARIANT_NATIVE 3u
ntt_status_t ntt_forward_variant(ntt_plan_t plan, uint64_t *data, unsigned batch, unsigned variant, void *stream);

/* ntt_execute_host -- the end-to-end path with HOST buffers: for each chunk of
 * ciphertexts, copy host_in -> device workspace, run the requested transforms
 * (flags: NTT_DIR_FORWARD, NTT_DIR_INVERSE, or both = forward then inverse),
 * copy back to host_out (may equal host_in).  Chunks are pipelined over three
 * internal streams (pipeline slots) so chunk k's H2D, chunk k-1's kernels and
 * chunk k-2's D2H overlap.
 *   host_in/host_out: HOST pointers to batch x L x N words (pinned memory gives
 *   overlap; pageable memory works but serialises).
 *   workspace: DEVICE pointer on the plan's device, 16-byte aligned, of at
 *   least ntt_workspace_words(plan, chunk) words; chunk = ciphertexts per
 *   pipeline step (0 = automatic).
 *   stream: cudaStream_t (as void*, NULL = legacy default stream) the
 *   workspace is ordered on: the internal streams wait for the work already
 *   queued on it before touching the workspace (e.g. a stream-ordered
 *   allocation that is still in use).
 *   Synchronous: returns when host_out holds the result.
 *   Errors: as ntt_forward, plus INVALID_ARG for a too-small workspace. */
ntt_status_t ntt_execute_host(ntt_plan_t plan, unsigned flags, const uint64_t *host_in, uint64_t *host_out,
                              unsigned batch, uint64_t *workspace, uint64_t workspace_words, unsigned chunk,
                              void *stream);

/* Words of device workspace ntt_execute_host needs for a given chunk (0 = auto). */
uint64_t ntt_workspace_words(ntt_plan_t plan, unsigned batch, unsigned chunk);

/* ntt_plan_destroy -- frees the plan's device tables and host state.
 * NULL is accepted (no-op).  Caller must have synchronised all work. */
ntt_status_t ntt_plan_destroy(ntt_plan_t plan);

/* ---------------------------------------------------------------- request graphs
 * Small requests (one ciphertext of a few primes, BASELINE config 5) are bound
 * by host launch cost, not by the kernels.  A request graph is
 * the CUDA graph of one fixed call -- the kernels of the forward and / or
 * inverse transform of `batch` ciphertexts at a fixed device buffer --
 * captured once and replayed with one cudaGraphLaunch per request: the caller
 * copies each request into the buffer (or produces it there) and launches.
 *
 * ntt_graph_create -- capture the transforms `flags` (NTT_DIR_FORWARD,
 * NTT_DIR_INVERSE, or both = forward then inverse; NTT_GRAPH_PRODUCT = the
 * negacyclic product b <- a * b of ntt_negacyclic_mul with a = data and
 * b = data2) of plan over data[0 .. batch*L*N) into *graph.  data / data2:
 * DEVICE pointers as for ntt_forward; they are baked into the graph and must
 * stay valid while it exists.  The graph holds a reference to the plan's
 * tables: destroy the graph before the plan.  Synchronous; enqueues nothing.
 *
 * NTT_GRAPH_ONE_KERNEL (or'ed with the direction flags): the request is ONE
 * cooperative kernel instead of two per direction -- the column and block
 * passes of the split run as phases of one persistent grid with
 * grid barriers between them (ntt_request.cu), for the
 * latency of small requests (BASELINE config 5).  Results are identical to
 * the two-kernel path's.  The graph then owns 8 bytes of device memory (the
 * barrier state).  Requires N = 2^14..2^17, OT off, and a job the device can
 * hold co-resident in one wave of its grid (any batch works; large jobs are
 * faster without the flag).
 * Errors: as ntt_forward, INVALID_ARG (graph NULL, flags 0 or unknown,
 * batch 0, data2 NULL with NTT_GRAPH_PRODUCT, ONE_KERNEL with PRODUCT, OT,
 * or N outside 2^14..2^17), CUDA (capture failed). */
typedef struct ntt_graph_s *ntt_graph_t;
#define NTT_GRAPH_PRODUCT 4u
#define NTT_GRAPH_ONE_KERNEL 8u
ntt_status_t ntt_graph_create(ntt_graph_t *graph, ntt_plan_t plan, uint64_t *data, uint64_t *data2, unsigned batch,
                              unsigned flags);

/* ntt_graph_launch -- enqueue one replay of the graph on `stream`
 * (cudaStream_t as void*, NULL = legacy default).  Asynchronous, ordered
 * after earlier work on `stream`.  A graph must not be replayed concurrently
 * with itself on two streams (its buffer is shared).  Errors: INVALID_ARG
 * (graph NULL), CUDA. */
ntt_status_t ntt_graph_launch(ntt_graph_t graph, void *stream);

/* ntt_graph_destroy -- frees the graph; NULL accepted.  Replays must be done. */
ntt_status_t ntt_graph_destroy(ntt_graph_t graph);

/* ---------------------------------------------------------------- host helpers for tests
 * ntt_shoup_companion -- *wb = floor(w 2^64 / p), the Shoup companion of w
 * (Algorithm 4 precompute; R6) exactly as the plan tables store it.
 * Host only.  Errors: INVALID_ARG (wb NULL, p < 2, w >= p). */
ntt_status_t ntt_shoup_companion(uint64_t w, uint64_t p, uint64_t *wb);

/* ntt_table_sizes -- the twiddle storage a plan with (n, L, OT base) holds,
 * from the same function plan creation sizes its allocations with.  Host only.
 *   *psi_bytes  = bytes of one direction's bit-reversed tables, L x N
 *                 (w, w_bar) pairs ("2 N np words" doubled by w_bar);
 *   *ot_entries = (w, w_bar) pairs of one prime's OT base tables,
 *                 B + N / B;
 *   *plan_bytes = all device bytes of a default (two-kernel) plan.
 * Any output may be NULL.  ot_base 0 = the default of ntt_opts_t.
 * Errors: INVALID_N, INVALID_ARG (L == 0, bad base). */
ntt_status_t ntt_table_sizes(unsigned n, unsigned L, unsigned ot_base, uint64_t *psi_bytes, uint64_t *ot_entries,
                             uint64_t *plan_bytes);

/* ntt_debug_corrupt_twiddle -- TESTING ONLY (fault injection for the parity
 * harness): XOR `mask` into the twiddle w (field 0) or its Shoup companion
 * w_bar (field 1) of Psi[index] (dir NTT_DIR_FORWARD) or Psi^-1[index]
 * (NTT_DIR_INVERSE) of prime l, in every device copy of the plan's
 * bit-reversed tables (the standard and the Kernel-2-ordered one; the OT base
 * tables are not touched).  XOR-ing the same mask again restores the plan.
 * Synchronous (device-wide).  Errors: INVALID_ARG (bad dir / l / index /
 * field), CUDA. */
ntt_status_t ntt_debug_corrupt_twiddle(ntt_plan_t plan, unsigned dir, unsigned l, unsigned index, unsigned field,
                                       uint64_t mask);

/* ---------------------------------------------------------------- 32-bit words
 * The paper's 32-bit-word alternative ("32b vs 64b"; SURVEY 8(f)
 * NEXT-4): residues of primes 2^29 <= p < 2^30 stored one per uint32 word, with
 * 32-bit Shoup pairs w_bar = floor(w 2^32 / p) (Algorithm 4, with
 * beta = 2^32).  A modulus Q of the same size needs about twice as many primes
 * as the 60-bit path.  The transform, its order and its canonical output are
 * those of ntt_forward / ntt_inverse (R4, R5, R10, R15); no
 * OT and no fused product on this path.  Same general rules as above. */
typedef struct ntt32_plan_s *ntt32_plan_t;

/* ntt_find_primes32 -- host helper: the first `count` primes p = 1 (mod 2N),
 * 2^29 <= p < 2^30, scanning downward from 2^30 - 2N + 1, into out[0..count).
 * Errors: INVALID_N, INVALID_ARG (out == NULL or count == 0), RANGE_EXHAUSTED. */
ntt_status_t ntt_find_primes32(unsigned n, unsigned count, uint32_t *out);

/* ntt_plan_create32 -- plan for N = n and primes[0..L) (each prime, = 1 mod 2N,
 * < 2^30, distinct; copied).  Builds, on the current device, Psi / Psi^-1
 * bit-reversed tables with 32-bit Shoup companions (8 bytes per entry), their
 * Kernel-2 ordered copies for N >= 2^14, and N^-1.  log_n1: two-kernel split
 * N = N1 N2; 0 = default (7 for N <= 2^15, else 8), otherwise one
 * of (N, log_n1) = (2^14, 7), (2^15, 7), (2^16, 8), (2^17, 8), (2^17, 9);
 * ignored for N <= 2^13 (one kernel holds the row).  Synchronous.
 * Errors: INVALID_ARG (NULLs, L == 0, unsupported split), INVALID_N,
 * INVALID_PRIME, CUDA (no device), OOM. */
ntt_status_t ntt_plan_create32(ntt32_plan_t *plan, unsigned n, const uint32_t *primes, unsigned L,
                               unsigned log_n1);

/* ntt_plan_info32 -- host query: L, log2 N, log2 N1 used (0 = one kernel),
 * the plan's psi per prime into psi_out[0..L) (host), device-table bytes.
 * Any output pointer may be NULL. */
ntt_status_t ntt_plan_info32(ntt32_plan_t plan, unsigned *L, unsigned *logn, unsigned *log_n1,
                             uint32_t *psi_out, uint64_t *table_bytes);

/* ntt_forward32 / ntt_inverse32 -- in-place forward / inverse over batch x L
 * rows of N uint32 words, [b][l][i] row-major, DEVICE pointer on the plan's
 * device, 16-byte aligned; inputs in [0, p) (precondition), outputs canonical
 * in [0, p), forward output bit-reversed as ntt_forward.  Asynchronous on
 * `stream` (cudaStream_t as void*).  batch == 0 is a no-op.
 * Errors: INVALID_ARG, MISALIGNED, WRONG_DEVICE, CUDA. */
ntt_status_t ntt_forward32(ntt32_plan_t plan, uint32_t *data, unsigned batch, void *stream);
ntt_status_t ntt_inverse32(ntt32_plan_t plan, uint32_t *data, unsigned batch, void *stream);

/* ntt_plan_destroy32 -- frees the plan (NULL accepted).  Work must be done. */
ntt_status_t ntt_plan_destroy32(ntt32_plan_t plan);

/* Static English text for a status code. */
const char *ntt_status_string(ntt_status_t s);

#ifdef __cplusplus
}
#endif
#endif /* NTT_B200_H */
