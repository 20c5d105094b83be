// ntt_api.cu -- the C ABI of include/ntt.h: plan lifecycle, argument checks,
// kernel dispatch and the pipelined host-buffer executor.
#include "../../include/ntt.h"
#include "ntt_launch.h"
#include "params.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

using ntt::KArgs;
using ntt::PrimeConst;
using ntt::Tw;

struct ntt_plan_s {
    int device = 0;
    unsigned logn = 0, L = 0, log_n1 = 0;  // log_n1 == 0: single kernel per row
    int ot_enable = 0;
    unsigned ot_base = 0, ot_logb = 0, ot_stages = 0;
    std::vector<uint64_t> primes, psis;
    Tw* d_fwd = nullptr;  // [L][N]
    Tw* d_inv = nullptr;  // [L][N]
    Tw* d_fwd2 = nullptr;  // [L][N] Kernel-2 order (K2Layout), two-kernel plans only
    Tw* d_inv2 = nullptr;
    Tw* d_ot_fwd = nullptr;  // [L][B + N/B]
    Tw* d_ot_inv = nullptr;
    PrimeConst* d_pc = nullptr;       // [L]
    PrimeConst* d_pc_mont = nullptr;  // [L] the same with N^-1 scaled by 2^64 (NTT-domain products)
    uint64_t table_bytes = 0;
    // Kernel-1 variant (4 = one tile per CTA, 5 = persistent pipelined); Kernel-2 variant (9 = shared-twiddle
    // CTA per block position on the remainder-last schedule, 7 = the same on the remainder-first schedule,
    // 5 = persistent pipelined, 6 = pipelined radix 8, 3/4 = one-shot radix 8/16)
    int loge_k1 = 4, loge_k2 = 9;
    int arith = ntt::kArithGeneral;  // prime-constant type of the kernels (ntt_launch.h)
    bool fused = false;            // single-pass cluster kernel per direction (log_n1 = log2 cluster size)
    bool dform = false;  // every prime p = 2^60 - d, d < 2^32 (R3 chain): the forward Kernel-2's d-form reduction
};

namespace {

unsigned ilog2(uint64_t v)
{
    unsigned l = 0;
    while ((1ull << l) < v) ++l;
    return l;
}

bool pow2_in(unsigned n, unsigned lo_log, unsigned hi_log)
{
    return n && (n & (n - 1)) == 0 && ilog2(n) >= lo_log && ilog2(n) <= hi_log;
}

// Two-kernel split: N1 = 2^log_n1 column transforms, N2 contiguous.
// Rows up to 2^13 words (64 KiB) are handled by one kernel in SMEM.
unsigned default_log_n1(unsigned logn)
{
    switch (logn) {
        case 14: return 7;
        case 15: return 7;
        case 16: return 8;
        case 17: return 8;
        default: return 0;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void free_plan_memory(ntt_plan_s* p)
{
    cudaFree(p->d_fwd);
    cudaFree(p->d_inv);
    cudaFree(p->d_ot_fwd);
    cudaFree(p->d_ot_inv);
    cudaFree(p->d_pc);
    cudaFree(p->d_pc_mont);
    p->d_pc_mont = nullptr;
    cudaFree(p->d_fwd2);
    cudaFree(p->d_inv2);
    p->d_fwd2 = p->d_inv2 = nullptr;
    p->d_fwd = p->d_inv = p->d_ot_fwd = p->d_ot_inv = nullptr;
    p->d_pc = nullptr;
}

ntt_status_t check_data(const ntt_plan_s* plan, const void* data)
{
    if (!plan || !data) return NTT_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(data) & 15u) return NTT_ERR_MISALIGNED;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, data) != cudaSuccess) {
        cudaGetLastError();
        return NTT_ERR_WRONG_DEVICE;
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return NTT_ERR_WRONG_DEVICE;
    if (at.device != plan->device) return NTT_ERR_WRONG_DEVICE;
    return NTT_OK;
}

// Kernel index arithmetic is 32-bit: batch * L * N1 (rows times column tiles
// or block positions) must stay below 2^31 on every entry point that enqueues.
ntt_status_t check_batch(const ntt_plan_s* plan, uint64_t batch)
{
    return (batch * plan->L << plan->log_n1) < (1ull << 31) ? NTT_OK : NTT_ERR_INVALID_ARG;
}

// NVTX range around one C-ABI call (visible under nsys / ncu --nvtx; a no-op
// without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

KArgs base_args(const ntt_plan_s* plan, uint64_t* data, unsigned batch, bool inverse)
{
    KArgs a{};
    a.data = data;
    a.tab = inverse ? plan->d_inv : plan->d_fwd;
    a.tab2 = inverse ? plan->d_inv2 : plan->d_fwd2;
    a.ot = inverse ? plan->d_ot_inv : plan->d_ot_fwd;
    a.pc = plan->d_pc;
    a.L = plan->L;
    a.batch = batch;
    a.logn = plan->logn;
    a.log_n1 = plan->log_n1;
    a.ot_logb = plan->ot_logb;
    a.iters = 1;
    return a;
}

// The two kernels of one direction over `rows` rows of `a` (pass < 0: both).
cudaError_t two_pass(const ntt_plan_s* plan, KArgs a, uint32_t rows, bool inverse, int ots, int pass, cudaStream_t st)
{
    a.total_blocks = rows << plan->log_n1;
    a.log_tiles = plan->logn - plan->log_n1 - 4;
    cudaError_t e = cudaSuccess;
    if (!inverse) {
        if (pass != 1 && (e = ntt::launch_k1(false, plan->loge_k1, a, rows, st, plan->arith)) != cudaSuccess)
            return e;
        const int k2_arith = plan->arith == ntt::kArithGeneral && plan->dform ? ntt::kArithGeneralD : plan->arith;
        if (pass != 0) e = ntt::launch_k2(false, plan->loge_k2, a, ots, 1, st, k2_arith);
        return e;
    }
    // Kernel-1' on PrimeConstD (exact-division N^-1) unless this inverse
    // carries the NTT-domain product, whose N^-1 is R-scaled (Montgomery)
    const int k1i_arith = a.mul_a                                               ? plan->arith
                          : plan->arith == ntt::kArithProth                      ? ntt::kArithProthD
                          : plan->arith == ntt::kArithGeneral && plan->dform ? ntt::kArithGeneralD
                                                                               : plan->arith;
    if (pass != 1) {
        e = ntt::launch_k2(true, plan->loge_k2, a, ots, 1, st, plan->arith);
        if (e == cudaErrorNotSupported && a.mul_a) {  // unfused: product kernel, then Kernel-2'
            cudaGetLastError();
            if ((e = ntt::launch_pointwise(a, st)) != cudaSuccess) return e;
            KArgs b = a;
            b.mul_a = nullptr;
            e = ntt::launch_k2(true, plan->loge_k2, b, ots, 1, st, plan->arith);
        }
        if (e != cudaSuccess) return e;
    }
    a.mul_a = nullptr;
    if (pass != 0) e = ntt::launch_k1(true, plan->loge_k1, a, rows, st, k1i_arith);
    return e;
}

// Enqueue one direction (pass < 0: all passes) on `st`; no checks.  mul_a:
// fuse data <- mul_a (.) data into the inverse's first kernel (Montgomery,
// with the R-scaled N^-1 constants).
cudaError_t enqueue(const ntt_plan_s* plan, uint64_t* data, unsigned batch, bool inverse, cudaStream_t st,
                    int pass = -1, const uint64_t* mul_a = nullptr)
{
    KArgs a = base_args(plan, data, batch, inverse);
    if (mul_a) {
        a.pc = plan->d_pc_mont;
        a.mul_a = mul_a;
    }
    const uint32_t rows = batch * plan->L;
    const int ots = plan->ot_enable ? (int)plan->ot_stages : 0;
    if (plan->fused) {
        if (mul_a) {  // the product is not fused into the cluster kernel: element-wise kernel first
            cudaError_t e = ntt::launch_pointwise(a, st);
            if (e != cudaSuccess) return e;
            a.mul_a = nullptr;
        }
        return ntt::launch_fused(inverse, a, rows, st, plan->arith);
    }
    if (plan->log_n1 == 0) {
        a.total_blocks = rows;
        cudaError_t e = ntt::launch_single(inverse, a, ots, 1, st, plan->arith);
        if (e == cudaErrorNotSupported && mul_a) {  // unfused: product kernel, then the inverse
            cudaGetLastError();
            if ((e = ntt::launch_pointwise(a, st)) != cudaSuccess) return e;
            a.mul_a = nullptr;
            e = ntt::launch_single(inverse, a, ots, 1, st, plan->arith);
        }
        return e;
    }
    return two_pass(plan, a, rows, inverse, ots, pass, st);
}

ntt_status_t run(ntt_plan_t plan, uint64_t* data, unsigned batch, void* stream, bool inverse, int pass = -1)
{
    if (!plan || !data) return NTT_ERR_INVALID_ARG;
    if (batch == 0) return NTT_OK;
    ntt_status_t s = check_data(plan, data);
    if (s == NTT_OK) s = check_batch(plan, batch);
    if (s != NTT_OK) return s;
    DeviceGuard g(plan->device);
    return enqueue(plan, data, batch, inverse, (cudaStream_t)stream, pass) == cudaSuccess ? NTT_OK : NTT_ERR_CUDA;
}

// Device bytes of a plan's twiddle storage (ntt_table_sizes and plan creation):
// per direction L x N Shoup pairs (doubled by w_bar), their Kernel-2
// ordered copies for the two-kernel / cluster paths, the OT bases
// (B + N/B pairs per prime and direction), and two PrimeConst
// arrays (plain and R-scaled N^-1).
struct TableSizes {
    uint64_t psi_dir, ot_per_prime, ot_dir, pc, total;
};
TableSizes table_sizes(uint64_t N, unsigned L, uint64_t ot_base, bool k2tab)
{
    TableSizes t;
    t.psi_dir = sizeof(Tw) * N * L;
    t.ot_per_prime = ot_base + N / ot_base;
    t.ot_dir = sizeof(Tw) * t.ot_per_prime * L;
    t.pc = sizeof(PrimeConst) * L;
    t.total = (k2tab ? 4 : 2) * t.psi_dir + 2 * t.ot_dir + 2 * t.pc;
    return t;
}

unsigned default_ot_base(unsigned logn) { return logn >= 11 ? 1024u : (1u << ((logn + 1) / 2)); }

}  // namespace

extern "C" {

const char* ntt_status_string(ntt_status_t s)
{
    switch (s) {
        case NTT_OK: return "ok";
        case NTT_ERR_INVALID_N: return "N must be a power of two in [2, 2^17]";
        case NTT_ERR_INVALID_PRIME: return "prime must be prime, = 1 mod 2N, < 2^60 (32-bit path: < 2^30) and distinct";
        case NTT_ERR_INVALID_ARG: return "invalid argument";
        case NTT_ERR_MISALIGNED: return "data pointer must be 16-byte aligned";
        case NTT_ERR_WRONG_DEVICE: return "data pointer is not device memory of the plan's device";
        case NTT_ERR_CUDA: return "CUDA error";
        case NTT_ERR_OOM: return "out of memory";
        case NTT_ERR_RANGE_EXHAUSTED: return "not enough NTT primes in the word's range ([2^59, 2^60) or [2^29, 2^30))";
    }
    return "unknown status";
}

ntt_status_t ntt_find_primes(unsigned n, unsigned count, uint64_t* out)
{
    if (!pow2_in(n, 1, 17)) return NTT_ERR_INVALID_N;
    if (!out || count == 0) return NTT_ERR_INVALID_ARG;
    std::vector<uint64_t> v;
    if (!nttp::ntt_primes(n, count, v)) return NTT_ERR_RANGE_EXHAUSTED;
    std::copy(v.begin(), v.end(), out);
    return NTT_OK;
}

ntt_status_t ntt_find_primes_ex(unsigned n, unsigned count, unsigned form, uint64_t* out)
{
    if (form == NTT_PRIMES_2N) return ntt_find_primes(n, count, out);
    if (form != NTT_PRIMES_PROTH32) return NTT_ERR_INVALID_ARG;
    if (!pow2_in(n, 1, 17)) return NTT_ERR_INVALID_N;
    if (!out || count == 0) return NTT_ERR_INVALID_ARG;
    std::vector<uint64_t> v;
    if (!nttp::proth_primes(count, v)) return NTT_ERR_RANGE_EXHAUSTED;
    std::copy(v.begin(), v.end(), out);
    return NTT_OK;
}

ntt_status_t ntt_find_psi(uint64_t p, unsigned n, uint64_t* psi)
{
    if (!pow2_in(n, 1, 17)) return NTT_ERR_INVALID_N;
    if (!psi) return NTT_ERR_INVALID_ARG;
    const uint64_t r = nttp::smallest_psi(p, n);
    if (!r) return NTT_ERR_INVALID_PRIME;
    *psi = r;
    return NTT_OK;
}

ntt_status_t ntt_plan_create(ntt_plan_t* plan, unsigned n, const uint64_t* primes, unsigned L)
{
    return ntt_plan_create_ex(plan, n, primes, L, nullptr);
}

ntt_status_t ntt_plan_create_ex(ntt_plan_t* out, unsigned n, const uint64_t* primes, unsigned L, const ntt_opts_t* o)
{
    if (!out) return NTT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!primes || L == 0 || L > 65535) return NTT_ERR_INVALID_ARG;  // L is a grid dimension of the kernels
    if (!pow2_in(n, 1, 17)) return NTT_ERR_INVALID_N;
    ntt_opts_t opts{};
    if (o) opts = *o;
    const unsigned logn = ilog2(n);

    std::vector<uint64_t> pr(primes, primes + L);
    for (unsigned i = 0; i < L; ++i) {
        if (!nttp::valid_ntt_prime(pr[i], n)) return NTT_ERR_INVALID_PRIME;
        for (unsigned j = 0; j < i; ++j)
            if (pr[j] == pr[i]) return NTT_ERR_INVALID_PRIME;
    }

    // options
    unsigned log_n1 = default_log_n1(logn);
    if (opts.log_n1) {
        if (logn <= 13) {
            log_n1 = 0;  // one kernel holds the row
        } else {
            const unsigned l1 = opts.log_n1, l2 = logn - opts.log_n1;
            if (l1 < 6 || l1 > 10 || l2 < 6 || l2 > 11) return NTT_ERR_INVALID_ARG;
            log_n1 = l1;
        }
    }
    if (opts.ot_enable < -1 || opts.ot_enable > 1) return NTT_ERR_INVALID_ARG;
    const int ot_enable = opts.ot_enable == 1;
    unsigned ot_base = opts.ot_base;
    if (ot_base == 0) ot_base = default_ot_base(logn);
    if ((ot_base & (ot_base - 1)) || ot_base > n) return NTT_ERR_INVALID_ARG;
    unsigned ot_stages = opts.ot_stages ? opts.ot_stages : 2;
    if (ot_stages > 2) return NTT_ERR_INVALID_ARG;
    const unsigned last_kernel_stages = log_n1 ? logn - log_n1 : logn;
    if (ot_stages > last_kernel_stages) ot_stages = last_kernel_stages;
    if (opts.prime_arith < -1 || opts.prime_arith > 0) return NTT_ERR_INVALID_ARG;
    // kernel variants (tuning and experiments): 0 = default
    int loge_k1 = 4, loge_k2 = 9;
    if (opts.k1_variant) {
        if (opts.k1_variant != 4 && opts.k1_variant != 5) return NTT_ERR_INVALID_ARG;
        loge_k1 = opts.k1_variant;
    }
    if (opts.k2_variant) {
        if (opts.k2_variant < 3 || opts.k2_variant > 9 || opts.k2_variant == 8) return NTT_ERR_INVALID_ARG;
        loge_k2 = opts.k2_variant;
    }
    if (opts.fused < -1 || opts.fused > 1) return NTT_ERR_INVALID_ARG;
    // single pass per direction (cluster kernel): N = 2^14..2^17, no OT, no explicit split
    const bool fused_ok = logn >= 14 && logn <= 17 && !ot_enable && opts.log_n1 == 0;
    if (opts.fused == 1 && !fused_ok) return NTT_ERR_INVALID_ARG;
    const bool fused = fused_ok && opts.fused == 1;
    if (fused) log_n1 = logn - 13;
    // Proth arithmetic when every prime has the form
    bool all_proth = opts.prime_arith == 0;
    for (unsigned i = 0; i < L; ++i) all_proth = all_proth && (uint32_t)pr[i] == 1u;

    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return NTT_ERR_CUDA;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return NTT_ERR_CUDA;
    }

    ntt_plan_s* p = new (std::nothrow) ntt_plan_s;
    if (!p) return NTT_ERR_OOM;
    p->device = dev;
    p->logn = logn;
    p->L = L;
    p->log_n1 = log_n1;
    p->ot_enable = ot_enable;
    p->ot_base = ot_base;
    p->ot_logb = ilog2(ot_base);
    p->ot_stages = ot_stages;
    p->primes = pr;
    p->psis.assign(L, 0);
    p->loge_k1 = loge_k1;
    p->loge_k2 = loge_k2;
    // the Proth kernels exist for the default variants only (ntt_kernels.cuh)
    const bool special_ok = ((loge_k1 == 4 || loge_k1 == 5) && (loge_k2 == 5 || loge_k2 == 7 || loge_k2 == 9)) || fused;
    p->arith = special_ok && all_proth ? ntt::kArithProth : ntt::kArithGeneral;
    p->fused = fused;
    p->dform = true;
    for (unsigned l = 0; l < L; ++l) p->dform = p->dform && ((0 - pr[l]) >> 32) == 0xF0000000ull;

    // host tables, one thread per hardware thread over primes
    const uint64_t N = n, NOT = ot_base + N / ot_base;
    std::vector<Tw> h_fwd(N * L), h_inv(N * L), h_otf(NOT * L), h_oti(NOT * L);
    std::vector<PrimeConst> h_pc(L), h_pcm(L);
    unsigned nth = std::max(1u, std::min(L, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; ++t)
        th.emplace_back([&, t] {
            for (unsigned l = t; l < L; l += nth) {
                const uint64_t q = pr[l];
                const uint64_t psi = nttp::smallest_psi(q, N);
                const uint64_t psi_inv = nttp::pow_mod(psi, q - 2, q);
                p->psis[l] = psi;
                static_assert(sizeof(nttp::Twiddle) == sizeof(Tw), "layout");
                nttp::bitrev_power_table(q, psi, logn, reinterpret_cast<nttp::Twiddle*>(&h_fwd[l * N]));
                nttp::bitrev_power_table(q, psi_inv, logn, reinterpret_cast<nttp::Twiddle*>(&h_inv[l * N]));
                nttp::ot_base_tables(q, psi, N, ot_base, reinterpret_cast<nttp::Twiddle*>(&h_otf[l * NOT]));
                nttp::ot_base_tables(q, psi_inv, N, ot_base, reinterpret_cast<nttp::Twiddle*>(&h_oti[l * NOT]));
                const uint64_t ninv = nttp::pow_mod(N % q, q - 2, q);
                const uint64_t ninv_psi = nttp::mul_mod(ninv, h_inv[l * N + (N > 1 ? 1 : 0)].w, q);
                PrimeConst c;
                c.p = q;
                c.p2 = 2 * q;
                c.p4 = 4 * q;
                c.np = 0 - q;
                c.p5 = 5 * q;
                c.p4_hi = (uint32_t)((4 * q) >> 32);
                c.rn = (uint32_t)((((unsigned __int128)1) << 90) / q);
                uint64_t inv = 1;  // p^-1 mod 2^64 by Newton iteration (p odd)
                for (int it = 0; it < 6; ++it) inv *= 2 - q * inv;
                c.pinv = 0 - inv;
                c.m1 = 0u - (uint32_t)(q >> 32);
                c.p8 = 8 * q;
                c.p8_hi = (uint32_t)((8 * q) >> 32);
                c.zero = 0;
                c.mN = (q - 1) >> logn;  // div_n (PrimeConstD Kernel-1'); p = 1 mod 2N
                c.logn = logn;
                c.nmask = (uint32_t)(N - 1);
                nttp::Twiddle t1 = nttp::shoup_pair(ninv, q), t2 = nttp::shoup_pair(ninv_psi, q);
                c.ninv = Tw{t1.w, t1.wb};
                c.ninv_psi = Tw{t2.w, t2.wb};
                h_pc[l] = c;
                // R-scaled copy for inverses fed by Montgomery products (R = 2^64)
                const uint64_t r_mod = (uint64_t)((((unsigned __int128)1) << 64) % q);
                PrimeConst cm = c;
                nttp::Twiddle t3 = nttp::shoup_pair(nttp::mul_mod(ninv, r_mod, q), q);
                nttp::Twiddle t4 = nttp::shoup_pair(nttp::mul_mod(ninv_psi, r_mod, q), q);
                cm.ninv = Tw{t3.w, t3.wb};
                cm.ninv_psi = Tw{t4.w, t4.wb};
                h_pcm[l] = cm;
            }
        });
    for (auto& t : th) t.join();

    // Kernel-2 ordered copies for the two-kernel path
    const bool k2tab = log_n1 != 0;
    std::vector<Tw> h_fwd2, h_inv2;
    if (k2tab) {
        const unsigned loge = (!fused && (p->loge_k2 == 3 || p->loge_k2 == 6)) ? 3
                              : (!fused && p->loge_k2 == 9) ? (4u | (unsigned)ntt::kRemLast) : 4;
        h_fwd2.resize(N * L);
        h_inv2.resize(N * L);
        std::vector<std::thread> th2;
        for (unsigned t = 0; t < nth; ++t)
            th2.emplace_back([&, t] {
                for (unsigned l = t; l < L; l += nth) {
                    nttp::k2_order(&h_fwd[l * N], logn, log_n1, loge, &h_fwd2[l * N]);
                    nttp::k2_order(&h_inv[l * N], logn, log_n1, loge, &h_inv2[l * N]);
                }
            });
        for (auto& t : th2) t.join();
    }

    const TableSizes ts = table_sizes(N, L, ot_base, k2tab);
    const size_t bt = ts.psi_dir, bo = ts.ot_dir, bp = ts.pc;
    if (cudaMalloc(&p->d_fwd, bt) != cudaSuccess || cudaMalloc(&p->d_inv, bt) != cudaSuccess ||
        cudaMalloc(&p->d_ot_fwd, bo) != cudaSuccess || cudaMalloc(&p->d_ot_inv, bo) != cudaSuccess ||
        cudaMalloc(&p->d_pc, bp) != cudaSuccess || cudaMalloc(&p->d_pc_mont, bp) != cudaSuccess ||
        (k2tab && (cudaMalloc(&p->d_fwd2, bt) != cudaSuccess || cudaMalloc(&p->d_inv2, bt) != cudaSuccess))) {
        cudaGetLastError();
        free_plan_memory(p);
        delete p;
        return NTT_ERR_OOM;
    }
    if (cudaMemcpy(p->d_fwd, h_fwd.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_inv, h_inv.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_ot_fwd, h_otf.data(), bo, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_ot_inv, h_oti.data(), bo, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_pc, h_pc.data(), bp, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_pc_mont, h_pcm.data(), bp, cudaMemcpyHostToDevice) != cudaSuccess ||
        (k2tab && (cudaMemcpy(p->d_fwd2, h_fwd2.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
                   cudaMemcpy(p->d_inv2, h_inv2.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess))) {
        cudaGetLastError();
        free_plan_memory(p);
        delete p;
        return NTT_ERR_CUDA;
    }
    p->table_bytes = ts.total;
    *out = p;
    return NTT_OK;
}

ntt_status_t ntt_plan_psi(ntt_plan_t plan, uint64_t* psi_out)
{
    if (!plan || !psi_out) return NTT_ERR_INVALID_ARG;
    std::copy(plan->psis.begin(), plan->psis.end(), psi_out);
    return NTT_OK;
}

ntt_status_t ntt_plan_info(ntt_plan_t plan, unsigned* L, unsigned* logn, unsigned* log_n1, int* ot_enable,
                           unsigned* ot_base, unsigned* ot_stages, uint64_t* table_bytes)
{
    if (!plan) return NTT_ERR_INVALID_ARG;
    if (L) *L = plan->L;
    if (logn) *logn = plan->logn;
    if (log_n1) *log_n1 = plan->log_n1;
    if (ot_enable) *ot_enable = plan->ot_enable;
    if (ot_base) *ot_base = plan->ot_base;
    if (ot_stages) *ot_stages = plan->ot_stages;
    if (table_bytes) *table_bytes = plan->table_bytes;
    return NTT_OK;
}

ntt_status_t ntt_plan_exec(ntt_plan_t plan, int* arith, unsigned* passes, unsigned* cluster)
{
    if (!plan) return NTT_ERR_INVALID_ARG;
    if (arith) *arith = plan->arith == ntt::kArithGeneral && plan->dform ? ntt::kArithGeneralD : plan->arith;
    if (passes) *passes = (plan->fused || plan->log_n1 == 0) ? 1u : 2u;
    if (cluster) *cluster = plan->fused ? (1u << plan->log_n1) : 1u;
    return NTT_OK;
}

ntt_status_t ntt_forward(ntt_plan_t plan, uint64_t* data, unsigned batch, void* stream)
{
    NvtxRange r("ntt_forward");
    return run(plan, data, batch, stream, false);
}

ntt_status_t ntt_inverse(ntt_plan_t plan, uint64_t* data, unsigned batch, void* stream)
{
    NvtxRange r("ntt_inverse");
    return run(plan, data, batch, stream, true);
}

ntt_status_t ntt_launch_pass(ntt_plan_t plan, uint64_t* data, unsigned batch, unsigned dir, unsigned pass,
                             void* stream)
{
    if (!plan || (dir != NTT_DIR_FORWARD && dir != NTT_DIR_INVERSE)) return NTT_ERR_INVALID_ARG;
    const bool one = plan->fused || plan->log_n1 == 0;
    if (pass > 1 || (pass == 1 && one)) return NTT_ERR_INVALID_ARG;
    return run(plan, data, batch, stream, dir == NTT_DIR_INVERSE, one ? -1 : (int)pass);
}

ntt_status_t ntt_pointwise_inverse(ntt_plan_t plan, const uint64_t* a_ntt, uint64_t* data, unsigned batch,
                                   void* stream)
{
    NvtxRange r("ntt_pointwise_inverse");
    if (!plan || !data || !a_ntt) return NTT_ERR_INVALID_ARG;
    if (batch == 0) return NTT_OK;
    ntt_status_t s = check_data(plan, data);
    if (s == NTT_OK) s = check_data(plan, a_ntt);
    if (s == NTT_OK) s = check_batch(plan, batch);
    if (s != NTT_OK) return s;
    DeviceGuard g(plan->device);
    return enqueue(plan, data, batch, true, (cudaStream_t)stream, -1, a_ntt) == cudaSuccess ? NTT_OK : NTT_ERR_CUDA;
}

ntt_status_t ntt_negacyclic_mul(ntt_plan_t plan, uint64_t* a, uint64_t* b, unsigned batch, void* stream)
{
    NvtxRange r("ntt_negacyclic_mul");
    if (!plan || !a || !b) return NTT_ERR_INVALID_ARG;
    if (a == b) return NTT_ERR_INVALID_ARG;
    ntt_status_t s;
    if ((s = ntt_forward(plan, a, batch, stream)) != NTT_OK) return s;
    if ((s = ntt_forward(plan, b, batch, stream)) != NTT_OK) return s;
    return ntt_pointwise_inverse(plan, a, b, batch, stream);
}

ntt_status_t ntt_forward_variant(ntt_plan_t plan, uint64_t* data, unsigned batch, unsigned variant, void* stream)
{
    if (variant == NTT_VARIANT_DEFAULT) return ntt_forward(plan, data, batch, stream);
    NvtxRange r("ntt_forward_variant");
    if (!plan || !data || variant > NTT_VARIANT_NATIVE) return NTT_ERR_INVALID_ARG;
    if (variant == NTT_VARIANT_NATIVE && (plan->fused || plan->ot_enable)) return NTT_ERR_INVALID_ARG;
    if (batch == 0) return NTT_OK;
    ntt_status_t s = check_data(plan, data);
    if (s == NTT_OK) s = check_batch(plan, batch);
    if (s != NTT_OK) return s;
    DeviceGuard g(plan->device);
    const KArgs a = base_args(plan, data, batch, false);
    cudaError_t e;
    if (variant == NTT_VARIANT_NATIVE) {
        e = ntt::launch_native_forward(a, batch * plan->L, (cudaStream_t)stream);
        if (e == cudaErrorNotSupported) return NTT_ERR_INVALID_ARG;  // non-default split
    } else {
        e = ntt::launch_baseline_forward((int)variant, a, (cudaStream_t)stream);
    }
    return e == cudaSuccess ? NTT_OK : NTT_ERR_CUDA;
}

// pipeline slots (stream + device buffer) of the host-buffer executor: with
// three, chunk k's H2D, chunk k-1's transforms and chunk k-2's D2H overlap
// without a slot waiting for its own previous D2H
static constexpr unsigned kHostSlots = 3;

static unsigned auto_chunk(const ntt_plan_s* plan, unsigned batch, unsigned chunk)
{
    if (chunk) return std::min(chunk, batch);
    const uint64_t ct_bytes = (uint64_t)plan->L * 8ull << plan->logn;
    uint64_t c = std::max<uint64_t>(1, (64ull << 20) / ct_bytes);  // ~64 MiB per pipeline step
    return (unsigned)std::min<uint64_t>(c, batch);
}

uint64_t ntt_workspace_words(ntt_plan_t plan, unsigned batch, unsigned chunk)
{
    if (!plan || batch == 0) return 0;
    const unsigned c = auto_chunk(plan, batch, chunk);
    const unsigned steps = (batch + c - 1) / c;
    const unsigned nbuf = std::min<unsigned>(kHostSlots, steps);
    return (uint64_t)nbuf * c * plan->L << plan->logn;
}

ntt_status_t ntt_execute_host(ntt_plan_t plan, unsigned flags, const uint64_t* host_in, uint64_t* host_out,
                              unsigned batch, uint64_t* workspace, uint64_t workspace_words, unsigned chunk,
                              void* stream)
{
    NvtxRange r("ntt_execute_host");
    if (!plan || !host_in || !host_out || (flags & ~3u)) return NTT_ERR_INVALID_ARG;
    if (batch == 0) return NTT_OK;
    ntt_status_t s = check_data(plan, workspace);
    if (s != NTT_OK) return s;
    const unsigned c = auto_chunk(plan, batch, chunk);
    if ((s = check_batch(plan, c)) != NTT_OK) return s;
    if (workspace_words < ntt_workspace_words(plan, batch, c)) return NTT_ERR_INVALID_ARG;
    DeviceGuard g(plan->device);
    const uint64_t ct_words = (uint64_t)plan->L << plan->logn;
    const unsigned nslot = std::min<unsigned>(kHostSlots, (batch + c - 1) / c);
    cudaStream_t st[kHostSlots] = {};
    cudaEvent_t ready = nullptr;
    for (unsigned i = 0; i < nslot; ++i)
        if (cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking) != cudaSuccess) {
            for (unsigned j = 0; j < i; ++j) cudaStreamDestroy(st[j]);
            cudaGetLastError();
            return NTT_ERR_CUDA;
        }
    // order the slots after the caller's stream (the workspace may still be in use there)
    cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ready, (cudaStream_t)stream);
    for (unsigned i = 0; i < nslot && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(st[i], ready, 0);
    unsigned k = 0;
    for (unsigned b0 = 0; b0 < batch && e == cudaSuccess; b0 += c, ++k) {
        const unsigned nb = std::min(c, batch - b0);
        cudaStream_t sk = st[k % nslot];
        uint64_t* buf = workspace + (uint64_t)(k % nslot) * c * ct_words;
        const size_t bytes = (size_t)nb * ct_words * 8;
        e = cudaMemcpyAsync(buf, host_in + (uint64_t)b0 * ct_words, bytes, cudaMemcpyHostToDevice, sk);
        if (e == cudaSuccess && (flags & NTT_DIR_FORWARD)) e = enqueue(plan, buf, nb, false, sk);
        if (e == cudaSuccess && (flags & NTT_DIR_INVERSE)) e = enqueue(plan, buf, nb, true, sk);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(host_out + (uint64_t)b0 * ct_words, buf, bytes, cudaMemcpyDeviceToHost, sk);
    }
    cudaError_t e0 = cudaSuccess;
    for (unsigned i = 0; i < nslot; ++i) {
        const cudaError_t ei = cudaStreamSynchronize(st[i]);
        if (ei != cudaSuccess) e0 = ei;
        cudaStreamDestroy(st[i]);
    }
    if (ready) cudaEventDestroy(ready);
    if (e == cudaSuccess) e = e0;
    if (e != cudaSuccess) cudaGetLastError();
    return e == cudaSuccess ? NTT_OK : NTT_ERR_CUDA;
}

// ---------------------------------------------------------------- request graphs

struct ntt_graph_s {
    int device = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned long long* bar = nullptr;  // NTT_GRAPH_ONE_KERNEL: grid barrier arrival counter
    bool one = false;                  // NTT_GRAPH_ONE_KERNEL: ...
    ntt::ReqArgs ra{};                 // its kernel arguments
    unsigned logn = 0;
    int arith = 0;
};
// NTT_REQ_DIRECT (experiment knob): replay a one-kernel request by launching
// its kernel directly instead of through cudaGraphLaunch
#ifndef NTT_REQ_DIRECT
#define NTT_REQ_DIRECT 0
#endif

static void free_graph(ntt_graph_s* gr)
{
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    if (gr->graph) cudaGraphDestroy(gr->graph);
    if (gr->bar) cudaFree(gr->bar);
    delete gr;
}

ntt_status_t ntt_graph_create(ntt_graph_t* out, ntt_plan_t plan, uint64_t* data, uint64_t* data2, unsigned batch,
                              unsigned flags)
{
    NvtxRange r("ntt_graph_create");
    if (!out) return NTT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!plan || !data || batch == 0 || (flags & ~15u)) return NTT_ERR_INVALID_ARG;
    const bool product = flags & NTT_GRAPH_PRODUCT;
    const bool one = flags & NTT_GRAPH_ONE_KERNEL;
    if ((flags & 7u) == 0) return NTT_ERR_INVALID_ARG;
    if (product && (flags != NTT_GRAPH_PRODUCT || !data2 || data2 == data)) return NTT_ERR_INVALID_ARG;
    if (one && (plan->logn < 14 || plan->logn > 17 || plan->ot_enable)) return NTT_ERR_INVALID_ARG;
    ntt_status_t s = check_data(plan, data);
    if (s == NTT_OK && product) s = check_data(plan, data2);
    if (s == NTT_OK) s = check_batch(plan, batch);
    if (s != NTT_OK) return s;
    DeviceGuard g(plan->device);
    ntt_graph_s* gr = new (std::nothrow) ntt_graph_s;
    if (!gr) return NTT_ERR_OOM;
    gr->device = plan->device;
    cudaStream_t st = nullptr;
    cudaError_t e = cudaSuccess;
    if (one) {
        e = cudaMalloc(&gr->bar, ntt::kReqBarrierBytes);
        if (e == cudaSuccess) e = cudaMemset(gr->bar, 0, ntt::kReqBarrierBytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            free_graph(gr);
            return NTT_ERR_OOM;
        }
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        cudaError_t ek = cudaSuccess;
        if (product) {  // b <- a * b: forward a, forward b, fused odot + inverse (ntt_negacyclic_mul)
            ek = enqueue(plan, data, batch, false, st);
            if (ek == cudaSuccess) ek = enqueue(plan, data2, batch, false, st);
            if (ek == cudaSuccess) ek = enqueue(plan, data2, batch, true, st, -1, data);
        } else if (one) {  // the whole request in one cooperative launch (ntt_request.cu)
            ntt::ReqArgs ra;
            ra.data = data;
            ra.tf = plan->d_fwd;
            ra.ti = plan->d_inv;
            ra.pc = plan->d_pc;
            ra.bar = gr->bar;
            ra.L = plan->L;
            ra.rows = batch * plan->L;
            ra.flags = flags & 3u;
            gr->one = true;
            gr->ra = ra;
            gr->logn = plan->logn;
            gr->arith = plan->arith;
            ek = ntt::launch_request(plan->logn, ra, st, plan->arith);
        } else {
            if (flags & NTT_DIR_FORWARD) ek = enqueue(plan, data, batch, false, st);
            if (ek == cudaSuccess && (flags & NTT_DIR_INVERSE)) ek = enqueue(plan, data, batch, true, st);
        }
        e = cudaStreamEndCapture(st, &gr->graph);  // ends the capture even after a failed launch
        if (ek != cudaSuccess) e = ek;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiateWithFlags(&gr->exec, gr->graph, 0);
    if (st) cudaStreamDestroy(st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_graph(gr);
        return NTT_ERR_CUDA;
    }
    *out = gr;
    return NTT_OK;
}

ntt_status_t ntt_graph_launch(ntt_graph_t graph, void* stream)
{
    if (!graph) return NTT_ERR_INVALID_ARG;
    if (NTT_REQ_DIRECT && graph->one) {
        DeviceGuard g(graph->device);
        return ntt::launch_request(graph->logn, graph->ra, (cudaStream_t)stream, graph->arith) == cudaSuccess
                   ? NTT_OK
                   : NTT_ERR_CUDA;
    }
    if (cudaGraphLaunch(graph->exec, (cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return NTT_ERR_CUDA;
    }
    return NTT_OK;
}

ntt_status_t ntt_graph_destroy(ntt_graph_t graph)
{
    if (!graph) return NTT_OK;
    {
        DeviceGuard g(graph->device);
        free_graph(graph);
    }
    return NTT_OK;
}

// ---------------------------------------------------------------- host helpers for tests

ntt_status_t ntt_shoup_companion(uint64_t w, uint64_t p, uint64_t* wb)
{
    if (!wb || p < 2 || w >= p) return NTT_ERR_INVALID_ARG;
    *wb = nttp::shoup_pair(w, p).wb;
    return NTT_OK;
}

ntt_status_t ntt_table_sizes(unsigned n, unsigned L, unsigned ot_base, uint64_t* psi_bytes, uint64_t* ot_entries,
                             uint64_t* plan_bytes)
{
    if (!pow2_in(n, 1, 17)) return NTT_ERR_INVALID_N;
    if (L == 0) return NTT_ERR_INVALID_ARG;
    const unsigned logn = ilog2(n);
    const unsigned b = ot_base ? ot_base : default_ot_base(logn);
    if ((b & (b - 1)) || b > n) return NTT_ERR_INVALID_ARG;
    const TableSizes t = table_sizes(n, L, b, default_log_n1(logn) != 0);
    if (psi_bytes) *psi_bytes = t.psi_dir;
    if (ot_entries) *ot_entries = t.ot_per_prime;
    if (plan_bytes) *plan_bytes = t.total;
    return NTT_OK;
}

ntt_status_t ntt_debug_corrupt_twiddle(ntt_plan_t plan, unsigned dir, unsigned l, unsigned index, unsigned field,
                                       uint64_t mask)
{
    if (!plan || (dir != NTT_DIR_FORWARD && dir != NTT_DIR_INVERSE) || l >= plan->L ||
        index >= (1u << plan->logn) || field > 1)
        return NTT_ERR_INVALID_ARG;
    DeviceGuard g(plan->device);
    const uint64_t N = 1ull << plan->logn;
    Tw* tab = (dir == NTT_DIR_FORWARD ? plan->d_fwd : plan->d_inv) + l * N;
    Tw* tab2 = (dir == NTT_DIR_FORWARD ? plan->d_fwd2 : plan->d_inv2);
    Tw orig;
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(&orig, tab + index, sizeof(Tw), cudaMemcpyDeviceToHost))
        return cudaGetLastError(), NTT_ERR_CUDA;
    Tw bad = orig;
    (field ? bad.wb : bad.w) ^= mask;
    if (cudaMemcpy(tab + index, &bad, sizeof(Tw), cudaMemcpyHostToDevice) != cudaSuccess)
        return cudaGetLastError(), NTT_ERR_CUDA;
    if (tab2) {  // the Kernel-2 ordered copy: every Psi entry appears once (entry 0 of a block is padding)
        std::vector<Tw> h(N);
        if (cudaMemcpy(h.data(), tab2 + l * N, N * sizeof(Tw), cudaMemcpyDeviceToHost) != cudaSuccess)
            return cudaGetLastError(), NTT_ERR_CUDA;
        for (uint64_t i = 0; i < N; ++i)
            if (h[i].w == orig.w && h[i].wb == orig.wb && (orig.w | orig.wb)) {
                if (cudaMemcpy(tab2 + l * N + i, &bad, sizeof(Tw), cudaMemcpyHostToDevice) != cudaSuccess)
                    return cudaGetLastError(), NTT_ERR_CUDA;
            }
    }
    return NTT_OK;
}

ntt_status_t ntt_plan_destroy(ntt_plan_t plan)
{
    if (!plan) return NTT_OK;
    {
        DeviceGuard g(plan->device);
        free_plan_memory(plan);
    }
    delete plan;
    return NTT_OK;
}

}  // extern "C"
