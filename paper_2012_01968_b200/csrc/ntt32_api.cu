// ntt32_api.cu -- C ABI of the 32-bit-word path (include/ntt.h, "32-bit
// words"; the paper's 32b-vs-64b comparison P:407-423).
// Plan creation mirrors ntt_api.cu with 32-bit Shoup pairs; no OT and no fused
// products on this path.
#include "../../include/ntt.h"
#include "ntt_launch.h"
#include "params.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <new>
#include <thread>
#include <vector>

using ntt::PrimeConst32;
using ntt::Tw32;

struct ntt32_plan_s {
    int device = 0;
    unsigned logn = 0, L = 0, log_n1 = 0;
    std::vector<uint32_t> primes, psis;
    Tw32* d_fwd = nullptr;  // [L][N] Psi (bit-reversed powers)
    Tw32* d_inv = nullptr;
    Tw32* d_fwd2 = nullptr;  // [L][N] Kernel-2 order, two-kernel plans only
    Tw32* d_inv2 = nullptr;
    PrimeConst32* d_pc = nullptr;
    uint64_t table_bytes = 0;
};

namespace {

unsigned ilog2_32(uint64_t v)
{
    unsigned l = 0;
    while ((1ull << l) < v) ++l;
    return l;
}

bool pow2_ok(unsigned n) { return n >= 2 && n <= (1u << 17) && (n & (n - 1)) == 0; }

// Splits with a compiled Kernel-1 / Kernel-2 pair (ntt32.cu K1Pairs32).
bool split_ok(unsigned logn, unsigned log_n1)
{
    return (logn == 14 && log_n1 == 7) || (logn == 15 && log_n1 == 7) || (logn == 16 && log_n1 == 8) ||
           (logn == 17 && (log_n1 == 8 || log_n1 == 9));
}

void free32(ntt32_plan_s* p)
{
    cudaFree(p->d_fwd);
    cudaFree(p->d_inv);
    cudaFree(p->d_fwd2);
    cudaFree(p->d_inv2);
    cudaFree(p->d_pc);
    p->d_fwd = p->d_inv = p->d_fwd2 = p->d_inv2 = nullptr;
    p->d_pc = nullptr;
}

ntt_status_t run32(ntt32_plan_t plan, uint32_t* data, unsigned batch, void* stream, bool inverse)
{
    if (!plan || !data) return NTT_ERR_INVALID_ARG;
    if (batch == 0) return NTT_OK;
    if (reinterpret_cast<uintptr_t>(data) & 15u) return NTT_ERR_MISALIGNED;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, data) != cudaSuccess) {
        cudaGetLastError();
        return NTT_ERR_WRONG_DEVICE;
    }
    if ((at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) || at.device != plan->device)
        return NTT_ERR_WRONG_DEVICE;
    const uint64_t rows = (uint64_t)batch * plan->L;
    if ((rows << plan->log_n1) >= (1ull << 31)) return NTT_ERR_INVALID_ARG;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != plan->device) cudaSetDevice(plan->device);
    ntt::KArgs32 a{};
    a.data = data;
    a.tab = inverse ? plan->d_inv : plan->d_fwd;
    a.tab2 = inverse ? plan->d_inv2 : plan->d_fwd2;
    a.pc = plan->d_pc;
    a.L = plan->L;
    a.batch = batch;
    a.logn = plan->logn;
    a.log_n1 = plan->log_n1;
    const cudaError_t e = ntt::launch32(inverse, a, (uint32_t)rows, (cudaStream_t)stream);
    if (prev >= 0 && prev != plan->device) cudaSetDevice(prev);
    return e == cudaSuccess ? NTT_OK : NTT_ERR_CUDA;
}

}  // namespace

extern "C" {

ntt_status_t ntt_find_primes32(unsigned n, unsigned count, uint32_t* out)
{
    if (!pow2_ok(n)) return NTT_ERR_INVALID_N;
    if (!out || count == 0) return NTT_ERR_INVALID_ARG;
    std::vector<uint32_t> v;
    if (!nttp::ntt_primes32(n, count, v)) return NTT_ERR_RANGE_EXHAUSTED;
    std::copy(v.begin(), v.end(), out);
    return NTT_OK;
}

ntt_status_t ntt_plan_create32(ntt32_plan_t* out, unsigned n, const uint32_t* primes, unsigned L, unsigned log_n1)
{
    if (!out) return NTT_ERR_INVALID_ARG;
    *out = nullptr;
    if (!primes || L == 0) return NTT_ERR_INVALID_ARG;
    if (!pow2_ok(n)) return NTT_ERR_INVALID_N;
    const unsigned logn = ilog2_32(n);
    std::vector<uint32_t> pr(primes, primes + L);
    for (unsigned i = 0; i < L; ++i) {
        if (!nttp::valid_ntt_prime32(pr[i], n)) return NTT_ERR_INVALID_PRIME;
        for (unsigned j = 0; j < i; ++j)
            if (pr[j] == pr[i]) return NTT_ERR_INVALID_PRIME;
    }
    unsigned l1 = 0;  // one kernel per row up to 2^13 words (32 KiB)
    if (logn > 13) {
        l1 = log_n1 ? log_n1 : (logn <= 15 ? 7u : 8u);
        if (!split_ok(logn, l1)) return NTT_ERR_INVALID_ARG;
    }
    int dev = 0, ndev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return NTT_ERR_CUDA;
    }
    ntt32_plan_s* p = new (std::nothrow) ntt32_plan_s;
    if (!p) return NTT_ERR_OOM;
    p->device = dev;
    p->logn = logn;
    p->L = L;
    p->log_n1 = l1;
    p->primes = pr;
    p->psis.assign(L, 0);

    const uint64_t N = n;
    std::vector<Tw32> h_fwd(N * L), h_inv(N * L), h_fwd2, h_inv2;
    std::vector<PrimeConst32> h_pc(L);
    if (l1) {
        h_fwd2.resize(N * L);
        h_inv2.resize(N * L);
    }
    const unsigned nth = std::max(1u, std::min(L, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nth; ++t)
        th.emplace_back([&, t] {
            std::vector<nttp::Twiddle> wide(N);
            for (unsigned l = t; l < L; l += nth) {
                const uint32_t q = pr[l];
                const uint64_t psi = nttp::smallest_psi(q, N);
                const uint64_t psi_inv = nttp::pow_mod(psi, q - 2, q);
                p->psis[l] = (uint32_t)psi;
                for (int dir = 0; dir < 2; ++dir) {
                    Tw32* tab = (dir ? h_inv.data() : h_fwd.data()) + l * N;
                    nttp::bitrev_power_table(q, dir ? psi_inv : psi, logn, wide.data());
                    for (uint64_t i = 0; i < N; ++i) {
                        const nttp::Twiddle32 t32 = nttp::shoup_pair32((uint32_t)wide[i].w, q);
                        tab[i] = Tw32{t32.w, t32.wb};
                    }
                    if (l1)  // remainder-last round order, as the 32-bit Kernel-2 runs it
                        nttp::k2_order(tab, logn, l1, 4u | (unsigned)ntt::kRemLast,
                                       (dir ? h_inv2.data() : h_fwd2.data()) + l * N);
                }
                const uint32_t ninv = (uint32_t)nttp::pow_mod(N % q, q - 2, q);
                const uint32_t ninv_psi = (uint32_t)nttp::mul_mod(ninv, h_inv[l * N + (N > 1 ? 1 : 0)].w, q);
                const nttp::Twiddle32 a = nttp::shoup_pair32(ninv, q), b = nttp::shoup_pair32(ninv_psi, q);
                PrimeConst32 c{};
                c.p = q;
                c.p2 = 2 * q;
                c.ninv = Tw32{a.w, a.wb};
                c.ninv_psi = Tw32{b.w, b.wb};
                h_pc[l] = c;
            }
        });
    for (auto& t : th) t.join();

    const size_t bt = sizeof(Tw32) * N * L, bp = sizeof(PrimeConst32) * L;
    if (cudaMalloc(&p->d_fwd, bt) != cudaSuccess || cudaMalloc(&p->d_inv, bt) != cudaSuccess ||
        cudaMalloc(&p->d_pc, bp) != cudaSuccess ||
        (l1 && (cudaMalloc(&p->d_fwd2, bt) != cudaSuccess || cudaMalloc(&p->d_inv2, bt) != cudaSuccess))) {
        cudaGetLastError();
        free32(p);
        delete p;
        return NTT_ERR_OOM;
    }
    if (cudaMemcpy(p->d_fwd, h_fwd.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_inv, h_inv.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->d_pc, h_pc.data(), bp, cudaMemcpyHostToDevice) != cudaSuccess ||
        (l1 && (cudaMemcpy(p->d_fwd2, h_fwd2.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(p->d_inv2, h_inv2.data(), bt, cudaMemcpyHostToDevice) != cudaSuccess))) {
        cudaGetLastError();
        free32(p);
        delete p;
        return NTT_ERR_CUDA;
    }
    p->table_bytes = (l1 ? 4 : 2) * bt + bp;
    *out = p;
    return NTT_OK;
}

ntt_status_t ntt_plan_info32(ntt32_plan_t plan, unsigned* L, unsigned* logn, unsigned* log_n1, uint32_t* psi_out,
                             uint64_t* table_bytes)
{
    if (!plan) return NTT_ERR_INVALID_ARG;
    if (L) *L = plan->L;
    if (logn) *logn = plan->logn;
    if (log_n1) *log_n1 = plan->log_n1;
    if (psi_out) std::copy(plan->psis.begin(), plan->psis.end(), psi_out);
    if (table_bytes) *table_bytes = plan->table_bytes;
    return NTT_OK;
}

ntt_status_t ntt_forward32(ntt32_plan_t plan, uint32_t* data, unsigned batch, void* stream)
{
    return run32(plan, data, batch, stream, false);
}

ntt_status_t ntt_inverse32(ntt32_plan_t plan, uint32_t* data, unsigned batch, void* stream)
{
    return run32(plan, data, batch, stream, true);
}

ntt_status_t ntt_plan_destroy32(ntt32_plan_t plan)
{
    if (!plan) return NTT_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != plan->device) cudaSetDevice(plan->device);
    free32(plan);
    if (prev >= 0 && prev != plan->device) cudaSetDevice(prev);
    delete plan;
    return NTT_OK;
}

}  // extern "C"
