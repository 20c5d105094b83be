// ntt_launch.h -- host-side launchers of the kernels in ntt_kernels.cuh.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <mutex>
#include "ntt_device.cuh"

namespace ntt {
// One-time, per-device setup of a kernel (cudaFuncSetAttribute, occupancy
// query), safe from any number of host threads: the first caller on a device
// runs `f` under the mutex and the device's bit is published only after `f`
// succeeded, so no thread launches before the attribute is in place; a failed
// setup is retried by the next call.  value(dev) holds what `f` stored.
struct DeviceOnce {
    std::atomic<uint64_t> done{0};
    std::mutex mu;
    int val[64] = {};
    template <class F>
    cudaError_t run(F&& f)
    {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
        std::lock_guard<std::mutex> lk(mu);
        if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
        const cudaError_t e = f(val[dev & 63]);
        if (e != cudaSuccess) {
            cudaGetLastError();  // consume it: reported once, here
            return e;
        }
        done.fetch_or(bit, std::memory_order_release);
        return cudaSuccess;
    }
    int value()
    {
        int dev = 0;
        cudaGetDevice(&dev);
        return val[dev & 63];
    }
};
// Error of the launch just made: cudaGetLastError consumes it, so one failed
// launch is reported once and does not poison later calls on the thread.
inline cudaError_t launch_status() { return cudaGetLastError(); }

// Launch a transform kernel with programmatic stream serialization (PDL, see
// pdl_trigger / pdl_wait in ntt_device.cuh); the status of the launch.
template <class K>
cudaError_t launch_pdl(void (*fn)(K), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const K& a,
                       const cudaLaunchAttribute* extra = nullptr)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    unsigned n = 1;
    if (extra) at[n++] = *extra;
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    return e != cudaSuccess ? (cudaGetLastError(), e) : launch_status();
}

// arith: the prime-constant type the kernels are instantiated on --
// kArithGeneral (PrimeConst, any prime) or kArithProth (PrimeConstP: every
// prime = 1 mod 2^32); DESIGN.md 5.1.  The Proth form exists for the default
// kernel variants only (ntt_kernels.cuh).
// kArithGeneralD: general arithmetic, every prime p = 2^60 - d with d < 2^32
// (the R3 chain); passed for the forward Kernel-2 (d-form final reduction)
// and for Kernel-1' outside the NTT-domain product path (exact-division N^-1);
// PrimeConstD, ntt_kernels_d.cu.
// kArithProthD: Proth arithmetic with Kernel-1''s exact-division N^-1 (PrimeConstPD).
enum { kArithGeneral = 0, kArithProth = 1, kArithGeneralD = 2, kArithProthD = 3 };
// One kernel per row: contiguous rows of N = 2^logn, N <= 2^13.
cudaError_t launch_single(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st,
                          int arith = kArithGeneral);
// Kernel-2 (forward) / Kernel-2' (inverse): contiguous N2-blocks.
// loge: the Kernel-2 variant (9 = default).
cudaError_t launch_k2(bool inverse, int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st,
                      int arith = kArithGeneral);
// Kernel-1 (forward) / Kernel-1' (inverse): stride-N2 columns, 16 per CTA.
cudaError_t launch_k1(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st,
                      int arith = kArithGeneral);
// per-family instantiations, one translation unit each (parallel compilation):
// _g general primes, _p Proth primes (ntt_single.cu, ntt_kernels_p.cu, ntt_k1.cu)
cudaError_t launch_single_g(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_single_p(bool inverse, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_k2_p(bool inverse, int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_k2_fwd_d(int loge, const KArgs& a, int ot_stages, uint32_t iters, cudaStream_t st);
cudaError_t launch_k1_inv_d(int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
cudaError_t launch_k1_inv_pd(int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
cudaError_t launch_k1_g(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
cudaError_t launch_k1_p(bool inverse, int loge, const KArgs& a, uint32_t rows, cudaStream_t st);
// Single-pass NTT / iNTT, one thread-block cluster per row (N = 2^14..2^17;
// ntt_fused.cuh).  a.tab2 must be the Kernel-2-ordered table of the split
// N = (N / 2^13) x 2^13.
cudaError_t launch_fused(bool inverse, const KArgs& a, uint32_t rows, cudaStream_t st, int arith);
// data <- mul_a (.) data 2^-64 (Montgomery), every word.
cudaError_t launch_pointwise(const KArgs& a, cudaStream_t st);
// The paper's comparison kernels, forward only: 1 = radix-2 per stage, 2 = register radix-16.
cudaError_t launch_baseline_forward(int variant, const KArgs& a, cudaStream_t st);
// The paper's "Native" arm: the default forward kernels with native-modulo twiddle products
// (ntt_native.cu); cudaErrorNotSupported for a non-default split.
cudaError_t launch_native_forward(KArgs a, uint32_t rows, cudaStream_t st);
// Single-launch request kernel (ntt_request.cu): forward and / or inverse of
// rows = batch * L rows of N = 2^14..2^17 in one cooperative launch with grid
// barriers between the column and block phases.
struct ReqArgs {
    uint64_t* data;        // [batch][L][N]
    const Tw* tf;          // [L][N] Psi, bit-reversed
    const Tw* ti;          // [L][N] Psi^-1, bit-reversed (R5)
    const PrimeConst* pc;  // [L]
    unsigned long long* bar;  // grid barrier arrival counter (kReqBarrierBytes), zeroed once, owned by the request object
    uint32_t L, rows;      // rows = batch * L
    uint32_t flags;        // NTT_DIR_FORWARD (1) | NTT_DIR_INVERSE (2)
};
constexpr size_t kReqBarrierBytes = 8;  // one 64-bit arrival counter (ntt_request.cu)
cudaError_t launch_request(unsigned logn, const ReqArgs& a, cudaStream_t st, int arith);
// 32-bit-word path: all passes of one direction.
cudaError_t launch32(bool inverse, const KArgs32& a, uint32_t rows, cudaStream_t st);
}  // namespace ntt
