// ntt_native.cu -- the paper's "Native" comparison arm (fig:native_shoup,
// P:437-447): the default forward kernels -- Kernel-1 +
// Kernel-2 of the default split, or the single-CTA kernel for N <= 2^13 --
// instantiated on PrimeConstN, whose twiddle product is the native 128-bit
// modulo (unsigned __int128)(b w) % p instead of Shoup's modmul.  Everything
// else (schedule, layout, SMEM exchange, final normalisation) is unchanged, so
// the time difference is the modmul alone.  Forward, no OT.
#include "ntt_kernels.cuh"

namespace ntt {
namespace {

template <int LOGN, int LOGN1>
cudaError_t native_split(const KArgs& a, uint32_t rows, cudaStream_t st)
{
    constexpr int LOGM = LOGN - LOGN1;
    constexpr int LE2 = 4 | kRemLast;
    if (a.log_n1 != (uint32_t)LOGN1) return cudaErrorNotSupported;  // default split only
    cudaError_t e = detail::launch_cols_t<LOGN1, LOGN, 4, false, PrimeConstN>(a, rows, st);
    if (e != cudaSuccess) return e;
    // Kernel-2 as launch_k2_t picks it for the default variant: the shared-twiddle
    // kernel when the batch fills its CTAs and N2 >= 2^8, else the persistent one
    if constexpr (LOGM >= 8) {
        if (a.batch >= (4096u >> LOGM))
            return detail::launch_shared_t<LOGM, false, 0, false, PrimeConstN, LE2>(a, st);
    }
    return detail::launch_blocks_t<LOGM, LE2, false, 0, false, PrimeConstN>(a, st);
}

}  // namespace

cudaError_t launch_native_forward(KArgs a, uint32_t rows, cudaStream_t st)
{
    if (a.log_n1 == 0) {
        a.total_blocks = rows;
        // single-CTA kernel (N <= 2^13)
        cudaError_t err = cudaErrorNotSupported;
        switch (a.logn) {
#define NATIVE_CASE(L)                                                                                        \
    case L: err = detail::launch_contig_t<L, 4, false, false, 0, false, false, PrimeConstN>(a, 1, st); break;
            NATIVE_CASE(1) NATIVE_CASE(2) NATIVE_CASE(3) NATIVE_CASE(4) NATIVE_CASE(5) NATIVE_CASE(6)
            NATIVE_CASE(7) NATIVE_CASE(8) NATIVE_CASE(9) NATIVE_CASE(10) NATIVE_CASE(11) NATIVE_CASE(12)
            NATIVE_CASE(13)
#undef NATIVE_CASE
            default: break;
        }
        return err;
    }
    a.total_blocks = rows << a.log_n1;
    a.log_tiles = a.logn - a.log_n1 - 4;
    switch (a.logn) {
        case 14: return native_split<14, 7>(a, rows, st);
        case 15: return native_split<15, 7>(a, rows, st);
        case 16: return native_split<16, 8>(a, rows, st);
        case 17: return native_split<17, 8>(a, rows, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace ntt
