"""ctypes binding of libntt.so (include/ntt.h).  Argument marshalling only:
every step of the transform runs in the CUDA kernels behind the C ABI.
There is no fallback -- if the library is missing, loading fails loudly."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libntt.so")

NTT_OK = 0
STATUS = {
    0: "NTT_OK", -1: "NTT_ERR_INVALID_N", -2: "NTT_ERR_INVALID_PRIME", -3: "NTT_ERR_INVALID_ARG",
    -4: "NTT_ERR_MISALIGNED", -5: "NTT_ERR_WRONG_DEVICE", -6: "NTT_ERR_CUDA", -7: "NTT_ERR_OOM",
    -8: "NTT_ERR_RANGE_EXHAUSTED",
}
NTT_DIR_FORWARD = 1
NTT_DIR_INVERSE = 2
NTT_VARIANT_DEFAULT, NTT_VARIANT_RADIX2, NTT_VARIANT_RADIX16, NTT_VARIANT_NATIVE = 0, 1, 2, 3
NTT_PRIMES_2N, NTT_PRIMES_PROTH32 = 0, 1
NTT_ARITH_GENERAL, NTT_ARITH_PROTH, NTT_ARITH_GENERAL_D = 0, 1, 2
NTT_GRAPH_PRODUCT = 4
NTT_GRAPH_ONE_KERNEL = 8

# every symbol include/ntt.h declares
EXPORTS = [
    "ntt_find_primes", "ntt_find_primes_ex", "ntt_plan_exec", "ntt_find_psi", "ntt_plan_create", "ntt_plan_create_ex", "ntt_plan_psi",
    "ntt_plan_info", "ntt_forward", "ntt_inverse", "ntt_launch_pass", "ntt_pointwise_inverse", "ntt_negacyclic_mul", "ntt_forward_variant",
    "ntt_execute_host", "ntt_workspace_words",
    "ntt_plan_destroy", "ntt_status_string",
    "ntt_graph_create", "ntt_graph_launch", "ntt_graph_destroy",
    "ntt_shoup_companion", "ntt_table_sizes", "ntt_debug_corrupt_twiddle",
    "ntt_find_primes32", "ntt_plan_create32", "ntt_plan_info32", "ntt_forward32", "ntt_inverse32",
    "ntt_plan_destroy32",
]


class NttError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        name = STATUS.get(status, str(status))
        msg = lib().ntt_status_string(status).decode()
        super().__init__(f"{what}: {name} ({msg})" if what else f"{name} ({msg})")


class Opts(ctypes.Structure):
    _fields_ = [("ot_enable", ctypes.c_int), ("ot_base", ctypes.c_uint),
                ("ot_stages", ctypes.c_uint), ("log_n1", ctypes.c_uint), ("prime_arith", ctypes.c_int),
                ("fused", ctypes.c_int), ("k1_variant", ctypes.c_int), ("k2_variant", ctypes.c_int)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2012_01968_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        u32, i32, u64, vp = ctypes.c_uint, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p
        p64 = ctypes.POINTER(ctypes.c_uint64)
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.ntt_find_primes.argtypes = [u32, u32, p64]
        L.ntt_find_primes_ex.argtypes = [u32, u32, u32, p64]
        L.ntt_plan_exec.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(u32), ctypes.POINTER(u32)]
        L.ntt_find_psi.argtypes = [u64, u32, p64]
        L.ntt_plan_create.argtypes = [pp, u32, p64, u32]
        L.ntt_plan_create_ex.argtypes = [pp, u32, p64, u32, ctypes.POINTER(Opts)]
        L.ntt_plan_psi.argtypes = [vp, p64]
        L.ntt_plan_info.argtypes = [vp, ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(u32),
                                    ctypes.POINTER(i32), ctypes.POINTER(u32), ctypes.POINTER(u32), p64]
        L.ntt_forward.argtypes = [vp, vp, u32, vp]
        L.ntt_inverse.argtypes = [vp, vp, u32, vp]
        L.ntt_launch_pass.argtypes = [vp, vp, u32, u32, u32, vp]
        L.ntt_forward_variant.argtypes = [vp, vp, u32, u32, vp]
        L.ntt_pointwise_inverse.argtypes = [vp, vp, vp, u32, vp]
        L.ntt_negacyclic_mul.argtypes = [vp, vp, vp, u32, vp]
        L.ntt_execute_host.argtypes = [vp, u32, vp, vp, u32, vp, u64, u32, vp]
        L.ntt_graph_create.argtypes = [pp, vp, vp, vp, u32, u32]
        L.ntt_graph_launch.argtypes = [vp, vp]
        L.ntt_graph_destroy.argtypes = [vp]
        L.ntt_shoup_companion.argtypes = [u64, u64, p64]
        L.ntt_table_sizes.argtypes = [u32, u32, u32, p64, p64, p64]
        L.ntt_debug_corrupt_twiddle.argtypes = [vp, u32, u32, u32, u32, u64]
        L.ntt_workspace_words.argtypes = [vp, u32, u32]
        L.ntt_workspace_words.restype = u64
        L.ntt_plan_destroy.argtypes = [vp]
        p32 = ctypes.POINTER(ctypes.c_uint32)
        L.ntt_find_primes32.argtypes = [u32, u32, p32]
        L.ntt_plan_create32.argtypes = [pp, u32, p32, u32, u32]
        L.ntt_plan_info32.argtypes = [vp, ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(u32), p32, p64]
        L.ntt_forward32.argtypes = [vp, vp, u32, vp]
        L.ntt_inverse32.argtypes = [vp, vp, u32, vp]
        L.ntt_plan_destroy32.argtypes = [vp]
        L.ntt_status_string.argtypes = [i32]
        L.ntt_status_string.restype = ctypes.c_char_p
        for name in ["ntt_find_primes", "ntt_find_primes_ex", "ntt_plan_exec", "ntt_find_psi", "ntt_plan_create", "ntt_plan_create_ex",
                     "ntt_plan_psi", "ntt_plan_info", "ntt_forward", "ntt_inverse", "ntt_launch_pass", "ntt_forward_variant",
                     "ntt_pointwise_inverse", "ntt_negacyclic_mul", "ntt_execute_host",
                     "ntt_plan_destroy", "ntt_find_primes32", "ntt_plan_create32", "ntt_plan_info32",
                     "ntt_forward32", "ntt_inverse32", "ntt_plan_destroy32", "ntt_graph_create",
                     "ntt_graph_launch", "ntt_graph_destroy", "ntt_shoup_companion", "ntt_table_sizes",
                     "ntt_debug_corrupt_twiddle"]:
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status != NTT_OK:
        raise NttError(status, what)
