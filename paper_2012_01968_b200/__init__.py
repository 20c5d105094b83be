"""B200-native batched negacyclic NTT / iNTT over RNS residue rows
(arxiv 2012.01968 hot path).

Thin Python layer over the C ABI in include/ntt.h (libntt.so).  PyTorch is
used only for device memory and streams; every arithmetic step runs in the
sm_100a kernels.  Layout of a batch: ``[batch][L][N]`` uint64 (or int64 with
the same bits), row (b, l) reduced mod ``primes[l]``.

    plan = Plan(1 << 17, find_primes(1 << 17, 60))
    plan.forward(x)   # in place, bit-reversed NTT domain
    plan.inverse(x)   # in place, back to coefficients
"""
from __future__ import annotations

import ctypes

from ._native import (NTT_ARITH_GENERAL_D, NTT_ARITH_PROTH, NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL, NTT_GRAPH_PRODUCT,
                      NTT_PRIMES_2N,
                      NTT_PRIMES_PROTH32, NttError, Opts, check, lib)

__all__ = ["Plan", "Plan32", "Graph", "find_primes", "find_primes32", "find_psi", "table_sizes", "shoup_companion",
           "NttError", "NTT_DIR_FORWARD", "NTT_DIR_INVERSE", "NTT_GRAPH_PRODUCT",
           "NTT_GRAPH_ONE_KERNEL"]


PRIME_FORMS = {"2n": NTT_PRIMES_2N, "proth": NTT_PRIMES_PROTH32}


def find_primes(N: int, count: int, form: str = "2n") -> list[int]:
    """First ``count`` primes in [2^59, 2^60), descending (host): form "2n" =
    p = 1 mod 2N from 2^60 - 2N + 1 (R3); "proth" = p = 1 mod 2^32."""
    out = (ctypes.c_uint64 * count)()
    check(lib().ntt_find_primes_ex(N, count, PRIME_FORMS[form], out), "ntt_find_primes_ex")
    return [int(v) for v in out]


def find_primes32(N: int, count: int) -> list[int]:
    """First ``count`` primes p = 1 mod 2N in [2^29, 2^30), descending (host)."""
    out = (ctypes.c_uint32 * count)()
    check(lib().ntt_find_primes32(N, count, out), "ntt_find_primes32")
    return [int(v) for v in out]


def find_psi(p: int, N: int) -> int:
    """Smallest primitive 2N-th root of unity mod p (host)."""
    v = ctypes.c_uint64()
    check(lib().ntt_find_psi(p, N, ctypes.byref(v)), "ntt_find_psi")
    return int(v.value)


def shoup_companion(w: int, p: int) -> int:
    """floor(w 2^64 / p), as the plan tables store it (host, R6)."""
    v = ctypes.c_uint64()
    check(lib().ntt_shoup_companion(w, p, ctypes.byref(v)), "ntt_shoup_companion")
    return int(v.value)


def table_sizes(N: int, L: int, ot_base: int = 0) -> dict:
    """Twiddle storage of a plan (host): bytes of one direction's Psi tables,
    OT base entries per prime, and all device bytes of a default plan."""
    a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().ntt_table_sizes(N, L, ot_base, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "ntt_table_sizes")
    return {"psi_bytes": int(a.value), "ot_entries": int(b.value), "plan_bytes": int(c.value)}


def _host_ptr(a, what: str) -> tuple[int, int]:
    """(address, 64-bit words) of a C-contiguous CPU buffer of 64-bit integers
    (numpy array or CPU torch tensor)."""
    import numpy as np

    if hasattr(a, "data_ptr"):  # torch
        import torch

        if a.device.type != "cpu":
            raise ValueError(f"{what} must be a CPU (host) tensor")
        if a.dtype not in (torch.int64, torch.uint64):
            raise TypeError(f"{what} must hold 64-bit integers, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        return a.data_ptr(), a.numel()
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{what} must be a numpy array or a CPU torch tensor")
    if a.dtype not in (np.uint64, np.int64):
        raise TypeError(f"{what} must hold 64-bit integers, got {a.dtype}")
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what} must be C-contiguous")
    return a.ctypes.data, a.size


def _dev_ptr(t, N: int, L: int, bits: int = 64) -> tuple[int, int]:
    """(data_ptr, batch) of a CUDA [batch][L][N] tensor of 64- (or 32-) bit words."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch CUDA tensor")
    ok = (torch.uint64, torch.int64) if bits == 64 else (torch.uint32, torch.int32)
    if t.dtype not in ok:
        raise TypeError(f"dtype must be uint{bits} or int{bits}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if t.numel() % (N * L):
        raise ValueError(f"numel {t.numel()} is not a multiple of L*N = {L * N}")
    return t.data_ptr(), t.numel() // (N * L)


def _stream_handle(stream, t=None) -> int:
    """cudaStream_t of `stream`, or of the current stream of t's device (the
    raw-stream query is several us cheaper than torch.cuda.current_stream())."""
    import torch

    if stream is None:
        dev = t.device.index if t is not None else torch.cuda.current_device()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return raw(dev)
        stream = torch.cuda.current_stream(dev)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Plan:
    """Owns the device twiddle tables of one (N, prime chain) on the current
    CUDA device (ntt_plan_create_ex)."""

    def __init__(self, N: int, primes, ot: bool = False, ot_base: int = 0, ot_stages: int = 0,
                 log_n1: int = 0, proth_arith: bool = True, fused: bool | None = None,
                 k1_variant: int = 0, k2_variant: int = 0):
        self.N = int(N)
        self.primes = [int(p) for p in primes]
        self.L = len(self.primes)
        arr = (ctypes.c_uint64 * max(self.L, 1))(*self.primes)
        opts = Opts(1 if ot else -1, ot_base, ot_stages, log_n1, 0 if proth_arith else -1,
                    0 if fused is None else (1 if fused else -1), k1_variant, k2_variant)
        h = ctypes.c_void_p()
        check(lib().ntt_plan_create_ex(ctypes.byref(h), self.N, arr, self.L, ctypes.byref(opts)),
              "ntt_plan_create")
        self._h = h

    # ---------------------------------------------------------------- queries
    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise ValueError("plan destroyed")
        return self._h

    @property
    def psis(self) -> list[int]:
        out = (ctypes.c_uint64 * self.L)()
        check(lib().ntt_plan_psi(self.handle, out), "ntt_plan_psi")
        return [int(v) for v in out]

    def info(self) -> dict:
        L, logn, logn1, ots, otb = (ctypes.c_uint() for _ in range(5))
        ote, pr = ctypes.c_int(), ctypes.c_int()
        tb = ctypes.c_uint64()
        check(lib().ntt_plan_info(self.handle, ctypes.byref(L), ctypes.byref(logn), ctypes.byref(logn1),
                                  ctypes.byref(ote), ctypes.byref(otb), ctypes.byref(ots), ctypes.byref(tb)))
        npass, ncl = ctypes.c_uint(), ctypes.c_uint()
        check(lib().ntt_plan_exec(self.handle, ctypes.byref(pr), ctypes.byref(npass), ctypes.byref(ncl)))
        return {"L": L.value, "logn": logn.value, "log_n1": logn1.value, "ot_enable": bool(ote.value),
                "ot_base": otb.value, "ot_stages": ots.value, "table_bytes": tb.value,
                "proth": pr.value == NTT_ARITH_PROTH,
                "arith": {NTT_ARITH_PROTH: "proth", NTT_ARITH_GENERAL_D: "general-d"}.get(pr.value, "general"),
                "passes": npass.value, "cluster": ncl.value}

    # ---------------------------------------------------------------- transforms
    def forward(self, x, stream=None):
        """In-place forward NTT of a CUDA [batch][L][N] tensor (asynchronous)."""
        ptr, batch = _dev_ptr(x, self.N, self.L)
        check(lib().ntt_forward(self.handle, ptr, batch, _stream_handle(stream, x)), "ntt_forward")
        return x

    def inverse(self, x, stream=None):
        """In-place inverse NTT of a CUDA [batch][L][N] tensor (asynchronous)."""
        ptr, batch = _dev_ptr(x, self.N, self.L)
        check(lib().ntt_inverse(self.handle, ptr, batch, _stream_handle(stream, x)), "ntt_inverse")
        return x

    @property
    def passes(self) -> int:
        """Kernels per direction: 2 for the two-kernel split, 1 otherwise."""
        return self.info()["passes"]

    def launch_pass(self, x, direction: int, pass_index: int, stream=None):
        """Enqueue one kernel of a direction (for per-kernel timing)."""
        ptr, batch = _dev_ptr(x, self.N, self.L)
        check(lib().ntt_launch_pass(self.handle, ptr, batch, direction, pass_index, _stream_handle(stream, x)),
              "ntt_launch_pass")
        return x

    def pointwise_inverse(self, a_ntt, x, stream=None):
        """x <- iNTT(a_ntt (.) x): both CUDA tensors in the NTT domain."""
        pa, batch_a = _dev_ptr(a_ntt, self.N, self.L)
        ptr, batch = _dev_ptr(x, self.N, self.L)
        if batch_a != batch:
            raise ValueError("operands must have the same batch")
        check(lib().ntt_pointwise_inverse(self.handle, pa, ptr, batch, _stream_handle(stream, x)),
              "ntt_pointwise_inverse")
        return x

    def negacyclic_mul(self, a, b, stream=None):
        """b <- a * b mod (X^N + 1) per row; a is left in the NTT domain."""
        pa, batch_a = _dev_ptr(a, self.N, self.L)
        pb, batch = _dev_ptr(b, self.N, self.L)
        if batch_a != batch:
            raise ValueError("operands must have the same batch")
        check(lib().ntt_negacyclic_mul(self.handle, pa, pb, batch, _stream_handle(stream, b)), "ntt_negacyclic_mul")
        return b

    def forward_variant(self, x, variant: int, stream=None):
        """Forward NTT through one of the paper's comparison kernels
        (1 = radix-2 per stage, 2 = register radix-16, 3 = default kernels with
        native-modulo twiddle products; 0 = default path)."""
        ptr, batch = _dev_ptr(x, self.N, self.L)
        check(lib().ntt_forward_variant(self.handle, ptr, batch, variant, _stream_handle(stream, x)),
              "ntt_forward_variant")
        return x

    def workspace_words(self, batch: int, chunk: int = 0) -> int:
        return int(lib().ntt_workspace_words(self.handle, batch, chunk))

    def execute_host(self, host_in, host_out, flags: int, workspace, chunk: int = 0, stream=None) -> None:
        """End-to-end transform of HOST buffers (C-contiguous 64-bit numpy
        arrays or CPU tensors, ideally pinned) through a CUDA workspace tensor
        of 64-bit words; synchronous.  The workspace is used after the work
        already queued on `stream` (default: the current stream)."""
        pin, n_in = _host_ptr(host_in, "host_in")
        pout, n_out = _host_ptr(host_out, "host_out")
        if n_in != n_out or n_in % (self.N * self.L):
            raise ValueError("host buffers must both hold batch*L*N words")
        batch = n_in // (self.N * self.L)
        wptr, _ = _dev_ptr(workspace, 1, 1)
        check(lib().ntt_execute_host(self.handle, flags, pin, pout, batch, wptr, workspace.numel(), chunk,
                                     _stream_handle(stream, workspace)), "ntt_execute_host")

    def graph(self, x, flags: int = NTT_DIR_FORWARD | NTT_DIR_INVERSE, other=None) -> "Graph":
        """Capture the transforms `flags` of the CUDA tensor x (or, with
        NTT_GRAPH_PRODUCT, the product other <- x * other) into a replayable
        request graph (ntt_graph_create).  | NTT_GRAPH_ONE_KERNEL: the whole
        request as one persistent kernel (N = 2^14..2^17, no OT)."""
        return Graph(self, x, flags, other)

    def corrupt_twiddle(self, direction: int, l: int, index: int, field: int, mask: int) -> None:
        """TESTING ONLY: XOR mask into Psi[index] (field 0 = w, 1 = w_bar) of
        prime l in the plan's device tables (ntt_debug_corrupt_twiddle)."""
        check(lib().ntt_debug_corrupt_twiddle(self.handle, direction, l, index, field, mask),
              "ntt_debug_corrupt_twiddle")

    # ---------------------------------------------------------------- lifetime
    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib().ntt_plan_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """A captured request (ntt_graph_create): replay with launch(); the tensor(s)
    it was captured on are baked in and kept alive with the plan."""

    def __init__(self, plan: Plan, x, flags: int, other=None):
        ptr, batch = _dev_ptr(x, plan.N, plan.L)
        ptr2 = 0
        if other is not None:
            ptr2, b2 = _dev_ptr(other, plan.N, plan.L)
            if b2 != batch:
                raise ValueError("operands must have the same batch")
        h = ctypes.c_void_p()
        check(lib().ntt_graph_create(ctypes.byref(h), plan.handle, ptr, ptr2 or None, batch, flags),
              "ntt_graph_create")
        self._h = h
        self._keep = (plan, x, other)

    def launch(self, stream=None) -> None:
        if self._h is None:
            raise ValueError("graph destroyed")
        check(lib().ntt_graph_launch(self._h, _stream_handle(stream, self._keep[1])), "ntt_graph_launch")

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib().ntt_graph_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan32:
    """The 32-bit-word path (ntt_plan_create32): primes in [2^29, 2^30), one
    uint32 (or int32) word per residue, ``[batch][L][N]``.  Same transform and
    output order as :class:`Plan`; no OT, no fused products."""

    def __init__(self, N: int, primes, log_n1: int = 0):
        self.N = int(N)
        self.primes = [int(p) for p in primes]
        self.L = len(self.primes)
        arr = (ctypes.c_uint32 * max(self.L, 1))(*self.primes)
        h = ctypes.c_void_p()
        check(lib().ntt_plan_create32(ctypes.byref(h), self.N, arr, self.L, log_n1), "ntt_plan_create32")
        self._h = h

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise ValueError("plan destroyed")
        return self._h

    def info(self) -> dict:
        L, logn, logn1 = (ctypes.c_uint() for _ in range(3))
        psi = (ctypes.c_uint32 * self.L)()
        tb = ctypes.c_uint64()
        check(lib().ntt_plan_info32(self.handle, ctypes.byref(L), ctypes.byref(logn), ctypes.byref(logn1), psi,
                                    ctypes.byref(tb)), "ntt_plan_info32")
        return {"L": L.value, "logn": logn.value, "log_n1": logn1.value, "psis": [int(v) for v in psi],
                "table_bytes": tb.value}

    @property
    def psis(self) -> list[int]:
        return self.info()["psis"]

    def forward(self, x, stream=None):
        ptr, batch = _dev_ptr(x, self.N, self.L, 32)
        check(lib().ntt_forward32(self.handle, ptr, batch, _stream_handle(stream, x)), "ntt_forward32")
        return x

    def inverse(self, x, stream=None):
        ptr, batch = _dev_ptr(x, self.N, self.L, 32)
        check(lib().ntt_inverse32(self.handle, ptr, batch, _stream_handle(stream, x)), "ntt_inverse32")
        return x

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib().ntt_plan_destroy32(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
