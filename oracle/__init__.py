"""CPU oracle for the batched negacyclic NTT / iNTT (arxiv 2012.01968).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2012_01968_b200`` never imports it, and
the two share no code.

The arithmetic lives in ``ntt_oracle.c`` (plain C, ``unsigned __int128 %``);
this module is ctypes marshalling only.  Each function cites the PAPER.md
passage it follows (``P:n`` = /root/reference/PAPER.md line n).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ntt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

P59 = 1 << 59
P60 = 1 << 60


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (checker build; not the product path)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, u32, i32 = ctypes.c_uint64, ctypes.c_uint, ctypes.c_int
        p64 = ctypes.POINTER(ctypes.c_uint64)
        L.oracle_mulmod.argtypes = [u64, u64, u64]
        L.oracle_mulmod.restype = u64
        L.oracle_powmod.argtypes = [u64, u64, u64]
        L.oracle_powmod.restype = u64
        L.oracle_is_prime.argtypes = [u64]
        L.oracle_is_prime.restype = i32
        L.oracle_find_primes.argtypes = [u64, u64, u64, u32, p64]
        L.oracle_find_primes.restype = i32
        L.oracle_find_psi.argtypes = [u64, u64]
        L.oracle_find_psi.restype = u64
        L.oracle_bitrev.argtypes = [u64, u32]
        L.oracle_bitrev.restype = u64
        L.oracle_psi_table.argtypes = [u64, u64, u64, p64]
        L.oracle_psi_table.restype = None
        L.oracle_ntt_forward.argtypes = [p64, u64, u64, u64]
        L.oracle_ntt_forward.restype = i32
        L.oracle_ntt_inverse.argtypes = [p64, u64, u64, u64]
        L.oracle_ntt_inverse.restype = i32
        L.oracle_negacyclic_mul.argtypes = [p64, p64, p64, u64, u64]
        L.oracle_negacyclic_mul.restype = None
        L.oracle_pointwise_mul.argtypes = [p64, p64, p64, u64, u64]
        L.oracle_pointwise_mul.restype = None
        L.oracle_ntt_batch.argtypes = [p64, u64, p64, p64, u32, u32, i32, u32]
        L.oracle_ntt_batch.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


# --------------------------------------------------------------- arithmetic

def mulmod(a: int, b: int, p: int) -> int:
    """(a*b) mod p by a 128-bit product and remainder."""
    return int(lib().oracle_mulmod(a, b, p))


def powmod(a: int, e: int, p: int) -> int:
    return int(lib().oracle_powmod(a, e, p))


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin, bases 2..37 (exact for 64-bit n)."""
    return bool(lib().oracle_is_prime(n))


def find_primes(N: int, count: int, lo: int = P59, hi: int = P60) -> list[int]:
    """First ``count`` primes p = 1 mod 2N in [lo, hi), descending (P:274, P:296,
    P:423; R1/R3).  Raises if the range runs out."""
    out = np.zeros(max(count, 1), dtype=np.uint64)
    got = lib().oracle_find_primes(N, lo, hi, count, _ptr(out))
    if got < count:
        raise ValueError(f"only {got} primes = 1 mod {2 * N} in [{lo}, {hi})")
    return [int(x) for x in out[:count]]


def find_psi(p: int, N: int) -> int:
    """Smallest primitive 2N-th root of unity mod p (R2)."""
    r = int(lib().oracle_find_psi(p, N))
    if r == 0:
        raise ValueError(f"p={p} is not an NTT prime for N={N}")
    return r


def bitrev(i: int, logn: int) -> int:
    return int(lib().oracle_bitrev(i, logn))


def psi_table(p: int, root: int, N: int) -> np.ndarray:
    """Psi[i] = root^bitrev(i)."""
    out = np.zeros(N, dtype=np.uint64)
    lib().oracle_psi_table(p, root, N, _ptr(out))
    return out


# --------------------------------------------------------------- transforms

def ntt_forward(a, p: int, psi: int) -> np.ndarray:
    """Algorithm 1; output bit-reversed.  Returns a copy."""
    x = _u64(a).copy()
    if lib().oracle_ntt_forward(_ptr(x), x.size, p, psi):
        raise ValueError("N must be a power of two")
    return x


def ntt_inverse(a, p: int, psi: int) -> np.ndarray:
    """Gentleman-Sande inverse with Psi^-1 and N^-1 (R5)."""
    x = _u64(a).copy()
    if lib().oracle_ntt_inverse(_ptr(x), x.size, p, psi):
        raise ValueError("N must be a power of two")
    return x


def negacyclic_mul(a, b, p: int) -> np.ndarray:
    """Schoolbook negacyclic product by its definition, O(N^2)."""
    a, b = _u64(a), _u64(b)
    c = np.zeros_like(a)
    lib().oracle_negacyclic_mul(_ptr(a), _ptr(b), _ptr(c), a.size, p)
    return c


def pointwise_mul(a, b, p: int) -> np.ndarray:
    a, b = _u64(a), _u64(b)
    c = np.zeros_like(a)
    lib().oracle_pointwise_mul(_ptr(a), _ptr(b), _ptr(c), a.size, p)
    return c


def ntt_batch(data: np.ndarray, primes, psis, direction: int, nthreads: int = 0) -> np.ndarray:
    """In-place batched transform of a [batch][L][N] uint64 array (P:264-287,
    P:479-481).  direction +1 forward, -1 inverse.  Returns ``data``."""
    assert data.dtype == np.uint64 and data.flags["C_CONTIGUOUS"] and data.ndim == 3
    batch, L, N = data.shape
    pr, ps = _u64(primes), _u64(psis)
    assert pr.size == L and ps.size == L
    s = lib().oracle_ntt_batch(_ptr(data), N, _ptr(pr), _ptr(ps), L, batch, direction, nthreads)
    if s:
        raise ValueError("oracle_ntt_batch failed")
    return data
