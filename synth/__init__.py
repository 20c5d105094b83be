"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the method's arithmetic: it maps a counter to a
uniform residue in [0, p) (see ``synth.c`` and DESIGN.md section 5).  The C
fill is used for speed; ``draw_numpy`` is an independent numpy rendering of
the same formula used by a test to check the C fill.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

SEED = 0x2012019680000000

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None

# config ids of BASELINE.json's configs (C1..C5) and of the paper's Table 2 setting
CONFIG_IDS = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "Cp": 6, "test": 15}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _l():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        p64 = ctypes.POINTER(ctypes.c_uint64)
        L.synth_fill_rows.argtypes = [p64, ctypes.c_uint64, p64, p64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint]
        L.synth_fill_rows.restype = None
        _lib = L
    return _lib


def _p(a):
    return ctypes.cast(ctypes.c_void_p(a.ctypes.data), ctypes.POINTER(ctypes.c_uint64))


def fill_rows(out: np.ndarray, row_ids, row_primes, seed: int = SEED, config_id: int = 15,
              nthreads: int = 0) -> np.ndarray:
    """Fill ``out`` (nrows x N uint64, C-contiguous; may be a view of pinned
    memory) with the seeded residues of the given global rows."""
    assert out.dtype == np.uint64 and out.flags["C_CONTIGUOUS"]
    N = out.shape[-1]
    nrows = out.size // N
    ids = np.ascontiguousarray(np.asarray(row_ids, dtype=np.uint64).reshape(-1))
    prs = np.ascontiguousarray(np.asarray(row_primes, dtype=np.uint64).reshape(-1))
    assert ids.size == nrows and prs.size == nrows
    _l().synth_fill_rows(_p(out), N, _p(ids), _p(prs), nrows, seed, config_id, nthreads)
    return out


def rns_rows(primes, batch: int, N: int, seed: int = SEED, config_id: int = 15,
             prime_offset: int = 0, L_total: int | None = None, batch_offset: int = 0,
             out: np.ndarray | None = None) -> np.ndarray:
    """A [batch][L][N] array of residues.  Row (b, l) has global id
    (batch_offset + b) * L_total + (prime_offset + l) so a shard of a larger
    job draws exactly the values the unsharded job would."""
    primes = [int(p) for p in primes]
    L = len(primes)
    L_total = L if L_total is None else L_total
    ids = np.array([(batch_offset + b) * L_total + prime_offset + l
                    for b in range(batch) for l in range(L)], dtype=np.uint64)
    prs = np.array([primes[l] for b in range(batch) for l in range(L)], dtype=np.uint64)
    if out is None:
        out = np.empty((batch, L, N), dtype=np.uint64)
    return fill_rows(out, ids, prs, seed, config_id)


# ------------------------------------------------- independent numpy rendering

_M32 = np.uint64(0xFFFFFFFF)


def _splitmix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _mulhi_np(a: np.ndarray, b: int) -> np.ndarray:
    b = np.uint64(b)
    a0, a1 = a & _M32, a >> np.uint64(32)
    b0, b1 = b & _M32, b >> np.uint64(32)
    with np.errstate(over="ignore"):
        lo = a0 * b0
        m1 = a1 * b0 + (lo >> np.uint64(32))
        m2 = a0 * b1 + (m1 & _M32)
        return a1 * b1 + (m1 >> np.uint64(32)) + (m2 >> np.uint64(32))


def draw_numpy(row_id: int, p: int, N: int, seed: int = SEED, config_id: int = 15) -> np.ndarray:
    i = np.arange(N, dtype=np.uint64)
    key = np.uint64((config_id << 48) | (row_id << 20))
    return _mulhi_np(_splitmix64_np(np.uint64(seed) ^ (key | i)), p)
