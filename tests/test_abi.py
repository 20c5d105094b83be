"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only logic (prime scan, psi, argument checks)
behaves; no compute call needs a GPU here."""
import ctypes
import glob
import os
import re

import pytest

import oracle
from paper_2012_01968_b200 import _native
from paper_2012_01968_b200 import find_primes, find_psi, NttError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = "".join(open(f).read() for f in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntt_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.lib()
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert sorted(declared) == sorted(_native.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    # exported with C linkage (no C++ mangling)
    out = os.popen(f"nm -D --defined-only {_native.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_status_strings():
    lib = _native.lib()
    for code in range(-8, 1):
        assert lib.ntt_status_string(code)


@pytest.mark.parametrize("logn,count", [(1, 3), (12, 4), (15, 15), (16, 45), (17, 60)])
def test_host_primes_match_oracle(logn, count):
    N = 1 << logn
    assert find_primes(N, count) == oracle.find_primes(N, count)


@pytest.mark.parametrize("logn", [1, 4, 12, 15, 16, 17])
def test_host_psi_matches_oracle(logn):
    N = 1 << logn
    for p in oracle.find_primes(N, 3):
        assert find_psi(p, N) == oracle.find_psi(p, N)


def test_host_helper_errors():
    with pytest.raises(NttError) as e:
        find_primes(3, 1)
    assert e.value.status == -1
    with pytest.raises(NttError) as e:
        find_primes(1 << 18, 1)
    assert e.value.status == -1
    with pytest.raises(NttError) as e:
        find_psi(19, 4)
    assert e.value.status == -2
    out = (ctypes.c_uint64 * 1)()
    assert _native.lib().ntt_find_primes(8, 0, out) == -3


def test_plan_create_argument_errors_before_device():
    lib = _native.lib()
    h = ctypes.c_void_p()
    p = oracle.find_primes(1 << 12, 2)
    arr = (ctypes.c_uint64 * 2)(*p)
    assert lib.ntt_plan_create(ctypes.byref(h), 3000, arr, 2) == -1          # N not a power of two
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 18, arr, 2) == -1       # N too large
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, None, 2) == -3      # no primes
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, arr, 0) == -3       # L = 0
    bad = (ctypes.c_uint64 * 2)(p[0], p[0])
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, bad, 2) == -2       # repeated prime
    bad = (ctypes.c_uint64 * 1)(p[0] + 2 * (1 << 12))                        # = 1 mod 2N, composite?
    if not oracle.is_prime(bad[0]):
        assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, bad, 1) == -2
    big = oracle.find_primes(1 << 12, 1, 1 << 60, 1 << 61)                 # >= 2^60: lazy headroom gone
    bad = (ctypes.c_uint64 * 1)(big[0])
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, bad, 1) == -2
    bad = (ctypes.c_uint64 * 1)(17)                                          # 17 != 1 mod 2^13
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, bad, 1) == -2
    assert lib.ntt_forward(None, None, 1, None) == -3
    assert lib.ntt_inverse(None, None, 1, None) == -3
    assert lib.ntt_plan_destroy(None) == 0


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    lib = _native.lib()
    h = ctypes.c_void_p()
    p = oracle.find_primes(1 << 12, 1)
    arr = (ctypes.c_uint64 * 1)(*p)
    assert lib.ntt_plan_create(ctypes.byref(h), 1 << 12, arr, 1) == -6      # NTT_ERR_CUDA, loudly


@pytest.mark.parametrize("logn,count", [(1, 3), (12, 8), (16, 60), (17, 120)])
def test_host_primes32_match_oracle(logn, count):
    from paper_2012_01968_b200 import find_primes32
    N = 1 << logn
    assert find_primes32(N, count) == oracle.find_primes(N, count, 1 << 29, 1 << 30)


def test_plan_create32_argument_errors():
    lib = _native.lib()
    h = ctypes.c_void_p()
    p = oracle.find_primes(1 << 12, 2, 1 << 29, 1 << 30)
    arr = (ctypes.c_uint32 * 2)(*p)
    assert lib.ntt_plan_create32(ctypes.byref(h), 3000, arr, 2, 0) == -1
    assert lib.ntt_plan_create32(ctypes.byref(h), 1 << 12, None, 2, 0) == -3
    assert lib.ntt_plan_create32(ctypes.byref(h), 1 << 12, arr, 0, 0) == -3
    bad = (ctypes.c_uint32 * 2)(p[0], p[0])
    assert lib.ntt_plan_create32(ctypes.byref(h), 1 << 12, bad, 2, 0) == -2      # repeated
    big = oracle.find_primes(1 << 12, 1, 1 << 30, 1 << 31)                     # >= 2^30: lazy headroom gone
    bad = (ctypes.c_uint32 * 1)(big[0])
    assert lib.ntt_plan_create32(ctypes.byref(h), 1 << 12, bad, 1, 0) == -2
    q = oracle.find_primes(1 << 16, 1, 1 << 29, 1 << 30)
    arr = (ctypes.c_uint32 * 1)(*q)
    assert lib.ntt_plan_create32(ctypes.byref(h), 1 << 16, arr, 1, 9) == -3      # split not compiled
    out = (ctypes.c_uint32 * 1)()
    assert lib.ntt_find_primes32(1 << 17, 10**6, (ctypes.c_uint32 * 10**6)()) == -8
    assert lib.ntt_find_primes32(8, 0, out) == -3
    assert lib.ntt_forward32(None, None, 1, None) == -3
    assert lib.ntt_plan_destroy32(None) == 0


def test_product_package_does_not_touch_oracle():
    """The product path never imports, links, includes or reads the oracle."""
    pkg = os.path.join(ROOT, "paper_2012_01968_b200")
    pat = re.compile(r"^\s*(import\s+oracle|from\s+oracle\b)|#include\s*[<\"].*oracle|liboracle|ntt_oracle",
                     re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not pat.search(src), f
    out = os.popen(f"nm -D {_native.LIB_PATH}").read()
    assert "oracle_" not in out


@pytest.mark.parametrize("logn,count", [(1, 2), (12, 4), (17, 60), (17, 64)])
def test_host_proth_primes_match_oracle(logn, count):
    """NTT_PRIMES_PROTH32: p = k 2^32 + 1 in [2^59, 2^60) (P:423 range; = 1 mod
    2N for every N <= 2^17, P:274 / R1), descending -- the oracle's own scan
    with step 2^32 finds the same list."""
    N = 1 << logn
    got = find_primes(N, count, "proth")
    assert got == oracle.find_primes(1 << 31, count)
    assert all(p % (1 << 32) == 1 and (1 << 59) <= p < (1 << 60) for p in got)
    assert got == sorted(got, reverse=True) and len(set(got)) == count
    # no prime of the family was skipped between the first and the last
    k_hi, k_lo = got[0] >> 32, got[-1] >> 32
    found = {p >> 32 for p in got}
    for k in range(k_lo, k_hi + 1):
        if k not in found:
            assert not oracle.is_prime((k << 32) + 1)
    assert (((1 << 28) - 1) << 32) + 1 >= got[0]


def test_proth_primes_errors():
    lib = _native.lib()
    out = (ctypes.c_uint64 * 2)()
    assert lib.ntt_find_primes_ex(1 << 12, 2, 7, out) == -3  # unknown form
    assert lib.ntt_find_primes_ex(3, 2, 1, out) == -1
    assert lib.ntt_find_primes_ex(1 << 12, 0, 1, out) == -3


# ------------------------------------------------------------------ round 2: ADVICE / golden / Python-side checks

def test_small_ntt_primes_rejected():
    """Primes below 2^59 are rejected with INVALID_PRIME before the device is
    touched (the 64-bit kernels need p > 2^58 for reduce_full's estimate and
    P:423 names [2^59, 2^60)); (N=4, p=17) is a valid NTT prime otherwise."""
    lib = _native.lib()
    h = ctypes.c_void_p()
    for n, p in [(4, 17), (256, 12289), (1 << 12, oracle.find_primes(1 << 12, 1, 1 << 58, 1 << 59)[0])]:
        arr = (ctypes.c_uint64 * 1)(p)
        assert lib.ntt_plan_create(ctypes.byref(h), n, arr, 1) == -2, (n, p)
    p59 = oracle.find_primes(1 << 12, 1, 1 << 59, (1 << 59) + (1 << 40))  # the lowest accepted range
    assert p59 and p59[0] >= 1 << 59


def test_golden_shoup_companion(golden):
    """w_bar(1,17) = floor(2^64/17), w_bar(0,17) = 0 -- the host
    routine the plan tables are built with."""
    from paper_2012_01968_b200 import shoup_companion
    for g in golden["shoup"]:
        assert shoup_companion(g["w"], g["p"]) == g["w_bar"], g["cite"]
    with pytest.raises(NttError):
        shoup_companion(17, 17)  # w >= p


def test_golden_table_sizes(golden):
    """P:92 / S:206-207 table bytes and P:795 OT entry count, from the function
    plan creation sizes its allocations with."""
    from paper_2012_01968_b200 import table_sizes
    for g in golden["table_bytes"]:
        t = table_sizes(g["N"], g["np"])
        assert t["psi_bytes"] * g["directions"] == g["bytes"], g["cite"]
    for g in golden["ot_entries"]:
        assert table_sizes(g["N"], 1, g["base"])["ot_entries"] == g["entries"], g["cite"]
    # a default C4 plan: Psi + Psi^-1, their Kernel-2 copies, OT bases, two 128-byte PrimeConst per prime
    t = table_sizes(1 << 17, 60)
    assert t["plan_bytes"] == 4 * 60 * (1 << 17) * 16 + 2 * 60 * 1152 * 16 + 2 * 60 * 128


def test_execute_host_validates_host_buffers():
    """Host buffers must be C-contiguous 64-bit integer CPU arrays:
    a float / int32 array or a strided view is refused before the C ABI."""
    import numpy as np
    from paper_2012_01968_b200 import Plan
    plan = Plan.__new__(Plan)  # no device here: only the argument checks run
    plan.N, plan.L, plan._h = 8, 1, None
    good = np.zeros(8, dtype=np.uint64)
    for bad, err in [(np.zeros(8, dtype=np.int32), TypeError), (np.zeros(8, dtype=np.float64), TypeError),
                     (np.zeros(16, dtype=np.uint64)[::2], ValueError), ([0] * 8, TypeError)]:
        with pytest.raises(err):
            plan.execute_host(bad, good, 3, None)
        with pytest.raises(err):
            plan.execute_host(good, bad, 3, None)


def test_library_reads_no_environment():
    """Kernel selection is an ntt_opts_t field, not an environment variable."""
    srcs = glob.glob(os.path.join(ROOT, "paper_2012_01968_b200", "csrc", "*"))
    for f in srcs:
        assert "getenv" not in open(f).read(), f
