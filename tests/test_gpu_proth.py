"""GPU parity of the Proth-prime arithmetic: plans whose
primes are all p = 1 mod 2^32 (ntt_find_primes_ex NTT_PRIMES_PROTH32) run
kernels that form lo64(q p) of Shoup's modmul as q + (q0 p1 << 32).
The outputs must equal the CPU oracle bit for bit, as for any prime."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


from paper_2012_01968_b200 import Plan  # noqa: E402


def variant_kw(variant: str) -> dict:
    """"k1,k2" -> the ntt_opts_t kernel-variant fields (k1 4 = the default)."""
    k1, k2 = (int(v) for v in variant.split(","))
    return {"k1_variant": k1, "k2_variant": k2}


def to_dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def to_host(t) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def chain(N, L):
    primes = oracle.find_primes(1 << 31, L)  # the oracle's own scan, step 2^32
    return primes, [oracle.find_psi(p, N) for p in primes]


def roundtrip(N, L, batch, config_id=21, expect_proth=True, **kw):
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=config_id)
    plan = Plan(N, primes, **kw)
    assert plan.info()["proth"] == expect_proth
    assert plan.psis == psis
    d = to_dev(x)
    plan.forward(d)
    want = oracle.ntt_batch(x.copy(), primes, psis, +1)
    got = to_host(d)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"forward mismatch at {bad[:5].tolist()} of {bad.shape[0]}"
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)
    y = synth.rns_rows(primes, batch, N, config_id=config_id + 1)
    d = to_dev(y)
    plan.inverse(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(y.copy(), primes, psis, -1))
    plan.close()


@pytest.mark.parametrize("logn", list(range(1, 18)))
def test_proth_every_size(logn):
    roundtrip(1 << logn, 3, 2)


@pytest.mark.parametrize("logn,log_n1", [(14, 6), (15, 8), (16, 10), (17, 7), (17, 9), (17, 10)])
def test_proth_splits(logn, log_n1):
    roundtrip(1 << logn, 2, 2, log_n1=log_n1)


@pytest.mark.parametrize("logn", [12, 16, 17])
@pytest.mark.parametrize("ot_stages", [1, 2])
def test_proth_ot(logn, ot_stages):
    roundtrip(1 << logn, 3, 2, ot=True, ot_stages=ot_stages)


def test_proth_arith_off_is_general_path():
    roundtrip(1 << 17, 2, 1, expect_proth=False, proth_arith=False)


def test_mixed_chain_uses_general_arithmetic():
    """One non-Proth prime in the chain: the plan keeps the general arithmetic."""
    N = 1 << 16
    primes = oracle.find_primes(1 << 31, 2) + oracle.find_primes(N, 1)
    psis = [oracle.find_psi(p, N) for p in primes]
    plan = Plan(N, primes)
    assert not plan.info()["proth"]
    x = synth.rns_rows(primes, 1, N, config_id=23)
    d = to_dev(x)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))


def test_plan_reports_the_d_form_arithmetic():
    """R3 chains (every prime 2^60 - d, d < 2^32) run the PrimeConstD kernels;
    Proth chains the Proth ones (ntt_plan_exec, ntt.h)."""
    N = 1 << 17
    assert Plan(N, oracle.find_primes(N, 4)).info()["arith"] == "general-d"
    assert Plan(N, oracle.find_primes(1 << 31, 4)).info()["arith"] == "proth"


@pytest.mark.parametrize("logn", [13, 16, 17])
def test_mixed_chain_shared_kernel_both_normalisations(logn):
    """General arithmetic with primes of both forms in one launch: R3 primes
    p = 2^60 - d, d < 2^32 (the d-form final reduction) and a
    Proth prime below 2^60 - 2^32 (reduce_full); batch 8 runs the
    shared-twiddle Kernel-2 (and the single-CTA kernel at 2^13), full rows
    compared with the oracle in both directions."""
    N = 1 << logn
    primes = oracle.find_primes(1 << 31, 3)[1:] + oracle.find_primes(N, 2)
    assert any((2**64 - p) >> 32 != 0xF0000000 for p in primes)
    assert any((2**64 - p) >> 32 == 0xF0000000 for p in primes)
    psis = [oracle.find_psi(p, N) for p in primes]
    plan = Plan(N, primes)
    assert plan.info()["arith"] == "general"  # not every prime is 2^60 - d, d < 2^32
    x = synth.rns_rows(primes, 8, N, config_id=29)
    x[0, :, :] = np.array([p - 1 for p in primes], dtype=np.uint64)[:, None]  # largest residues
    d = to_dev(x)
    plan.forward(d)
    X = oracle.ntt_batch(x.copy(), primes, psis, +1)
    assert np.array_equal(to_host(d), X)
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("logn", [12, 17])
def test_proth_edge_rows(logn):
    """zeros, delta_0, delta_{N-1}, all p-1 (largest residues: the lazy bounds)."""
    N = 1 << logn
    primes, psis = chain(N, 2)
    x = np.zeros((4, 2, N), dtype=np.uint64)
    for l, p in enumerate(primes):
        x[1, l, 0] = 1
        x[2, l, N - 1] = p - 1
        x[3, l, :] = p - 1
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("logn", [10, 14, 17])
def test_proth_negacyclic_mul(logn):
    N = 1 << logn
    primes, psis = chain(N, 2)
    a = synth.rns_rows(primes, 2, N, config_id=24)
    b = synth.rns_rows(primes, 2, N, config_id=25)
    plan = Plan(N, primes)
    da, db = to_dev(a), to_dev(b)
    plan.negacyclic_mul(da, db)
    got = to_host(db)
    A = oracle.ntt_batch(a.copy(), primes, psis, +1)
    B = oracle.ntt_batch(b.copy(), primes, psis, +1)
    C = np.stack([np.stack([oracle.pointwise_mul(A[bi, l], B[bi, l], primes[l]) for l in range(2)])
                  for bi in range(2)])
    assert np.array_equal(got, oracle.ntt_batch(C, primes, psis, -1))


def test_proth_full_size_c4():
    """C4 at full size (N=2^17, 60 Proth primes, batch 32), the configuration
    bench.py times with --primes proth: every row against the oracle."""
    N, L, B = 1 << 17, 60, 32
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"])
    plan = Plan(N, primes)
    assert plan.info()["proth"]
    d = to_dev(x)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("variant", ["4,5", "4,7", "4,9", "5,7"])
@pytest.mark.parametrize("logn,log_n1", [(14, 7), (16, 8), (17, 8), (17, 6), (17, 9)])
def test_proth_kernel_variants(variant, logn, log_n1):
    """Kernel variants with Proth instantiations (k1_variant / k2_variant), OT on and off."""
    kv = variant_kw(variant)
    roundtrip(1 << logn, 3, 2, log_n1=log_n1, **kv)
    roundtrip(1 << logn, 2, 3, log_n1=log_n1, ot=True, **kv)
