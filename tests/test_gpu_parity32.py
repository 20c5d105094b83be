"""GPU parity of the 32-bit-word path (NEXT-4) against the CPU
oracle: primes in [2^29, 2^30), bit-exact forward and inverse, every size the
path supports and every compiled two-kernel split."""
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


from paper_2012_01968_b200 import Plan32, NttError  # noqa: E402


def chain32(N, L):
    primes = oracle.find_primes(N, L, 1 << 29, 1 << 30)
    return primes, [oracle.find_psi(p, N) for p in primes]


def to_dev32(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x.astype(np.uint32)).view(np.int32)).cuda()


def to_host32(t) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32).astype(np.uint64)


def check32(N, L, batch, log_n1=0, config_id=15):
    primes, psis = chain32(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=config_id)
    plan = Plan32(N, primes, log_n1=log_n1)
    assert plan.psis == psis
    d = to_dev32(x)
    plan.forward(d)
    got = to_host32(d)
    want = oracle.ntt_batch(x.copy(), primes, psis, +1)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"forward mismatch at {bad[:5].tolist()} of {bad.shape[0]}"
    plan.inverse(d)
    bad = np.argwhere(to_host32(d) != x)
    assert bad.size == 0, f"round trip mismatch at {bad[:5].tolist()} of {bad.shape[0]}"
    y = synth.rns_rows(primes, batch, N, config_id=config_id + 1)
    d = to_dev32(y)
    plan.inverse(d)
    assert np.array_equal(to_host32(d), oracle.ntt_batch(y.copy(), primes, psis, -1))
    info = plan.info()
    plan.close()
    return info


@pytest.mark.parametrize("logn", list(range(1, 18)))
def test_every_size(logn):
    N = 1 << logn
    L = 3 if logn <= 14 else 2
    info = check32(N, L, 2)
    assert info["log_n1"] == (0 if logn <= 13 else (7 if logn <= 15 else 8))


@pytest.mark.parametrize("logn,log_n1", [(14, 7), (15, 7), (16, 8), (17, 8), (17, 9)])
def test_every_split(logn, log_n1):
    assert check32(1 << logn, 2, 1, log_n1=log_n1)["log_n1"] == log_n1


def test_ragged_batch_and_extreme_values():
    N, L = 1 << 16, 3
    primes, psis = chain32(N, L)
    x = synth.rns_rows(primes, 5, N, config_id=15)
    for l, p in enumerate(primes):  # p-1 and 0 everywhere in some rows
        x[0, l, :] = p - 1
        x[1, l, :] = 0
    plan = Plan32(N, primes)
    d = to_dev32(x)
    plan.forward(d)
    assert np.array_equal(to_host32(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    assert np.array_equal(to_host32(d), x)
    plan.close()


def test_full_size_c4_q_equivalent_sampled():
    """C4's modulus with 30-bit words: N=2^17, 120 primes, batch 2 -- the whole
    round trip must be exact and sampled rows must match the oracle."""
    N, L, batch = 1 << 17, 120, 2
    primes, psis = chain32(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=4)
    plan = Plan32(N, primes)
    d = to_dev32(x)
    plan.forward(d)
    got = to_host32(d)
    for b, l in [(0, 0), (1, 59), (1, 119)]:
        want = oracle.ntt_batch(x[b:b + 1, l:l + 1].copy(), [primes[l]], [psis[l]], +1)
        assert np.array_equal(got[b:b + 1, l:l + 1], want), (b, l)
    plan.inverse(d)
    assert np.array_equal(to_host32(d), x)
    plan.close()


def test_errors_32():
    N = 1 << 12
    primes, _ = chain32(N, 2)
    plan = Plan32(N, primes)
    with pytest.raises(TypeError):
        plan.forward(torch.zeros(2 * N, dtype=torch.int64, device="cuda"))
    t = torch.zeros(2 * N + 1, dtype=torch.int32, device="cuda")
    with pytest.raises(NttError) as e:
        plan.forward(t[1:])  # 4-byte offset: misaligned
    assert e.value.status == -4
    plan.close()


@pytest.mark.parametrize("logn,batch", [(17, 8), (17, 11), (16, 16), (16, 21), (15, 16), (14, 32), (14, 35)])
def test_shared_kernel2_32(logn, batch):
    """Batches that fill the 32-bit shared-twiddle Kernel-2 (2^12 / N2
    ciphertexts per CTA), including a ragged last group: forward against the
    oracle on every row, exact round trip -- the remainder-last schedule with
    its direct global ends (single-stage remainder at N2 = 2^9) and without."""
    N = 1 << logn
    check32(N, 2, batch, config_id=40)
