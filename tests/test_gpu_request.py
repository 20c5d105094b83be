"""GPU parity of the single-launch request kernel (NTT_GRAPH_ONE_KERNEL,
ntt_request.cu): the forward (Algorithm 1) and the
inverse (R5) of a small job as ONE cooperative kernel with grid
barriers between the column and block phases, checked word for word against
the CPU oracle -- every size it covers, both prime families, forward only,
inverse only and both, replayed (the barrier state is reused across
replays), and jobs larger than one wave of the grid (units looped per CTA)."""
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


from paper_2012_01968_b200 import (NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL,  # noqa: E402
                                   NTT_GRAPH_PRODUCT, NttError, Plan)

BOTH = NTT_DIR_FORWARD | NTT_DIR_INVERSE


def to_dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def to_host(t) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def chain(N, L, form="2n"):
    primes = oracle.find_primes(N, L) if form == "2n" else oracle.find_primes(1 << 31, L)
    return primes, [oracle.find_psi(p, N) for p in primes]


@pytest.mark.parametrize("form", ["2n", "proth"])
@pytest.mark.parametrize("logn,L,batch", [(14, 1, 1), (14, 3, 2), (15, 1, 1), (15, 2, 3), (16, 1, 1), (16, 4, 1),
                                          (17, 1, 1), (17, 2, 2)])
@pytest.mark.parametrize("flags", [NTT_DIR_FORWARD, NTT_DIR_INVERSE, BOTH])
def test_one_kernel_request(form, logn, L, batch, flags):
    """Each replay on fresh data equals the oracle: the forward output
    (bit-reversed, canonical), the inverse of an oracle forward, and the
    round trip."""
    N = 1 << logn
    primes, psis = chain(N, L, form)
    plan = Plan(N, primes)
    buf = torch.empty(batch * L * N, dtype=torch.int64, device="cuda")
    g = plan.graph(buf, flags | NTT_GRAPH_ONE_KERNEL)
    for rep in range(3):
        x = synth.rns_rows(primes, batch, N, config_id=60 + rep)
        src = x.copy()
        if flags == NTT_DIR_INVERSE:  # the inverse of a forward-domain input
            oracle.ntt_batch(src, primes, psis, +1)
        buf.copy_(to_dev(src).view(-1))
        g.launch()
        want = src.copy()
        if flags & NTT_DIR_FORWARD:
            oracle.ntt_batch(want, primes, psis, +1)
        if flags & NTT_DIR_INVERSE:
            oracle.ntt_batch(want, primes, psis, -1)
        assert np.array_equal(to_host(buf).reshape(want.shape), want), rep
        if flags == NTT_DIR_INVERSE:
            assert np.array_equal(to_host(buf).reshape(x.shape), x)
    g.close()
    plan.close()


@pytest.mark.parametrize("logn,L,batch", [(16, 45, 1), (17, 60, 2), (14, 30, 8)])
def test_one_kernel_many_units(logn, L, batch):
    """Jobs with more units than co-resident CTAs (each CTA loops over units
    in every phase): forward equals the oracle on sampled rows, the two-kernel
    path's output exactly on every row, and the round trip restores the input."""
    N = 1 << logn
    primes, psis = chain(N, L)
    plan = Plan(N, primes)
    x = synth.rns_rows(primes, batch, N, config_id=63)
    a = to_dev(x)
    g = plan.graph(a, NTT_DIR_FORWARD | NTT_GRAPH_ONE_KERNEL)
    g.launch()
    b = to_dev(x)
    plan.forward(b)
    got = to_host(a).reshape(x.shape)
    assert np.array_equal(got, to_host(b).reshape(x.shape))
    for bi, l in [(0, 0), (batch - 1, L - 1), (batch // 2, L // 2)]:
        want = oracle.ntt_batch(x[bi, l][None, None].copy(), [primes[l]], [psis[l]], +1)[0, 0]
        assert np.array_equal(got[bi, l], want), (bi, l)
    gi = plan.graph(a, NTT_DIR_INVERSE | NTT_GRAPH_ONE_KERNEL)
    gi.launch()
    assert np.array_equal(to_host(a).reshape(x.shape), x)
    g.close()
    gi.close()
    plan.close()


def test_one_kernel_edge_rows():
    """Zero, delta, all p-1 and constant rows through the one-kernel request."""
    N = 1 << 16
    primes, psis = chain(N, 1)
    p = primes[0]
    rows = np.zeros((5, 1, N), dtype=np.uint64)
    rows[1, 0, 0] = 1
    rows[2, 0, N - 1] = 1
    rows[3, 0, :] = p - 1
    rows[4, 0, :] = 12345
    plan = Plan(N, primes)
    d = to_dev(rows)
    g = plan.graph(d, NTT_DIR_FORWARD | NTT_GRAPH_ONE_KERNEL)
    g.launch()
    want = oracle.ntt_batch(rows.copy(), primes, psis, +1)
    assert np.array_equal(to_host(d).reshape(rows.shape), want)
    g.close()
    plan.close()


def test_one_kernel_argument_errors():
    N = 1 << 12
    primes, _ = chain(N, 1)
    plan = Plan(N, primes)  # N = 2^12: one kernel per row already, not this path
    d = torch.zeros(N, dtype=torch.int64, device="cuda")
    with pytest.raises(NttError) as e:
        plan.graph(d, BOTH | NTT_GRAPH_ONE_KERNEL)
    assert e.value.status == -3
    N = 1 << 14
    primes, _ = chain(N, 1)
    d = torch.zeros(N, dtype=torch.int64, device="cuda")
    ot = Plan(N, primes, ot=True)
    with pytest.raises(NttError) as e:
        ot.graph(d, BOTH | NTT_GRAPH_ONE_KERNEL)
    assert e.value.status == -3
    plan = Plan(N, primes)
    for flags in (NTT_GRAPH_ONE_KERNEL, NTT_GRAPH_PRODUCT | NTT_GRAPH_ONE_KERNEL, 16 | NTT_DIR_FORWARD):
        with pytest.raises(NttError) as e:
            plan.graph(d, flags, other=d.clone())
        assert e.value.status == -3
