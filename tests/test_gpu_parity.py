"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element
by element, bit-exact (the method is exact, so every row has exactly one
correct canonical output)."""
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


from paper_2012_01968_b200 import Plan, NttError, NTT_DIR_FORWARD, NTT_DIR_INVERSE  # noqa: E402


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
    primes = oracle.find_primes(N, L)
    return primes, [oracle.find_psi(p, N) for p in primes]


def check_roundtrip(N, L, batch, config_id=15, **plan_kw):
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=config_id)
    plan = Plan(N, primes, **plan_kw)
    assert plan.psis == psis  # the plan and the oracle picked the same root (R2)
    d = to_dev(x)
    plan.forward(d)
    got_f = to_host(d)
    want_f = oracle.ntt_batch(x.copy(), primes, psis, +1)
    bad = np.argwhere(got_f != want_f)
    assert bad.size == 0, f"forward mismatch at {bad[:5].tolist()} of {bad.shape[0]}"
    plan.inverse(d)
    got_i = to_host(d)
    bad = np.argwhere(got_i != x)
    assert bad.size == 0, f"inverse mismatch at {bad[:5].tolist()} of {bad.shape[0]}"
    # inverse alone, against the oracle, on an arbitrary NTT-domain input
    y = synth.rns_rows(primes, batch, N, config_id=config_id + 1)
    d = to_dev(y)
    plan.inverse(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(y.copy(), primes, psis, -1))
    plan.close()


@pytest.mark.parametrize("logn", list(range(1, 18)))
def test_every_size(logn):
    N = 1 << logn
    check_roundtrip(N, 3, 2)


@pytest.mark.parametrize("logn,log_n1", [(14, 6), (14, 7), (14, 8), (15, 6), (15, 7), (15, 8), (15, 9),
                                         (16, 6), (16, 7), (16, 8), (16, 9), (16, 10),
                                         (17, 6), (17, 7), (17, 8), (17, 9), (17, 10)])
def test_every_split(logn, log_n1):
    """Every supported (N1, N2) combination."""
    check_roundtrip(1 << logn, 2, 2, log_n1=log_n1)


@pytest.mark.parametrize("logn", [10, 12, 13, 14, 16, 17])
@pytest.mark.parametrize("ot_stages", [1, 2])
def test_ot_on(logn, ot_stages):
    """OT on the last 1 or 2 forward / first 1 or 2 inverse stages."""
    check_roundtrip(1 << logn, 3, 2, ot=True, ot_stages=ot_stages)


@pytest.mark.parametrize("base", [2, 64, 1024, 4096])
def test_ot_bases(base):
    """OT base sweep: result independent of the factorisation."""
    check_roundtrip(1 << 15, 2, 1, ot=True, ot_base=base)


def test_ot_with_split_128x1024():
    """The split the paper singles out for OT."""
    check_roundtrip(1 << 17, 2, 1, ot=True, ot_stages=2, log_n1=7)
    check_roundtrip(1 << 17, 2, 1, ot=True, ot_stages=1, log_n1=7)


@pytest.mark.parametrize("logn", [4, 12, 14, 17])
def test_edge_rows(logn):
    """zeros, delta_0, delta_{N-1}, all p-1, a constant; and the closed forms."""
    N = 1 << logn
    primes, psis = chain(N, 5)
    x = np.zeros((1, 5, N), dtype=np.uint64)
    x[0, 1, 0] = 1
    x[0, 2, N - 1] = 1
    x[0, 3, :] = primes[3] - 1
    x[0, 4, :] = 12345
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward(d)
    got = to_host(d)
    assert np.array_equal(got, oracle.ntt_batch(x.copy(), primes, psis, +1))
    assert not got[0, 0].any()
    assert np.all(got[0, 1] == 1)  # delta_0 -> all ones
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


def test_convolution_theorem_on_gpu():
    """iNTT(NTT(a) . NTT(b)) on the GPU equals the schoolbook negacyclic
    product."""
    N = 256
    primes, psis = chain(N, 2)
    a = synth.rns_rows(primes, 1, N, config_id=3)
    b = synth.rns_rows(primes, 1, N, config_id=4)
    plan = Plan(N, primes)
    da, db = to_dev(a), to_dev(b)
    plan.forward(da)
    plan.forward(db)
    A, B = to_host(da), to_host(db)
    C = np.stack([oracle.pointwise_mul(A[0, l], B[0, l], primes[l]) for l in range(2)])[None]
    dc = to_dev(C)
    plan.inverse(dc)
    got = to_host(dc)
    for l in range(2):
        assert np.array_equal(got[0, l], oracle.negacyclic_mul(a[0, l], b[0, l], primes[l]))


def test_errors_on_device():
    N = 1 << 12
    primes, _ = chain(N, 2)
    plan = Plan(N, primes)
    d = torch.zeros(2 * 2 * N + 2, dtype=torch.int64, device="cuda")
    with pytest.raises(NttError) as e:  # misaligned by 8 bytes
        from paper_2012_01968_b200 import _native
        _native.check(_native.lib().ntt_forward(plan.handle, d.data_ptr() + 8, 1, None))
    assert e.value.status == -4
    h = np.zeros(2 * N, dtype=np.uint64)
    from paper_2012_01968_b200 import _native
    assert _native.lib().ntt_forward(plan.handle, h.ctypes.data, 1, None) == -5  # host pointer
    assert _native.lib().ntt_forward(plan.handle, d.data_ptr(), 0, None) == 0    # batch 0: no-op
    with pytest.raises(ValueError):
        plan.forward(torch.zeros(3 * N, dtype=torch.int64, device="cuda"))      # not a multiple of L*N
    with pytest.raises(ValueError):
        plan.forward(torch.zeros(2 * N, dtype=torch.int64))                     # CPU tensor: no fallback


def test_streams_and_concurrency():
    """One plan, two streams, disjoint buffers (plans are immutable)."""
    N = 1 << 16
    primes, psis = chain(N, 4)
    plan = Plan(N, primes)
    xs = [synth.rns_rows(primes, 2, N, config_id=7 + i) for i in range(2)]
    ds = [to_dev(x) for x in xs]
    st = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(3):
        for d, s in zip(ds, st):
            plan.forward(d, stream=s)
            plan.inverse(d, stream=s)
    torch.cuda.synchronize()
    for d, x in zip(ds, xs):
        assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("flags", [NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_DIR_FORWARD | NTT_DIR_INVERSE])
def test_execute_host(flags):
    """The host-buffer end-to-end path (the e2e API) equals the oracle."""
    N, L, batch = 1 << 14, 3, 5
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=9)
    plan = Plan(N, primes)
    hin = torch.from_numpy(x.view(np.int64)).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ws = torch.empty(plan.workspace_words(batch, 2), dtype=torch.int64, device="cuda")
    plan.execute_host(hin, hout, flags, ws, chunk=2)
    want = x.copy()
    if flags & NTT_DIR_FORWARD:
        oracle.ntt_batch(want, primes, psis, +1)
    if flags & NTT_DIR_INVERSE:
        oracle.ntt_batch(want, primes, psis, -1)
    assert np.array_equal(hout.numpy().view(np.uint64), want)


# ------------------------------------------------- full-size configs (bench launch config)

FULL = {
    "C1": (12, 1, 1),
    "C2": (15, 15, 16),
    "C3": (16, 45, 64),
    "C4": (17, 60, 32),
}


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("ot", [False, True])
def test_full_size_configs(name, ot):
    """BASELINE.json configs at full size, every row against the oracle
    (multi-threaded), in the plan configuration bench.py times."""
    if ot and name in ("C1", "C2"):
        pytest.skip("OT exercised at full size on C3/C4")
    logn, L, batch = FULL[name]
    N = 1 << logn
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=synth.CONFIG_IDS[name])
    plan = Plan(N, primes, ot=ot)
    d = to_dev(x)
    plan.forward(d)
    got = to_host(d)
    want = oracle.ntt_batch(x.copy(), primes, psis, +1)
    assert np.array_equal(got, want)
    del want
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("logn,kw", [(1, {}), (4, {}), (8, {}), (10, {}), (10, {"ot": True}), (13, {}),
                                     (14, {}), (14, {"ot": True}), (16, {}), (17, {"log_n1": 9})])
def test_negacyclic_mul(logn, kw):
    """NEXT-2: b <- a*b mod (X^N+1) with the product fused into the inverse:
    equals the oracle's schoolbook product for small N and, for large
    N, the oracle pipeline NTT -> odot -> iNTT (whose convolution-theorem
    equality the oracle tests pin)."""
    N = 1 << logn
    primes, psis = chain(N, 2)
    a = synth.rns_rows(primes, 2, N, config_id=12)
    b = synth.rns_rows(primes, 2, N, config_id=13)
    plan = Plan(N, primes, **kw)
    da, db = to_dev(a), to_dev(b)
    plan.negacyclic_mul(da, db)
    got = to_host(db)
    A = oracle.ntt_batch(a.copy(), primes, psis, +1)
    assert np.array_equal(to_host(da), A)  # a left in the NTT domain
    if logn <= 10:
        for bi in range(2):
            for l in range(2):
                assert np.array_equal(got[bi, l], oracle.negacyclic_mul(a[bi, l], b[bi, l], primes[l]))
    else:
        B = oracle.ntt_batch(b.copy(), primes, psis, +1)
        C = np.stack([np.stack([oracle.pointwise_mul(A[bi, l], B[bi, l], primes[l]) for l in range(2)])
                      for bi in range(2)])
        assert np.array_equal(got, oracle.ntt_batch(C, primes, psis, -1))


@pytest.mark.parametrize("variant", ["4,3", "4,6", "4,4", "4,5"])
def test_negacyclic_mul_unfused_variants(variant):
    """Kernel-2 variants without the fused product fall back to a separate
    element-wise kernel: same result."""
    kv = variant_kw(variant)
    N = 1 << 15
    primes, psis = chain(N, 2)
    a = synth.rns_rows(primes, 1, N, config_id=12)
    b = synth.rns_rows(primes, 1, N, config_id=13)
    plan = Plan(N, primes, **kv)
    da, db = to_dev(a), to_dev(b)
    plan.negacyclic_mul(da, db)
    A = oracle.ntt_batch(a.copy(), primes, psis, +1)
    B = oracle.ntt_batch(b.copy(), primes, psis, +1)
    C = np.stack([oracle.pointwise_mul(A[0, l], B[0, l], primes[l]) for l in range(2)])[None]
    assert np.array_equal(to_host(db), oracle.ntt_batch(C, primes, psis, -1))


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("logn", [1, 3, 4, 6, 10, 13, 14, 17])
def test_paper_baseline_kernels(variant, logn):
    """The paper's radix-2 (Algorithm 1 per stage) and register radix-16
    comparison kernels (NEXT-3) are bit-exact with the oracle."""
    N = 1 << logn
    primes, psis = chain(N, 3)
    x = synth.rns_rows(primes, 2, N, config_id=11)
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward_variant(d, variant)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("L", [1, 2, 7, 16, 45])
def test_c5_prime_sweep(L):
    """BASELINE.json C5 (mixed stream): N=2^16, one ciphertext per request,
    L swept over 1..45 -- every L in the two-kernel path."""
    check_roundtrip(1 << 16, L, 1)


@pytest.mark.parametrize("variant", ["4,3", "4,4", "4,5", "4,6", "4,7", "4,9", "5,5"])
@pytest.mark.parametrize("logn,log_n1", [(14, 7), (15, 7), (16, 8), (17, 8), (17, 7), (17, 9)])
def test_kernel2_variants(variant, logn, log_n1):
    """Kernel-2 implementations (radix 8 / 16, one-shot / pipelined persistent)
    selected with ntt_opts_t.k1_variant / k2_variant: all bit-exact, OT on and off."""
    kv = variant_kw(variant)
    check_roundtrip(1 << logn, 3, 2, log_n1=log_n1, **kv)
    check_roundtrip(1 << logn, 2, 1, log_n1=log_n1, ot=True, **kv)


@pytest.mark.parametrize("logn", [14, 15, 16, 17])
@pytest.mark.parametrize("L,batch", [(1, 1), (3, 2), (5, 3)])
def test_fused_cluster_kernel(logn, L, batch):
    """NEXT-1: the single-pass cluster kernel (N/2^13 CTAs per row, DSMEM
    exchange) equals the oracle for every cluster size 2..16."""
    plan = Plan(1 << logn, chain(1 << logn, L)[0], fused=True)
    info = plan.info()
    assert info["passes"] == 1 and info["cluster"] == 1 << (logn - 13)
    plan.close()
    check_roundtrip(1 << logn, L, batch, config_id=31, fused=True)


@pytest.mark.parametrize("logn", [14, 17])
def test_fused_vs_two_kernel_identical(logn):
    """The fused and the two-kernel paths give the same words (both equal the
    oracle, which is exact)."""
    N = 1 << logn
    primes, psis = chain(N, 2)
    x = synth.rns_rows(primes, 2, N, config_id=33)
    outs = []
    for fused in (True, False):
        plan = Plan(N, primes, fused=fused)
        assert plan.info()["passes"] == (1 if fused else 2)
        d = to_dev(x)
        plan.forward(d)
        outs.append(to_host(d))
        plan.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], oracle.ntt_batch(x.copy(), primes, psis, +1))


def test_fused_option_errors():
    N = 1 << 13
    with pytest.raises(NttError):
        Plan(N, chain(N, 1)[0], fused=True)  # one CTA holds the row: no cluster kernel
    N = 1 << 16
    with pytest.raises(NttError):
        Plan(N, chain(N, 1)[0], fused=True, ot=True)


@pytest.mark.parametrize("form", ["proth", "2n"])
def test_fused_full_size_c4_sampled(form):
    """The single-pass cluster kernel at BASELINE.json's full C4 size (N=2^17,
    60 primes, batch 32) in the launch configuration bench.py would time with
    fused=True: 48 sampled rows against the oracle, and the exact roundtrip of
    every row."""
    from paper_2012_01968_b200 import find_primes as lib_find_primes
    N, L, B = 1 << 17, 60, 32
    primes = lib_find_primes(N, L, form)
    assert primes == (oracle.find_primes(1 << 31, L) if form == "proth" else oracle.find_primes(N, L))
    x = synth.rns_rows(primes, B, N, config_id=synth.CONFIG_IDS["C4"])
    plan = Plan(N, primes, fused=True)
    assert plan.info()["passes"] == 1 and plan.info()["cluster"] == 16
    d = to_dev(x)
    plan.forward(d)
    got = to_host(d)
    rng = np.random.default_rng(7)
    for r in rng.choice(B * L, 48, replace=False):
        b, l = divmod(int(r), L)
        want = oracle.ntt_forward(x[b, l].copy(), primes[l], oracle.find_psi(primes[l], N))
        assert np.array_equal(got[b, l], want), (b, l)
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)


@pytest.mark.parametrize("logn,batch", [(17, 13), (15, 20), (16, 17), (14, 40)])
@pytest.mark.parametrize("form", ["2n", "proth"])
def test_shared_kernel2_ragged_groups(logn, batch, form):
    """Batches that fill the shared-twiddle Kernel-2's CTAs except the last
    (2^12 / N2 ciphertexts per CTA): the idle block groups of the last CTA must
    neither store nor disturb the others."""
    from paper_2012_01968_b200 import find_primes as lib_find_primes
    N = 1 << logn
    primes = lib_find_primes(N, 2, form)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, batch, N, config_id=35)
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    plan.inverse(d)
    assert np.array_equal(to_host(d), x)
    # the inverse alone on fresh NTT-domain words (no state left from the forward)
    y = synth.rns_rows(primes, batch, N, config_id=36)
    d = to_dev(y)
    plan.inverse(d)
    assert np.array_equal(to_host(d), oracle.ntt_batch(y.copy(), primes, psis, -1))
