"""GPU tests of the round-2 library features, each against the CPU oracle:
the native-modulo comparison variant, request graphs (C5 small
requests), the stream-ordered host executor, fault injection into the plan
tables (the parity harness must catch a bad twiddle), and first calls from
many host threads at once."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


from paper_2012_01968_b200 import (NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_PRODUCT, NttError,  # noqa: E402
                                   Plan)
from paper_2012_01968_b200._native import NTT_VARIANT_NATIVE  # noqa: E402


def to_dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def to_host(t) -> np.ndarray:
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def chain(N, L, form="2n"):
    primes = oracle.find_primes(N, L) if form == "2n" else oracle.find_primes(1 << 31, L)
    return primes, [oracle.find_psi(p, N) for p in primes]


# ------------------------------------------------------------------ native modulo (NEXT-4)

@pytest.mark.parametrize("logn,batch", [(1, 1), (5, 2), (12, 3), (13, 1), (14, 9), (15, 2), (16, 1), (17, 2),
                                        (17, 8)])
def test_native_modulo_variant(logn, batch):
    """NTT_VARIANT_NATIVE (the default kernels with (u128)(b w) % p twiddle
    products) equals the oracle bit for bit: single-CTA sizes, the
    persistent and the shared-twiddle Kernel-2 (batch 8 at 2^17)."""
    N = 1 << logn
    primes, psis = chain(N, 3)
    x = synth.rns_rows(primes, batch, N, config_id=31)
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward_variant(d, NTT_VARIANT_NATIVE)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))


def test_native_modulo_variant_proth_and_refusals():
    N = 1 << 17
    primes, psis = chain(N, 2, "proth")
    x = synth.rns_rows(primes, 1, N, config_id=32)
    plan = Plan(N, primes)
    d = to_dev(x)
    plan.forward_variant(d, NTT_VARIANT_NATIVE)
    assert np.array_equal(to_host(d), oracle.ntt_batch(x.copy(), primes, psis, +1))
    for kw in ({"ot": True}, {"fused": True}, {"log_n1": 9}):
        p2 = Plan(N, primes, **kw)
        with pytest.raises(NttError) as e:
            p2.forward_variant(d, NTT_VARIANT_NATIVE)
        assert e.value.status == -3


# ------------------------------------------------------------------ request graphs

@pytest.mark.parametrize("logn,L,batch", [(12, 1, 1), (16, 1, 1), (16, 8, 1), (16, 45, 1), (17, 3, 2), (14, 2, 9)])
@pytest.mark.parametrize("flags", [NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_DIR_FORWARD | NTT_DIR_INVERSE])
def test_graph_replay(logn, L, batch, flags):
    """A captured request replays the same transforms as the direct calls: each
    replay on fresh data equals the oracle."""
    N = 1 << logn
    primes, psis = chain(N, L)
    plan = Plan(N, primes)
    buf = torch.empty(batch * L * N, dtype=torch.int64, device="cuda")
    g = plan.graph(buf, flags)
    for rep in range(3):
        x = synth.rns_rows(primes, batch, N, config_id=40 + rep)
        buf.copy_(to_dev(x).view(-1))
        g.launch()
        want = x.copy()
        if flags & NTT_DIR_FORWARD:
            oracle.ntt_batch(want, primes, psis, +1)
        if flags & NTT_DIR_INVERSE:
            oracle.ntt_batch(want, primes, psis, -1)
        assert np.array_equal(to_host(buf).reshape(want.shape), want), rep
    g.close()


def test_graph_product():
    """NTT_GRAPH_PRODUCT: b <- a * b mod (X^N + 1), the captured
    ntt_negacyclic_mul, equals the oracle's schoolbook product."""
    N = 1 << 10
    primes, psis = chain(N, 2)
    a = synth.rns_rows(primes, 2, N, config_id=44)
    b = synth.rns_rows(primes, 2, N, config_id=45)
    plan = Plan(N, primes)
    da, db = to_dev(a), to_dev(b)
    g = plan.graph(da, NTT_GRAPH_PRODUCT, other=db)
    g.launch()
    got = to_host(db).reshape(b.shape)
    for bi in range(2):
        for l in range(2):
            assert np.array_equal(got[bi, l], oracle.negacyclic_mul(a[bi, l], b[bi, l], primes[l]))
    g.close()


def test_graph_argument_errors():
    N = 1 << 12
    primes, _ = chain(N, 1)
    plan = Plan(N, primes)
    d = torch.zeros(N, dtype=torch.int64, device="cuda")
    for flags in (0, 8, NTT_GRAPH_PRODUCT):  # no transform, unknown flag, product without b
        with pytest.raises(NttError) as e:
            plan.graph(d, flags)
        assert e.value.status == -3
    with pytest.raises(NttError):
        plan.graph(d, NTT_GRAPH_PRODUCT | NTT_DIR_FORWARD, other=d.clone())


# ------------------------------------------------------------------ host executor ordering

def test_execute_host_orders_after_caller_stream():
    """The workspace is written only after the caller stream's queued work:
    a long kernel chain still writing the workspace on the current stream
    does not race the executor's first H2D copy."""
    N, L, batch = 1 << 14, 2, 4
    primes, psis = chain(N, L)
    x = synth.rns_rows(primes, batch, N, config_id=46)
    plan = Plan(N, primes)
    hin = torch.from_numpy(x.view(np.int64)).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ws = torch.empty(plan.workspace_words(batch, 1), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(200):
            ws.fill_(7)  # queued work on the caller stream that touches the workspace
        plan.execute_host(hin, hout, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws, chunk=1, stream=s)
    assert np.array_equal(hout.numpy().view(np.uint64), x)


# ------------------------------------------------------------------ fault injection

@pytest.mark.parametrize("logn,index,field", [(12, 5, 1), (12, 3000, 0), (17, 7, 1), (17, 100000, 1),
                                              (17, 65537, 0)])
@pytest.mark.parametrize("direction", [NTT_DIR_FORWARD, NTT_DIR_INVERSE])
def test_fault_injection_is_caught(logn, index, field, direction):
    """Corrupting ONE twiddle (or its Shoup companion) of the plan makes the
    oracle comparison fail -- so the parity harness has teeth -- and restoring
    it makes the output bit-exact again."""
    N = 1 << logn
    primes, psis = chain(N, 2)
    x = synth.rns_rows(primes, 2, N, config_id=47)
    want = oracle.ntt_batch(x.copy(), primes, psis, +1)
    plan = Plan(N, primes)

    def run():
        d = to_dev(want if direction == NTT_DIR_INVERSE else x)
        (plan.inverse if direction == NTT_DIR_INVERSE else plan.forward)(d)
        return to_host(d).reshape(x.shape)

    ref = x if direction == NTT_DIR_INVERSE else want
    assert np.array_equal(run(), ref)
    mask = (1 << 40) if field == 0 else (1 << 33)
    plan.corrupt_twiddle(direction, 1, index, field, mask)
    bad = run()
    assert not np.array_equal(bad, ref), "a corrupted twiddle went unnoticed"
    assert np.array_equal(bad[:, 0], ref[:, 0])  # prime 0 untouched
    plan.corrupt_twiddle(direction, 1, index, field, mask)  # XOR again: restored
    assert np.array_equal(run(), ref)


# ------------------------------------------------------------------ concurrency of first calls

def test_first_calls_from_many_threads():
    """Eight host threads make their FIRST calls at once (fresh process), each
    on its own stream, with kernels needing > 48 KiB of dynamic SMEM (the
    per-device attribute setup must complete before any launch)."""
    code = r'''
import threading, numpy as np, torch, sys
sys.path.insert(0, "%s")
import oracle, synth
from paper_2012_01968_b200 import Plan
torch.cuda.init()
cases = [(13, 2, 3), (17, 2, 2), (16, 3, 8), (15, 2, 1)]
errs = []
def work(i):
    try:
        logn, L, B = cases[i %% len(cases)]
        N = 1 << logn
        primes = oracle.find_primes(N, L)
        psis = [oracle.find_psi(p, N) for p in primes]
        x = synth.rns_rows(primes, B, N, config_id=50 + i)
        plan = Plan(N, primes)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            d = torch.from_numpy(x.view(np.int64)).cuda()
            plan.forward(d)
        s.synchronize()
        if not np.array_equal(d.cpu().numpy().view(np.uint64), oracle.ntt_batch(x.copy(), primes, psis, +1)):
            errs.append(i)
    except Exception as e:
        errs.append((i, repr(e)))
ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
[t.start() for t in ts]
[t.join() for t in ts]
print("ERRS", errs)
sys.exit(1 if errs else 0)
''' % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
