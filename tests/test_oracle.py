"""Pins for the CPU oracle (oracle/): each check compares it with something
other than itself -- the paper's definitions evaluated a different way in
Python big integers, closed forms, brute force on tiny inputs, worked
examples from the cited text (tests/golden/), or number-theoretic facts.

P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
"""
import math
import random

import numpy as np
import pytest

import oracle
import synth

P60 = 1 << 60


# --------------------------------------------------------- independent helpers
# Everything below is written from the paper's *definitions* with Python ints,
# not from the oracle's algorithm (Algorithm 1 / GS), so a mistake in one does
# not repeat in the other.

def brev(i, bits):
    return int(format(i, f"0{bits}b")[::-1], 2) if bits else 0


def direct_forward(a, p, psi):
    """A_k = sum_n a_n psi^{n(2k+1)}, stored at position bitrev(k)
    (P:298).  O(N^2)."""
    N = len(a)
    bits = N.bit_length() - 1
    out = [0] * N
    for k in range(N):
        w = pow(psi, 2 * k + 1, p)
        s, x = 0, 1
        for n in range(N):
            s += a[n] * x
            x = x * w % p
        out[brev(k, bits)] = s % p
    return out


def direct_inverse(C_bitrev, p, psi):
    """c_k = N^-1 sum_n C_n psi^{-k(2n+1)}, reading C_n from
    position bitrev(n)."""
    N = len(C_bitrev)
    bits = N.bit_length() - 1
    C = [C_bitrev[brev(n, bits)] for n in range(N)]
    ninv = pow(N, -1, p)
    pinv = pow(psi, -1, p)
    out = []
    for k in range(N):
        s = sum(C[n] * pow(pinv, k * (2 * n + 1), p) for n in range(N))
        out.append(s * ninv % p)
    return out


def schoolbook(a, b, p):
    """P:227 via polynomial product then reduction by X^N = -1."""
    N = len(a)
    full = [0] * (2 * N)
    for i in range(N):
        for j in range(N):
            full[i + j] += a[i] * b[j]
    return [(full[k] - full[k + N]) % p for k in range(N)]


def trial_division_prime(n):
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    r = math.isqrt(n)
    f = 3
    while f <= r:
        if n % f == 0:
            return False
        f += 2
    return True


def pollard_rho(n, seed=1):
    """A nontrivial factor of composite n (Brent/Floyd variant)."""
    if n % 2 == 0:
        return 2
    for f in (3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % f == 0:
            return f
    rng = random.Random(seed)
    while True:
        c = rng.randrange(1, n)
        x = y = rng.randrange(2, n)
        d = 1
        while d == 1:
            x = (x * x + c) % n
            y = (y * y + c) % n
            y = (y * y + c) % n
            d = math.gcd(abs(x - y), n)
        if d != n:
            return d


def rand_vec(rng, N, p):
    return [rng.randrange(p) for _ in range(N)]


SMALL_CASES = [(17, 4), (97, 8), (193, 16), (257, 32), (7681, 64), (12289, 256)]


# ------------------------------------------------------------ golden examples

def test_golden_psi_table(golden):
    for g in golden["psi_table"]:
        assert list(oracle.psi_table(g["p"], g["psi"], g["N"])) == g["Psi"], g["cite"]


def test_golden_psi(golden):
    for g in golden["psi"]:
        assert oracle.find_psi(g["p"], g["N"]) == g["psi"], g["cite"]


def test_golden_forward_inverse(golden):
    for g in golden["forward"]:
        assert list(oracle.ntt_forward(g["in"], g["p"], g["psi"])) == g["out"], g["cite"]
        assert list(oracle.ntt_inverse(g["out"], g["p"], g["psi"])) == g["in"], g["cite"]
    for g in golden["inverse"]:
        assert list(oracle.ntt_inverse(g["in"], g["p"], g["psi"])) == g["out"], g["cite"]


def test_golden_negacyclic(golden):
    for g in golden["negacyclic"]:
        assert list(oracle.negacyclic_mul(g["a"], g["b"], g["p"])) == g["c"], g["cite"]


def test_golden_primes(golden):
    for g in golden["primes"]:
        assert oracle.find_primes(g["N"], g["count"], g["lo"], g["hi"]) == g["primes"], g["cite"]
        # the full descending list, by trial division
        want = [c for c in range(g["hi"] - 1, g["lo"] - 1, -1)
                if c % (2 * g["N"]) == 1 and trial_division_prime(c)][: g["count"]]
        assert want == g["primes"]


# ------------------------------------------------------------- number theory

def test_mulmod_powmod_against_python():
    rng = random.Random(7)
    for _ in range(2000):
        p = rng.randrange(2, 1 << 64)
        a, b = rng.randrange(1 << 64), rng.randrange(1 << 64)
        assert oracle.mulmod(a, b, p) == a * b % p
        e = rng.randrange(1 << 64)
        assert oracle.powmod(a, e, p) == pow(a, e, p)


def test_is_prime_small_exhaustive():
    sieve = np.ones(20000, dtype=bool)
    sieve[:2] = False
    for i in range(2, 142):
        if sieve[i]:
            sieve[i * i::i] = False
    for n in range(20000):
        assert oracle.is_prime(n) == bool(sieve[n]), n


def test_is_prime_strong_pseudoprimes_and_known_primes():
    # strong pseudoprimes to the first prime bases (textbook list); all composite
    spsp = [2047, 1373653, 25326001, 3215031751, 2152302898747, 3474749660383,
            341550071728321, 3825123056546413051]
    for n in spsp:
        assert not oracle.is_prime(n), n
        assert n % pollard_rho(n) == 0 and 1 < pollard_rho(n) < n
    for n in [(1 << 61) - 1, (1 << 31) - 1, (1 << 19) - 1, 18446744073709551557]:
        assert oracle.is_prime(n), n  # Mersenne primes; largest 64-bit prime
    assert not oracle.is_prime(((1 << 31) - 1) * ((1 << 29) - 3))


@pytest.mark.parametrize("logn,count", [(12, 4), (15, 15), (16, 8), (17, 60)])
def test_find_primes_properties(logn, count):
    """R1/R3: descending p = 1 mod 2N in [2^59, 2^60); every skipped candidate
    in between is composite (a factor is exhibited), every kept one passes
    Fermat tests to random bases."""
    N = 1 << logn
    ps = oracle.find_primes(N, count)
    assert len(set(ps)) == count
    assert ps == sorted(ps, reverse=True)
    rng = random.Random(logn)
    c = ((P60 - 2) // (2 * N)) * 2 * N + 1
    assert ps[0] <= c
    expect_next = c
    for p in ps:
        assert (1 << 59) <= p < P60 and p % (2 * N) == 1
        for _ in range(8):
            a = rng.randrange(2, p - 1)
            assert pow(a, p - 1, p) == 1
        while expect_next > p:  # skipped candidates are composite
            f = pollard_rho(expect_next)
            assert 1 < f < expect_next and expect_next % f == 0
            expect_next -= 2 * N
        assert expect_next == p
        expect_next -= 2 * N


def test_find_proth_primes_properties():
    """R18: the oracle's own scan at step 2^32 (N = 2^31) yields descending
    primes p = k 2^32 + 1 in [2^59, 2^60); every skipped candidate in between
    is composite (a factor is exhibited), every kept one passes Fermat tests."""
    ps = oracle.find_primes(1 << 31, 64)
    step = 1 << 32
    rng = random.Random(31)
    expect_next = ((P60 - 2) // step) * step + 1
    for p in ps:
        assert (1 << 59) <= p < P60 and p % step == 1 and p % (1 << 18) == 1
        for _ in range(8):
            a = rng.randrange(2, p - 1)
            assert pow(a, p - 1, p) == 1
        while expect_next > p:
            f = pollard_rho(expect_next)
            assert 1 < f < expect_next and expect_next % f == 0
            expect_next -= step
        assert expect_next == p
        expect_next -= step


def test_closed_forms_full_size_proth():
    """The closed forms of test_closed_forms_full_size at N = 2^17 for a Proth
    prime (the bench's default family): delta_j and constant inputs."""
    N, logn = 1 << 17, 17
    p = oracle.find_primes(1 << 31, 3)[2]
    psi = oracle.find_psi(p, N)
    assert pow(psi, N, p) == p - 1
    rng = random.Random(18)
    idx = rng.sample(range(N), 48) + [0, N - 1]
    j = rng.randrange(N)
    a = np.zeros(N, dtype=np.uint64)
    a[j] = 1
    out = oracle.ntt_forward(a, p, psi)
    for i in idx:
        assert int(out[i]) == pow(psi, j * (2 * brev(i, logn) + 1), p)
    c = rng.randrange(1, p)
    out = oracle.ntt_forward(np.full(N, c, dtype=np.uint64), p, psi)
    for i in idx:
        assert int(out[i]) == 2 * c * pow(1 - pow(psi, 2 * brev(i, logn) + 1, p), -1, p) % p


def test_find_primes_range_exhausted():
    with pytest.raises(ValueError):
        oracle.find_primes(4, 10, 17, 128)


@pytest.mark.parametrize("p,N", SMALL_CASES)
def test_psi_is_smallest_primitive_root_bruteforce(p, N):
    """R2: psi = smallest x with order exactly 2N, by brute force over Z_p."""
    want = next(x for x in range(2, p) if pow(x, N, p) == p - 1)
    # x^N = -1 implies order exactly 2N for N a power of two
    assert oracle.find_psi(p, N) == want


@pytest.mark.parametrize("logn", [12, 15, 16, 17])
def test_psi_order_large(logn):
    N = 1 << logn
    p = oracle.find_primes(N, 1)[0]
    psi = oracle.find_psi(p, N)
    assert pow(psi, N, p) == p - 1 and pow(psi, 2 * N, p) == 1
    if logn == 12:  # minimality: no odd power of psi (= every primitive root) is smaller
        assert min(pow(psi, k, p) for k in range(1, 2 * N, 2)) == psi


def test_find_psi_rejects_non_ntt_prime():
    with pytest.raises(ValueError):
        oracle.find_psi(19, 4)  # 19 != 1 mod 8


def test_bitrev_and_table_structure():
    for bits in range(0, 11):
        for i in range(1 << bits):
            assert oracle.bitrev(i, bits) == brev(i, bits)
    p, N = 12289, 256
    psi = oracle.find_psi(p, N)
    T = oracle.psi_table(p, psi, N)
    assert T[0] == 1 and int(T[1]) ** 2 % p == p - 1  # Psi[1] = psi^(N/2), a square root of -1
    for i in range(N):
        assert int(T[i]) == pow(psi, brev(i, 8), p)


# ------------------------------------------------------------- transforms

@pytest.mark.parametrize("p,N", SMALL_CASES + [(0, 2), (0, 1024)])
def test_forward_equals_direct_sum(p, N):
    """Algorithm 1 == the P:242 definition (bit-reversed order)."""
    if p == 0:
        p = oracle.find_primes(N, 1)[0]
    psi = oracle.find_psi(p, N)
    rng = random.Random(N)
    reps = 1 if N >= 1024 else 3
    for _ in range(reps):
        a = rand_vec(rng, N, p)
        assert list(map(int, oracle.ntt_forward(a, p, psi))) == direct_forward(a, p, psi)


@pytest.mark.parametrize("p,N", SMALL_CASES[:5] + [(0, 128)])
def test_inverse_equals_direct_sum(p, N):
    """GS inverse (R5) == the P:252-255 formula."""
    if p == 0:
        p = oracle.find_primes(N, 1)[0]
    psi = oracle.find_psi(p, N)
    rng = random.Random(N + 1)
    C = rand_vec(rng, N, p)
    assert list(map(int, oracle.ntt_inverse(C, p, psi))) == direct_inverse(C, p, psi)


def test_forward_degenerate_sizes():
    p = 17
    assert list(oracle.ntt_forward([5], p, 16)) == [5]  # N=1: identity
    assert list(oracle.ntt_inverse([5], p, 16)) == [5]
    psi = oracle.find_psi(p, 2)  # N=2: one butterfly, A_k = a0 + a1 psi^(2k+1)
    a = [3, 11]
    out = oracle.ntt_forward(a, p, psi)
    assert list(out) == [(3 + 11 * psi) % p, (3 + 11 * pow(psi, 3, p)) % p]


@pytest.mark.parametrize("logn", [12, 17])
def test_closed_forms_full_size(logn):
    """Delta and constant inputs at full size (any N): delta_j maps to
    out[i] = psi^{j(2 bitrev(i)+1)}; constant c maps to
    out[i] = 2c (1 - psi^{2 bitrev(i)+1})^-1 (geometric sum with psi^N = -1)."""
    N = 1 << logn
    p = oracle.find_primes(N, 2)[1]
    psi = oracle.find_psi(p, N)
    rng = random.Random(logn)
    idx = rng.sample(range(N), 64) + [0, 1, N - 1]
    for j in (0, 1, N - 1, rng.randrange(N)):
        a = np.zeros(N, dtype=np.uint64)
        a[j] = 1
        out = oracle.ntt_forward(a, p, psi)
        for i in idx:
            assert int(out[i]) == pow(psi, j * (2 * brev(i, logn) + 1), p)
    c = rng.randrange(1, p)
    out = oracle.ntt_forward(np.full(N, c, dtype=np.uint64), p, psi)
    for i in idx:
        k = brev(i, logn)
        assert int(out[i]) == 2 * c * pow(1 - pow(psi, 2 * k + 1, p), -1, p) % p
    back = oracle.ntt_inverse(out, p, psi)
    assert np.all(back == c)


@pytest.mark.parametrize("logn", [1, 2, 5, 10, 13, 17])
def test_roundtrip_and_linearity(logn):
    N = 1 << logn
    p = oracle.find_primes(N, 3)[-1]
    psi = oracle.find_psi(p, N)
    rng = np.random.default_rng(logn)
    a = synth.draw_numpy(3, p, N)
    b = synth.draw_numpy(4, p, N)
    A, B = oracle.ntt_forward(a, p, psi), oracle.ntt_forward(b, p, psi)
    assert np.array_equal(oracle.ntt_inverse(A, p, psi), a)
    s = np.array([(int(x) + int(y)) % p for x, y in zip(a, b)], dtype=np.uint64)
    S = oracle.ntt_forward(s, p, psi)
    assert all(int(S[i]) == (int(A[i]) + int(B[i])) % p for i in rng.integers(0, N, 32))
    # edge rows: zeros and all p-1
    assert not oracle.ntt_forward(np.zeros(N, dtype=np.uint64), p, psi).any()
    m = np.full(N, p - 1, dtype=np.uint64)
    assert np.array_equal(oracle.ntt_inverse(oracle.ntt_forward(m, p, psi), p, psi), m)


@pytest.mark.parametrize("p,N", [(17, 2), (17, 4), (97, 8), (7681, 64), (0, 256)])
def test_convolution_theorem(p, N):
    """iNTT(NTT(a) . NTT(b)) = negacyclic product (P:232-236 with both psi
    merges) = schoolbook c_k."""
    if p == 0:
        p = oracle.find_primes(N, 1)[0]
    psi = oracle.find_psi(p, N)
    rng = random.Random(p + N)
    for _ in range(3):
        a, b = rand_vec(rng, N, p), rand_vec(rng, N, p)
        want = schoolbook(a, b, p)
        assert list(map(int, oracle.negacyclic_mul(a, b, p))) == want
        C = oracle.pointwise_mul(oracle.ntt_forward(a, p, psi), oracle.ntt_forward(b, p, psi), p)
        assert list(map(int, oracle.ntt_inverse(C, p, psi))) == want


def test_batch_matches_rows_and_thread_count():
    N, L, batch = 256, 3, 4
    primes = oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, batch, N)
    ref = np.stack([np.stack([oracle.ntt_forward(x[b, l], primes[l], psis[l]) for l in range(L)])
                    for b in range(batch)])
    for nth in (1, 3, 0):
        y = oracle.ntt_batch(x.copy(), primes, psis, +1, nth)
        assert np.array_equal(y, ref)
        assert np.array_equal(oracle.ntt_batch(y, primes, psis, -1, nth), x)


# ------------------------------------------------------------------ synth

def test_synth_c_matches_numpy_and_is_in_range():
    N = 1 << 12
    primes = oracle.find_primes(N, 3)
    x = synth.rns_rows(primes, 2, N, config_id=1)
    for b in range(2):
        for l in range(3):
            want = synth.draw_numpy(b * 3 + l, primes[l], N, config_id=1)
            assert np.array_equal(x[b, l], want)
            assert int(x[b, l].max()) < primes[l]
    # a shard draws exactly the unsharded values
    sh = synth.rns_rows(primes[1:], 1, N, config_id=1, prime_offset=1, L_total=3, batch_offset=1)
    assert np.array_equal(sh[0], x[1, 1:])
