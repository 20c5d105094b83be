"""Multi-rank host logic on CPU (gloo, world size 2): the strong (contiguous
prime ranges) and weak (prime x ciphertext grid) sharding of bench.py covers
every row of the job exactly once, per-rank shards transformed independently
equal the unsharded job, and bench.py's checksum gather (Dist.gather_rows,
ragged shards) brings every rank's rows to rank 0 (no collective is needed on
the data path; gloo here stands in for NCCL's verification gather)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from bench import balanced_pieces, gather_rows, my_shard, prime_ranges, row_checksums_np, sample_rows, shard_grid


@pytest.mark.parametrize("G", range(1, 9))
def test_strong_shards_partition_the_c4_job(G):
    """the fixed C4 job (32 ciphertexts x 60 primes) in contiguous
    prime ranges -- 30/30, 15x4, 8/8/8/8/7/7/7/7 -- every row exactly once."""
    L, batch = 60, 32
    seen = {}
    sizes = []
    for r in range(G):
        sh = my_shard(r, G, L, batch, "strong")
        assert sh["batch"] == batch and sh["batch_offset"] == 0
        sizes.append(sh["L"])
        for b in range(batch):
            for l in range(sh["prime_offset"], sh["prime_offset"] + sh["L"]):
                assert (b, l) not in seen
                seen[(b, l)] = r
        for (b, l) in sample_rows(sh):
            assert 0 <= b < batch and 0 <= l < sh["L"]
    assert len(seen) == L * batch
    assert sizes == {1: [60], 2: [30, 30], 4: [15] * 4, 8: [8, 8, 8, 8, 7, 7, 7, 7]}.get(G, sizes)
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == L
    assert [n for _, n in prime_ranges(G, L)] == sizes


@pytest.mark.parametrize("G", range(1, 9))
@pytest.mark.parametrize("L,batch", [(60, 32), (45, 64), (15, 16), (7, 3)])
def test_balanced_pieces_partition_the_job(G, L, batch):
    """SURVEY 8(e)'s balanced variant: the prime-major rows split into G equal
    ranges (240 rows per rank for C4 at G = 8), each a run of whole primes and
    at most two partial primes; every row exactly once, and the pieces' rows
    in prime-major order are exactly the rank's range."""
    seen = set()
    for r in range(G):
        pcs = balanced_pieces(r, G, L, batch)
        rows = []
        for pc in pcs:
            assert pc["L"] >= 1 and pc["batch"] >= 1
            assert pc["L"] == 1 or (pc["batch_offset"] == 0 and pc["batch"] == batch)
            for l in range(pc["prime_offset"], pc["prime_offset"] + pc["L"]):
                for b in range(pc["batch_offset"], pc["batch_offset"] + pc["batch"]):
                    rows.append(l * batch + b)
        lo, hi = L * batch * r // G, L * batch * (r + 1) // G
        assert rows == list(range(lo, hi))
        assert sum(1 for pc in pcs if pc["batch"] < batch) <= 2
        seen.update(rows)
    assert seen == set(range(L * batch))
    if (G, L, batch) == (8, 60, 32):
        assert all(len(balanced_pieces(r, 8, 60, 32)) <= 3 for r in range(8))


def test_checksums_detect_single_word_changes():
    rng = np.random.default_rng(1)
    p = oracle.find_primes(1 << 17, 1)[0]
    x = rng.integers(0, p, size=(2, 1 << 17), dtype=np.uint64)
    base = row_checksums_np(x)
    for i, delta in [(0, 1), (77, 1 << 40), ((1 << 17) - 1, p - 1 - int(x[0, -1])), (5, 1 << 28)]:
        y = x.copy()
        y[0, i] = (int(y[0, i]) + delta) % (1 << 60)
        got = row_checksums_np(y)
        assert not np.array_equal(got[0], base[0]) and np.array_equal(got[1], base[1])


@pytest.mark.parametrize("G", range(1, 9))
def test_weak_shards_partition_the_job(G):
    L, per_gpu = 60, 32
    seen = {}
    for r in range(G):
        sh = my_shard(r, G, L, per_gpu, "weak")
        assert sh["L"] * sh["batch"] == L * per_gpu  # weak scaling: fixed rows per rank
        for b in range(sh["batch_offset"], sh["batch_offset"] + sh["batch"]):
            for l in range(sh["prime_offset"], sh["prime_offset"] + sh["L"]):
                assert (b, l) not in seen
                seen[(b, l)] = r
    assert len(seen) == L * per_gpu * G
    gp, gb = shard_grid(G, L)
    assert gp * gb == G and L % gp == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, L, per = 64, 4, 2
    primes = oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    sh = my_shard(rank, world, L, per, "weak")
    pr = primes[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    ps = psis[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    x = synth.rns_rows(pr, sh["batch"], N, config_id=5, prime_offset=sh["prime_offset"], L_total=L,
                       batch_offset=sh["batch_offset"])
    oracle.ntt_batch(x, pr, ps, +1)
    # per-row checksums with their global (b, l), gathered to every rank
    rows = []
    for b in range(sh["batch"]):
        for l in range(sh["L"]):
            rows.append([sh["batch_offset"] + b, sh["prime_offset"] + l, int(x[b, l].sum() % (1 << 62))])
    t = torch.tensor(rows, dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        q.put(torch.cat(out).tolist())
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_unsharded():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference: the whole job (2 GPUs x 2 ciphertexts) in one process
    N, L, per = 64, 4, 2
    primes = oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, per * world, N, config_id=5)
    oracle.ntt_batch(x, primes, psis, +1)
    want = {(b, l): int(x[b, l].sum() % (1 << 62)) for b in range(per * world) for l in range(L)}
    assert len(got) == len(want)
    assert {(b, l): s for b, l, s in got} == want


def _gather_worker(rank, world, port, q):
    """bench.py's verification gather with ragged strong shards: C4's 60 primes
    over 8 ranks is 8/8/8/8/7/7/7/7; here 5 primes over 2 ranks (3/2) at a
    small N, checksums of oracle-transformed rows."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, L, B = 256, 5, 3
    primes = oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    sh = my_shard(rank, world, L, B, "strong")
    pr = primes[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    ps = psis[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    x = synth.rns_rows(pr, B, N, config_id=5, prime_offset=sh["prime_offset"], L_total=L)
    oracle.ntt_batch(x, pr, ps, +1)
    got = gather_rows(dist, torch.from_numpy(row_checksums_np(x)), world, "cpu")
    if rank == 0:
        q.put([g.numpy().tolist() for g in got])
    dist.destroy_process_group()


def test_gloo_world2_ragged_checksum_gather():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, L, B = 256, 5, 3
    primes = oracle.find_primes(N, L)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, B, N, config_id=5)
    oracle.ntt_batch(x, primes, psis, +1)
    for r in range(world):
        sh = my_shard(r, world, L, B, "strong")
        want = row_checksums_np(x[:, sh["prime_offset"]: sh["prime_offset"] + sh["L"]])
        assert np.array_equal(np.array(got[r]), want), r
