"""Multi-rank host logic on CPU (gloo, world size 2): the prime x ciphertext
sharding of bench.py covers every row of the job exactly once, and per-rank
shards transformed independently equal the unsharded job (no collective is
needed on the data path; gloo here stands in for NCCL's verification gather)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from bench import my_shard, shard_grid


@pytest.mark.parametrize("G", range(1, 9))
def test_shards_partition_the_job(G):
    L, per_gpu = 60, 32
    seen = {}
    for r in range(G):
        sh = my_shard(r, G, L, per_gpu)
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
    sh = my_shard(rank, world, L, per)
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
