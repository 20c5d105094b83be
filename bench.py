#!/usr/bin/env python3
"""bench.py -- the headline measurement of the batched negacyclic NTT + iNTT.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--scaling strong|weak]
                    [--primes 2n|proth] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (python bench.py --gpus N re-launches itself so)

A "step" is one pass of the whole hot path over one batch: ntt_forward then
ntt_inverse of every residue row.  Workload at N=1:
BASELINE.json configs[3] ("C4": N=2^17, 60 primes of 60 bits, batch 32),
primes = the R3 chain (p = 1 mod 2N scanned down from 2^60 - 2N + 1, SURVEY
8(c)#3); the Proth chain is reported beside it at equal rank ("proth").

Multi-GPU: the rows are independent, so the job shards with no
data-path collective.  --scaling strong (default): the fixed C4 job (32
ciphertexts x 60 primes) is split into contiguous prime ranges, one per rank
(30/30, 15x4, 8/8/8/8/7/7/7/7); at N>1 the line also carries "balanced",
SURVEY 8(e)'s variant (the prime-major rows split evenly, 240 per rank at
G=8: whole primes plus at most two partial primes, timed and oracle-checked
the same way).  --scaling weak: 32 ciphertexts per GPU.
NCCL (torch.distributed) carries the barriers, the max-over-ranks time and,
after timing, the per-row checksums that rank 0 checks against the oracle.

--config C5 (mixed request stream, N=2^16, L swept over 1..45): throughput
mode (whole requests round-robin to ranks, batched per L) and latency mode
(one request at a time, its primes sharded over the ranks, replayed from a
request graph -- the split's kernels or the one-kernel request, the faster
per L), microseconds per request for each L.

Prints ONE JSON line on rank 0 (DESIGN.md section 7 explains every key).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs per NTT+iNTT (N=2^17, all primes) & HBM GB/s vs 8 TB/s, 1/2/4/8 B200"

CONFIGS = {
    # name: (logN, L, batch of the job, BASELINE.json text)
    "C1": (12, 1, 1, "N=2^12, 1 prime (~60-bit), batch 1"),
    "C2": (15, 15, 16, "N=2^15, 15 primes (~Q=2^881, SEAL-like), batch 16"),
    "C3": (16, 45, 64, "N=2^16, 45 primes (bootstrappable CKKS-size), batch 64"),
    "C4": (17, 60, 32, "N=2^17, ~60 primes (large bootstrappable set), batch 32"),
    "C5": (16, 45, 64, "mixed ciphertext stream: N=2^16, L sweep 1-45 primes, latency vs throughput"),
}
C5_LS = [1, 2, 4, 8, 15, 30, 45]
C5_REQUESTS = 64  # requests per L in throughput mode
PRIME_TEXT = {"2n": "p = 1 mod 2N descending from 2^60 - 2N + 1 (SURVEY 8(c)#3, DESIGN.md R3)",
              "proth": "p = 1 mod 2^32 descending from 2^60 - 2^32 + 1 (DESIGN.md R18)"}
L2_BYTES = 126 * 2**20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# Multiply-pipe cost of one warp-instruction per SMSP, in clocks: IMAD from the
# guide (rt_SMSP = 2); IMAD.WIDE / IMAD.HI measured on B200 with independent
# chains (profiles/r01_alu_roof.jsonl: 24 and 28 per clk per SM; confirmed by
# the 2 WIDE + 2 HI + 3 IMAD mix at 25.7 clk, profiles/r01g_bf_roof_variants.txt).
CLK_IMAD, CLK_WIDE, CLK_HI = 2.0, 16 / 3.0, 32 / 7.0
SM_COUNT, SM_GHZ = 148, 1.965


def alu_floor_clk(form: str) -> float:
    """Multiply-pipe clocks per warp-modmul of the truncated-quotient Shoup
    multiply: general primes 3 WIDE + 2 HI + 4 IMAD, Proth
    primes 2 WIDE + 2 HI + 3 IMAD."""
    if form == "proth":
        return 2 * CLK_WIDE + 2 * CLK_HI + 3 * CLK_IMAD
    return 3 * CLK_WIDE + 2 * CLK_HI + 4 * CLK_IMAD


def alu_peak(form: str) -> float:
    """Derived integer roof in G modmul/s: 148 SMs x 4 SMSPs x 32 lanes /
    (multiply-pipe clk per warp-modmul) x 1.965 GHz."""
    return SM_COUNT * 4 * 32 / alu_floor_clk(form) * SM_GHZ


def butterfly_ceiling():
    """The practical ceiling, measured live: tools/libs/bf_roof runs the
    kernels' own CT / GS butterflies (radix-16 rounds on registers, twiddles
    broadcast from SMEM, 32 warps/SM, no memory).  {"ct_2n": G/s, ...}."""
    exe = os.path.join(ROOT, "tools", "libs", "bf_roof")
    out = {}
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
        for line in r.stdout.splitlines():
            d = json.loads(line)
            out[f"{d['butterfly']}_{d['primes']}"] = d["Gbutterfly_s"]
    except Exception as e:  # reported, not hidden
        out["error"] = repr(e)
    return out


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ sharding

def prime_ranges(G: int, L: int) -> list[tuple[int, int]]:
    """Contiguous prime ranges (offset, count) of L primes over G ranks, the
    first L mod G ranks one prime larger: 60 over 8 -> 8,8,8,8,7,7,7,7."""
    base, extra = divmod(L, G)
    out, off = [], 0
    for r in range(G):
        n = base + (1 if r < extra else 0)
        out.append((off, n))
        off += n
    return out


def strong_shard(rank: int, G: int, L: int, batch: int) -> dict:
    """Strong scaling: the fixed job (batch ciphertexts x L primes) split into
    contiguous prime ranges; every rank holds all ciphertexts of its primes."""
    off, n = prime_ranges(G, L)[rank]
    return {"prime_offset": off, "L": n, "batch_offset": 0, "batch": batch, "Gp": G, "Gb": 1}


def shard_grid(G: int, L: int):
    """(Gp, Gb) for weak scaling: the largest Gp <= G dividing both G and L, Gb = G / Gp."""
    gp = max(d for d in range(1, G + 1) if G % d == 0 and L % d == 0)
    return gp, G // gp


def weak_shard(rank: int, G: int, L: int, batch_per_gpu: int) -> dict:
    """Weak scaling: batch_per_gpu * G ciphertexts over a Gp x Gb grid of
    (prime range, ciphertext range) shards, every rank batch_per_gpu * L rows."""
    gp, gb = shard_grid(G, L)
    rp, rb = rank % gp, rank // gp
    Lp = L // gp
    Bb = batch_per_gpu * G // gb
    return {"Gp": gp, "Gb": gb, "prime_offset": rp * Lp, "L": Lp, "batch_offset": rb * Bb, "batch": Bb}


def my_shard(rank: int, G: int, L: int, batch: int, scaling: str = "strong") -> dict:
    return strong_shard(rank, G, L, batch) if scaling == "strong" else weak_shard(rank, G, L, batch)


def balanced_pieces(rank: int, G: int, L: int, batch: int) -> list[dict]:
    """SURVEY 8(e)'s balanced variant of the strong split: the job's L*batch
    rows in prime-major order (row r = (l, b), l = r // batch), cut into G
    equal ranges; a rank's range is a run of whole primes (all ciphertexts)
    plus at most two partial primes (a ciphertext range of one prime) at its
    ends -- one plan and one buffer per piece.  60 x 32 over 8: 240 rows each."""
    total = L * batch
    lo, hi = total * rank // G, total * (rank + 1) // G
    out, r = [], lo
    while r < hi:
        l, b = divmod(r, batch)
        if b == 0 and hi - r >= batch:
            n = (hi - r) // batch
            out.append({"prime_offset": l, "L": n, "batch_offset": 0, "batch": batch})
            r += n * batch
        else:
            end = min(hi, (l + 1) * batch)
            out.append({"prime_offset": l, "L": 1, "batch_offset": b, "batch": end - r})
            r = end
    return out


def sample_rows(sh: dict) -> list[tuple[int, int]]:
    """Local (b, l) rows of a shard that rank 0 checks against the oracle: the
    first, the last, and two interior ones (deterministic)."""
    B, L = sh["batch"], sh["L"]
    cand = [(0, 0), (B - 1, L - 1), (B // 2, L // 2), ((B * 7) // 11, (L * 5) // 7)]
    out = []
    for c in cand:
        if c not in out:
            out.append(c)
    return out


# ------------------------------------------------------------------ checksums

# per-row checksum of 64-bit words x_i (no overflow in int64 for N <= 2^17):
#   s0 = sum (x_i & (2^28 - 1)) (i + 1),  s1 = sum (x_i >> 28),  s2 = sum (x_i >> 28) ((7 i + 3) & 1023)
def row_checksums_np(rows: np.ndarray) -> np.ndarray:
    r = rows.reshape(-1, rows.shape[-1]).astype(np.uint64)
    N = r.shape[-1]
    i = np.arange(N, dtype=np.int64)
    lo = (r & np.uint64(0xFFFFFFF)).astype(np.int64)
    hi = (r >> np.uint64(28)).astype(np.int64)
    return np.stack([(lo * (i + 1)).sum(-1), hi.sum(-1), (hi * ((7 * i + 3) & 1023)).sum(-1)], -1)


def row_checksums_torch(dev, B: int, L: int, N: int):
    import torch
    x = dev.view(B * L, N)
    i = torch.arange(N, dtype=torch.int64, device=dev.device)
    lo = x & 0xFFFFFFF
    hi = torch.bitwise_right_shift(x, 28) & 0xFFFFFFFFF  # logical shift of the 64-bit word
    return torch.stack([(lo * (i + 1)).sum(-1), hi.sum(-1), (hi * ((7 * i + 3) & 1023)).sum(-1)], -1)


# ------------------------------------------------------------------ host info + oracle timing

def host_info() -> dict:
    model, phys = None, set()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model is None:
                model = line.split(":", 1)[1].strip()
            if line.startswith("physical id"):
                phys.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    return {"cpu_model": model, "sockets": max(1, len(phys)), "nproc": os.cpu_count(),
            "cores": len(os.sched_getaffinity(0))}


def oracle_chain(logn: int, L: int, form: str):
    import oracle
    N = 1 << logn
    primes = oracle.find_primes(1 << 31, L) if form == "proth" else oracle.find_primes(N, L)
    return primes, [oracle.find_psi(p, N) for p in primes]


def oracle_fwd_inv_seconds(x: np.ndarray, primes, psis, nthreads: int) -> float:
    import oracle
    t0 = time.perf_counter()
    oracle.ntt_batch(x, primes, psis, +1, nthreads)
    oracle.ntt_batch(x, primes, psis, -1, nthreads)
    return time.perf_counter() - t0


def cpu_baseline(logn: int, L: int, batch: int, cfg_id: int, form: str, reps: int = 2) -> dict:
    """The oracle as it stands (SURVEY 8(d) "Oracle"): after a warm-up, the
    whole job (batch ciphertexts x L primes, NTT + iNTT) on all host cores,
    `reps` times; and one ciphertext on one core.  us per full-L ciphertext."""
    import synth
    N = 1 << logn
    primes, psis = oracle_chain(logn, L, form)
    info = host_info()
    cores = info["cores"]
    x1 = synth.rns_rows(primes, 1, N, config_id=cfg_id)
    xb = synth.rns_rows(primes, batch, N, config_id=cfg_id)
    # warm-up on the whole job, as the reference arm does (threads, and the
    # first-touch page faults of the job's buffers, which a one-ciphertext
    # warm-up leaves inside the first timed rep)
    oracle_fwd_inv_seconds(xb, primes, psis, cores)
    ts = [oracle_fwd_inv_seconds(xb, primes, psis, cores) for _ in range(reps)]
    one = oracle_fwd_inv_seconds(x1.copy(), primes, psis, 1)
    T = statistics.mean(ts)
    return {"value": round(T / batch * 1e6, 1), "unit": "us", "cores": cores, "kind": "oracle",
            "sample": f"whole job: {batch} ciphertexts x {L} primes x N=2^{logn}, fwd+inv, {reps} reps after "
                      f"a whole-job warm-up, {cores} threads ({T:.2f} s per rep)",
            "one_core_us": round(one * 1e6, 1), "cpu_model": info["cpu_model"], "sockets": info["sockets"],
            "nproc": info["nproc"]}


# ------------------------------------------------------------------ reference arm

def run_reference(args):
    """The tier's reference arm: the oracle (the paper's algorithm written
    plainly, CPU) as it stands, each step one whole C4 job (or the config's),
    the same routine as the GPU arm's cpu_baseline.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synth
    cfg = "C4" if args.config == "C5" else args.config
    logn, L, batch, text = CONFIGS[cfg]
    N = 1 << logn
    cfg_id = synth.CONFIG_IDS[cfg]
    primes, psis = oracle_chain(logn, L, args.primes)
    info = host_info()
    cores = info["cores"]
    xb = synth.rns_rows(primes, batch, N, config_id=cfg_id)
    for _ in range(args.warmup):
        oracle_fwd_inv_seconds(xb, primes, psis, cores)
    times = [oracle_fwd_inv_seconds(xb, primes, psis, cores) for _ in range(args.steps)]
    T = statistics.mean(times)
    value = T / batch * 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "us", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(T * 1e3, 3), "higher_is_better": False,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{cfg}: {text}; NTT+iNTT of every row", "N": N, "L": L, "batch": batch,
                   "primes": PRIME_TEXT[args.primes], "sample": f"the whole {cfg} job per step"},
        "cpu_baseline": {"value": round(value, 3), "unit": "us", "cores": cores, "kind": "oracle",
                         "sample": f"{batch} ciphertexts x {L} primes x N=2^{logn}, fwd+inv per step, {cores} threads",
                         "cpu_model": info["cpu_model"], "sockets": info["sockets"], "nproc": info["nproc"]},
        "e2e": {"value": round(value, 3), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ self-launch

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`python bench.py --gpus N` without torchrun: re-run this script under
    torch.distributed.run with N local ranks (the driver's own launch line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ own arm

def gather_rows(dist, t, world: int, dev: str):
    """all_gather of a [rows, k] int64 tensor whose row count differs per rank
    (ragged prime ranges): counts first, then zero-padded rows; returns every
    rank's rows on the CPU, in rank order."""
    import torch
    if world == 1:
        return [t.cpu()]
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    m = int(max(v.item() for v in ns))
    pad = torch.zeros((m, t.shape[1]), dtype=torch.int64, device=dev)
    pad[: t.shape[0]] = t.to(dev)
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    return [o[: int(k.item())].cpu() for o, k in zip(outs, ns)]


class Dist:
    """Rank / world / reductions.  Backend: NCCL, one rank per GPU; gloo when
    ranks share a GPU (fewer visible devices than ranks -- tests, one-GPU
    boxes) or BENCH_DIST_BACKEND=gloo."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % ndev
        torch.cuda.set_device(self.local)
        self.backend = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if ndev >= self.world else "gloo")
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group("gloo")
        self.dev = "cuda" if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def allreduce(self, vals, op="max"):
        if self.world == 1:
            return list(vals)
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX, "min": self.dist.ReduceOp.MIN,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return t.tolist()

    def gather_rows(self, t):
        return gather_rows(self.dist, t, self.world, self.dev)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def timed_steps(D, plan, dev, steps, warmup, flush_l2=False, scratch=None, sample_clocks=False):
    """W untimed (fwd, inv) steps, then K steps timed with CUDA events on the
    launching stream between barriers; per-kernel times from events between
    the ntt_launch_pass calls.  Returns (this rank's ms, per-kernel ms, clocks, launches)."""
    from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE
    torch = D.torch
    stream = torch.cuda.current_stream()
    passes = plan.passes
    seq = [(NTT_DIR_FORWARD, i) for i in range(passes)] + [(NTT_DIR_INVERSE, i) for i in range(passes)]
    for _ in range(warmup):
        plan.forward(dev)
        plan.inverse(dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(steps)]
    D.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(D.local) if sample_clocks else None
    if sampler:
        sampler.__enter__()
    start.record(stream)
    for s in range(steps):
        if flush_l2:
            scratch.fill_(s)  # untimed: between ev[s-1][-1] and ev[s][0]
        ev[s][0].record(stream)
        for j, (d, p) in enumerate(seq):
            plan.launch_pass(dev, d, p)
            ev[s][j + 1].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    D.barrier()
    if flush_l2:  # the sum of the per-step spans, flushes excluded
        ms = sum(ev[s][0].elapsed_time(ev[s][-1]) for s in range(steps))
    else:
        ms = start.elapsed_time(end)
    per_kernel = [statistics.mean(ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(steps)) for j in range(len(seq))]
    names = [("fwd" if d == NTT_DIR_FORWARD else "inv") + f"_pass{p}" for d, p in seq]
    # median and min of the per-step spans, forward and inverse separately
    spans = [ev[s][0].elapsed_time(ev[s][-1]) for s in range(steps)]
    fwd = [ev[s][0].elapsed_time(ev[s][passes]) for s in range(steps)]
    inv = [ev[s][passes].elapsed_time(ev[s][-1]) for s in range(steps)]
    D.step_stats = {"step_ms_median": round(statistics.median(spans), 4), "step_ms_min": round(min(spans), 4),
                    "fwd_ms_median": round(statistics.median(fwd), 4), "inv_ms_median": round(statistics.median(inv), 4)}
    return ms, dict(zip(names, per_kernel)), (sampler.summary() if sampler else None), len(seq) * steps


def modmuls_per_launch(name: str, rows: int, N: int, logn: int, log_n1: int, passes: int, ots: int = 0) -> int:
    """Shoup modmuls of one kernel launch: one per butterfly,
    + N/2 per OT stage (the second factor), + N/2 for the fused N^-1 (the last
    inverse stage multiplies both outputs)."""
    if passes == 2:
        st = {"fwd_pass0": log_n1, "fwd_pass1": logn - log_n1, "inv_pass0": logn - log_n1, "inv_pass1": log_n1}[name]
        ot_here = name in ("fwd_pass1", "inv_pass0")
        last_inv = name == "inv_pass1"
    else:
        st, ot_here, last_inv = logn, True, name.startswith("inv")
    per_row = (N // 2) * st + (N // 2) * (ots if ot_here else 0) + (N // 2 if last_inv else 0)
    return rows * per_row


def balanced_run(D, args, logn, L_total, batch_job, cfg_id):
    """Time and verify the balanced split (balanced_pieces): every rank runs
    forward then inverse over its pieces, timed with CUDA events between
    barriers, max over ranks; per-row checksums of one forward, in global
    prime-major order, are gathered for rank 0's oracle check."""
    torch = D.torch
    import synth
    from paper_2012_01968_b200 import Plan, find_primes

    N = 1 << logn
    chain = find_primes(N, L_total, args.primes)
    pieces = []
    for pc in balanced_pieces(D.rank, D.world, L_total, batch_job):
        pr = chain[pc["prime_offset"]: pc["prime_offset"] + pc["L"]]
        host = torch.empty(pc["batch"] * pc["L"] * N, dtype=torch.int64)
        synth.rns_rows(pr, pc["batch"], N, config_id=cfg_id, prime_offset=pc["prime_offset"], L_total=L_total,
                       batch_offset=pc["batch_offset"],
                       out=host.numpy().view(np.uint64).reshape(pc["batch"], pc["L"], N))
        pieces.append((pc, Plan(N, pr), host.cuda()))
    ref = [d.clone() for _, _, d in pieces]

    def step():
        for _, pl, d in pieces:
            pl.forward(d)
        for _, pl, d in pieces:
            pl.inverse(d)

    for _ in range(args.warmup):
        step()
    steps = max(3, args.steps // 2)
    D.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    mine = e0.elapsed_time(e1) / steps
    ok = all(bool(torch.equal(d, r)) for (_, _, d), r in zip(pieces, ref))
    cs = []
    for pc, pl, d in pieces:  # one forward; checksums in prime-major order
        pl.forward(d)
        c = row_checksums_torch(d, pc["batch"], pc["L"], N).view(pc["batch"], pc["L"], 3)
        cs.append(c.transpose(0, 1).reshape(-1, 3))
        pl.inverse(d)
    torch.cuda.synchronize()
    ok = ok and all(bool(torch.equal(d, r)) for (_, _, d), r in zip(pieces, ref))
    gathered = D.gather_rows(torch.cat(cs))
    per_rank = [0.0] * D.world
    per_rank[D.rank] = mine
    per_rank = D.allreduce(per_rank, "sum")
    ok = bool(D.allreduce([float(ok)], "min")[0])
    for _, pl, _ in pieces:
        pl.close()
    return per_rank, ok, gathered, len(pieces)


def transform_line(D, args, logn, L_total, batch_job, text):
    """C1-C4: time the job, verify, and build rank 0's line."""
    torch = D.torch
    import synth
    from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes

    rank, world = D.rank, D.world
    N = 1 << logn
    sh = my_shard(rank, world, L_total, batch_job, args.scaling)
    units = batch_job if args.scaling == "strong" else batch_job * world  # full-L ciphertexts per step
    cfg_id = synth.CONFIG_IDS[args.config]

    def make_inputs(form):
        primes = find_primes(N, L_total, form)[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
        host = torch.empty(sh["batch"] * sh["L"] * N, dtype=torch.int64).pin_memory()
        synth.rns_rows(primes, sh["batch"], N, config_id=cfg_id, prime_offset=sh["prime_offset"], L_total=L_total,
                       batch_offset=sh["batch_offset"],
                       out=host.numpy().view(np.uint64).reshape(sh["batch"], sh["L"], N))
        return primes, host

    B, L = sh["batch"], sh["L"]
    rows = B * L
    words = rows * N
    primes, host = make_inputs(args.primes)
    dev = host.cuda()
    flush_l2 = words * 8 < 2 * L2_BYTES
    scratch = torch.empty(256 * 2**20 // 4, dtype=torch.int32, device="cuda") if flush_l2 else None

    plan = Plan(N, primes)
    info = plan.info()
    ms, kern, clocks, launches = timed_steps(D, plan, dev, args.steps, args.warmup, flush_l2, scratch, True)
    ms_step_rank = ms / args.steps
    step_stats = D.step_stats
    l2_warm = None
    if flush_l2:  # small configs also timed L2-warm (no flush between steps)
        ms_w, _, _, _ = timed_steps(D, plan, dev, args.steps, 1)
        l2_warm = max(D.allreduce([ms_w / args.steps], "max"))

    # ---- verification (untimed): the roundtrip restored every row; then one
    # forward, per-row checksums gathered to rank 0, checked against the oracle
    torch.cuda.synchronize()
    ok_roundtrip = bool(torch.equal(dev, host.cuda()))
    plan.forward(dev)
    cs = row_checksums_torch(dev, B, L, N)
    plan.inverse(dev)
    torch.cuda.synchronize()
    ok_roundtrip = ok_roundtrip and bool(torch.equal(dev, host.cuda()))
    gathered = D.gather_rows(cs)
    per_rank_ms = [0.0] * world
    per_rank_ms[rank] = ms_step_rank
    per_rank_ms = D.allreduce(per_rank_ms, "sum")
    ms_step = max(per_rank_ms)  # the job's step time: max over ranks (device time)
    ok_roundtrip = bool(D.allreduce([float(ok_roundtrip)], "min")[0])

    # ---- the other prime family at equal rank, OT on, the negacyclic product, e2e
    alt_form = "proth" if args.primes == "2n" else "2n"
    alt_primes, alt_host = make_inputs(alt_form)
    alt_dev = alt_host.cuda()
    alt_plan = Plan(N, alt_primes)
    alt_steps = max(3, args.steps // 2)
    ms_alt, kern_alt, _, _ = timed_steps(D, alt_plan, alt_dev, alt_steps, 2, flush_l2, scratch)
    torch.cuda.synchronize()
    alt_ok = bool(D.allreduce([float(torch.equal(alt_dev, alt_host.cuda()))], "min")[0])
    alt_ms_step = max(D.allreduce([ms_alt / alt_steps], "max"))
    alt_info = alt_plan.info()
    alt_key = "proth" if alt_info["arith"] == "proth" else "2n"
    alt_plan.close()
    del alt_dev, alt_host

    ot_plan = Plan(N, primes, ot=True)
    ot_steps = max(3, args.steps // 2)
    ms_ot, kern_ot, _, _ = timed_steps(D, ot_plan, dev, ot_steps, 2, flush_l2, scratch)
    ot_ms_step = max(D.allreduce([ms_ot / ot_steps], "max"))
    ot_stages = ot_plan.info()["ot_stages"]
    ot_plan.close()

    pm_steps = max(2, min(args.steps, 5))
    other = dev.clone()
    for _ in range(2):
        plan.negacyclic_mul(other, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(pm_steps):
        plan.negacyclic_mul(other, dev)
    e1.record()
    torch.cuda.synchronize()
    pm_ms = max(D.allreduce([e0.elapsed_time(e1) / pm_steps], "max"))
    del other
    dev.copy_(host.cuda())

    # e2e: host buffers through the public C-ABI host path, H2D + fwd + inv + D2H per step
    out_host = torch.empty_like(host).pin_memory()
    ws = torch.empty(plan.workspace_words(B), dtype=torch.int64, device="cuda")
    plan.execute_host(host, out_host, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)  # warm
    e2e_steps = max(2, min(args.steps, 5))
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.execute_host(host, out_host, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)
    e2e_s = max(D.allreduce([(time.perf_counter() - t0) / e2e_steps], "max"))
    e2e_ok = bool(D.allreduce([float(torch.equal(out_host, host))], "min")[0])
    del ws

    bal = None
    if world > 1 and args.scaling == "strong":  # SURVEY 8(e)'s balanced variant, reported beside
        del dev
        bal = balanced_run(D, args, logn, L_total, batch_job, cfg_id)

    if rank != 0:
        plan.close()
        return None

    # ---- rank 0: check sampled rows of every rank against the oracle
    import oracle
    checked, bad = 0, []
    chain_primes, chain_psis = oracle_chain(logn, L_total, args.primes)
    for r in range(world):
        shr = my_shard(r, world, L_total, batch_job, args.scaling)
        cs_r = gathered[r].numpy()
        for (b, l) in sample_rows(shr):
            gl = shr["prime_offset"] + l
            x = synth.rns_rows([chain_primes[gl]], 1, N, config_id=cfg_id, prime_offset=gl, L_total=L_total,
                               batch_offset=shr["batch_offset"] + b)
            want = row_checksums_np(oracle.ntt_batch(x, [chain_primes[gl]], [chain_psis[gl]], +1))[0]
            checked += 1
            if not np.array_equal(cs_r[b * shr["L"] + l], want):
                bad.append([r, shr["batch_offset"] + b, gl])

    balanced = None
    if bal is not None:
        per_rank_b, ok_b, gathered_b, _ = bal
        b_checked, b_bad = 0, []
        for r in range(world):
            lo = L_total * batch_job * r // world
            n_r = L_total * batch_job * (r + 1) // world - lo
            cs_r = gathered_b[r].numpy()
            for k in sorted({0, n_r - 1, n_r // 2, (n_r * 7) // 11}):
                gl, gb = divmod(lo + k, batch_job)
                x = synth.rns_rows([chain_primes[gl]], 1, N, config_id=cfg_id, prime_offset=gl, L_total=L_total,
                                   batch_offset=gb)
                want = row_checksums_np(oracle.ntt_batch(x, [chain_primes[gl]], [chain_psis[gl]], +1))[0]
                b_checked += 1
                if not np.array_equal(cs_r[k], want):
                    b_bad.append([r, gb, gl])
        ms_b = max(per_rank_b)
        balanced = {
            "value": round(ms_b * 1e3 / units, 3), "unit": "us", "ms_per_step": round(ms_b, 4),
            "per_rank_ms": [round(v, 4) for v in per_rank_b],
            "imbalance": round(max(per_rank_b) / min(per_rank_b), 4),
            "shard": f"prime-major rows split {L_total * batch_job // world} per rank: whole primes plus at most two "
                     "partial primes (one plan and one buffer per piece; SURVEY 8(e) variant)",
            "pieces_per_rank": [len(balanced_pieces(r, world, L_total, batch_job)) for r in range(world)],
            "roundtrip_exact": ok_b,
            "verify": {"rows_checked_vs_oracle": b_checked, "mismatched": b_bad, "verified_rows": b_checked - len(b_bad)},
        }
        bad = bad + [["balanced"] + m for m in b_bad]

    value_us = ms_step * 1e3 / units
    hbm_peak, peak_kind = peaks()
    ceil = butterfly_ceiling()
    form = info["arith"] if info["arith"] == "proth" else "2n"

    def roofline_of(kern_ms, form_, ots=0):
        dom = max(kern_ms, key=kern_ms.get)
        mm = modmuls_per_launch(dom, rows, N, logn, info["log_n1"], plan.passes, ots)
        ach = mm / (kern_ms[dom] * 1e-3) / 1e9
        peak = alu_peak(form_)
        c = ceil.get(("ct_" if dom.startswith("fwd") else "gs_") + form_)
        return dom, mm, ach, peak, c

    dom, mm, achieved, peak, c_dom = roofline_of(kern, form)
    dom_bytes = 2 * 8 * N * rows  # compulsory bytes of one pass: read + write every word
    per_kernel = {}
    for k, t in kern.items():
        m = modmuls_per_launch(k, rows, N, logn, info["log_n1"], plan.passes)
        g = m / (t * 1e-3) / 1e9
        cc = ceil.get(("ct_" if k.startswith("fwd") else "gs_") + form)
        per_kernel[k] = {"ms": round(t, 4), "modmuls": m, "Gmodmul_s": round(g, 1), "frac_of_peak": round(g / peak, 4),
                         "frac_of_ceiling": round(g / cc, 4) if cc else None,
                         "hbm_gbs": round(dom_bytes / (t * 1e-3) / 1e9, 1)}
    traffic, traffic_src = None, None
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            if tr.get("primes") == args.primes and tr.get("config") == args.config and args.scaling == "strong" \
                    and world == 1:
                traffic = tr["kernels"].get(dom)
                traffic_src = {k: tr.get(k) for k in ("file", "commit", "primes", "config")}
        except Exception:
            traffic = None
    # step-level HBM fractions and the ceilings of section 5.4
    ct_bytes = lambda per_row: per_row * N * L_total  # bytes per full-L ciphertext
    two_pass_step = 2 * 2 * 16  # 2 directions x 2 passes x (read + write 8 B)
    step_modmuls_ct = L_total * ((N // 2) * logn * 2 + N // 2)
    cc_ct, cc_gs = ceil.get("ct_" + form), ceil.get("gs_" + form)
    floor_us = None
    if cc_ct and cc_gs:
        floor_us = (L_total * (N // 2) * logn / cc_ct + L_total * ((N // 2) * logn + N // 2) / cc_gs) / 1e3
    line = {
        "metric": METRIC,
        "value": round(value_us, 3),
        "unit": "us",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": False,
        "scaling": "strong" if args.scaling == "strong" else "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic: seeded splitmix64 residues uniform mod each prime (synth/)",
        "config": {
            "workload": f"{args.config}: {text}; one step = NTT + iNTT of every row of the job",
            "N": N, "L": L_total, "global_batch": units,
            "shard": (f"contiguous prime ranges {[n for _, n in prime_ranges(world, L_total)]}, all "
                      f"{batch_job} ciphertexts per rank" if args.scaling == "strong"
                      else f"{sh['Gp']} prime ranges x {sh['Gb']} ciphertext ranges, {batch_job} ciphertexts per GPU"),
            "parallelism": f"prime-sharded x{world}" if world > 1 else "1 GPU",
            "log_n1": info["log_n1"], "passes": info["passes"], "ot": False,
            "primes": PRIME_TEXT[args.primes], "arith": info["arith"],
            "l2": ("L2 flushed between timed steps (256 MiB write, untimed; inputs %.0f MiB per GPU)" % (words * 8 / 2**20)
                   if flush_l2 else "inputs larger than L2 (%.0f MiB per GPU vs 126 MB L2)" % (words * 8 / 2**20)),
            "dist_backend": D.backend if world > 1 else None,
        },
        "residue_ntts_per_s": round(2 * units * L_total / (ms_step * 1e-3), 1),
        "step_stats": {**step_stats, "what": "rank 0's per-step CUDA-event spans: median, min, and the forward "
                                            "(Kernel-1 + Kernel-2) and inverse halves"},
        "l2_warm": ({"value": round(l2_warm * 1e3 / units, 3), "unit": "us", "ms_per_step": round(l2_warm, 4)}
                    if l2_warm is not None else None),
        "per_rank_ms": [round(v, 4) for v in per_rank_ms],
        "imbalance": round(max(per_rank_ms) / min(per_rank_ms), 4),
        "verify": {"rows_checked_vs_oracle": checked, "mismatched": bad, "verified_rows": checked - len(bad),
                   "roundtrip_exact_all_rows": ok_roundtrip,
                   "how": "after timing: one forward, per-row checksums all_gathered to rank 0, sampled rows of "
                          "every rank recomputed by the oracle; inverse restores every row exactly"},
        "roofline": {
            "bound": "alu", "kernel": dom, "achieved": round(achieved, 1), "peak": round(peak, 1),
            "unit": "Gmodmul/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": traffic_src,
            "units": f"{mm} Shoup modmuls per launch of {dom} (SURVEY 8(d): one per butterfly, "
                     "+N/2 per row for the fused N^-1)",
            "peak_kind": "derived: multiply-pipe clk per Shoup modmul (IMAD 2 clk per guide; IMAD.WIDE 5.33, "
                         "IMAD.HI 4.57 clk measured) x 148 SMs x 1.965 GHz (DESIGN.md 7)",
            "ceiling": {"value": c_dom, "unit": "Gbutterfly/s",
                        "what": "the kernels' own butterflies in a register-only loop, measured live "
                                "(tools/libs/bf_roof, 32 warps/SM, no memory)", "all": ceil},
            "frac_of_ceiling": round(achieved / c_dom, 4) if c_dom else None,
            "hbm": {"achieved": round(dom_bytes / (kern[dom] * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(dom_bytes / (kern[dom] * 1e-3) / 1e9 / hbm_peak, 4), "peak_kind": peak_kind,
                    "bytes": "compulsory 16N per row per pass"},
            "step": {
                "hbm_two_pass_gbs": round(ct_bytes(two_pass_step) * units / (ms_step * 1e-3) / 1e9, 1),
                "hbm_two_pass_frac": round(ct_bytes(two_pass_step) * units / (ms_step * 1e-3) / 1e9 / hbm_peak, 4),
                "hbm_compulsory_frac": round(ct_bytes(32) * units / (ms_step * 1e-3) / 1e9 / hbm_peak, 4),
                "modmuls_per_ciphertext": step_modmuls_ct,
            },
            "target": {
                "hbm_frac": 0.70,
                "us_per_ciphertext_needed": round(ct_bytes(two_pass_step) / (0.70 * hbm_peak * 1e9) * 1e6, 1),
                "butterfly_ceiling_floor_us": round(floor_us, 1) if floor_us else None,
                "note": "a two-pass step at 70% of HBM needs the first number; the kernels' own butterflies at "
                        "their register-only rate (CT for forward, GS for inverse) need the second",
            },
            "per_kernel": per_kernel,
        },
        "kernels_ms": {k: round(v, 4) for k, v in kern.items()},
        alt_form: {"primes": PRIME_TEXT[alt_form], "arith": alt_info["arith"],
                   "value": round(alt_ms_step * 1e3 / units, 3), "unit": "us",
                   "ms_per_step": round(alt_ms_step, 4), "roundtrip_exact": alt_ok,
                   "kernels_ms": {k: round(v, 4) for k, v in kern_alt.items()},
                   "roofline_frac": round(roofline_of(kern_alt, alt_key)[2] / alu_peak(alt_key), 4),
                   "frac_of_ceiling": (round(roofline_of(kern_alt, alt_key)[2] / roofline_of(kern_alt, alt_key)[4], 4)
                                       if roofline_of(kern_alt, alt_key)[4] else None)},
        "ot_on": {"value": round(ot_ms_step * 1e3 / units, 3), "unit": "us", "ms_per_step": round(ot_ms_step, 4),
                  "ot_stages": ot_stages, "kernels_ms": {k: round(v, 4) for k, v in kern_ot.items()}},
        "negacyclic_mul": {"ms_per_step": round(pm_ms, 4), "us_per_ct": round(pm_ms * 1e3 / units, 3),
                           "what": "b <- a*b mod (X^N+1): 2 forward NTTs + fused odot/inverse, per ciphertext pair"},
        "cpu_baseline": None,
        "e2e": {"value": round(e2e_s * 1e6 / units, 3), "unit": "us",
                "h2d_bytes_per_step": units * L_total * N * 8, "d2h_bytes_per_step": units * L_total * N * 8,
                "ms_per_step": round(e2e_s * 1e3, 3), "ok": e2e_ok,
                "what": "ntt_execute_host: pinned host in -> H2D -> fwd -> inv -> D2H, every rank its shard"},
        "gpu_launches": launches,
        "clocks": clocks,
        "roundtrip_exact": ok_roundtrip and (balanced is None or balanced["roundtrip_exact"]),
    }
    if balanced is not None:
        line["balanced"] = balanced
    plan.close()
    return line


def c5_line(D, args):
    """C5, the mixed request stream at N = 2^16 (BASELINE config 5):
    per L, throughput mode (requests round-robin to ranks, each rank's
    requests of one L batched into one call) and latency mode (one request at
    a time, its primes sharded over the ranks, replayed from a request
    graph: the split's kernels, or the one-kernel request of
    NTT_GRAPH_ONE_KERNEL -- both timed, the faster one reported per L).  value = mixed-stream latency-mode us per request (the mean over
    the L sweep, one request per L in turn)."""
    torch = D.torch
    import synth
    from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, NTT_GRAPH_ONE_KERNEL, Plan, find_primes

    rank, world = D.rank, D.world
    logn = 16
    N = 1 << logn
    cfg_id = synth.CONFIG_IDS["C5"]
    sweep, launches = {}, 0
    ok_all = True
    for L in C5_LS:
        primes_all = find_primes(N, L, args.primes)
        # throughput: requests r = rank, rank + world, ... ; all of this rank's requests share the chain -> one batch
        mine = list(range(rank, C5_REQUESTS, world))
        tp_plan = Plan(N, primes_all)
        x = torch.empty(len(mine) * L * N, dtype=torch.int64)
        synth.rns_rows(primes_all, len(mine), N, config_id=cfg_id, out=x.numpy().view(np.uint64).reshape(len(mine), L, N))
        xd = x.cuda()
        ref = xd.clone()
        for _ in range(args.warmup):
            tp_plan.forward(xd)
            tp_plan.inverse(xd)
        D.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            tp_plan.forward(xd)
            tp_plan.inverse(xd)
        e1.record()
        torch.cuda.synchronize()
        tp_ms = max(D.allreduce([e0.elapsed_time(e1) / args.steps], "max"))
        launches += 2 * tp_plan.passes * args.steps
        ok_all = ok_all and bool(torch.equal(xd, ref))
        tp_plan.close()
        # latency: this rank's prime range of ONE request, replayed from a request graph
        off, n = prime_ranges(world, L)[rank] if world <= L else ((rank, 1) if rank < L else (0, 0))
        forms = {"graph": 0.0, "graph_n1_2^7": 0.0, "one_kernel": 0.0}
        serial, means = dict(forms), dict(forms)
        if n > 0:
            lp = Plan(N, primes_all[off: off + n])
            lp7 = Plan(N, primes_all[off: off + n], log_n1=7)  # the split with the shorter Kernel-1 columns
            y = torch.empty(n * N, dtype=torch.int64)
            synth.rns_rows(primes_all[off: off + n], 1, N, config_id=cfg_id, prime_offset=off, L_total=L,
                           out=y.numpy().view(np.uint64).reshape(1, n, N))
            yd = y.cuda()
            yref = yd.clone()
            # request forms: the split's kernels (2 per direction) captured as a
            # graph -- the default split (2^8 x 2^8) and 2^7 x 2^9 -- and the
            # one-kernel request (NTT_GRAPH_ONE_KERNEL)
            for form, pl, flag, kernels in (("graph", lp, 0, 4), ("graph_n1_2^7", lp7, 0, 4),
                                            ("one_kernel", lp, NTT_GRAPH_ONE_KERNEL, 1)):
                g = pl.graph(yd, NTT_DIR_FORWARD | NTT_DIR_INVERSE | flag)
                for _ in range(max(3, args.warmup)):
                    g.launch()
                reps = max(20, args.steps * 4)
                D.barrier()
                torch.cuda.synchronize()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
                evs[0].record()
                for i in range(reps):  # one request in flight: each replay waits for the previous on the stream
                    g.launch()
                    evs[i + 1].record()
                torch.cuda.synchronize()
                spans = [evs[i].elapsed_time(evs[i + 1]) for i in range(reps)]
                forms[form] = statistics.median(spans)
                # the event spans come in steps of the timer's granularity (2.048 us
                # on the B200 boxes): the mean is the finer estimate of the same latency
                means[form] = statistics.mean(spans)
                # the same serial stream with events only at its ends: the per-request
                # device time without a completion event after every request
                torch.cuda.synchronize()
                evs[0].record()
                for i in range(reps):
                    g.launch()
                evs[1].record()
                torch.cuda.synchronize()
                serial[form] = evs[0].elapsed_time(evs[1]) / reps
                launches += 2 * reps * kernels
                ok_all = ok_all and bool(torch.equal(yd, yref))
                g.close()
            lp.close()
            lp7.close()
        else:
            for _ in range(3):
                D.barrier()
        forms = {k: max(D.allreduce([v], "max")) for k, v in sorted(forms.items())}
        serial = {k: max(D.allreduce([v], "max")) for k, v in sorted(serial.items())}
        means = {k: max(D.allreduce([v], "max")) for k, v in sorted(means.items())}
        lat_form = min(forms, key=forms.get)  # the faster request form at this L
        lat_ms = forms[lat_form]
        sweep[str(L)] = {"throughput_us_per_request": round(tp_ms * 1e3 / C5_REQUESTS, 3),
                         "latency_us_per_request": round(lat_ms * 1e3, 3),
                         "latency_form": lat_form,
                         "latency_us_by_form": {k: round(v * 1e3, 3) for k, v in forms.items()},
                         "latency_mean_us_by_form": {k: round(v * 1e3, 3) for k, v in means.items()},
                         "serial_us_by_form": {k: round(v * 1e3, 3) for k, v in serial.items()},
                         "latency_primes_per_rank": [c for _, c in prime_ranges(world, L)] if world <= L
                         else [1 if r < L else 0 for r in range(world)]}
    ok_all = bool(D.allreduce([float(ok_all)], "min")[0])
    if rank != 0:
        return None
    lat_mean = statistics.mean(v["latency_us_per_request"] for v in sweep.values())
    tp_mean = statistics.mean(v["throughput_us_per_request"] for v in sweep.values())
    return {
        "metric": METRIC, "value": round(lat_mean, 3), "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(lat_mean * len(C5_LS) / 1e3, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: seeded splitmix64 residues uniform mod each prime (synth/)",
        "config": {"workload": "C5: mixed ciphertext stream, N=2^16, one request = NTT + iNTT of one ciphertext of "
                               f"L primes, L in {C5_LS}; value = latency mode, mean over the sweep",
                   "latency_how": "one request in flight (each replay waits for the previous on the stream), CUDA "
                                  "events after every request, median (latency_mean_us_by_form: their mean -- the spans come in steps of "
                                  "the 2.048 us event granularity); serial_us_by_form: the same stream timed "
                                  "with events only at its ends (no per-request completion event)",
                   "N": N, "requests_per_L_throughput": C5_REQUESTS, "primes": PRIME_TEXT[args.primes],
                   "parallelism": f"x{world}" if world > 1 else "1 GPU"},
        "sweep": sweep,
        "throughput_mode_mean_us_per_request": round(tp_mean, 3),
        "roundtrip_exact": ok_all,
        "gpu_launches": launches,
        "e2e": None,
        "cpu_baseline": None,
    }


def run_own(args):
    D = Dist()
    if D.world != args.gpus and D.rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {D.world}", file=sys.stderr)
    if args.config == "C5":
        line = c5_line(D, args)
    else:
        logn, L_total, batch, text = CONFIGS[args.config]
        line = transform_line(D, args, logn, L_total, batch, text)
    if D.rank == 0 and line is not None:
        if D.world == 1 and not args.no_cpu and args.config != "C5":
            import synth
            logn, L_total, batch, _ = CONFIGS[args.config]
            line["cpu_baseline"] = cpu_baseline(logn, L_total, batch, synth.CONFIG_IDS[args.config], args.primes)
        print(json.dumps(line), flush=True)
    D.close()
    bad = line is not None and (line.get("verify", {}).get("mismatched") or not line.get("roundtrip_exact", True))
    return 1 if bad else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--primes", default="2n", choices=["2n", "proth"],
                    help="prime chain: 2n = SURVEY 8(c)#3 (default), proth = p = 1 mod 2^32")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    return run_own(args)


if __name__ == "__main__":
    sys.exit(main())
