#!/usr/bin/env python3
"""bench.py -- the headline measurement of the batched negacyclic NTT + iNTT.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one pass of the whole hot path over one batch: ntt_forward then
ntt_inverse of every residue row.  Workload at N=1:
BASELINE.json configs[3] ("C4": N=2^17, 60 primes of 60 bits, batch 32).
Multi-GPU is weak-scaled and prime-sharded: G ranks process 32*G ciphertexts,
split over a Gp x Gb grid of (prime range, ciphertext range) shards so every
rank holds exactly 1920 rows; there is no collective on the data path
(SURVEY 8(e)); NCCL carries only the timing barrier / max.

Prints ONE JSON line on rank 0 (see DESIGN.md section 7 for every key).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs per NTT+iNTT (N=2^17, all primes) & HBM GB/s vs 8 TB/s, 1/2/4/8 B200"

CONFIGS = {
    # name: (logN, L, batch per GPU, BASELINE.json text)
    "C1": (12, 1, 1, "N=2^12, 1 prime (~60-bit), batch 1"),
    "C2": (15, 15, 16, "N=2^15, 15 primes (~Q=2^881, SEAL-like), batch 16"),
    "C3": (16, 45, 64, "N=2^16, 45 primes (bootstrappable CKKS-size), batch 64"),
    "C4": (17, 60, 32, "N=2^17, ~60 primes (large bootstrappable set), batch 32"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# Multiply-pipe cost of one warp-instruction per SMSP, in clocks: IMAD from the
# guide (rt_SMSP = 2); IMAD.WIDE / IMAD.HI measured on B200 with independent
# chains (profiles/r01_alu_roof.jsonl: 24 and 28 per clk per SM; confirmed by
# the 2 WIDE + 2 HI + 3 IMAD mix at 25.7 clk, profiles/r01g_bf_roof_variants.txt).
CLK_IMAD, CLK_WIDE, CLK_HI = 2.0, 16 / 3.0, 32 / 7.0


def alu_floor_clk(form: str = "2n") -> float:
    """Multiply-pipe clocks per warp-butterfly of the truncated-quotient Shoup
    butterfly: general primes 3 WIDE + 2 HI + 4 IMAD, Proth
    primes 2 WIDE + 2 HI + 3 IMAD."""
    if form == "proth":
        return 2 * CLK_WIDE + 2 * CLK_HI + 3 * CLK_IMAD
    return 3 * CLK_WIDE + 2 * CLK_HI + 4 * CLK_IMAD


def alu_peak(form: str = "2n", nominal: bool = False):
    """Derived integer roof in G butterflies/s: 148 SMs x 4 SMSPs x 32 lanes /
    (clk per warp-butterfly) x 1.965 GHz.  nominal=True uses quarter-rate
    (4 clk) WIDE/HI instead of the measured rates (an upper bound)."""
    sm_clk_ghz = 1.965
    clk = (22.0 if form == "proth" else 28.0) if nominal else alu_floor_clk(form)
    return 148 * 4 * 32 / clk * sm_clk_ghz


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

def shard_grid(G: int, L: int):
    """(Gp, Gb): the largest Gp <= G dividing both G and L, Gb = G / Gp."""
    gp = max(d for d in range(1, G + 1) if G % d == 0 and L % d == 0)
    return gp, G // gp


def my_shard(rank: int, G: int, L: int, batch_per_gpu: int):
    gp, gb = shard_grid(G, L)
    rp, rb = rank % gp, rank // gp
    Lp = L // gp
    Bb = batch_per_gpu * G // gb
    return {"Gp": gp, "Gb": gb, "prime_offset": rp * Lp, "L": Lp, "batch_offset": rb * Bb, "batch": Bb}


# ------------------------------------------------------------------ reference arm

def cpu_oracle_sample(logn: int, L_total: int, ciphertexts: int, config_id: int, form: str = "proth"):
    """Time the oracle (as it stands) on `ciphertexts` full-L ciphertexts
    (fwd+inv) on all host cores, with the same prime family as the GPU arm
    (the oracle's own scans: step 2N for "2n", step 2^32 for "proth").
    Returns (us_per_ntt_intt, seconds, cores)."""
    import oracle
    import synth
    N = 1 << logn
    primes = oracle.find_primes(1 << 31, L_total) if form == "proth" else oracle.find_primes(N, L_total)
    psis = [oracle.find_psi(p, N) for p in primes]
    x = synth.rns_rows(primes, ciphertexts, N, config_id=config_id)
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    oracle.ntt_batch(x, primes, psis, +1, cores)
    oracle.ntt_batch(x, primes, psis, -1, cores)
    dt = time.perf_counter() - t0
    return dt / ciphertexts * 1e6, dt, cores


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    logn, L, batch, text = CONFIGS[args.config]
    import synth
    cfg_id = synth.CONFIG_IDS[args.config]
    for _ in range(args.warmup):
        cpu_oracle_sample(logn, L, 1, cfg_id, args.primes)
    times = []
    cores = None
    for _ in range(args.steps):
        us, dt, cores = cpu_oracle_sample(logn, L, 1, cfg_id, args.primes)
        times.append(dt)
    T = sum(times) / len(times)
    value = T * 1e6  # one full-L ciphertext per step
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "us", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(T * 1e3, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {text}; NTT+iNTT", "N": 1 << logn, "L": L,
                   "sample": "1 full-L ciphertext per step"},
        "cpu_baseline": {"value": round(value, 3), "unit": "us", "cores": cores, "kind": "oracle",
                         "sample": f"1 ciphertext x {L} primes x N=2^{logn}, fwd+inv per step"},
        "e2e": {"value": round(value, 3), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ own arm

def run_own(args):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2012_01968_b200 import NTT_DIR_FORWARD, NTT_DIR_INVERSE, Plan, find_primes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 needs torchrun --nproc-per-node N")
    # BENCH_DIST_BACKEND=gloo (testing only): several ranks sharing the visible
    # GPUs, reductions on CPU tensors; the default is one rank per GPU over NCCL.
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    logn, L_total, batch_per_gpu, text = CONFIGS[args.config]
    N = 1 << logn
    sh = my_shard(rank, world, L_total, batch_per_gpu)
    all_primes = find_primes(N, L_total, args.primes)
    primes = all_primes[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    L, B = sh["L"], sh["batch"]
    words = B * L * N
    cfg_id = synth.CONFIG_IDS[args.config]

    # inputs: seeded residues, pinned host (for e2e) and device-resident (for value)
    host = torch.empty(words, dtype=torch.int64).pin_memory()
    synth.rns_rows(primes, B, N, config_id=cfg_id, prime_offset=sh["prime_offset"], L_total=L_total,
                   batch_offset=sh["batch_offset"], out=host.numpy().view(np.uint64).reshape(B, L, N))
    dev = host.cuda()
    ref_sum = None

    # Inputs smaller than 2x L2 (C1, C2): flush L2 between timed steps by writing a
    # 256 MiB scratch buffer, outside the timed spans (timing rule); C3/C4 inputs
    # are larger than L2 and run back to back.
    L2_BYTES = 126 * 2**20
    flush_l2 = words * 8 < 2 * L2_BYTES
    scratch = torch.empty(256 * 2**20 // 4, dtype=torch.int32, device="cuda") if flush_l2 else None

    def timed(plan, steps, warmup):
        stream = torch.cuda.current_stream()
        passes = plan.passes
        seq = [(NTT_DIR_FORWARD, i) for i in range(passes)] + [(NTT_DIR_INVERSE, i) for i in range(passes)]
        for _ in range(warmup):
            plan.forward(dev)
            plan.inverse(dev)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local)
        with sampler:
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
        if world > 1:
            dist.barrier()
        if flush_l2:  # the sum of the per-step spans, flushes excluded
            ms = sum(ev[s][0].elapsed_time(ev[s][-1]) for s in range(steps))
        else:
            ms = start.elapsed_time(end)
        per_kernel = [statistics.mean(ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(steps))
                      for j in range(len(seq))]
        if world > 1:
            t = torch.tensor([ms], device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        names = [("fwd" if d == NTT_DIR_FORWARD else "inv") + f"_pass{p}" for d, p in seq]
        return ms, dict(zip(names, per_kernel)), sampler.summary(), len(seq) * steps

    plan = Plan(N, primes)
    info = plan.info()
    ms, kern, clocks, launches = timed(plan, args.steps, args.warmup)
    # the roundtrip restores the input exactly: a free correctness check
    torch.cuda.synchronize()
    ok_roundtrip = bool(torch.equal(dev, host.cuda()))

    ms_step = ms / args.steps
    units = batch_per_gpu * world  # full-L ciphertexts the whole job processed per step
    value_us = ms_step * 1e3 / units
    rows = B * L
    bytes_alg = 2 * 2 * 8 * N * rows  # compulsory: read+write each word once, fwd and inv
    hbm_peak, peak_kind = peaks()
    dom = max(kern, key=kern.get)
    dom_ms = kern[dom]
    bfly_per_launch = rows * (N // 2) * (logn // 2 if plan.passes == 2 else logn)
    # stages per kernel: Kernel-1 holds log N1, Kernel-2 log N2
    if plan.passes == 2:
        ln1 = info["log_n1"]
        st = {"fwd_pass0": ln1, "fwd_pass1": logn - ln1, "inv_pass0": logn - ln1, "inv_pass1": ln1}[dom]
    else:
        st = logn
    bfly_per_launch = rows * (N // 2) * st
    achieved = bfly_per_launch / (dom_ms * 1e-3) / 1e9
    form = args.primes if info.get("proth") else "2n"
    peak = alu_peak(form)
    dom_bytes = 2 * 8 * N * rows  # compulsory bytes of one pass: read + write every word
    hbm_dom = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(dom)
        except Exception:
            traffic = None

    # the paper's two-kernel split (two HBM passes per direction), same primes and inputs
    tk_plan = Plan(N, primes, fused=False)
    tk_steps = max(3, args.steps // 2)
    ms_tk, kern_tk, _, _ = timed(tk_plan, tk_steps, 2)
    tk_plan.close()

    # the other prime family, same workload, reported beside
    alt_form = "2n" if args.primes == "proth" else "proth"
    alt_primes = find_primes(N, L_total, alt_form)[sh["prime_offset"]: sh["prime_offset"] + sh["L"]]
    alt_host = torch.empty(words, dtype=torch.int64)
    synth.rns_rows(alt_primes, B, N, config_id=cfg_id, prime_offset=sh["prime_offset"], L_total=L_total,
                   batch_offset=sh["batch_offset"], out=alt_host.numpy().view(np.uint64).reshape(B, L, N))
    dev.copy_(alt_host.cuda())
    alt_plan = Plan(N, alt_primes)
    alt_steps = max(3, args.steps // 2)
    ms_alt, kern_alt, _, _ = timed(alt_plan, alt_steps, 2)
    alt_ok = bool(torch.equal(dev, alt_host.cuda()))
    alt_proth = alt_plan.info()["proth"]
    alt_plan.close()
    del alt_host
    dev.copy_(host.cuda())

    # OT on: same workload, reported beside (north_star: OT on/off)
    ot_plan = Plan(N, primes, ot=True)
    ms_ot, kern_ot, _, _ = timed(ot_plan, max(3, args.steps // 2), 2)
    ot_plan.close()
    ot_steps = max(3, args.steps // 2)

    # NEXT-2 context: negacyclic product of two full-L ciphertext batches (fwd a, fwd b, fused odot+inv)
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
    pm_ms = e0.elapsed_time(e1) / pm_steps
    del other
    dev.copy_(host.cuda())

    # e2e: host buffers through the public C-ABI host path, H2D + fwd + inv + D2H per step
    out_host = torch.empty_like(host).pin_memory()
    ws = torch.empty(plan.workspace_words(B), dtype=torch.int64, device="cuda")
    plan.execute_host(host, out_host, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)  # warm
    e2e_steps = max(2, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.execute_host(host, out_host, NTT_DIR_FORWARD | NTT_DIR_INVERSE, ws)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_ok = bool(torch.equal(out_host, host))
    if world > 1:  # every rank's exactness flags to rank 0 (NCCL carries verification, not data)
        t = torch.tensor([int(ok_roundtrip), int(e2e_ok)], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok_roundtrip, e2e_ok = bool(t[0].item()), bool(t[1].item())
    del ws

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        us, dt, cores = cpu_oracle_sample(logn, L_total, 1, cfg_id, args.primes)
        cpu = {"value": round(us, 1), "unit": "us", "cores": cores, "kind": "oracle",
               "sample": f"1 ciphertext x {L_total} primes x N=2^{logn}, fwd+inv ({dt:.2f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value_us, 3),
            "unit": "us",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u64",
            "data": "synthetic: seeded splitmix64 residues uniform mod each prime (synth/)",
            "config": {
                "workload": f"{args.config}: {text} per GPU; one step = NTT + iNTT of every row",
                "N": N, "L": L_total, "batch_per_gpu": batch_per_gpu, "global_batch": units,
                "shard": f"{sh['Gp']} prime ranges x {sh['Gb']} ciphertext ranges",
                "log_n1": info["log_n1"], "passes": info["passes"], "cluster": info["cluster"], "ot": False,
                "primes": {"2n": "p = 1 mod 2N descending from 2^60 - 2N + 1 (DESIGN.md R3)",
                           "proth": "p = 1 mod 2^32 descending from 2^60 - 2^32 + 1 (DESIGN.md 5.1)"}[args.primes],
                "proth_arith": bool(info.get("proth")),
                "l2": ("L2 flushed between timed steps (256 MiB write, untimed; inputs %.0f MiB per GPU)" if flush_l2
                       else "inputs larger than L2 (%.0f MiB per GPU vs 126 MB L2)") % (words * 8 / 2**20),
            },
            "residue_ntts_per_s": round(2 * rows * world / (ms_step * 1e-3), 1),
            "hbm_gbs_compulsory": round(bytes_alg / (ms_step * 1e-3) / 1e9, 1),
            "roofline": {
                "bound": "alu", "kernel": dom, "achieved": round(achieved, 1), "peak": round(peak, 1),
                "unit": "Gbutterfly/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_kind": "derived: multiply-pipe clk per Shoup butterfly (IMAD 2 clk per guide; IMAD.WIDE 5.33, "
                             "IMAD.HI 4.57 clk measured) x 148 SMs x 1.965 GHz (DESIGN.md 7)",
                "peak_nominal_quarter_rate": round(alu_peak(form, nominal=True), 1),
                "hbm": {"achieved": round(hbm_dom, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(hbm_dom / hbm_peak, 4), "peak_kind": peak_kind,
                        "bytes": "compulsory 16N per row per pass"},
            },
            "kernels_ms": {k: round(v, 4) for k, v in kern.items()},
            "two_kernel": {"value": round(ms_tk / tk_steps * 1e3 / units, 3), "unit": "us",
                           "ms_per_step": round(ms_tk / tk_steps, 4),
                           "kernels_ms": {k: round(v, 4) for k, v in kern_tk.items()}},
            "other_primes": {"primes": alt_form, "proth_arith": alt_proth,
                             "value": round(ms_alt / alt_steps * 1e3 / units, 3), "unit": "us",
                             "ms_per_step": round(ms_alt / alt_steps, 4), "roundtrip_exact": alt_ok,
                             "kernels_ms": {k: round(v, 4) for k, v in kern_alt.items()}},
            "ot_on": {"value": round(ms_ot / ot_steps * 1e3 / units, 3), "unit": "us",
                      "ms_per_step": round(ms_ot / ot_steps, 4),
                      "kernels_ms": {k: round(v, 4) for k, v in kern_ot.items()}},
            "negacyclic_mul": {"ms_per_step": round(pm_ms, 4), "us_per_ct": round(pm_ms * 1e3 / units, 3),
                               "what": "b <- a*b mod (X^N+1): 2 forward NTTs + fused odot/inverse, per ciphertext pair"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_s * 1e6 / units, 3), "unit": "us",
                    "h2d_bytes_per_step": words * 8, "d2h_bytes_per_step": words * 8,
                    "ms_per_step": round(e2e_s * 1e3, 3), "ok": e2e_ok},
            "gpu_launches": launches,
            "clocks": clocks,
            "roundtrip_exact": ok_roundtrip,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--primes", default="proth", choices=["2n", "proth"],
                    help="prime family: proth = p = 1 mod 2^32 (default), 2n = DESIGN.md R3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_own(args)


if __name__ == "__main__":
    sys.exit(main())
