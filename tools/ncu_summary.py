"""Summarise ncu reports for profiles/ (committed evidence).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep] > profiles/rNN_ncu_summary.md
    (every report argument may also be the CSV export of its raw page)
    python tools/ncu_summary.py --launches gpurun_out/launches.csv          (launch list -> shares)
    python tools/ncu_summary.py --traffic gpurun_out/prof.ncu-rep           (per-kernel DRAM bytes JSON)
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("smsp__inst_executed.sum", "warp-instr"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def raw(rep):
    """The raw page of a report (.ncu-rep, read with ncu) or of its CSV export
    (`ncu -i rep --page raw --csv > raw.csv`, e.g. made on the GPU box)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(h, r):
    items = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled"):
            try:
                items.append((float(r[i]), n.replace("smsp__average_warps_issue_stalled_", "")
                              .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    return ", ".join(f"{n} {v:.2f}" for v, n in sorted(items, reverse=True)[:6])


def summary(reps):
    for rep in reps:
        h, u, rows = raw(rep)
        print(f"### {rep}\n")
        print("| kernel | " + " | ".join(k for _, k in KEYS) + " | top stalls (per issue) |")
        print("|---" * (len(KEYS) + 2) + "|")
        for r in rows:
            name = r[h.index("Kernel Name")]
            vals = []
            for m, _ in KEYS:
                if m in h:
                    v, un = r[h.index(m)], u[h.index(m)]
                    vals.append(f"{v} {un}".strip())
                else:
                    vals.append("-")
            print(f"| `{name}` | " + " | ".join(vals) + f" | {stalls(h, r)} |")
        print()


def traffic(rep):
    h, u, rows = raw(rep)
    out = {}
    for r in rows:
        name = r[h.index("Kernel Name")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[h.index("dram__bytes_read.sum")]) * scale[u[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * scale[u[h.index("dram__bytes_write.sum")]]
        out.setdefault(name, rd + wr)
    print(json.dumps(out, indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    for r in rows[hdr + 1:]:
        tot.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    allns = sum(sum(v) for v in tot.values())
    print("| kernel | launches | mean ns | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda t: -sum(t[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / allns:.3f} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--traffic":
        traffic(sys.argv[2])
    else:
        summary(sys.argv[1:])
