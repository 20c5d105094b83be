"""Hottest SASS instructions (by warp-stall samples) of one kernel in an ncu
report, with the per-reason breakdown columns ncu provides.

    python tools/sass_hot.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
end = next((i for i in range(2, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rd = list(csv.reader(io.StringIO("\n".join(lines[1:end]))))
hdr, rows = rd[0], rd[1:]
si = hdr.index("Source")
smp = hdr.index("Warp Stall Sampling (All Samples)")
reason_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
tot = sum(int(r[smp] or 0) for r in rows)
print(f"total samples {tot}; columns: {[hdr[i] for i in reason_cols][:12]}")
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][smp] or 0))[:top]
for i in sorted(order):
    r = rows[i]
    print(f"{i:5d} {int(r[smp]):7d} {100 * int(r[smp]) / tot:5.1f}%  {r[si].strip()[:90]}")
