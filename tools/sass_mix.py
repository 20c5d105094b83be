"""Instruction mix of a kernel from an ncu report's SASS source page,
weighted by executed warp-instructions, with pipe classes.
usage: python tools/sass_mix.py report.ncu-rep kernel_regex [per_unit]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# first kernel only
start = 1
end = next((i for i in range(2, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rd = csv.reader(io.StringIO("\n".join(lines[start:end])))
hdr = next(rd)
si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
stall_i = hdr.index("Warp Stall Sampling (All Samples)")
mix, stalls = Counter(), Counter()
total = 0
for r in rd:
    src = r[si].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    if not m:
        continue
    op = m.group(2)
    n = int(r[ei] or 0)
    mix[op] += n
    stalls[op] += int(r[stall_i] or 0)
    total += n

def pipe(op):
    if op.startswith(("IMAD.WIDE", "IMAD.HI")):
        return "fmaheavy-x2"
    if op.startswith(("IMAD", "HFMA2", "FFMA", "FMUL")):
        return "fmaheavy"
    if op.startswith(("IADD3", "LOP3", "SHF", "SEL", "ISETP", "MOV", "PRMT", "VIADD", "IABS", "LEA", "FSEL", "IMNMX", "VIMNMX")):
        return "alu"
    if op.startswith(("LDS", "STS", "LDG", "STG", "LDC", "SHFL", "ATOMS", "LDSM")):
        return "mem"
    return "other"

byp = Counter()
for op, n in mix.items():
    byp[pipe(op)] += n
print(f"total warp-instr {total:.4g}  per unit {total / per:.2f}")
for p, n in byp.most_common():
    print(f"  {p:12s} {n / per:8.2f}")
for op, n in mix.most_common(30):
    print(f"  {op:22s} {n / per:8.2f}   stall-samples {stalls[op]}")
