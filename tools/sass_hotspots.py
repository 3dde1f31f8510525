"""Warp-stall samples aggregated per SASS instruction (no -lineinfo needed).

usage: python tools/sass_hotspots.py report.ncu-rep kernel_regex [top]
Prints the top instructions by stall samples plus a per-opcode summary and the
stall-reason columns that dominate.
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
tot = sum(float(r[si] or 0) for r in data) or 1.0
print(f"total samples {tot:.0f}, instructions {len(data)}")
ops = collections.Counter()
opi = collections.Counter()
for idx, r in enumerate(data):
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    ops[op.split(".")[0]] += float(r[si] or 0)
    opi[op.split(".")[0]] += float(r[ei] or 0)
print("per-opcode stall share / executed warp-instr:")
for op, v in ops.most_common(20):
    print(f"  {op:10s} {v / tot:6.3f}  {opi[op]:12.0f}")
print("top instructions:")
order = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:top]
for i in order:
    r = data[i]
    print(f"  {i:5d} {float(r[si] or 0) / tot:6.3f} {r[1].strip()[:90]}")
