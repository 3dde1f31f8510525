"""Per-CUDA-line warp-stall attribution from an ncu report (sass,cuda view).

usage: python tools/src_hotspots.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = "?"
hdr = None
last_line, last_src = "?", ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        v = float(r[4])
        ex = float(r[7]) if r[7] else 0.0
    except ValueError:
        continue
    if r[0]:
        last_line, last_src = r[0], r[1].strip()[:80]
    key = (fname, last_line)
    a = agg.setdefault(key, [0.0, 0.0, last_src])
    a[0] += v
    a[1] += ex
tot = sum(a[0] for a in agg.values()) or 1.0
tex = sum(a[1] for a in agg.values()) or 1.0
for (f, ln), (v, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v / tot:6.3f} stall  {ex / tex:6.3f} instr  {f}:{ln}  {src}")
