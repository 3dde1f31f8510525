"""Summarise ncu outputs into profiles/ (run in the build container).

  python tools/summarize_ncu.py launches gpurun_out/launches.csv  > profiles/<tag>_launches.json
  python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep      > profiles/<tag>_ncu_full.json
"""

import collections
import csv
import io
import json
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    return {k: {"launches": cnt[k], "avg_us": round(tot[k] / cnt[k], 2), "share": round(tot[k] / T, 4)}
            for k in sorted(tot, key=lambda k: -tot[k])}


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    res = []
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    for r in data:
        rec = {"kernel": r[ki].split("(")[0]}
        for m in WANT:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = r[i] + (" " + units[i] if units[i] else "")
        st = []
        for i in stall_cols:
            try:
                st.append((hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i].replace(",", ""))))
            except ValueError:
                pass
        tot = sum(v for _, v in st) or 1.0
        rec["top_stalls"] = [(k, round(v / tot, 3)) for k, v in sorted(st, key=lambda x: -x[1])[:6]]
        res.append(rec)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
