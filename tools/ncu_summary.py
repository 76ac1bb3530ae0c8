"""Summaries of ncu output for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py rep  <file.ncu-rep>     key metrics + stall mix of each kernel
    python tools/ncu_summary.py launches <launches.csv> per-kernel launch totals and shares
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__block_size",
    "launch__grid_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        print(f"== {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        st = {k.split("stalled_")[1]: float(v or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
        tot = sum(st.values()) or 1.0
        mix = sorted(((k, 100.0 * v / tot) for k, v in st.items() if v), key=lambda x: -x[1])
        print("  stall mix (% of pc samples): " + ", ".join(f"{k} {v:.1f}" for k, v in mix[:9]))


def launches(path):
    agg = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(r["Kernel Name"][:100], [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("(cold-cache, serialised launches: compare shares, not absolutes)")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:4d} {t:10.1f} us {100 * t / tot:5.1f}%  {n}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
