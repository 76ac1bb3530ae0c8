"""Warp-stall samples of one ncu report attributed to CUDA source lines, from
ncu's own source page (--import-source on): top lines with their dominant
stall reasons, and totals per opcode from the SASS page.

    python tools/ncu_src.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
STALLS = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_mio", "stall_math", "stall_branch_resolving",
          "stall_no_inst", "stall_selected", "stall_not_selected", "stall_dispatch", "stall_lg", "stall_barrier",
          "stall_membar", "stall_drain", "stall_misc", "stall_sleep", "stall_tex"]


def blocks(text):
    """Split the multi-table CSV of the source page into (header rows, data rows) per file."""
    cur_file, head, rows = None, None, []
    for r in csv.reader(io.StringIO(text)):
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            if head is not None:
                yield cur_file, head, rows
            cur_file, head, rows = r[1], None, []
        elif r[0] in ("Line No", "Address") and head is None:
            head = r
        elif head is not None:
            rows.append(r)
    if head is not None:
        yield cur_file, head, rows


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = []
tot = 0
for f, head, rows in blocks(out):
    idx = {}
    for i, k in enumerate(head):
        idx.setdefault(k, i)
    for r in rows:
        if r[idx["Address"]] != "-":
            continue
        try:
            s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        if s <= 0:
            continue
        tot += s
        st = {k: float(r[idx[k]] or 0) for k in STALLS if k in idx}
        ins = float(r[idx["Instructions Executed"]] or 0)
        lines.append((s, f.split("/")[-1], r[0], r[1].strip()[:70], st, ins))
lines.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for s, f, ln, src, st, ins in lines[:top]:
    mix = ", ".join(f"{k[6:]} {100 * v / s:.0f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<4} inst {ins:9.0f}  [{mix}]  {src}")
