"""Attribute ncu warp-stall samples and executed instructions of one kernel to
CUDA source lines (the SASS page joined with nvdisasm line info).

    python tools/ncu_lines.py <report.ncu-rep> <file.cubin> <mangled kernel name> [top]

The cubin must be the one the profiled library was built from
(cuobjdump -xelf all build_obj/hf_cells3d.o)."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

# offset -> (file, line) from nvdisasm; with inlining, the outermost call site
# (the kernel body line) is kept
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
cur = None
inside = False
line_of = {}
for ln in dis.splitlines():
    if ln.startswith(".text."):
        inside = ln.strip().rstrip(":") == ".text." + fn
        continue
    if not inside:
        continue
    if "//##" in ln:
        locs = re.findall(r'"([^"]+)", line (\d+)', ln)
        if locs:
            f, l = locs[-1]
            cur = (f.split("/")[-1], int(l))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isamp, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = rows[2:]
base = int(data[0][ia], 16)
per = defaultdict(lambda: [0, 0])
tot_s = tot_e = 0
miss = 0
for r in data:
    off = int(r[ia], 16) - base
    s, e = int(r[isamp] or 0), int(r[iex] or 0)
    tot_s += s
    tot_e += e
    key = line_of.get(off)
    if key is None:
        miss += s
        key = ("?", 0)
    per[key][0] += s
    per[key][1] += e
print(f"samples {tot_s}, instructions {tot_e}, unattributed samples {miss}")
for (f, l), (s, e) in sorted(per.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * s / tot_s:5.1f}% samples {100 * e / max(tot_e, 1):5.1f}% inst  {f}:{l}")
