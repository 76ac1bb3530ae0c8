"""Summarise gpurun_out/ab2.log (tools/gpu/ab2.sh): median b2b / clean-flushed us per arm."""
import json
import sys
from collections import defaultdict

import numpy as np

d = defaultdict(list)
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab2.log"):
    arm, _, js = line.strip().partition(" ")
    js = js.strip()
    if not js.startswith("{"):
        continue
    r = json.loads(js)
    d[(r["cfg"], r["strategy"], arm)].append((r["b2b_us"], r["clean_flushed_us"]))
keys = sorted({(c, s) for c, s, _ in d})
for c, s in keys:
    out = []
    for arm in ("base", "new"):
        v = np.array(d.get((c, s, arm), [(np.nan, np.nan)]))
        out.append(f"{arm} b2b {np.median(v[:, 0]):6.2f} flushed {np.median(v[:, 1]):6.2f}")
    b, n = np.median(np.array(d[(c, s, 'base')])[:, 0]), np.median(np.array(d[(c, s, 'new')])[:, 0])
    print(f"cfg{c} {s:8s} " + " | ".join(out) + f" | new/base {n / b:.3f}")
