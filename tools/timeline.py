"""Per-warp timeline of one apply (instrumented build):

    HF_TIMELINE=1 python -m paper_1904_13131_b200.build
    HF_LIB=paper_1904_13131_b200/libhf_tl.so python tools/timeline.py [strategy] [cfg]

Runs a few back-to-back applies, then one more whose per-warp timestamps
(hf_timeline_fetch) are summarised: when warps start and end relative to the
first warp, the mean tile period and its split (gather+evaluation / point
phase / integration+scatter), the first tile's wait, and the end skew."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200._lib import check, lib
from paper_1904_13131_b200.workloads import make_workload

s = sys.argv[1] if len(sys.argv) > 1 else "tensor4"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
WARPS, SLOTS = 148 * 16, 72
wl = make_workload(cfg, seed=0)
op = MatrixFreeTangent(wl.fine, wl.ubar, s)
x = torch.from_numpy(wl.x).cuda()
y = torch.empty_like(x)
buf = np.zeros(WARPS * SLOTS, dtype=np.uint64)
for _ in range(5):
    op.apply_into(x, y)
torch.cuda.synchronize()
check(lib().hf_timeline_fetch(buf.ctypes.data, buf.size, 1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
op.apply_into(x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
check(lib().hf_timeline_fetch(buf.ctypes.data, buf.size, 1))
raw = buf.reshape(WARPS, SLOTS)
t = raw.astype(np.float64)
used = t[:, 0] > 0
smid = raw[used, SLOTS - 5].astype(np.int64) - 1  # the SM of each warp's block (-1: not recorded)
t = t[used]
t[:, SLOTS - 5] = 0
t0 = t[:, 0].min()
t = np.where(t > 0, t - t0, np.nan)
entry, exit_ = t[:, 0], t[:, SLOTS - 1]
per = []  # (start, evaluated, point done, end) per tile
for k in range(16):
    c = t[:, 1 + 4 * k: 5 + 4 * k]
    if c.shape[1] < 4 or np.all(np.isnan(c[:, 0])):
        break
    per.append(c)
per = np.stack(per, axis=1)  # warps, tiles, 4
dur = per[:, :, 3] - per[:, :, 0]
ev = per[:, :, 1] - per[:, :, 0]
pt = per[:, :, 2] - per[:, :, 1]
ig = per[:, :, 3] - per[:, :, 2]
res = {"strategy": s, "cfg": cfg, "event_ms": ms, "warps": int(used.sum()),
       "span_us": float(np.nanmax(exit_)) / 1e3,
       "entry_us": {"max": float(np.nanmax(entry)) / 1e3, "p50": float(np.nanmedian(entry)) / 1e3},
       "first_tile_start_us_p50": float(np.nanmedian(per[:, 0, 0])) / 1e3,
       "prologue_us_p50": {"gather_issued": float(np.nanmedian(t[:, SLOTS - 4])) / 1e3,
                           "tma_issued": float(np.nanmedian(t[:, SLOTS - 3])) / 1e3,
                           "offsets_loaded": float(np.nanmedian(t[:, SLOTS - 2])) / 1e3},
       "exit_us": {"min": float(np.nanmin(exit_)) / 1e3, "p10": float(np.nanpercentile(exit_, 10)) / 1e3,
                   "p50": float(np.nanmedian(exit_)) / 1e3, "max": float(np.nanmax(exit_)) / 1e3},
       "tiles_per_warp": {"min": int(np.min(np.sum(~np.isnan(dur), 1))), "max": int(np.max(np.sum(~np.isnan(dur), 1)))},
       "tile0_us": {"eval": float(np.nanmedian(ev[:, 0])) / 1e3, "point": float(np.nanmedian(pt[:, 0])) / 1e3,
                    "integ": float(np.nanmedian(ig[:, 0])) / 1e3},
       "tile_us_steady": {"total": float(np.nanmedian(dur[:, 1:])) / 1e3, "eval": float(np.nanmedian(ev[:, 1:])) / 1e3,
                          "point": float(np.nanmedian(pt[:, 1:])) / 1e3, "integ": float(np.nanmedian(ig[:, 1:])) / 1e3},
       "busy_frac": float(np.nansum(exit_ - entry) / (len(exit_) * np.nanmax(exit_)))}
print(json.dumps(res))
np.save(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                     f"timeline_{s}_{cfg}.npy"), t)
np.save(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                     f"timeline_{s}_{cfg}_smid.npy"), smid)
