"""Benchmark: tangent vmult GDoF/s (fp64) of the matrix-free Neo-Hookean
operator on B200, plus the GMG-CG Newton-iteration time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one MatrixFreeTangent.apply (tensor4 cache, the paper's
"Algorithm 3") on BASELINE config 2 (3D 32^3 Q2, 823,875 DoFs, seeded
synthetic inputs).  L2 is flushed (256 MiB write) before every
timed step; each step is bracketed by CUDA events on the launching stream.
Extra keys report the other caching variants, config 3 (16^3 Q4) and one
Newton iteration of config 4.  Under torchrun every rank runs an independent
replica (weak scaling, no data-path collective), timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tangent vmult GDoF/s (fp64) + GMG-CG Newton-step time at 1/2/4/8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _time_apply(op, x, y, steps, warmup, flush):
    """Per step: flush L2, init y (mask copy), apply kernel; events around each."""
    import torch

    from paper_1904_13131_b200 import _lib
    from paper_1904_13131_b200 import device as dv

    L = _lib.lib()
    n = x.numel()
    mask = op.problem.mask_ptr()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for _ in range(warmup):
        flush.zero_()
        op.apply_into(x, y)
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()
        ev[k][0].record()
        _lib.check(L.hf_fill_masked(n, dv.ptr(y), dv.ptr(x), mask, 0.0, dv.stream()))
        ev[k][1].record()
        op.apply_raw(x, y)
        ev[k][2].record()
    torch.cuda.synchronize()
    step_ms = [ev[k][0].elapsed_time(ev[k][2]) for k in range(steps)]
    kern_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(steps)]
    return float(np.mean(step_ms)), float(np.mean(kern_ms)), 2 * steps


def _e2e(op, x_np, steps, warmup):
    """Public API with pinned host buffers: H2D + apply + D2H inside the timed region."""
    import torch

    xh = torch.from_numpy(x_np.copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    for _ in range(warmup):
        op.apply(xh, out=yh)
    torch.cuda.synchronize()
    t = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(xh, out=yh)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return float(np.mean(t)), xh.numel() * 8, yh.numel() * 8


def cpu_baseline(cfg_id=2, strategy="tensor4", budget_s=20.0, threads=1):
    """Oracle (numpy port of the reference) on a bounded sample: cache build +
    as many applies as fit in the budget (at least one)."""
    from threadpoolctl import threadpool_limits

    from oracle import hf_oracle as O
    from paper_1904_13131_b200.workloads import CONFIGS, MATERIAL, clamp_weighted_sine, AMP_VMULT
    from paper_1904_13131_b200.mesh import build_benchmark_mesh
    from paper_1904_13131_b200.fespace import build_dof_map, face_dofs

    cfg = CONFIGS[cfg_id]
    rng = np.random.default_rng(0)
    centres = rng.random((cfg["n_inc"], cfg["dim"]))
    phases = 2.0 * np.pi * rng.random((cfg["dim"], cfg["dim"]))
    d, m, p = cfg["dim"], cfg["m"], cfg["degree"]
    mesh = build_benchmark_mesh(d, m, [(c, cfg["radius"]) for c in centres], side=1.0)
    inc = mesh.material_id == 1
    mu = np.where(inc, MATERIAL.inclusion.mu, MATERIAL.matrix.mu)
    lam = np.where(inc, MATERIAL.inclusion.lam, MATERIAL.matrix.lam)
    dm = build_dof_map(mesh, p, d)
    mask = np.zeros(dm.n_dofs, dtype=bool)
    mask[face_dofs(dm, cfg["clamp_axis"], 0)] = True
    ubar = clamp_weighted_sine(d, m, p, phases, AMP_VMULT, cfg["clamp_axis"])
    x = rng.standard_normal(dm.n_dofs)
    with threadpool_limits(threads):
        prob = O.OProblem(d, p, mesh.cells, mesh.vertices, mu, lam, mask)
        prob.geometry()
        op = O.Tangent(prob, ubar, strategy)
        t0 = time.perf_counter()
        n = 0
        while True:
            op.apply(x)
            n += 1
            if time.perf_counter() - t0 > budget_s / 2 or n >= 10:
                break
        dt = (time.perf_counter() - t0) / n
    return dm.n_dofs / dt / 1e9, dt, n, dm.n_dofs


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for _ in range(max(args.steps, 1)):
        v, dt, n, ndofs = cpu_baseline(2, "tensor4", budget_s=6.0, threads=threads)
        vals.append(v)
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": v, "unit": "GDoF/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ndofs / v / 1e6, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 3D 32^3 Q2 tensor4 tangent vmult (823,875 DoFs)", "strategy": "tensor4"},
            "cpu_baseline": {"value": v, "unit": "GDoF/s", "cores": threads, "kind": "port",
                             "sample": f"oracle/hf_oracle.py (numpy port of the reference) apply, "
                                       f"{n} applies after a cache build per step"},
            "e2e": {"value": v, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import algorithmic_bytes, make_workload, meter_flops

    hbm, peak_kind = _peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    wl = make_workload(2, seed=rank)
    p = wl.fine
    x = torch.from_numpy(wl.x).cuda()
    y = torch.empty_like(x)
    nqp = p.mesh.n_elements * p.n_qpoints_per_cell
    variants = {}
    head = None
    for s in ("tensor4", "tensor2", "scalar"):
        op = MatrixFreeTangent(p, wl.ubar, s)
        if s == "tensor4":
            if ws > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            with Clocks(torch.cuda.current_device()) as clk:
                step_ms, kern_ms, launches = _time_apply(op, x, y, args.steps, args.warmup, flush)
            torch.cuda.synchronize()
            if ws > 1:
                t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device="cuda")
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                step_ms, kern_ms = t.tolist()
            head = (op, step_ms, kern_ms, launches, clk.summary())
        else:
            sm, km, _ = _time_apply(op, x, y, max(args.steps // 2, 3), 3, flush)
            ab = algorithmic_bytes(s, 3, p.n_dofs, nqp)
            variants[s] = {"GDoF_s": p.n_dofs / sm / 1e6, "kernel_ms": km, "step_ms": sm,
                           "achieved_GBs": ab / km / 1e6, "frac_hbm": ab / km / 1e6 / hbm,
                           "meter_GFLOP_s": meter_flops(3, 2, p.mesh.n_elements, s) / km / 1e6}
        del op
    op, step_ms, kern_ms, launches, clocks = head
    ab = algorithmic_bytes("tensor4", 3, p.n_dofs, nqp)
    variants["tensor4"] = {"GDoF_s": p.n_dofs / step_ms / 1e6, "kernel_ms": kern_ms, "step_ms": step_ms,
                           "achieved_GBs": ab / kern_ms / 1e6, "frac_hbm": ab / kern_ms / 1e6 / hbm,
                           "meter_GFLOP_s": meter_flops(3, 2, p.mesh.n_elements, "tensor4") / kern_ms / 1e6}
    e2e_ms, h2d, d2h = _e2e(op, wl.x, max(args.steps // 2, 3), 2)
    value = ws * p.n_dofs / step_ms / 1e6  # GDoF/s over all ranks
    extra = {}
    if not args.no_extra and rank == 0:
        extra = _extras(args, hbm)
    line = {"metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 3D 32^3 Q2 tensor4 tangent vmult (823,875 DoFs)", "strategy": "tensor4",
                       "l2": "256 MiB flush before every timed step", "parallelism": f"replicas x{ws}"},
            "roofline": {"bound": "hbm", "achieved": ab / kern_ms / 1e6, "peak": hbm, "unit": "GB/s",
                         "frac": ab / kern_ms / 1e6 / hbm, "traffic": None, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": ab, "kernel": "hf::k_apply_line<3,3,TENSOR4>"},
            "e2e": {"value": ws * p.n_dofs / e2e_ms / 1e6, "unit": "GDoF/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "clocks": clocks, "variants": variants}
    line.update(extra)
    if rank == 0 and ws == 1 and not args.no_cpu:
        v, dt, n, _ = cpu_baseline(2, "tensor4", budget_s=20.0, threads=1)
        line["cpu_baseline"] = {"value": v, "unit": "GDoF/s", "cores": 1, "kind": "port",
                                "sample": f"oracle numpy port, cfg2 tensor4 apply x{n} (1 BLAS thread)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _extras(args, hbm):
    """Config 3 (16^3 Q4) vmult and one config-4 Newton iteration."""
    import torch

    from paper_1904_13131_b200 import MatrixFreeTangent
    from paper_1904_13131_b200.workloads import algorithmic_bytes, make_workload

    out = {}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    wl = make_workload(3, seed=0)
    p = wl.fine
    x = torch.from_numpy(wl.x).cuda()
    y = torch.empty_like(x)
    nqp = p.mesh.n_elements * p.n_qpoints_per_cell
    c3 = {}
    for s in ("tensor4", "tensor2", "scalar"):
        op = MatrixFreeTangent(p, wl.ubar, s)
        sm, km, _ = _time_apply(op, x, y, 10, 3, flush)
        ab = algorithmic_bytes(s, 3, p.n_dofs, nqp)
        c3[s] = {"GDoF_s": p.n_dofs / sm / 1e6, "kernel_ms": km, "achieved_GBs": ab / km / 1e6,
                 "frac_hbm": ab / km / 1e6 / hbm}
        del op
    out["cfg3_q4"] = c3
    if not args.no_newton:
        out["newton"] = _newton_iteration()
    return out


def _newton_iteration():
    """Time the first Newton iteration of load step 1 of config 4 (64^3 Q2,
    levels 4..64, prescribed top displacement): tangent + GMG build, CG to
    1e-6, residual."""
    import torch

    from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, build_transfers, cg, compute_residual
    from paper_1904_13131_b200.fespace import node_coordinates
    from paper_1904_13131_b200.workloads import make_workload

    wl = make_workload(4, seed=0, levels=True, with_x=False)
    probs = wl.problems
    fine = probs[-1]
    d = 3
    X = node_coordinates(fine.mesh, fine.dofmap)
    u = torch.zeros(fine.n_dofs, dtype=torch.float64, device="cuda")
    u.view(-1, d)[:, 2] += (-0.05 / 5) * torch.from_numpy(X[:, 2]).cuda()
    transfers = build_transfers(probs)
    res = compute_residual(fine, u)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = MatrixFreeTangent(fine, u, "tensor4")
    gmg = build_gmg(probs, u, "tensor4", seed=0, transfers=transfers, keep_constrained=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    du, rep = cg(op, -res, rel_tol=1e-6, preconditioner=gmg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    u += du
    res = compute_residual(fine, u)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return {"workload": "cfg4 64^3 Q2 levels 4..64, load step 1, iteration 1", "n_dofs": fine.n_dofs,
            "newton_iteration_s": t3 - t0, "setup_s": t1 - t0, "cg_s": t2 - t1, "cg_iterations": rep.iterations,
            "s_per_cg_iteration": (t2 - t1) / max(rep.iterations, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
