"""Multi-rank GPU parity driver for the slab decomposition (run under torchrun).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port P tests/dist_worker.py [--backend gloo|nccl] [--cells 16]

Every rank builds the global single-GPU result itself (small meshes) and its
own slab of the distributed one, then compares: tangent apply (3 strategies),
diagonal, residual, and the GMG-preconditioned CG solve (iteration count and
solution).  Rank 0 prints one JSON line.  With fewer GPUs than ranks the
ranks share cuda:0 and exchange through gloo (host-staged; no kernel waits on
another rank), which is how the tests run on the one-GPU box.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--cells", type=int, default=16)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--newton", action="store_true", help="config-4 prescribed-displacement Newton instead")
    ap.add_argument("--partition", default="slab", choices=["slab", "morton"])
    ap.add_argument("--graph-check", action="store_true", help="captured vs eager distributed V-cycle")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    dist.init_process_group(args.backend)
    from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, cg, compute_residual
    from paper_1904_13131_b200.distributed import TorchComm, build_dist_gmg, dist_cg
    from paper_1904_13131_b200.fespace import ConstraintSet
    from paper_1904_13131_b200.operators import Problem
    from paper_1904_13131_b200.workloads import AMP_SOLVE, MATERIAL, host_workload

    comm = TorchComm()
    if args.newton:
        return newton_main(args, comm)
    if args.graph_check:
        return graph_main(args, comm)
    wl = host_workload(args.config, seed=0, amp=AMP_SOLVE, levels=True, m=args.cells)
    p = wl.cfg["degree"]
    probs = []
    for mesh, mask in zip(wl.meshes, wl.masks):
        pr = Problem(mesh, p, MATERIAL)
        pr.constraints = ConstraintSet.from_dofs(pr.n_dofs, np.flatnonzero(mask))
        probs.append(pr)
    fine = probs[-1]
    ubar = torch.from_numpy(wl.ubar).cuda()
    x = torch.from_numpy(wl.x).cuda()

    gmg_d, dp, op_d = build_dist_gmg(wl.meshes, p, MATERIAL, wl.masks, dp_slice(wl.ubar, comm, wl, p, args.partition),
                                     comm, partition=args.partition)
    sl = dp.slab
    res = {"rank": comm.rank, "size": comm.size, "n_global_dofs": int(fine.n_dofs), "n_local_dofs": int(dp.n_dofs)}

    def rel(a, b):
        return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))

    xl = sl.local(x).contiguous()
    for s in ("scalar", "tensor2", "tensor4"):
        from paper_1904_13131_b200.distributed import DistributedTangent

        yg = MatrixFreeTangent(fine, ubar, s).apply(x)
        yl = DistributedTangent(dp, sl.local(ubar).contiguous(), s).apply(xl)
        res[f"apply_{s}"] = rel(yl, sl.local(yg))
    dg = MatrixFreeTangent(fine, ubar, "tensor4").diagonal()
    res["diagonal"] = rel(op_d.diagonal(), sl.local(dg))
    rg = compute_residual(fine, ubar)
    res["residual"] = rel(dp.residual(sl.local(ubar).contiguous()), sl.local(rg))

    # GMG-CG (config-1 style rtol 1e-8) on b = A x with constrained entries zeroed
    op_g = MatrixFreeTangent(fine, ubar, "tensor4")
    b = op_g.apply(x)
    b[fine.mask_dev] = 0.0
    gmg = build_gmg(probs, ubar, "tensor4", seed=0)
    xs, rep = cg(op_g, b, rel_tol=1e-8, preconditioner=gmg)
    xd, it_d, relres_d, _ = dist_cg(dp, op_d, sl.local(b).contiguous(), rel_tol=1e-8, preconditioner=gmg_d)
    res.update(cg_iterations_single=rep.iterations, cg_iterations_dist=it_d, cg_relres_dist=relres_d,
               cg_solution=rel(xd, sl.local(xs)))
    # worst case over ranks
    keys = [k for k in res if k.startswith(("apply_", "diagonal", "residual", "cg_solution"))]
    t = torch.tensor([res[k] for k in keys] + [float(it_d)], dtype=torch.float64, device="cuda")
    worst = t.clone()
    if comm.size > 1:
        h = worst.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        worst = h
    out = dict(zip(keys, worst[:-1].tolist()))
    out.update(cg_iterations_single=rep.iterations, cg_iterations_dist=int(worst[-1].item()), size=comm.size,
               backend=args.backend, n_global_dofs=res["n_global_dofs"], levels=[m.cells[-1] for m in wl.meshes])
    if comm.rank == 0:
        print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


def newton_main(args, comm):
    """Single-GPU newton_solve_prescribed vs newton_solve_prescribed_dist (config 4 recipe)."""
    from paper_1904_13131_b200 import NewtonSettings, newton_solve_prescribed
    from paper_1904_13131_b200.distributed import DistHierarchy, newton_solve_prescribed_dist
    from paper_1904_13131_b200.fespace import ConstraintSet, build_dof_map, node_coordinates
    from paper_1904_13131_b200.operators import Problem
    from paper_1904_13131_b200.workloads import MATERIAL, host_workload

    wl = host_workload(4, seed=0, levels=True, m=args.cells, with_x=False)
    probs = []
    for mesh, mask in zip(wl.meshes, wl.masks):
        pr = Problem(mesh, 2, MATERIAL)
        pr.constraints = ConstraintSet.from_dofs(pr.n_dofs, np.flatnonzero(mask))
        probs.append(pr)
    settings = NewtonSettings(n_load_steps=2)
    single = newton_solve_prescribed(probs, settings, -0.05)
    h = DistHierarchy(wl.meshes, 2, MATERIAL, wl.masks, comm, partition=args.partition)
    fine = wl.meshes[-1]
    X = node_coordinates(fine, build_dof_map(fine, 2, 3))
    hgt = X[:, 2] / X[:, 2].max()
    sl = h.fine.slab
    hl = torch.from_numpy(np.ascontiguousarray(sl.local(np.repeat(hgt, 3))[::3])).cuda()
    u, recs = newton_solve_prescribed_dist(h, settings, -0.05, hl)
    a = np.array([(r.load_step, r.iteration, r.residual_norm, r.cg_iterations) for r in single.records])
    b = np.array([(r.load_step, r.iteration, r.residual_norm, r.cg_iterations) for r in recs])
    ul = sl.local(single.u)
    out = dict(size=comm.size, newton=True, single=a.tolist(), dist=b.tolist(),
               u_rel=float(torch.linalg.norm(u - ul) / torch.linalg.norm(ul)))
    t = torch.tensor([out["u_rel"]], dtype=torch.float64)
    if comm.size > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["u_rel"] = t.item()
    if comm.rank == 0:
        print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


def graph_main(args, comm):
    """The distributed V-cycle replayed as a CUDA graph (NCCL calls inside) vs the
    same V-cycle run eagerly: identical preconditioned vectors and CG history."""
    from paper_1904_13131_b200.distributed import build_dist_gmg, dist_cg
    from paper_1904_13131_b200.workloads import AMP_SOLVE, MATERIAL, host_workload

    wl = host_workload(args.config, seed=0, amp=AMP_SOLVE, levels=True, m=args.cells)
    p = wl.cfg["degree"]
    u = dp_slice(wl.ubar, comm, wl, p, args.partition)
    gmg, dp, op = build_dist_gmg(wl.meshes, p, MATERIAL, wl.masks, u, comm, partition=args.partition)
    b = torch.from_numpy(np.ascontiguousarray(dp.slab.local(wl.x))).cuda()
    b[dp.mask_dev.bool()] = 0.0
    ze, zg = torch.empty_like(b), torch.empty_like(b)
    gmg._graph = False  # eager
    gmg.apply_into(b, ze)
    _, it_e, _, _ = dist_cg(dp, op, b, rel_tol=1e-8, preconditioner=gmg)
    gmg._graph = None  # capture on the next call
    diffs = []
    for _ in range(3):  # first call captures, later calls replay
        gmg.apply_into(b, zg)
        diffs.append(float(torch.linalg.norm(zg - ze) / torch.linalg.norm(ze)))
    _, it_g, _, _ = dist_cg(dp, op, b, rel_tol=1e-8, preconditioner=gmg)
    out = dict(size=comm.size, backend=args.backend, graph=gmg._graph not in (None, False), diffs=diffs,
               cg_eager=it_e, cg_graph=it_g, error=gmg.graph_error)
    if comm.rank == 0:
        print("DISTRESULT " + json.dumps(out), flush=True)
    dist.destroy_process_group()


def dp_slice(v, comm, wl, p, partition="slab"):
    from paper_1904_13131_b200.distributed import level_parts

    sl = level_parts(wl.cfg["dim"], p, wl.meshes[-1].cells, len(wl.meshes), comm.rank, comm.size,
                     partition=partition)[-1]
    return np.ascontiguousarray(sl.local(v))


if __name__ == "__main__":
    main()
