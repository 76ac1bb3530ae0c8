import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from _cases import golden, product_levels, rel
from paper_1904_13131_b200 import MatrixFreeTangent, build_gmg, cg, build_transfers
for name in ["mg_2d_16.npz", "mg_2d_32_cfg1.npz", "mg_3d_8.npz"]:
    g = golden(name); probs = product_levels(g)
    for k in range(3):
        gmg = build_gmg(probs, g["ubar"], str(g["strategy"]), seed=0)
        op = MatrixFreeTangent(probs[-1], g["ubar"], str(g["strategy"]))
        x, rep = cg(op, g["b"], rel_tol=1e-8, preconditioner=gmg)
        print(name, k, rep.iterations, int(g["cg_iterations"]), rel(x, g["cg_solution"]))
