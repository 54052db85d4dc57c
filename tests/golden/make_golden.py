"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists and
oracle/_ref/libtsref.so is built):  python tests/golden/make_golden.py
Outputs small .npz files next to this script. The GPU box never needs the
reference: the port oracle is checked against these fixtures there.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import Oracle, SolverConfig  # noqa: E402
from conftest import TWO_LAYER, lame  # noqa: E402

R = Oracle("reference")
lam, mu = lame(TWO_LAYER)

# 1) EBE products, block Jacobi on a 2x2x2 two-layer box
m = R.box_mesh((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1)
mask = m.dirichlet_mask()
out = dict(coords=m.coords, tets10=m.tets10, material_id=m.material_id, vertex_count=m.vertex_count,
           bc_node=m.bc_node, bc_axis=m.bc_axis, lam=lam, mu=mu)
for prec in (32, 64):
    for order in (1, 2):
        nn = m.vertex_count if order == 1 else m.n_nodes
        u = R.rng_sym(11 if prec == 64 else 12, 3 * nn * 4).reshape(3 * nn, 4)
        out[f"u_{prec}_{order}"] = u.astype(np.float32 if prec == 32 else np.float64)
        out[f"f_{prec}_{order}"] = R.ebe_apply(m, order, lam, mu, mask[: 3 * nn], prec, u)
        out[f"bj_{prec}_{order}"] = R.ebe_block_jacobi(m, order, lam, mu, mask[: 3 * nn], prec)
np.savez_compressed(os.path.join(HERE, "ebe_2x2x2.npz"), **out)

# 2) full multigrid solve + PCGE on a 4x4x4 two-layer box (test_solver.cpp:137-181 setup)
m = R.box_mesh((400.0, 400.0, 200.0), (4, 4, 4), (100.0,), 1)
mask = m.dirichlet_mask()
cfg = SolverConfig.default(batch_size=2)
lv = R.levels(m, lam, mu, cfg)
us = R.rng_sym(31, 3 * m.n_nodes * 2).reshape(-1, 2) * 0.05
us[mask == 1] = 0.0
f = lv.outer_apply(us)
u, rep = lv.solve(f, history=200)
up, repp = lv.solve_pcge(f)
ex = lv.export()
np.savez_compressed(os.path.join(HERE, "solve_4x4x4.npz"), f=f, u=u, u_pcge=up,
                    outer=rep["outer_iterations"], inner=np.array(rep["inner_iterations"]),
                    final=rep["final_rel_residual"], history=rep["history"],
                    pcge_outer=repp["outer_iterations"], agg=ex["agg"], n2=lv.n2,
                    blocks2=ex["blocks2"], row_ptr2=ex["row_ptr2"], col_idx2=ex["col_idx2"])
print("golden fixtures written to", HERE)
