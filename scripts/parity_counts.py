"""Iteration-count parity at a size the reference solves in minutes: reference solve()
(oracle/_ref, all host cores) vs ours with the assembled and the EBE level-1 operator.
args: cells batch"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch
import paper_1710_08679_b200 as ts
import bench
from oracle import Oracle, SolverConfig as OCfg
cells = tuple(int(x) for x in sys.argv[1].split(","))
B = int(sys.argv[2])
ext = tuple(c * bench.CELL_KM * 1e3 for c in cells)
ifs = (0.4 * ext[2], 0.75 * ext[2])
table = bench.THREE_LAYER
mesh = ts.generate_box_mesh(ext, cells, ifs)
us = bench.manufactured(mesh, ext, mesh.dirichlet_mask(), B, 31, torch).cpu().numpy()
out = {"cells": cells, "dof": 3 * mesh.node_count(), "batch": B}
for l1 in ("assembled", "ebe"):
    os.environ["TSGPU_L1"] = "ebe" if l1 == "ebe" else "bcsr"
    cfg = ts.SolverConfig(batch_size=B)
    model = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in table], cfg)
    f = model.levels.outer.apply(torch.from_numpy(us).cuda()).cpu().numpy()
    t0 = time.time()
    u, rep = ts.solve(model.levels, f, np.zeros_like(f), cfg, history=0)
    out[l1] = {"outer": rep.outer_iterations, "inner": list(rep.inner_iterations), "s": round(time.time() - t0, 3),
               "err": float(np.linalg.norm(u - us) / np.linalg.norm(us))}
    del model
ref = Oracle("reference")
om = ref.box_mesh(ext, cells, ifs, 1)
lam = [rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in table]
mu = [rho * vs * vs for vp, vs, rho in table]
olv = ref.levels(om, lam, mu, OCfg.default(batch_size=B), workers=ref.hw_threads())
fo = olv.outer_apply(us)
t0 = time.time()
uo, ro = olv.solve(fo)
out["reference"] = {"outer": ro["outer_iterations"], "inner": ro["inner_iterations"], "s": round(time.time() - t0, 2),
                    "cores": ref.hw_threads()}
print(json.dumps(out), flush=True)
