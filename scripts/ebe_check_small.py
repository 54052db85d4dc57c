"""Small EBE apply for sanitizer runs. args: prec r cells"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
prec, r = int(sys.argv[1]), int(sys.argv[2])
cells = tuple(int(x) for x in sys.argv[3].split(","))
m = ts.generate_box_mesh(tuple(c * 1000.0 for c in cells), cells, (cells[2] * 500.0,), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
op = ts.EbeOperator(m, 2, mats, m.dirichlet_mask(), prec=prec)
u = torch.rand(3 * op.n_nodes(), r, device="cuda", dtype=torch.float32 if prec == 32 else torch.float64)
f = op.apply(u)
torch.cuda.synchronize()
os.environ["TSGPU_EBE_KERNEL"] = "fast"
op2 = ts.EbeOperator(m, 2, mats, m.dirichlet_mask(), prec=prec)
g = op2.apply(u)
print("reldiff", float((f.double() - g.double()).norm() / g.double().norm()))
