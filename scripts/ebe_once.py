"""Run a few EBE applies (for ncu captures). args: prec order r [cells...]"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
prec, order, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cells = tuple(int(x) for x in sys.argv[4:7]) if len(sys.argv) > 6 else (82, 123, 41)
m = ts.generate_box_mesh((cells[0] * 1e3, cells[1] * 1e3, cells[2] * 1e3), cells, (cells[2] * 500.0,), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
mk = m.dirichlet_mask()
op = ts.EbeOperator(m, order, mats, mk if order == 2 else mk[:3 * m.vertex_count], prec=prec)
dt = torch.float32 if prec == 32 else torch.float64
u = torch.rand(3 * op.n_nodes(), r, device="cuda", dtype=dt)
f = torch.empty_like(u)
for _ in range(4):
    op.apply(u, f)
torch.cuda.synchronize()
print("done")
