"""A few level-2 products (ts_levels_apply 3) on the configs[2]-size box (for ncu captures)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
cells = (140, 210, 70)
ext = tuple(c * 2800.0 for c in cells)
mesh = ts.generate_box_mesh(ext, cells, (0.4 * ext[2], 0.75 * ext[2]))
table = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0), (6800.0, 3900.0, 2900.0)]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lv = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in table], ts.SolverConfig(batch_size=B)).levels
u = torch.rand(3 * lv.n2, B, device="cuda", dtype=torch.float32)
f = torch.empty_like(u)
for _ in range(4):
    lv.apply(3, u, f)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    lv.apply(3, u, f)
b.record(); b.synchronize()
print("level-2 product ms", a.elapsed_time(b) / 20)
