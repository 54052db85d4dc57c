"""Whole-apply time (init + sweep, CUDA events) of the configs[1] EBE product, fp32 r=16 by default.
args: [r=16] [prec=32] [kernel env] — TSGPU_* variants are taken from the environment."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cells = (82, 123, 41)
ext = tuple(c * 2800.0 for c in cells)
m = ts.generate_box_mesh(ext, cells, (0.75 * ext[2],), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
op = ts.EbeOperator(m, 2, mats, m.dirichlet_mask(), prec=prec)
dt = torch.float32 if prec == 32 else torch.float64
g = torch.Generator(device="cuda").manual_seed(5)
u = torch.rand(3 * op.n_nodes(), r, device="cuda", dtype=dt, generator=g) * 2 - 1
f = torch.empty_like(u)
for _ in range(5):
    op.apply(u, f)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts_ = []
for _ in range(20):
    a.record(); op.apply(u, f); b.record(); b.synchronize(); ts_.append(a.elapsed_time(b))
ts_.sort()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TSGPU_")}, "r": r, "prec": prec,
                  "apply_ms_median": round(ts_[len(ts_) // 2], 4), "apply_ms_min": round(ts_[0], 4),
                  "f_sum": float(f.double().sum()), "f_norm": float(f.double().norm())}))
