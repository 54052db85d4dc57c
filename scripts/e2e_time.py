"""Host-buffer apply time (ts_ebe_apply_host, pinned u / f; the e2e path) on the configs[1] box, fp32 r=16."""
import sys, os, time, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1710_08679_b200 as ts
cells = (82, 123, 41); ext = tuple(c * 2800.0 for c in cells)
m = ts.generate_box_mesh(ext, cells, (0.75 * ext[2],), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
op = ts.EbeOperator(m, 2, mats, m.dirichlet_mask(), prec=32)
uh = torch.rand(3 * op.n_nodes(), 16, dtype=torch.float32).pin_memory()
fh = torch.empty_like(uh).pin_memory()
a, b = uh.numpy(), fh.numpy()
for _ in range(3): op.apply(a, b)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): op.apply(a, b)
torch.cuda.synchronize()
print("e2e ms", (time.perf_counter() - t) * 100)
