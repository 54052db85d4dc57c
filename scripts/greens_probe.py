import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench
import paper_1710_08679_b200 as ts
from paper_1710_08679_b200.greens import DIP, STRIKE, FaultedModel, find_plane_fault_faces
cells = (82, 123, 41)
ext, div, ifs = bench.mesh_spec(cells)
h = bench.CELL_KM * 1e3
xm = (cells[0] // 2) * h
mesh = ts.generate_box_mesh(ext, div, ifs)
lo = (xm, 4 * h, 4 * h); hi = (xm, (cells[1] - 4) * h, (cells[2] - 8) * h)
faces = find_plane_fault_faces(mesh, 0, xm, lo, hi)
cfg = ts.SolverConfig(batch_size=16)
t = time.perf_counter()
fm = FaultedModel(mesh, [ts.material_from_wavespeeds(*x) for x in bench.TWO_LAYER], faces, cfg)
print("setup", time.perf_counter() - t)
ny, nz = 6, 4
ys = np.linspace(lo[1] + 0.15 * (hi[1] - lo[1]), hi[1] - 0.15 * (hi[1] - lo[1]), ny)
zs = np.linspace(lo[2] + 0.2 * (hi[2] - lo[2]), hi[2] - 0.2 * (hi[2] - lo[2]), nz)
centers = np.array([[xm, y, z] for y in ys for z in zs for _ in (DIP, STRIKE)])
dirs = np.array([d for _ in ys for _ in zs for d in (DIP, STRIKE)], np.int32)
radii = np.full(len(dirs), 0.6 * (hi[1] - lo[1]) / ny)
gx, gy = np.meshgrid(np.linspace(0.1, 0.9, 10) * ext[0], np.linspace(0.1, 0.9, 10) * ext[1])
pts100 = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, ext[2])], 1); axes100 = (np.arange(100) % 3).astype(np.int32)
pts1 = pts100[:1]; axes1 = axes100[:1]
for label, pts, axes, sampler in (("1pt", pts1, axes1, False), ("100pt", pts100, axes100, False), ("100pt+clk", pts100, axes100, True)):
    for rep in range(2):
        ctx = bench.ClockSampler(0) if sampler else None
        if ctx: ctx.__enter__()
        torch.cuda.synchronize(); t = time.perf_counter()
        bank, calls, outer = fm.greens_bank(centers, dirs, radii, pts, axes, cfg)
        dt = time.perf_counter() - t
        if ctx: ctx.__exit__(None, None, None)
        print("sweep", label, rep, round(dt, 3), calls, outer, flush=True)
