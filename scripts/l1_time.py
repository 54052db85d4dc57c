"""Level-1 assembled SpMV (K1 block CSR) and solve level times, natural vs Morton row order
(TSGPU_L1_ORDER), on the configs[2] box. args: [cells=140,210,70] [batch=16]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1710_08679_b200 as ts
cells = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "140,210,70").split(","))
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ext = tuple(c * 2800.0 for c in cells)
mesh = ts.generate_box_mesh(ext, cells, (0.4 * ext[2], 0.75 * ext[2]))
table = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0), (6800.0, 3900.0, 2900.0)]
mats = [ts.material_from_wavespeeds(*t) for t in table]
V = mesh.vertex_count
out = {}
ref = None
for order in ("natural", "brick"):
    os.environ["TSGPU_L1_ORDER"] = order
    cfg = ts.SolverConfig(batch_size=B)
    lv = ts.build_crust_model(mesh, mats, cfg).levels
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.rand(3 * V, B, device="cuda", dtype=torch.float32, generator=g) * 2 - 1
    f = torch.empty_like(u)
    for _ in range(3):
        lv.apply(2, u, f)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        lv.apply(2, u, f)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    same = None if ref is None else bool(torch.equal(ref, f))
    ref = f.clone()
    # a solve for the level times (manufactured smooth field)
    N = mesh.node_count()
    us = torch.rand(3 * N, B, device="cuda", dtype=torch.float64, generator=g) * 1e-3
    fo = lv.outer.apply(us)
    ud, rep = ts.solve(lv, fo, torch.zeros_like(fo), cfg, history=0)
    t0 = time.perf_counter()
    ud, rep = ts.solve(lv, fo, torch.zeros_like(fo), cfg, history=0)
    torch.cuda.synchronize()
    out[order] = {"l1_spmv_ms": round(ms, 4), "bitwise_equal_to_natural": same, "solve_s": round(time.perf_counter() - t0, 3),
                  "inner": list(rep.inner_iterations), "outer": rep.outer_iterations,
                  "time_inner_s": [round(x, 3) for x in rep.time_inner_s]}
    print(order, json.dumps(out[order]), flush=True)
    del lv
print(json.dumps({"cells": cells, "batch": B, "vertices": V, **out}))
