"""Time the full multigrid solve (setup + solve) on layered boxes. args: cells(csv) batch [cells batch ...]"""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1710_08679_b200 as ts
args = sys.argv[1:]
for i in range(0, len(args), 2):
    cells = tuple(int(x) for x in args[i].split(","))
    batch = int(args[i + 1])
    ext = tuple(c * 2800.0 for c in cells)
    t0 = time.time()
    mesh = ts.generate_box_mesh(ext, cells, (0.75 * ext[2],))
    mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
    t1 = time.time()
    cfg = ts.SolverConfig(batch_size=batch)
    model = ts.build_crust_model(mesh, mats, cfg)
    torch.cuda.synchronize(); t2 = time.time()
    lv = model.levels
    N = mesh.node_count()
    xyz = torch.from_numpy(np.asarray(mesh.coords).reshape(-1, 3)).cuda()
    g = torch.Generator(device="cuda").manual_seed(31)
    amp = 0.05 * (1 + 0.2 * (torch.rand(batch, device="cuda", dtype=torch.float64, generator=g) * 2 - 1))
    ky = 1.0 + (torch.rand(batch, device="cuda", dtype=torch.float64, generator=g) > 0.5).double()
    X, Y, Z = [xyz[:, k:k + 1] / ext[k] for k in range(3)]
    sz = torch.sin(0.5 * torch.pi * Z)
    us = torch.stack([amp * torch.sin(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz,
                      amp * torch.cos(torch.pi * X) * torch.sin(ky * torch.pi * Y) * sz,
                      amp * torch.cos(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz], 1).reshape(3 * N, batch).contiguous()
    mk = torch.from_numpy(model.mask).cuda().bool()
    us[mk] = 0
    f = lv.outer.apply(us)
    u0 = torch.zeros_like(f)
    torch.cuda.synchronize()
    t3 = time.time()
    u, rep = ts.solve(lv, f, u0, cfg, history=0)
    torch.cuda.synchronize()
    t4 = time.time()
    err = float((u - us).norm() / us.norm())
    print(json.dumps({"cells": cells, "dof": 3 * N, "batch": batch, "mesh_s": round(t1 - t0, 2), "setup_s": round(t2 - t1, 2),
                      "solve_s": round(t4 - t3, 3), "s_per_case": round((t4 - t3) / batch, 4),
                      "outer": rep.outer_iterations, "inner": rep.inner_iterations,
                      "t_inner": [round(x, 3) for x in rep.time_inner_s], "t_outer": round(rep.time_outer_s, 3),
                      "max_res": rep.max_final_residual(), "err_vs_manufactured": err}), flush=True)
    del model, lv, u, f, u0, us
