"""The configs[3] mesh (405M DOF) on ONE B200: EBE product timing at fp32 r=8 and r=4
(supplementary to bench.py; correctness is tests/test_maxsize_gpu.py). Prints one JSON line.

  python scripts/maxsize_bench.py [--steps 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_08679_b200 as ts  # noqa: E402

EXT = (792e3, 1192e3, 400e3)
DIV = (281, 423, 141)
LAYERS = [(5500.0, 3200.0, 2600.0), (6800.0, 3900.0, 2900.0), (8000.0, 4500.0, 3300.0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    t0 = time.perf_counter()
    mesh = ts.generate_box_mesh(EXT, DIV, (160e3, 300e3))
    t1 = time.perf_counter()
    mats = [ts.material_from_wavespeeds(*m) for m in LAYERS]
    op = ts.EbeOperator(mesh, 2, mats, mesh.dirichlet_mask(), prec=32)
    t2 = time.perf_counter()
    N, E = mesh.node_count(), mesh.element_count()
    out = {"workload": f"configs[3] mesh {list(DIV)} on one B200: {E} tet10, {N} nodes, {3 * N} DOF, fp32",
           "mesh_s": round(t1 - t0, 2), "operator_setup_s": round(t2 - t1, 2),
           "device_mem_gb_after_setup": round(torch.cuda.memory_allocated() / 1e9, 2)}
    op.set_timing(True)
    for r in (8, 4):
        u = torch.empty(3 * N, r, device="cuda").uniform_(-1, 1)
        f = torch.empty_like(u)
        for _ in range(3):
            op.apply(u, f)
        torch.cuda.synchronize()
        ks = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            op.apply(u, f)
            ks.append(op.last_kernel_ms())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        s = 4
        alg = E * (40 + 14 * s) + 3 * N * (2 * r * s + 1)  # DESIGN.md §4 B_tet10
        out[f"fp32_r{r}"] = {"apply_ms": round(ms, 3), "kernel_ms": round(float(np.mean(ks)), 3),
                             "alg_gb": round(alg / 1e9, 3), "apply_gb_s": round(alg / ms / 1e6, 1),
                             "kernel_gb_s": round(alg / float(np.mean(ks)) / 1e6, 1),
                             "vector_gb": round(3 * N * r * 4 / 1e9, 2)}
        if r == 8:  # end to end through the host entry: pinned u in, pinned f out
            uh = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
            uh.copy_(u)
            fh = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
            op.apply(uh.numpy(), fh.numpy())
            t = time.perf_counter()
            for _ in range(3):
                op.apply(uh.numpy(), fh.numpy())
            ms_h = (time.perf_counter() - t) / 3 * 1e3
            out[f"fp32_r{r}"]["e2e"] = {"ms": round(ms_h, 1), "gb_s": round(alg / ms_h / 1e6, 1),
                                        "pcie_bytes": 2 * u.numel() * 4, "entry": "ts_ebe_apply_host"}
            del uh, fh
        del u, f
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
