"""Time EBE sweep kernels (TSGPU_EBE_KERNEL variants) on the config-2 box; also checks variant agreement.
args: [variants=pair,fan] [cells=82,123,41]"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
variants = (sys.argv[1] if len(sys.argv) > 1 else "pair,fan").split(",")
cells = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "82,123,41").split(","))
ext = tuple(c * 2800.0 for c in cells)
m = ts.generate_box_mesh(ext, cells, (0.75 * ext[2],), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
mk = m.dirichlet_mask()
res = {}
for order in (2, 1):
    for prec in (32, 64):
        ops = {}
        for v in variants:
            os.environ["TSGPU_EBE_KERNEL"] = v
            ops[v] = ts.EbeOperator(m, order, mats, mk if order == 2 else mk[:3 * m.vertex_count], prec=prec)
            ops[v].set_timing(True)
        N, E = ops[variants[0]].n_nodes(), ops[variants[0]].n_elements()
        s = prec // 8
        npe = 10 if order == 2 else 4
        for r in ((1, 4, 8, 16) if order == 2 else (16,)):
            dt = torch.float32 if prec == 32 else torch.float64
            u = torch.rand(3 * N, r, device="cuda", dtype=dt) * 2 - 1
            outs = {}
            for v, op in ops.items():
                f = torch.empty_like(u)
                for _ in range(3): op.apply(u, f)
                torch.cuda.synchronize()
                ks = []
                for _ in range(10):
                    op.apply(u, f); ks.append(op.last_kernel_ms())
                k = sorted(ks)[len(ks) // 2]
                B = E * (npe * 4 + 14 * s) + 3 * N * (2 * r * s + 1)
                outs[v] = f.double()
                res[f"o{order}_fp{prec}_r{r}_{v}"] = {"kernel_ms": round(k, 4), "GBps": round(B / k / 1e6, 1)}
            if len(outs) > 1:
                a, b = list(outs.values())[:2]
                res[f"o{order}_fp{prec}_r{r}_reldiff"] = float((a - b).norm() / a.norm())
            print(json.dumps({k2: v2 for k2, v2 in res.items() if f"o{order}_fp{prec}_r{r}_" in k2}), flush=True)
