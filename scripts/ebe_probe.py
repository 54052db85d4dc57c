"""Quick EBE matvec timing probe (development aid; bench.py is the contract)."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1710_08679_b200 as ts

PEAK = 6547.8
def alg_bytes(E, N, r, s, npe=10):
    return E * (npe * 4 + 14 * s) + 3 * N * (2 * r * s + 1)

t0 = time.time()
cells = tuple(int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (82, 123, 41)))
m = ts.generate_box_mesh((cells[0] * 1e3, cells[1] * 1e3, cells[2] * 1e3), cells, (cells[2] * 500.0,), 1)
print(f"mesh {cells}: N={m.node_count()} E={m.element_count()} gen {time.time()-t0:.1f}s", flush=True)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
mk = m.dirichlet_mask()
res = []
for prec in (32, 64):
    for order in (2, 1):
        t0 = time.time()
        op = ts.EbeOperator(m, order, mats, mk if order == 2 else mk[:3 * m.vertex_count], prec=prec)
        op.set_timing(True)
        nn = op.n_nodes()
        dt = torch.float32 if prec == 32 else torch.float64
        for r in (1, 4, 8, 16):
            u = torch.rand(3 * nn, r, device="cuda", dtype=dt)
            f = torch.empty_like(u)
            for _ in range(3):
                op.apply(u, f)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 10
            ks = []
            e0.record()
            for _ in range(K):
                op.apply(u, f)
                ks.append(op.last_kernel_ms())
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            kms = float(np.mean(ks))
            B = alg_bytes(op.n_elements(), nn, r, prec // 8, 10 if order == 2 else 4)
            d = dict(prec=prec, order=order, r=r, ms=round(ms, 4), kernel_ms=round(kms, 4),
                     GBs=round(B / ms / 1e6, 1), frac=round(B / ms / 1e6 / PEAK, 3), kernel_frac=round(B / kms / 1e6 / PEAK, 3))
            res.append(d)
            print(json.dumps(d), flush=True)
        del op
