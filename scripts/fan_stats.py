"""Unit-plan statistics (fans vs pairs) and kernel timing on a box mesh. args: [cells=82,123,41]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1710_08679_b200 as ts
cells = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "82,123,41").split(","))
ext = tuple(c * 2800.0 for c in cells)
m = ts.generate_box_mesh(ext, cells, (0.75 * ext[2],), 1)
mats = [ts.material_from_wavespeeds(1600, 400, 1850), ts.material_from_wavespeeds(5800, 3000, 2700)]
for k in ("fan", "pair"):
    os.environ["TSGPU_EBE_KERNEL"] = k
    op = ts.EbeOperator(m, 2, mats, m.dirichlet_mask(), prec=32)
    print(k, json.dumps(op.unit_stats()), flush=True)
