"""Setup breakdown at a given size: mesh generation, then
build_crust_model with TSGPU_SETUP_PROFILE=1 (per-stage marks on stderr).
args: cells (default 140,210,70 = configs[2])."""
import os, sys, time
os.environ["TSGPU_SETUP_PROFILE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_08679_b200 as ts

cells = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "140,210,70").split(","))
ext = tuple(c * 2800.0 for c in cells)
t = time.perf_counter()
m = ts.generate_box_mesh(ext, cells, (ext[2] / 3, 2 * ext[2] / 3))
tg = time.perf_counter() - t
mats = [ts.material_from_wavespeeds(*x) for x in ((1600, 400, 1850), (3500, 1900, 2400), (5800, 3000, 2700))]
t = time.perf_counter()
model = ts.build_crust_model(m, mats, ts.SolverConfig(batch_size=16))
tb = time.perf_counter() - t
print(f"cells={cells} nodes={m.node_count()} elems={m.element_count()} generate_s={tg:.3f} build_crust_model_s={tb:.3f}",
      flush=True)
