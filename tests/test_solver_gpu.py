"""GPU parity of the full solve path: setup (build_solver_levels), the
multigrid-preconditioned flexible outer CG (solve) and the PCGE baseline
(solve_pcge) against the reference on the same meshes and loads.

North-star bars: per-case displacement within 1e-6 relative L2 of the
reference, CG iteration counts within +-2 %. Re-states test_solver.cpp:137-266.
"""
import numpy as np
import pytest
from conftest import STIFF, TWO_LAYER, lame

import paper_1710_08679_b200 as ts
from oracle import SolverConfig as OCfg

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def mats(table):
    return [ts.material_from_wavespeeds(*t) for t in table]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def smooth_batch(coords, extents, mask, batch, seed, orc):
    """acceptance_main.cpp:82-102 smooth fields with per-column amplitude / ky."""
    r = orc.rng_sym(seed, 2 * batch)
    u = np.zeros((coords.shape[0], 3, batch))
    x, y, z = coords[:, 0], coords[:, 1], coords[:, 2]
    sz = np.sin(0.5 * np.pi * z / extents[2])
    for b in range(batch):
        amp = 0.05 * (1.0 + 0.2 * r[2 * b])
        ky = 1.0 + (0.0 if (r[2 * b + 1] + 1) / 2 < 0.5 else 1.0)
        u[:, 0, b] = amp * np.sin(np.pi * x / extents[0]) * np.cos(ky * np.pi * y / extents[1]) * sz
        u[:, 1, b] = amp * np.cos(np.pi * x / extents[0]) * np.sin(ky * np.pi * y / extents[1]) * sz
        u[:, 2, b] = amp * np.cos(np.pi * x / extents[0]) * np.cos(ky * np.pi * y / extents[1]) * sz
    u = u.reshape(-1, batch)
    u[mask == 1] = 0.0
    return u


CASES = [
    # (extents, divisions, interfaces, table, batch)
    ((400.0, 400.0, 200.0), (4, 4, 4), (100.0,), TWO_LAYER, 2),
    ((16000.0, 16000.0, 10000.0), (8, 8, 5), (7000.0,), TWO_LAYER, 4),
    ((100.0, 100.0, 100.0), (3, 3, 3), (), STIFF, 3),
]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: "x".join(map(str, c[1])))
def problem(request, checker):
    ext, div, ifs, table, batch = request.param
    mesh = ts.generate_box_mesh(ext, div, ifs)
    om = checker.box_mesh(ext, div, ifs, 1)
    lam, mu = lame(table)
    cfg = ts.SolverConfig(batch_size=batch)
    model = ts.build_crust_model(mesh, mats(table), cfg)
    olv = checker.levels(om, lam, mu, OCfg.default(batch_size=batch))
    ustar = smooth_batch(om.coords, ext, om.dirichlet_mask(), batch, 31, checker)
    f = olv.outer_apply(ustar)
    return dict(mesh=mesh, om=om, model=model, olv=olv, cfg=cfg, ustar=ustar, f=f, batch=batch)


def test_setup_matches_reference(problem):
    """aggregation (sequential greedy), level-2 Galerkin operator, coarse mask, M2."""
    got = problem["model"].levels.export()
    want = problem["olv"].export()
    assert problem["model"].levels.n2 == problem["olv"].n2
    assert np.array_equal(got["agg"], want["agg"])
    assert np.array_equal(got["row_ptr2"], want["row_ptr2"])
    assert np.array_equal(got["col_idx2"], want["col_idx2"])
    assert np.array_equal(got["blocks2"], want["blocks2"])
    assert np.array_equal(got["mask2"], want["mask2"])
    assert np.array_equal(got["m2"], want["m2"])


def test_solve_matches_reference(problem):
    lv, cfg, f = problem["model"].levels, problem["cfg"], problem["f"]
    u, rep = ts.solve(lv, f, np.zeros_like(f), cfg)
    uo, ro = problem["olv"].solve(f, history=256)
    assert rep.converged and rep.method == "amg" and rep.inner_precision == "float32"
    assert rep.max_final_residual() <= 1e-8
    for b in range(problem["batch"]):
        assert rel(u[:, b], uo[:, b]) <= 1e-6
    assert abs(rep.outer_iterations - ro["outer_iterations"]) <= max(1, round(0.02 * ro["outer_iterations"]))
    for lvl in range(3):
        want = ro["inner_iterations"][lvl]
        assert abs(rep.inner_iterations[lvl] - want) <= max(2, 0.02 * want), (lvl, rep.inner_iterations, want)
    assert len(rep.residual_history) == rep.outer_iterations


def test_manufactured_solution(problem):
    """test_solver.cpp:137-181: u* recovered to 1e-7, all levels active, warm start exits at once."""
    lv, cfg, f, ustar = problem["model"].levels, problem["cfg"], problem["f"], problem["ustar"]
    u, rep = ts.solve(lv, f, np.zeros_like(f), cfg)
    assert rel(u, ustar) < 1e-7
    assert min(rep.inner_iterations) > 0
    u2, rep2 = ts.solve(lv, f, u, cfg)
    assert rep2.outer_iterations == 0


def test_device_entry_matches_host_entry(problem):
    import torch
    lv, cfg, f = problem["model"].levels, problem["cfg"], problem["f"]
    uh, rh = ts.solve(lv, f, np.zeros_like(f), cfg)
    fd = torch.from_numpy(f).cuda()
    ud, rd = ts.solve(lv, fd, torch.zeros_like(fd), cfg)
    assert rh.outer_iterations == rd.outer_iterations
    assert rel(ud.cpu().numpy(), uh) < 1e-12


def test_pcge_matches_reference(problem):
    """solve_pcge: test_solver.cpp:203-226 (agrees with AMG, needs more iterations)."""
    lv, f = problem["model"].levels, problem["f"]
    u, rep = ts.solve_pcge(lv.outer, f, np.zeros_like(f), 1e-8, 100000)
    uo, ro = problem["olv"].solve_pcge(f)
    assert rep.method == "pcge" and rep.inner_precision == "float64" and rep.converged
    assert rel(u, uo) <= 1e-6
    assert abs(rep.outer_iterations - ro["outer_iterations"]) <= max(1, round(0.02 * ro["outer_iterations"]))
    ua, ra = ts.solve(lv, f, np.zeros_like(f), problem["cfg"])
    assert rel(u, ua) < 1e-6
    assert rep.outer_iterations >= ra.outer_iterations


def test_identical_columns_stay_identical():
    """test_solver.cpp:183-201."""
    mesh = ts.generate_box_mesh((100.0, 100.0, 100.0), (2, 2, 2))
    cfg = ts.SolverConfig(batch_size=16)
    model = ts.build_crust_model(mesh, mats(STIFF), cfg)
    rng = np.random.default_rng(67)
    col = rng.uniform(-1, 1, 3 * mesh.node_count())
    col[model.mask == 1] = 0
    f = np.repeat(col[:, None], 16, axis=1)
    u, rep = ts.solve(model.levels, f, np.zeros_like(f), cfg)
    assert rep.converged
    for b in range(1, 16):
        assert np.array_equal(u[:, b], u[:, 0])


def test_zero_rhs():
    """test_solver.cpp:228-244."""
    mesh = ts.generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 1))
    model = ts.build_crust_model(mesh, mats(STIFF), ts.SolverConfig())
    f = np.zeros((3 * mesh.node_count(), 2))
    u, rep = ts.solve_pcge(model.levels.outer, f[:, :1], f[:, :1], 1e-8, 100)
    assert rep.outer_iterations == 0 and not u.any()
    with pytest.raises(ts.ValidationError):
        ts.solve(model.levels, f, f, ts.SolverConfig())


def test_convergence_error_carries_report():
    """test_solver.cpp:246-266."""
    ext = (400.0, 400.0, 200.0)
    mesh = ts.generate_box_mesh(ext, (3, 3, 2), (100.0,))
    cfg = ts.SolverConfig(batch_size=1, outer_max_iter=1)
    model = ts.build_crust_model(mesh, mats(TWO_LAYER), cfg)
    rng = np.random.default_rng(5)
    us = rng.uniform(-0.05, 0.05, (3 * mesh.node_count(), 1))
    us[model.mask == 1] = 0
    f = model.levels.outer.apply(us)
    with pytest.raises(ts.ConvergenceError) as ei:
        ts.solve(model.levels, f, np.zeros_like(f), cfg)
    rep = ei.value.report
    assert rep.outer_iterations == 1 and not rep.converged and len(rep.final_rel_residual) == 1


@pytest.mark.parametrize("which", [0, 1, 2])
@pytest.mark.parametrize("batch", [1, 3, 8, 16])
def test_level_operators_match_reference(checker, which, batch):
    """The operators the solve applies (ts_levels_apply) against the reference's
    EbeOperator<double> order 2 (outer), <float> order 2 (level 0) and <float>
    order 1 (level 1 — assembled K1 on the device) on the same inputs."""
    import torch
    ext, div, ifs = (16000.0, 20000.0, 10000.0), (6, 7, 4), (7000.0,)
    mesh = ts.generate_box_mesh(ext, div, ifs)
    om = checker.box_mesh(ext, div, ifs, 1)
    lam, mu = lame(TWO_LAYER)
    lv = ts.build_crust_model(mesh, mats(TWO_LAYER), ts.SolverConfig(batch_size=batch)).levels
    order, prec = [(2, 64), (2, 32), (1, 32)][which]
    nn = mesh.vertex_count if order == 1 else mesh.node_count()
    mask = mesh.dirichlet_mask()[: 3 * nn]
    dt = np.float64 if prec == 64 else np.float32
    u = checker.rng_sym(40 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(dt)
    want = checker.ebe_apply(om, order, lam, mu, mask, prec, u)
    got = lv.apply(which, torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got.astype(np.float64), want.astype(np.float64)) <= (1e-12 if prec == 64 else 1e-5)
    assert np.array_equal(got[mask == 1], u[mask == 1])


_STAGE_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/oracle"); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np, torch
import paper_1710_08679_b200 as ts
from oracle import Oracle
from conftest import TWO_LAYER, lame
chk = Oracle("port")
ext, div, ifs = (16000.0, 20000.0, 10000.0), (6, 7, 4), (7000.0,)
mesh = ts.generate_box_mesh(ext, div, ifs)
om = chk.box_mesh(ext, div, ifs, 1)
lam, mu = lame(TWO_LAYER)
worst = 0.0
for batch in (8, 16):
    lv = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in TWO_LAYER],
                              ts.SolverConfig(batch_size=batch)).levels
    nn = mesh.vertex_count
    mask = mesh.dirichlet_mask()[: 3 * nn]
    u = chk.rng_sym(60 + batch, 3 * nn * batch).reshape(3 * nn, batch).astype(np.float32)
    want = chk.ebe_apply(om, 1, lam, mu, mask, 32, u)
    got = lv.apply(2, torch.from_numpy(u).cuda()).cpu().numpy().astype(np.float64)
    worst = max(worst, float(np.linalg.norm(got - want) / np.linalg.norm(want)) / 1e-5)
print(worst)
"""


def test_staged_level1_global_path_matches_reference():
    """TSGPU_STAGE_FORCE_GLOBAL (read once per process, so in a child process): every warp of
    the staged level-1 product takes its unstaged path (the one a warp whose block range
    exceeds the staging capacity takes) and still gives the reference's tet4 product."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSGPU_STAGE_FORCE_GLOBAL="1")
    out = subprocess.run([sys.executable, "-c", _STAGE_SCRIPT, root], capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1.0


_FALLBACK_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
import paper_1710_08679_b200 as ts
from conftest import TWO_LAYER
mesh = ts.generate_box_mesh((24000.0, 28000.0, 12000.0), (8, 9, 5), (7000.0,))
cfg = ts.SolverConfig(batch_size=8)
model = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in TWO_LAYER], cfg)
rng = np.random.default_rng(9)
us = rng.uniform(-0.05, 0.05, (3 * mesh.node_count(), 8))
us[model.mask == 1] = 0
f = model.levels.outer.apply(us)
u, rep = ts.solve(model.levels, f, np.zeros_like(f), cfg)
print(json.dumps({"inner": list(rep.inner_iterations), "outer": rep.outer_iterations,
                  "err": float(np.linalg.norm(u - us) / np.linalg.norm(us))}))
"""


def test_fused_gamma_fallback_matches_separate_pass():
    """The level-0 fused (p, Ap) path's fallback (need_full: skip the update, rerun gamma with the full dot
    pass), forced on every iteration by TSGPU_TEST_FUSED_FALLBACK in a child process, gives the same solve as
    the separate gamma pass (TSGPU_EBE_FUSED_DOTS=0): same iteration counts, same solution."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for name, extra in (("separate", {"TSGPU_EBE_FUSED_DOTS": "0"}), ("fallback", {"TSGPU_TEST_FUSED_FALLBACK": "1"}),
                        ("fused", {})):
        env = dict(os.environ, **extra)
        out = subprocess.run([sys.executable, "-c", _FALLBACK_SCRIPT, root], capture_output=True, text=True, env=env,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        runs[name] = json.loads(out.stdout.strip().splitlines()[-1])
    assert runs["fallback"]["inner"] == runs["separate"]["inner"]
    assert runs["fallback"]["outer"] == runs["separate"]["outer"]
    for r in runs.values():
        assert r["err"] < 1e-6
    a, b = runs["fused"]["inner"], runs["separate"]["inner"]
    assert all(abs(x - y) <= max(2, 0.02 * y) for x, y in zip(a, b))
