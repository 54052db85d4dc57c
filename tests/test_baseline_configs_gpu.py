"""The BASELINE.json configs themselves under reference parity (B200).

* configs[0] (8^3 cells, 14,739 DOF, r = 4 — the one config the CPU reference
  solves in full): solve() and solve_pcge() against the reference's own, u
  within 1e-6 relative L2 per case, outer and per-level inner iteration
  counts within +-2 % (north_star bars).
* configs[1] (82 x 123 x 41 cells, 10.1M DOF): the headline matvec against the
  reference's own EbeOperator<T>::apply at r = 1/4/8/16 in both tiers, 1e-5
  (fp32) / 1e-12 (fp64) relative L2, constrained rows exact.
* configs[2] (140 x 210 x 70 cells, 50M DOF): the first outer iteration of
  solve() capped at outer_max_iter = 1 against the committed reference run
  (tests/golden/config2_outer1_reference.json, made by
  tests/golden/make_config2_capped.py): same loads, per-level inner counts
  within +-2 %, residual after the iteration within 1e-4.
"""
import json
import os

import numpy as np
import pytest
from config_specs import CONFIG0, CONFIG1, CONFIG2, lame, smooth_batch

import paper_1710_08679_b200 as ts
from oracle import SolverConfig as OCfg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def within(got, want, frac=0.02, floor=1):
    return abs(got - want) <= max(floor, round(frac * want))


# ---------------------------------------------------------------- configs[0]
@pytest.fixture(scope="module")
def config0(checker):
    c = CONFIG0
    mesh = ts.generate_box_mesh(c["extents"], c["cells"], c["interfaces"])
    om = checker.box_mesh(c["extents"], c["cells"], c["interfaces"], 1)
    assert 3 * om.n_nodes == 14739
    lam, mu = lame(c["table"])
    cfg = ts.SolverConfig(batch_size=c["batch"])
    model = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in c["table"]], cfg)
    olv = checker.levels(om, lam, mu, OCfg.default(batch_size=c["batch"]), workers=checker_workers(checker))
    us = smooth_batch(checker, om.coords, c["extents"], om.dirichlet_mask(), c["batch"])
    f = olv.outer_apply(us)
    return dict(model=model, olv=olv, cfg=cfg, f=f, us=us)


def checker_workers(checker):
    return checker.hw_threads() if checker.kind == "reference" else 1


def test_config0_solve_matches_reference(config0):
    lv, cfg, f = config0["model"].levels, config0["cfg"], config0["f"]
    u, rep = ts.solve(lv, f, np.zeros_like(f), cfg)
    uo, ro = config0["olv"].solve(f)
    assert rep.converged and ro["converged"]
    for b in range(f.shape[1]):
        assert rel(u[:, b], uo[:, b]) <= 1e-6, b
    assert within(rep.outer_iterations, ro["outer_iterations"])
    for lvl in range(3):
        assert within(rep.inner_iterations[lvl], ro["inner_iterations"][lvl], floor=2), (
            lvl, list(rep.inner_iterations), ro["inner_iterations"])
    assert rel(u, config0["us"]) < 1e-7  # the manufactured solution itself


def test_config0_pcge_matches_reference(config0):
    lv, f = config0["model"].levels, config0["f"]
    u, rep = ts.solve_pcge(lv.outer, f, np.zeros_like(f), 1e-8, 100000)
    uo, ro = config0["olv"].solve_pcge(f)
    assert rep.converged and ro["converged"]
    for b in range(f.shape[1]):
        assert rel(u[:, b], uo[:, b]) <= 1e-6, b
    assert within(rep.outer_iterations, ro["outer_iterations"])


# ---------------------------------------------------------------- configs[1]
@pytest.fixture(scope="module")
def config1(checker):
    cells = CONFIG1["cells"]
    ext, ifs = CONFIG1["extents"](cells), CONFIG1["interfaces"](cells)
    mesh = ts.generate_box_mesh(ext, cells, ifs)
    om = checker.box_mesh(ext, cells, ifs, 1)
    assert 3 * om.n_nodes == 10147995 and om.n_elems == 2481156
    mats = [ts.material_from_wavespeeds(*t) for t in CONFIG1["table"]]
    mask = mesh.dirichlet_mask()
    ops = {p: ts.EbeOperator(mesh, 2, mats, mask, prec=p) for p in (32, 64)}
    return dict(om=om, ops=ops, mask=mask, lam_mu=lame(CONFIG1["table"]))


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("r", [1, 4, 8, 16])
def test_config1_matvec_matches_reference(checker, config1, prec, r):
    """The headline workload against the reference's EbeOperator<T>::apply
    (colored std::thread path on all host cores when the reference is the checker)."""
    om, mask = config1["om"], config1["mask"]
    lam, mu = config1["lam_mu"]
    dt = np.float32 if prec == 32 else np.float64
    n = 3 * om.n_nodes
    u = checker.rng_sym(12 if prec == 32 else 11, n * r).reshape(n, r).astype(dt)  # acceptance_main.cpp:132-133 seeds
    want = checker.ebe_apply(om, 2, lam, mu, mask, prec, u, workers=checker_workers(checker))
    got = config1["ops"][prec].apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got, want) <= (1e-5 if prec == 32 else 1e-12)
    assert np.array_equal(got[mask == 1], u[mask == 1])


# ---------------------------------------------------------------- configs[2]
def test_config2_first_outer_iteration():
    """First outer iteration of the 50M-DOF solve against the reference's own capped
    solve (outer_max_iter = 1 -> ConvergenceError carrying the report)."""
    with open(os.path.join(HERE, "golden", "config2_outer1_reference.json")) as fh:
        ref = json.load(fh)
    from oracle import Oracle
    cells = tuple(ref["cells"])
    assert cells == CONFIG2["cells"]
    ext, ifs = CONFIG2["extents"](cells), CONFIG2["interfaces"](cells)
    mesh = ts.generate_box_mesh(ext, cells, ifs)
    batch = ref["batch"]
    cfg = ts.SolverConfig(batch_size=batch, outer_max_iter=1)
    model = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in CONFIG2["table"]], cfg)
    coords = np.asarray(mesh.coords).reshape(-1, 3)
    us = smooth_batch(Oracle("port"), coords, ext, model.mask, batch)
    f = model.levels.outer.apply(torch.from_numpy(us).cuda())
    del us
    norms = f.norm(dim=0).cpu().numpy()
    assert rel(norms, ref["f_column_norms"]) <= 1e-12  # the same loads as the reference run
    with pytest.raises(ts.ConvergenceError) as ei:
        ts.solve(model.levels, f, torch.zeros_like(f), cfg)
    rep = ei.value.report
    assert rep.outer_iterations == 1 == ref["outer_iterations"]
    for lvl in range(3):
        assert within(rep.inner_iterations[lvl], ref["inner_iterations"][lvl], floor=2), (
            lvl, list(rep.inner_iterations), ref["inner_iterations"])
    assert rel(rep.final_rel_residual, ref["final_rel_residual"]) <= 1e-4
