"""GPU parity of the Green's-function sweep against the
reference's own pipeline (find_plane_fault_faces -> build_faulted_model ->
unit_slip_basis -> slip_to_rhs -> compute_greens_bank, fault.hpp / model.hpp /
greens.hpp) on the same faulted layered box: identical fault faces, split
counts and batch plan; right-hand sides within 1e-12; bank within 1e-6
(displacements of 1e-8-converged solves); outer iterations within +-2 %.
Re-states acceptance_main.cpp:390-504 (C8) at test size."""
import numpy as np
import pytest
from conftest import TWO_LAYER, lame

import paper_1710_08679_b200 as ts
from paper_1710_08679_b200.greens import DIP, STRIKE, FaultedModel, find_plane_fault_faces
from oracle import SolverConfig as OCfg

pytestmark = pytest.mark.gpu

EXT, DIV, IFS = (8000.0, 8000.0, 6000.0), (8, 8, 6), (4500.0,)
PLANE = dict(axis=0, coord=4000.0, lo=(4000.0, 2000.0, 1000.0), hi=(4000.0, 6000.0, 5000.0))
CENTERS = np.array([[4000.0, 4000.0, 3000.0], [4000.0, 3000.0, 2500.0], [4000.0, 5000.0, 4000.0],
                    [4000.0, 4000.0, 3000.0], [4000.0, 3500.0, 2000.0]])
DIRS = np.array([DIP, DIP, STRIKE, STRIKE, DIP], np.int32)
RADII = np.array([1500.0, 1000.0, 1200.0, 1500.0, 900.0])
OBS = np.array([[1000.0, 2000.0, 6000.0], [3000.0, 4000.0, 6000.0], [5000.0, 4000.0, 6000.0],
                [6500.0, 1500.0, 6000.0], [4000.0, 7000.0, 6000.0], [2500.0, 2500.0, 5500.0]])
AXES = np.array([0, 1, 2, 0, 2, 1], np.int32)


def mats():
    return [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def setup(reference):
    mesh = ts.generate_box_mesh(EXT, DIV, IFS)
    om = reference.box_mesh(EXT, DIV, IFS, 1)
    faces = find_plane_fault_faces(mesh, PLANE["axis"], PLANE["coord"], PLANE["lo"], PLANE["hi"])
    ref_faces = reference.fault_plane_faces(om, PLANE["axis"], PLANE["coord"], PLANE["lo"], PLANE["hi"])
    return mesh, om, faces, ref_faces


def test_fault_faces_match(setup):
    _, _, faces, ref_faces = setup
    assert np.array_equal(faces, ref_faces)


def test_slip_to_rhs_matches(setup, reference):
    mesh, om, faces, _ = setup
    lam, mu = lame(TWO_LAYER)
    fm = FaultedModel(mesh, mats(), faces, ts.SolverConfig(batch_size=4))
    got = fm.slip_to_rhs(CENTERS, DIRS, RADII)
    want, info = reference.slip_to_rhs(om, lam, mu, faces, CENTERS, DIRS, RADII)
    assert (fm.n_split_nodes, fm.split_mesh_nodes) == tuple(info)
    assert rel(got, want) <= 1e-12
    assert np.linalg.norm(got) > 0


@pytest.mark.parametrize("batch", [2, 4])
def test_greens_bank_matches(setup, reference, batch):
    mesh, om, faces, _ = setup
    lam, mu = lame(TWO_LAYER)
    cfg = ts.SolverConfig(batch_size=batch)
    fm = FaultedModel(mesh, mats(), faces, cfg)
    bank, calls, outer = fm.greens_bank(CENTERS, DIRS, RADII, OBS, AXES, cfg)
    rbank, rcalls, router = reference.greens_bank(om, lam, mu, faces, CENTERS, DIRS, RADII, OBS, AXES,
                                                  OCfg.default(batch_size=batch))
    assert calls == rcalls == -(-len(DIRS) // batch)
    assert abs(outer - router) <= max(1, 0.02 * router)
    assert rel(bank, rbank) <= 1e-6
    assert np.abs(bank).max() > 0


def test_validation_errors(setup):
    mesh, _, faces, _ = setup
    fm = FaultedModel(mesh, mats(), faces)
    with pytest.raises(ts.ValidationError):
        fm.slip_to_rhs([[3000.0, 4000.0, 3000.0]], [DIP], [1000.0])  # center off the fault plane
    with pytest.raises(ts.ValidationError):
        fm.greens_bank(CENTERS[:1], DIRS[:1], RADII[:1], [[1e6, 0.0, 0.0]], [0])  # observation outside
    with pytest.raises(ts.ValidationError):
        find_plane_fault_faces(mesh, 0, 4500.0, (4500.0, 0.0, 0.0), (4500.0, 8000.0, 6000.0))  # not a mesh plane


def test_reconstruct_split_solution(setup, reference):
    """reconstruct_split_solution (fault.hpp:392-411; test_fault.cpp:360-376): the split-mesh
    displacement carries the prescribed jump exactly; on the same base solution it equals the
    reference's reconstruction bit for bit."""
    mesh, om, faces, _ = setup
    lam, mu = lame(TWO_LAYER)
    cfg = ts.SolverConfig(batch_size=4)
    fm = FaultedModel(mesh, mats(), faces, cfg)
    f = fm.slip_to_rhs(CENTERS, DIRS, RADII)
    u, _ = ts.solve(fm.levels, f, np.zeros_like(f), ts.SolverConfig(batch_size=len(DIRS)))
    us = fm.reconstruct_split_solution(CENTERS, DIRS, RADII, u)
    want = reference.reconstruct_split(om, lam, mu, faces, CENTERS, DIRS, RADII, u, fm.split_mesh_nodes)
    assert np.array_equal(us.view(np.uint64), want.view(np.uint64))
    assert np.abs(us).max() > 0


def test_fault_rejections_match_reference(setup, reference):
    """test_fault.cpp:119-143: a fault touching a Dirichlet boundary, and a boundary triangle, are
    rejected — by the reference and by the library (ValidationError)."""
    mesh, om, _, _ = setup
    lam, mu = lame(TWO_LAYER)
    full = find_plane_fault_faces(mesh, 0, 4000.0, (4000.0, 0.0, 0.0), (4000.0, 8000.0, 6000.0))
    t = np.asarray(om.tets10)[:, :4]
    z = np.asarray(om.coords)[:, 2]
    bottom = None
    for tet in t:
        for fv in ((1, 2, 3), (0, 3, 2), (0, 1, 3), (0, 2, 1)):
            tri = tet[list(fv)]
            if (z[tri] == 0.0).all():
                bottom = np.array([tri], np.int32)
                break
        if bottom is not None:
            break
    for faces in (full, bottom):
        with pytest.raises(Exception):
            reference.slip_to_rhs(om, lam, mu, faces, CENTERS[:1], DIRS[:1], RADII[:1])
        with pytest.raises(ts.ValidationError):
            FaultedModel(mesh, mats(), faces)


def test_sampling_at_a_node_returns_the_nodal_value(setup):
    """test_fault.cpp 'sampling at a node returns the nodal value': an observation placed on a
    surface vertex samples exactly that vertex's displacement."""
    mesh, _, faces, _ = setup
    cfg = ts.SolverConfig(batch_size=len(DIRS))
    fm = FaultedModel(mesh, mats(), faces, cfg)
    coords = np.asarray(mesh.coords)
    top = np.flatnonzero((coords[:, 2] == 6000.0) & (np.arange(len(coords)) < mesh.vertex_count)
                         & (coords[:, 0] > 0) & (coords[:, 0] < 8000.0) & (coords[:, 1] > 0) & (coords[:, 1] < 8000.0))
    node = int(top[len(top) // 2])
    bank, _, _ = fm.greens_bank(CENTERS, DIRS, RADII, coords[node:node + 1].repeat(3, 0), np.arange(3, dtype=np.int32),
                                cfg)
    f = fm.slip_to_rhs(CENTERS, DIRS, RADII)
    u, _ = ts.solve(fm.levels, f, np.zeros_like(f), cfg)
    want = u[3 * node:3 * node + 3]
    # the two solves agree to solver tolerance (the EBE scatter order is not fixed), the sampling itself is exact
    assert rel(bank, want) <= 1e-8
