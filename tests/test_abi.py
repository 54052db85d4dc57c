"""CPU-side checks of the C-ABI library (no GPU needed).

* libtsgpu.so loads and exports every function declared in include/tsgpu.h;
* the host-side mesh generator reproduces the reference numbering bit-exactly;
* validation errors surface as the reference's exception classes;
* with no CUDA device, compute entry points fail loudly (no CPU fallback).
"""
import ctypes as C

import numpy as np
import pytest
from conftest import has_cuda

import paper_1710_08679_b200 as ts
from paper_1710_08679_b200 import _lib


def test_library_exports_every_declared_symbol():
    syms = _lib.declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, f"declared in include/tsgpu.h but not exported: {missing}"


def test_version_string():
    assert b"sm_100a" in _lib.lib.ts_version()


@pytest.mark.parametrize("spec", [
    ((2.0, 2.0, 2.0), (2, 2, 2), (1.0,), 1),
    ((400.0, 400.0, 200.0), (4, 3, 2), (100.0,), 1),
    ((1.0, 2.0, 3.0), (3, 2, 1), (1.0, 2.0), 2),
    ((1.0, 1.0, 1.0), (1, 1, 1), (), 0),
    ((16000.0, 16000.0, 10000.0), (8, 8, 5), (7000.0,), 1),
])
def test_box_mesh_matches_reference_numbering(checker, spec):
    m = ts.generate_box_mesh(spec[0], spec[1], spec[2], spec[3])
    o = checker.box_mesh(*spec)
    a = m.arrays()
    assert m.vertex_count == o.vertex_count
    assert np.array_equal(a["coords"], o.coords)
    assert np.array_equal(a["tets10"], o.tets10)
    assert np.array_equal(a["material_id"], o.material_id)
    assert np.array_equal(a["bc_node"], o.bc_node)
    assert np.array_equal(a["bc_axis"], o.bc_axis)
    assert np.array_equal(m.dirichlet_mask(), o.dirichlet_mask())


def test_mesh_from_arrays_roundtrip(checker):
    o = checker.box_mesh((1.0, 1.0, 1.0), (2, 1, 1), (), 1)
    m = ts.Mesh.from_arrays(o.coords, o.tets10, o.material_id, o.vertex_count, o.bc_node, o.bc_axis)
    assert m.node_count() == o.n_nodes and m.element_count() == o.n_elems
    assert np.array_equal(m.tets10, o.tets10)


def test_box_mesh_validation():
    with pytest.raises(ts.ValidationError):
        ts.generate_box_mesh((1.0, 1.0, 1.0), (0, 1, 1))
    with pytest.raises(ts.ValidationError):
        ts.generate_box_mesh((1.0, -1.0, 1.0), (1, 1, 1))
    with pytest.raises(ts.ValidationError):
        ts.generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 2), (0.7, 0.5))


def test_material_from_wavespeeds():
    m = ts.material_from_wavespeeds(5800.0, 3000.0, 2700.0)
    assert m.mu == 2700.0 * 3000.0 ** 2
    assert m.lam == 2700.0 * (5800.0 ** 2 - 2 * 3000.0 ** 2)
    with pytest.raises(ts.ValidationError):
        ts.material_from_wavespeeds(1000.0, 800.0, 2000.0)


def test_solver_config_defaults_and_validation():
    cfg = ts.SolverConfig()
    cfg.validate()
    c = C.create_string_buffer(C.sizeof(_lib.SolverConfig))
    _lib.lib.ts_config_default(c)
    d = _lib.SolverConfig.from_buffer(c)
    assert d.outer_tol == 1e-8 and d.outer_max_iter == 5000
    assert list(d.level_tol) == [0.1, 0.05, 0.025] and list(d.level_max_iter) == [30, 300, 3000]
    assert d.batch_size == 16 and d.aggregate_target == 8
    bad = ts.SolverConfig(outer_tol=0.0)
    with pytest.raises(ts.ValidationError):
        bad.validate()
    with pytest.raises(ts.ValidationError):
        ts.SolverConfig(batch_size=0).validate()


@pytest.mark.skipif(has_cuda(), reason="checks the no-device path")
def test_compute_fails_loudly_without_gpu():
    m = ts.generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 1))
    mat = ts.material_from_wavespeeds(5800.0, 3000.0, 2700.0)
    with pytest.raises(ts.DeviceError):
        ts.EbeOperator(m, 2, [mat], m.dirichlet_mask(), prec=64)
