"""The C++ drop-in headers (include/tetsolve_b200/tetsolve.hpp) compile against
libtsgpu.so here (CPU), the reference's file-format tests written against them
run here (host-only), and the reference's manufactured-solution test written
against them runs on the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_demo")
LIBDIR = os.path.join(ROOT, "paper_1710_08679_b200")


def build(src=SRC, out=BIN):
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-ltsgpu",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


def test_dropin_header_compiles_and_links():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_manufactured_solution_on_gpu():
    build()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["converged"] == 1 and res["rel_err"] < 1e-7 and res["max_final"] <= 1e-8
    assert res["method"] == "pcge" and res["pcge_outer"] >= res["outer"]
    assert res["history"] == res["outer"] and res["validation_throw"] == 1


def test_dropin_file_formats(tmp_path):
    """test_mesh.cpp:120-188 + the TSVEC round trip through the drop-in header (no GPU needed)."""
    out_bin = str(tmp_path / "dropin_io")
    build(os.path.join(ROOT, "tests", "cpp", "dropin_io.cpp"), out_bin)
    out = subprocess.run([out_bin, str(tmp_path / "work")], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["failures"] == 0 and res["parse_throw"] == 1 and res["volume_throw"] == 1


def test_dropin_greens_compiles():
    build(os.path.join(ROOT, "tests", "cpp", "dropin_greens.cpp"), os.path.join(ROOT, "tests", "cpp", "dropin_greens"))


@pytest.mark.gpu
def test_dropin_greens_matches_reference(reference, tmp_path):
    """A Green's sweep written against the reference's fault/model/greens API, compiled against the
    drop-in header, reproduces the reference's own bank (compute_greens_bank, greens.hpp:114-145)."""
    import numpy as np
    from conftest import TWO_LAYER, lame
    from oracle import SolverConfig as OCfg
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_greens")
    build(os.path.join(ROOT, "tests", "cpp", "dropin_greens.cpp"), exe)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300, cwd=tmp_path)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["files_ok"] == 1
    om = reference.box_mesh((8000.0, 8000.0, 6000.0), (8, 8, 6), (4500.0,), 1)
    faces = reference.fault_plane_faces(om, 0, 4000.0, (4000.0, 2000.0, 1000.0), (4000.0, 6000.0, 5000.0))
    assert res["faces"] == len(faces)
    lam, mu = lame(TWO_LAYER)
    centers = np.array([[4000.0, 4000.0, 3000.0], [4000.0, 3000.0, 2500.0], [4000.0, 5000.0, 4000.0],
                        [4000.0, 4000.0, 3000.0], [4000.0, 3500.0, 2000.0]])
    dirs = np.array([0, 0, 1, 1, 0], np.int32)
    radii = np.array([1500.0, 1000.0, 1200.0, 1500.0, 900.0])
    pts = np.array([[1000.0, 2000.0, 6000.0], [3000.0, 4000.0, 6000.0], [5000.0, 4000.0, 6000.0],
                    [6500.0, 1500.0, 6000.0], [4000.0, 7000.0, 6000.0], [2500.0, 2500.0, 5500.0]])
    axes = np.array([0, 1, 2, 0, 2, 1], np.int32)
    rbank, rcalls, router = reference.greens_bank(om, lam, mu, faces, centers, dirs, radii, pts, axes,
                                                  OCfg.default(batch_size=2))
    f, info = reference.slip_to_rhs(om, lam, mu, faces, centers[:1], dirs[:1], radii[:1])
    assert (res["split_nodes"], res["split_mesh_nodes"]) == tuple(info)
    assert abs(res["f0_norm2"] - float((f ** 2).sum())) <= 1e-12 * float((f ** 2).sum())
    assert res["calls"] == rcalls and abs(res["outer"] - router) <= max(1, 0.02 * router)
    bank = np.array(res["bank"]).reshape(rbank.shape)
    assert float(np.linalg.norm(bank - rbank) / np.linalg.norm(rbank)) <= 1e-6
    assert res["solve_outer"] >= 1
