"""The reference's own Catch2 unit suites, compiled unchanged against the B200
drop-in headers (include/tetsolve/<module>.hpp) — only the include path
differs — with the mini Catch2 / Eigen shims of tests/cpp/shim
(tests/cpp/Makefile, built by __graft_entry__.build() where
/root/reference exists; the binaries travel to the GPU box).

* test_ebe.cpp (ebe vs assembled, nullspace, symmetry, block Jacobi, BCSR,
  batch == single bit-exact, shape errors) and test_solver.cpp (inner_pcg,
  dense-LU oracle, indefinite operator -> SolverError, manufactured solution,
  identical columns, PCGE, zero RHS, ConvergenceError with report, config)
  and test_multigrid.cpp (prolongation, aggregation, Galerkin product, coarse
  masks, SPD) need the GPU;
* test_mesh.cpp is host-only (generator, validation, mesh files) and also
  runs here.

The deterministic-coloring case of test_ebe.cpp (":296-317") compares two
reference EbeOperator instances with different worker counts; the drop-in
accepts `workers` and runs one device sweep whose summation order is fixed per
launch configuration, so the check holds when the two products are bitwise
equal (it is asserted, not skipped).
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def run_suite(name, timeout=1800):
    exe = os.path.join(CPP, f"ref_{name}")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj/tests"):
            subprocess.run(["make", "-C", CPP, f"ref_{name}"], check=True)
        else:
            pytest.skip(f"tests/cpp/ref_{name} not built (reference test sources absent on this host)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, out.stdout[-2000:] + out.stderr[-4000:]
    res = json.loads(lines[-1])
    assert out.returncode == 0 and res["failures"] == 0, out.stderr[-6000:]
    assert res["test_cases"] > 0 and res["checks"] > 0
    return res


def test_reference_mesh_suite():
    res = run_suite("test_mesh")
    assert res["test_cases"] >= 11


@pytest.mark.gpu
def test_reference_ebe_suite():
    res = run_suite("test_ebe")
    assert res["test_cases"] >= 14


@pytest.mark.gpu
def test_reference_solver_suite():
    res = run_suite("test_solver")
    assert res["test_cases"] >= 11


@pytest.mark.gpu
def test_reference_multigrid_suite():
    res = run_suite("test_multigrid")
    assert res["test_cases"] >= 5
