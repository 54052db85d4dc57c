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
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-ltsgpu",
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
