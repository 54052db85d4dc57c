"""Capped reference solve at BASELINE configs[2] (the 50M-DOF 3-layer crust box).

BASELINE.md §3: a full CPU solve of configs[2] takes on the order of a day, so
the reference's own solve() is run with outer_max_iter = 1; the
ConvergenceError it raises still carries the timed report
(adaptive_cg.hpp:179-188). This script runs the UNMODIFIED reference
(oracle/_ref/libtsref.so) in the build container, where /root/reference
exists, and writes tests/golden/config2_outer1_reference.json:

* per-level inner iteration counts of outer iteration 1 (the GPU test
  tests/test_baseline_configs_gpu.py::test_config2_first_outer_iteration
  compares its own counts with them, +-2 %),
* the per-column relative residual after outer iteration 1,
* column norms of f (so the GPU side can check it lifted the same loads),
* the reference's wall times (setup, the capped solve, per level), used by
  bench.py for the LABELLED per-outer-iteration CPU extrapolation.

Memory forces r = 4 here (r = 16 needs ~9 fp64 batches of 6.4 GB plus the
fp32 level vectors, more than this 62 GB host); the GPU comparison uses the
same r = 4 batch, since max-over-columns termination makes the counts depend
on the batch.

Usage: python tests/golden/make_config2_capped.py [cells...]
"""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import Oracle, OracleError, SolverConfig  # noqa: E402
from config_specs import CONFIG2, THREE_LAYER, config2_rhs, lame  # noqa: E402


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def main():
    cells = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else CONFIG2["cells"]
    batch = CONFIG2["batch"]
    R = Oracle("reference")
    workers = R.hw_threads()
    ext, ifs = CONFIG2["extents"](cells), CONFIG2["interfaces"](cells)
    lam, mu = lame(THREE_LAYER)
    t0 = time.perf_counter()
    m = R.box_mesh(ext, cells, ifs, 1)
    t_mesh = time.perf_counter() - t0
    cfg = SolverConfig.default(batch_size=batch, outer_max_iter=1)
    t0 = time.perf_counter()
    lv = R.levels(m, lam, mu, cfg, workers=workers)
    t_levels = time.perf_counter() - t0
    us = config2_rhs(R, m.coords, ext, m.dirichlet_mask(), batch)
    t0 = time.perf_counter()
    f = lv.outer_apply(us)
    t_rhs = time.perf_counter() - t0
    del us
    t0 = time.perf_counter()
    try:
        lv.solve(f, history=4)
        raise SystemExit("expected ConvergenceError after one outer iteration")
    except OracleError as err:
        assert err.code == 4, str(err)
        rep = err.report
    t_solve = time.perf_counter() - t0
    out = {
        "what": "reference solve() capped at outer_max_iter=1 (ConvergenceError report), BASELINE configs[2]",
        "generated_by": "tests/golden/make_config2_capped.py (UNMODIFIED reference, oracle/_ref/libtsref.so)",
        "cells": list(cells), "extents": list(ext), "interfaces": list(ifs), "batch": batch,
        "dof": 3 * m.n_nodes, "elements": m.n_elems, "n2": lv.n2,
        "outer_iterations": rep["outer_iterations"], "inner_iterations": rep["inner_iterations"],
        "final_rel_residual": [float(x) for x in rep["final_rel_residual"]],
        "f_column_norms": [float(x) for x in np.linalg.norm(f, axis=0)],
        "host": {"cpu_model": cpu_model(), "workers": workers, "note": "build container, not the GPU box"},
        "seconds": {"mesh": round(t_mesh, 2), "levels_setup": round(t_levels, 2), "rhs_apply": round(t_rhs, 2),
                    "capped_solve": round(t_solve, 2), "report_total": rep["time_total_s"],
                    "report_inner": rep["time_inner_s"]},
    }
    with open(os.path.join(HERE, "config2_outer1_reference.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
