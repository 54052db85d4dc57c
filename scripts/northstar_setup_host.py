"""Host side of the north-star partitioned setup at BASELINE configs[3] (405M DOF),
measured without GPUs: what each of P ranks does on the host before any
device work in ts_dist_levels_create (dist_solver.cu), run here rank by rank
in one process.

  mesh       generate_box_mesh of the global mesh (every rank)
  partition  recursive coordinate bisection into P parts (every rank)
  plan[r]    build_dist_plan of rank r: local mesh, halos, ownership (every rank)
  level2     K1 assembly + sequential aggregation + Galerkin product + M2 +
             coarse mask of the GLOBAL mesh (rank 0 only; broadcast to the others)

Reports wall time and resident memory (current RSS after the step and the
process peak) per step as one JSON line; profiles/r02_northstar_setup_host.json
keeps the committed run. Usage: python scripts/northstar_setup_host.py [P] [cells...]
"""
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import paper_1710_08679_b200 as ts  # noqa: E402
from paper_1710_08679_b200._lib import lib  # noqa: E402
from paper_1710_08679_b200.dist import dist_plan, partition_rcb  # noqa: E402

CELL_KM = 2.8
FOUR_LAYER = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0), (6800.0, 3900.0, 2900.0), (8000.0, 4500.0, 3300.0)]


def rss_gb():
    with open("/proc/self/statm") as fh:
        return int(fh.read().split()[1]) * os.sysconf("SC_PAGE_SIZE") / 1e9


def peak_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    cells = tuple(int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (281, 423, 141)
    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    ifs = (0.2 * ext[2], 0.45 * ext[2], 0.8 * ext[2])
    out = {"what": "host side of ts_dist_levels_create at configs[3], rank by rank, no GPU",
           "cells": list(cells), "ranks": P, "host_threads": os.cpu_count(), "steps": {}}

    def step(name, fn):
        t0 = time.perf_counter()
        r = fn()
        out["steps"][name] = {"s": round(time.perf_counter() - t0, 2), "rss_gb": round(rss_gb(), 2),
                              "peak_gb": round(peak_gb(), 2)}
        print(name, out["steps"][name], file=sys.stderr, flush=True)
        return r

    mesh = step("mesh", lambda: ts.generate_box_mesh(ext, cells, ifs))
    out["dof"] = 3 * mesh.node_count()
    out["elements"] = mesh.element_count()
    part = step("partition", lambda: partition_rcb(mesh, P))
    plans = {}
    for r in range(P):
        p = step(f"plan[{r}]", lambda r=r: dist_plan(mesh, part, P, r))
        plans[r] = {"n_local": int(len(p["l2g"])), "elements": int(len(p["elems"])), "neighbours": int(len(p["nbr"])),
                    "interface_rows": int(p["nbr_rows"].sum())}
        del p
    out["plans"] = plans
    mats = [ts.material_from_wavespeeds(*t) for t in FOUR_LAYER]
    lam = np.array([m.lam for m in mats])
    mu = np.array([m.mu for m in mats])
    n2, nz = C.c_int32(), C.c_int64()

    def level2():
        rc = lib.ts_level2_setup_host(mesh._h, len(lam), lam.ctypes.data_as(C.c_void_p), mu.ctypes.data_as(C.c_void_p),
                                      None, 8, C.byref(n2), C.byref(nz))
        if rc:
            raise RuntimeError(lib.ts_last_error().decode())

    step("level2 (rank 0)", level2)
    out["n2"], out["nnzb2"] = n2.value, nz.value
    out["broadcast_bytes"] = int(4 * 3 * (mesh.vertex_count // 3) + 4 * (n2.value + 1) + (4 + 36) * nz.value +
                                 36 * n2.value + 3 * n2.value)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
