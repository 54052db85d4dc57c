"""Green's-function sweep — Python mirror of include/tsgpu.h's ts_fault_* /
ts_faulted_* / ts_greens_bank (reference fault.hpp,
model.hpp:34-56, greens.hpp:114-145)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib
from .tetsolve import Mesh, SolverConfig, SolverLevels, _ck, _lame, _p

DIP, STRIKE = 0, 1  # SlipDirection (fault.hpp:304)


def find_plane_fault_faces(mesh: Mesh, axis: int, coord: float, lo, hi) -> np.ndarray:
    """find_plane_fault_faces (fault.hpp:86-118): [F, 3] base-mesh vertex ids."""
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    n = C.c_int32(0)
    _ck(lib.ts_fault_plane_faces(mesh._h, int(axis), float(coord), _p(lo), _p(hi), C.byref(n), None))
    out = np.zeros((n.value, 3), np.int32)
    _ck(lib.ts_fault_plane_faces(mesh._h, int(axis), float(coord), _p(lo), _p(hi), C.byref(n), _p(out)))
    return out


class FaultedModel:
    """build_faulted_model (model.hpp:41-51): split mesh + base crust hierarchy on the device."""

    def __init__(self, mesh: Mesh, materials, faces, cfg: SolverConfig | None = None):
        cfg = cfg or SolverConfig()
        lam, mu = _lame(materials)
        faces = np.ascontiguousarray(faces, np.int32)
        c = cfg.to_c()
        h = C.c_void_p()
        _ck(lib.ts_faulted_model_create(mesh._h, len(lam), _p(lam), _p(mu), _p(faces), len(faces), C.byref(c),
                                        C.byref(h)))
        self._h, self.mesh = h, mesh
        ns, nsm, nf = C.c_int32(), C.c_int32(), C.c_int32()
        _ck(lib.ts_faulted_info(self._h, C.byref(ns), C.byref(nsm), C.byref(nf)))
        self.n_split_nodes, self.split_mesh_nodes, self.n_faces = ns.value, nsm.value, nf.value
        lv = C.c_void_p()
        _ck(lib.ts_faulted_levels(self._h, C.byref(lv)))
        self.levels = SolverLevels(lv, mesh, owner=self)  # FaultedModel::base.levels

    def slip_to_rhs(self, centers, directions, radii) -> np.ndarray:
        """slip_to_rhs (fault.hpp:363-388) of each unit slip: [3N, n_slips]."""
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        directions = np.ascontiguousarray(directions, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        f = np.zeros((3 * self.mesh.node_count(), len(directions)), np.float64)
        _ck(lib.ts_slip_to_rhs(self._h, len(directions), _p(centers), _p(directions), _p(radii), _p(f)))
        return f

    def reconstruct_split_solution(self, centers, directions, radii, u_base) -> np.ndarray:
        """reconstruct_split_solution (fault.hpp:392-411): base-mesh solutions [3N, n] of the n unit
        slips -> split-mesh displacements [3 NS, n] with the prescribed jumps."""
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        directions = np.ascontiguousarray(directions, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        ub = np.ascontiguousarray(u_base, np.float64).reshape(3 * self.mesh.node_count(), len(directions))
        out = np.zeros((3 * self.split_mesh_nodes, len(directions)), np.float64)
        _ck(lib.ts_reconstruct_split_solution(self._h, len(directions), _p(centers), _p(directions), _p(radii),
                                              _p(ub), _p(out)))
        return out

    def greens_bank(self, centers, directions, radii, points, axes, cfg: SolverConfig | None = None):
        """compute_greens_bank (greens.hpp:114-145): (bank [n_obs, n_slips], solver_calls, outer_iterations)."""
        cfg = cfg or SolverConfig()
        c = cfg.to_c()
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        directions = np.ascontiguousarray(directions, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        points = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        axes = np.ascontiguousarray(axes, np.int32)
        bank = np.zeros((len(axes), len(directions)), np.float64)
        calls, outer = C.c_int32(), C.c_int64()
        _ck(lib.ts_greens_bank(self._h, len(directions), _p(centers), _p(directions), _p(radii), len(axes), _p(points),
                               _p(axes), C.byref(c), _p(bank), C.byref(calls), C.byref(outer)))
        return bank, calls.value, outer.value

    def __del__(self):
        try:
            lib.ts_faulted_model_destroy(self._h)
        except Exception:
            pass


# ------------------------------------------------------------------ files
def _path(p) -> bytes:
    import os

    return os.fsencode(p)


def write_fault_faces(faces, path) -> None:
    """write_fault_faces (fault.hpp:414-419): TSFAULT 1, one "v0 v1 v2" line per face."""
    f = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
    _ck(lib.ts_fault_faces_write(_path(path), _p(f), f.shape[0]))


def read_fault_faces(path) -> np.ndarray:
    """read_fault_faces (fault.hpp:47-78) -> (F, 3) int32."""
    n = C.c_int32(0)
    _ck(lib.ts_fault_faces_read(_path(path), C.byref(n), None))
    out = np.zeros((n.value, 3), np.int32)
    _ck(lib.ts_fault_faces_read(_path(path), C.byref(n), _p(out)))
    return out


def read_observations(path):
    """read_observations (greens.hpp:20-44) -> (points (R, 3), axes (R,))."""
    n = C.c_int32(0)
    _ck(lib.ts_observations_read(_path(path), C.byref(n), None, None))
    pts = np.zeros((n.value, 3), np.float64)
    ax = np.zeros(n.value, np.int32)
    _ck(lib.ts_observations_read(_path(path), C.byref(n), _p(pts), _p(ax)))
    return pts, ax


def write_greens_bank(path, bank, obs_points, obs_axes, centers, directions, radii) -> None:
    """write_greens_bank (greens.hpp:147-165): TSGREENS 1 text header + row-major fp64 matrix."""
    b = np.ascontiguousarray(bank, np.float64)
    rows, cols = b.shape
    pts = np.ascontiguousarray(obs_points, np.float64).reshape(rows, 3)
    ax = np.ascontiguousarray(obs_axes, np.int32).reshape(rows)
    c = np.ascontiguousarray(centers, np.float64).reshape(cols, 3)
    d = np.ascontiguousarray(directions, np.int32).reshape(cols)
    r = np.ascontiguousarray(radii, np.float64).reshape(cols)
    _ck(lib.ts_greens_bank_write(_path(path), rows, cols, _p(pts), _p(ax), _p(c), _p(d), _p(r), _p(b)))


def read_greens_bank(path) -> dict:
    """read_greens_bank (greens.hpp:167-222) -> dict(values, obs_points, obs_axes, centers, directions, radii)."""
    rows, cols = C.c_int32(0), C.c_int32(0)
    _ck(lib.ts_greens_bank_read(_path(path), C.byref(rows), C.byref(cols), None, None, None, None, None, None))
    R, K = rows.value, cols.value
    out = dict(values=np.zeros((R, K)), obs_points=np.zeros((R, 3)), obs_axes=np.zeros(R, np.int32),
               centers=np.zeros((K, 3)), directions=np.zeros(K, np.int32), radii=np.zeros(K))
    _ck(lib.ts_greens_bank_read(_path(path), C.byref(rows), C.byref(cols), _p(out["obs_points"]), _p(out["obs_axes"]),
                                _p(out["centers"]), _p(out["directions"]), _p(out["radii"]), _p(out["values"])))
    return out
