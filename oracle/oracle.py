"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end over the two CPU checkers of the reference solve path:

* ``kind="port"``      -> oracle/libtsoracle.so, the plain-C restatement
                          (oracle/tsoracle.c, every function cites the
                          reference file:line it follows);
* ``kind="reference"`` -> oracle/_ref/libtsref.so, the UNMODIFIED reference
                          headers (/root/reference/proj/include/tetsolve)
                          compiled in place through oracle/ref_shim.cpp.

Both expose the same functions, so tests can pin the port against the
reference (tests/test_oracle_pin.py) and then use the port (or the reference
when present) as the checker for the CUDA path. Only tests/, smoke() and
bench.py (cpu_baseline / --impl reference) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libtsoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class SolverConfig(C.Structure):
    """ts_solver_config (include/tsgpu.h) == tetsolve::SolverConfig (solver_config.hpp:21-48)."""

    _fields_ = [
        ("outer_tol", C.c_double),
        ("outer_max_iter", C.c_int32),
        ("level_tol", C.c_double * 3),
        ("level_max_iter", C.c_int32 * 3),
        ("batch_size", C.c_int32),
        ("aggregate_target", C.c_int32),
        ("residual_history_stride", C.c_int32),
    ]

    @classmethod
    def default(cls, **kw):
        c = cls()
        c.outer_tol = 1e-8
        c.outer_max_iter = 5000
        c.level_tol[:] = [0.1, 0.05, 0.025]
        c.level_max_iter[:] = [30, 300, 3000]
        c.batch_size = 16
        c.aggregate_target = 8
        c.residual_history_stride = 1
        for k, v in kw.items():
            if k in ("level_tol", "level_max_iter"):
                getattr(c, k)[:] = v
            else:
                setattr(c, k, v)
        return c


class SolveReport(C.Structure):
    """ts_solve_report (include/tsgpu.h) == tetsolve::SolveReport (solver_config.hpp:50-63)."""

    _fields_ = [
        ("converged", C.c_int32),
        ("outer_iterations", C.c_int32),
        ("inner_iterations", C.c_int64 * 3),
        ("time_setup_s", C.c_double),
        ("time_outer_s", C.c_double),
        ("time_inner_s", C.c_double * 3),
        ("time_total_s", C.c_double),
        ("batch_size", C.c_int32),
        ("method", C.c_int32),
        ("inner_precision", C.c_int32),
        ("history_count", C.c_int32),
        ("history_capacity", C.c_int32),
        ("final_rel_residual", C.POINTER(C.c_double)),
        ("history_iter", C.POINTER(C.c_int32)),
        ("history", C.POINTER(C.c_double)),
    ]


def make_report(batch: int, capacity: int = 0):
    """Allocate a report plus the numpy buffers it points into."""
    rep = SolveReport()
    final = np.zeros(batch, np.float64)
    hist_it = np.zeros(max(capacity, 1), np.int32)
    hist = np.zeros((max(capacity, 1), batch), np.float64)
    rep.final_rel_residual = final.ctypes.data_as(C.POINTER(C.c_double))
    rep.history_iter = hist_it.ctypes.data_as(C.POINTER(C.c_int32))
    rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
    rep.history_capacity = capacity
    return rep, (final, hist_it, hist)


def report_dict(rep: SolveReport, bufs) -> dict:
    final, hist_it, hist = bufs
    n = rep.history_count
    return {
        "converged": bool(rep.converged),
        "outer_iterations": int(rep.outer_iterations),
        "inner_iterations": [int(x) for x in rep.inner_iterations],
        "final_rel_residual": final.copy(),
        "history_iter": hist_it[:n].copy(),
        "history": hist[:n].copy(),
        "method": "pcge" if rep.method == 1 else "amg",
        "inner_precision": "float64" if rep.inner_precision == 64 else "float32",
        "time_total_s": float(rep.time_total_s),
        "time_inner_s": [float(x) for x in rep.time_inner_s],
    }


@dataclass
class MeshArrays:
    """Plain arrays of a tetsolve::Mesh (mesh.hpp:26-42)."""

    coords: np.ndarray      # [N,3] f64
    tets10: np.ndarray      # [E,10] i32
    material_id: np.ndarray  # [E] i32
    vertex_count: int
    bc_node: np.ndarray     # [nbc] i32
    bc_axis: np.ndarray     # [nbc] i8

    @property
    def n_nodes(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_elems(self) -> int:
        return int(self.tets10.shape[0])

    def dirichlet_mask(self) -> np.ndarray:
        m = np.zeros(3 * self.n_nodes, np.uint8)
        m[3 * self.bc_node.astype(np.int64) + self.bc_axis.astype(np.int64)] = 1
        return m


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Same interface over the C port (``port``) or the reference (``reference``)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run __graft_entry__.build())")
        self.lib = C.CDLL(path)
        self.pre = "or_" if kind == "port" else "ref_"
        L = self.lib
        vp = C.c_void_p
        self._f("last_error").restype = C.c_char_p
        self._f("box_mesh").restype = vp
        self._f("box_mesh").argtypes = [vp, vp, C.c_int32, vp, C.c_int32]
        self._f("mesh_from_arrays").restype = vp
        self._f("mesh_from_arrays").argtypes = [C.c_int32, C.c_int32, vp, C.c_int32, vp, vp, C.c_int32, vp, vp]
        self._f("mesh_sizes").argtypes = [vp, vp, vp, vp, vp]
        self._f("mesh_export").argtypes = [vp] * 6
        self._f("mesh_mask").argtypes = [vp, vp]
        self._f("mesh_destroy").argtypes = [vp]
        self._f("element_matrix").argtypes = [C.c_int32, vp, C.c_double, C.c_double, vp]
        self._f("ebe_apply").argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, C.c_int32]
        self._f("assemble_bcsr").restype = vp
        self._f("assemble_bcsr").argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int32]
        self._f("bcsr_sizes").argtypes = [vp, vp, vp]
        self._f("bcsr_export").argtypes = [vp, vp, vp, vp]
        self._f("bcsr_destroy").argtypes = [vp]
        self._f("bcsr_apply").argtypes = [C.c_int32, vp, vp, vp, C.c_int32, vp, vp, C.c_int32]
        self._f("ebe_block_jacobi").argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int32, vp]
        self._f("bj_apply").argtypes = [C.c_int32, vp, C.c_int32, vp, vp, C.c_int32]
        self._f("geo_prolong").argtypes = [vp, C.c_int32, vp, vp, C.c_int32]
        self._f("inner_pcg_ebe").argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, C.c_int32,
                                             C.c_double, C.c_int32, vp, vp]
        self._f("levels_create").restype = vp
        self._f("levels_create").argtypes = [vp, C.c_int32, vp, vp, vp, C.c_int32, vp]
        self._f("levels_sizes").argtypes = [vp, vp, vp, vp, vp]
        self._f("levels_export").argtypes = [vp] * 9
        self._f("levels_destroy").argtypes = [vp]
        self._f("levels_outer_apply").argtypes = [vp, vp, vp, C.c_int32]
        self._f("solve").argtypes = [vp, vp, vp, vp, C.c_int32, vp, vp]
        self._f("solve_pcge").argtypes = [vp, vp, vp, vp, C.c_int32, C.c_double, C.c_int32, vp]
        self._f("rng_sym").argtypes = [C.c_uint64, C.c_int64, vp]
        if kind == "reference":
            # every pointer argument needs its argtypes: an undeclared handle would be passed as a 32-bit int
            L.ref_fault_plane_faces.argtypes = [vp, C.c_int32, C.c_double, vp, vp, vp, vp]
            L.ref_slip_to_rhs.argtypes = [vp, C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]
            L.ref_greens_bank.argtypes = [vp, C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int32, vp, vp,
                                          vp, vp, vp, vp]
            L.ref_time_ebe_apply.argtypes = [vp, C.c_int32, C.c_int32, vp, vp, C.c_int32, C.c_int32,
                                             C.c_int32, C.c_int32, C.c_int32, C.c_uint64, vp, vp]
            L.ref_hw_threads.restype = C.c_int

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._f("last_error")().decode())

    # ------------------------------------------------------------ meshes
    def box_mesh(self, extents, divisions, interfaces=(), fixed=1) -> MeshArrays:
        ext = np.ascontiguousarray(extents, np.float64)
        div = np.ascontiguousarray(divisions, np.int32)
        ifs = np.ascontiguousarray(interfaces, np.float64) if len(interfaces) else np.zeros(1)
        h = self._f("box_mesh")(_p(ext), _p(div), len(interfaces), _p(ifs), fixed)
        if not h:
            raise OracleError(1, self._f("last_error")().decode())
        try:
            return self._export(h)
        finally:
            self._f("mesh_destroy")(h)

    def _export(self, h) -> MeshArrays:
        nn, nv, ne, nbc = (C.c_int32() for _ in range(4))
        self._f("mesh_sizes")(h, C.byref(nn), C.byref(nv), C.byref(ne), C.byref(nbc))
        coords = np.zeros((nn.value, 3), np.float64)
        tets = np.zeros((ne.value, 10), np.int32)
        mat = np.zeros(ne.value, np.int32)
        bn = np.zeros(max(nbc.value, 1), np.int32)
        ba = np.zeros(max(nbc.value, 1), np.int8)
        self._f("mesh_export")(h, _p(coords), _p(tets), _p(mat), _p(bn), _p(ba))
        return MeshArrays(coords, tets, mat, nv.value, bn[: nbc.value].copy(), ba[: nbc.value].copy())

    def _mesh(self, m: MeshArrays):
        c = np.ascontiguousarray(m.coords, np.float64)
        t = np.ascontiguousarray(m.tets10, np.int32)
        mat = np.ascontiguousarray(m.material_id, np.int32)
        bn = np.ascontiguousarray(m.bc_node, np.int32)
        ba = np.ascontiguousarray(m.bc_axis, np.int8)
        h = self._f("mesh_from_arrays")(m.n_nodes, m.vertex_count, _p(c), m.n_elems, _p(t), _p(mat),
                                        len(bn), _p(bn), _p(ba))
        return h

    # --------------------------------------------------------- operators
    def element_matrix(self, order, v12, lam, mu):
        n = 12 if order == 1 else 30
        k = np.zeros((n, n), np.float64)
        v = np.ascontiguousarray(v12, np.float64)
        self._check(self._f("element_matrix")(order, _p(v), lam, mu, _p(k)))
        return k

    def ebe_apply(self, m: MeshArrays, order, lam, mu, mask, prec, u, workers=1):
        dt = np.float32 if prec == 32 else np.float64
        u = np.ascontiguousarray(u, dt)
        f = np.zeros_like(u)
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        h = self._mesh(m)
        try:
            self._check(self._f("ebe_apply")(h, order, len(lam), _p(lam), _p(mu), _p(mk), prec, workers,
                                             _p(u), _p(f), u.shape[-1]))
        finally:
            self._f("mesh_destroy")(h)
        return f

    def assemble_bcsr(self, m: MeshArrays, order, lam, mu, mask, prec):
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        h = self._mesh(m)
        try:
            a = self._f("assemble_bcsr")(h, order, len(lam), _p(lam), _p(mu), _p(mk), prec)
        finally:
            self._f("mesh_destroy")(h)
        if not a:
            raise OracleError(1, self._f("last_error")().decode())
        nr, nz = C.c_int32(), C.c_int64()
        self._f("bcsr_sizes")(a, C.byref(nr), C.byref(nz))
        rp = np.zeros(nr.value + 1, np.int32)
        ci = np.zeros(nz.value, np.int32)
        bl = np.zeros((nz.value, 9), np.float64)
        self._f("bcsr_export")(a, _p(rp), _p(ci), _p(bl))
        self._f("bcsr_destroy")(a)
        return rp, ci, bl

    def bcsr_apply(self, rp, ci, blocks, prec, u):
        dt = np.float32 if prec == 32 else np.float64
        u = np.ascontiguousarray(u, dt)
        f = np.zeros_like(u)
        bl = np.ascontiguousarray(blocks, dt)
        rp = np.ascontiguousarray(rp, np.int32)
        ci = np.ascontiguousarray(ci, np.int32)
        self._check(self._f("bcsr_apply")(len(rp) - 1, _p(rp), _p(ci), _p(bl), prec, _p(u), _p(f), u.shape[-1]))
        return f

    def ebe_block_jacobi(self, m: MeshArrays, order, lam, mu, mask, prec):
        dt = np.float32 if prec == 32 else np.float64
        nn = m.vertex_count if order == 1 else m.n_nodes
        inv = np.zeros((nn, 9), dt)
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        h = self._mesh(m)
        try:
            self._check(self._f("ebe_block_jacobi")(h, order, len(lam), _p(lam), _p(mu), _p(mk), prec, _p(inv)))
        finally:
            self._f("mesh_destroy")(h)
        return inv

    def bj_apply(self, inv, prec, r):
        dt = np.float32 if prec == 32 else np.float64
        inv = np.ascontiguousarray(inv, dt)
        r = np.ascontiguousarray(r, dt)
        z = np.zeros_like(r)
        self._check(self._f("bj_apply")(inv.shape[0], _p(inv), prec, _p(r), _p(z), r.shape[-1]))
        return z

    def geo_prolong(self, m: MeshArrays, x, transpose: bool):
        x = np.ascontiguousarray(x, np.float32)
        nb = x.shape[-1]
        n_out = m.vertex_count if transpose else m.n_nodes
        out = np.zeros((3 * n_out, nb), np.float32)
        h = self._mesh(m)
        try:
            self._check(self._f("geo_prolong")(h, int(transpose), _p(x), _p(out), nb))
        finally:
            self._f("mesh_destroy")(h)
        return out

    def inner_pcg_ebe(self, m: MeshArrays, order, lam, mu, mask, r, u0, tol, max_iter):
        r = np.ascontiguousarray(r, np.float32)
        u = np.array(u0, np.float32, copy=True)
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        it, cv = C.c_int32(), C.c_int32()
        h = self._mesh(m)
        try:
            self._check(self._f("inner_pcg_ebe")(h, order, len(lam), _p(lam), _p(mu), _p(mk), _p(r), _p(u),
                                                 r.shape[-1], tol, max_iter, C.byref(it), C.byref(cv)))
        finally:
            self._f("mesh_destroy")(h)
        return u, it.value, bool(cv.value)

    def levels(self, m: MeshArrays, lam, mu, cfg: SolverConfig | None = None, workers: int = 1):
        return Levels(self, m, lam, mu, cfg or SolverConfig.default(), workers)

    def rng_sym(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._f("rng_sym")(seed, n, _p(out))
        return out

    def time_ebe_apply_box(self, extents, divisions, interfaces, fixed, order, lam, mu, prec, workers, batch, reps,
                           seed=12):
        """Reference EbeOperator<T>::apply timing on a box mesh generated by the
        reference itself (no array round trip). Returns (sec/apply, checksum)."""
        assert self.kind == "reference"
        ext = np.ascontiguousarray(extents, np.float64)
        div = np.ascontiguousarray(divisions, np.int32)
        ifs = np.ascontiguousarray(interfaces, np.float64) if len(interfaces) else np.zeros(1)
        h = self._f("box_mesh")(_p(ext), _p(div), len(interfaces), _p(ifs), fixed)
        if not h:
            raise OracleError(1, self._f("last_error")().decode())
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        sec, chk = C.c_double(), C.c_double()
        try:
            self._check(self.lib.ref_time_ebe_apply(h, order, len(lam), _p(lam), _p(mu), 1, prec, workers, batch,
                                                    reps, seed, C.byref(sec), C.byref(chk)))
        finally:
            self._f("mesh_destroy")(h)
        return sec.value, chk.value

    # ---- Green's-function sweep (reference only: fault.hpp / greens.hpp)
    def fault_plane_faces(self, m: MeshArrays, axis, coord, lo, hi) -> np.ndarray:
        assert self.kind == "reference"
        h = self._mesh(m)
        try:
            n = C.c_int32(0)
            lo = np.ascontiguousarray(lo, np.float64)
            hi = np.ascontiguousarray(hi, np.float64)
            self._check(self.lib.ref_fault_plane_faces(h, axis, C.c_double(coord), _p(lo), _p(hi), C.byref(n), None))
            out = np.zeros((n.value, 3), np.int32)
            self._check(self.lib.ref_fault_plane_faces(h, axis, C.c_double(coord), _p(lo), _p(hi), C.byref(n), _p(out)))
        finally:
            self._f("mesh_destroy")(h)
        return out

    def slip_to_rhs(self, m: MeshArrays, lam, mu, faces, centers, dirs, radii):
        assert self.kind == "reference"
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        faces = np.ascontiguousarray(faces, np.int32)
        centers = np.ascontiguousarray(centers, np.float64)
        dirs = np.ascontiguousarray(dirs, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        f = np.zeros((3 * m.n_nodes, len(dirs)), np.float64)
        info = np.zeros(2, np.int32)
        h = self._mesh(m)
        try:
            self._check(self.lib.ref_slip_to_rhs(h, len(lam), _p(lam), _p(mu), _p(faces), len(faces), len(dirs),
                                                 _p(centers), _p(dirs), _p(radii), _p(f), _p(info)))
        finally:
            self._f("mesh_destroy")(h)
        return f, info

    def reconstruct_split(self, m: MeshArrays, lam, mu, faces, centers, dirs, radii, u_base, n_split_mesh_nodes):
        assert self.kind == "reference"
        arrs = [np.ascontiguousarray(x, t) for x, t in ((lam, np.float64), (mu, np.float64), (faces, np.int32),
                                                          (centers, np.float64), (dirs, np.int32), (radii, np.float64),
                                                          (u_base, np.float64))]
        lam_, mu_, faces_, centers_, dirs_, radii_, ub = arrs
        out = np.zeros((3 * n_split_mesh_nodes, len(dirs_)), np.float64)
        h = self._mesh(m)
        try:
            vp = C.c_void_p
            self.lib.ref_reconstruct_split.argtypes = [vp, C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]
            self._check(self.lib.ref_reconstruct_split(h, len(lam_), _p(lam_), _p(mu_), _p(faces_), len(faces_),
                                                       len(dirs_), _p(centers_), _p(dirs_), _p(radii_), _p(ub),
                                                       _p(out)))
        finally:
            self._f("mesh_destroy")(h)
        return out

    def greens_bank(self, m: MeshArrays, lam, mu, faces, centers, dirs, radii, points, axes, cfg: SolverConfig):
        assert self.kind == "reference"
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        faces = np.ascontiguousarray(faces, np.int32)
        centers = np.ascontiguousarray(centers, np.float64)
        dirs = np.ascontiguousarray(dirs, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        points = np.ascontiguousarray(points, np.float64)
        axes = np.ascontiguousarray(axes, np.int32)
        bank = np.zeros((len(axes), len(dirs)), np.float64)
        calls, outer = C.c_int32(), C.c_int64()
        h = self._mesh(m)
        try:
            self._check(self.lib.ref_greens_bank(h, len(lam), _p(lam), _p(mu), _p(faces), len(faces), len(dirs),
                                                 _p(centers), _p(dirs), _p(radii), len(axes), _p(points), _p(axes),
                                                 C.byref(cfg), _p(bank), C.byref(calls), C.byref(outer)))
        finally:
            self._f("mesh_destroy")(h)
        return bank, calls.value, outer.value

    # ------------------------------------------------------ file formats (reference only)
    def _io(self):
        if self.kind != "reference":
            raise OracleError(9, "file formats are checked against the reference itself (mesh_io.hpp, solution_io.hpp)")
        L = self.lib
        vp, cp = C.c_void_p, C.c_char_p
        L.ref_write_mesh.argtypes = [vp, cp]
        L.ref_read_mesh.argtypes = [cp, vp]
        L.ref_write_dirichlet.argtypes = [vp, cp]
        L.ref_read_dirichlet.argtypes = [vp, cp]
        L.ref_write_solution.argtypes = [cp, vp, C.c_int32, C.c_int32]
        L.ref_read_solution.argtypes = [cp, vp, vp, vp]
        L.ref_write_fault_faces.argtypes = [cp, vp, C.c_int32]
        L.ref_read_fault_faces.argtypes = [cp, vp, vp]
        L.ref_read_observations.argtypes = [cp, vp, vp, vp]
        L.ref_write_greens_bank.argtypes = [cp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp]
        L.ref_read_greens_bank.argtypes = [cp, vp, vp, vp, vp, vp, vp, vp, vp]
        return L

    def write_fault_faces(self, path, faces) -> None:
        L = self._io()
        f = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
        self._check(L.ref_write_fault_faces(os.fsencode(path), _p(f), f.shape[0]))

    def read_fault_faces(self, path) -> np.ndarray:
        L = self._io()
        n = C.c_int32()
        self._check(L.ref_read_fault_faces(os.fsencode(path), C.byref(n), None))
        out = np.zeros((n.value, 3), np.int32)
        self._check(L.ref_read_fault_faces(os.fsencode(path), C.byref(n), _p(out)))
        return out

    def read_observations(self, path):
        L = self._io()
        n = C.c_int32()
        self._check(L.ref_read_observations(os.fsencode(path), C.byref(n), None, None))
        pts, ax = np.zeros((n.value, 3)), np.zeros(n.value, np.int32)
        self._check(L.ref_read_observations(os.fsencode(path), C.byref(n), _p(pts), _p(ax)))
        return pts, ax

    def write_greens_bank(self, path, bank, pts, axes, centers, dirs, radii) -> None:
        L = self._io()
        b = np.ascontiguousarray(bank, np.float64)
        arr = [np.ascontiguousarray(x, t) for x, t in ((pts, np.float64), (axes, np.int32), (centers, np.float64),
                                                         (dirs, np.int32), (radii, np.float64))]
        self._check(L.ref_write_greens_bank(os.fsencode(path), b.shape[0], b.shape[1], *[_p(x) for x in arr], _p(b)))

    def read_greens_bank(self, path) -> dict:
        L = self._io()
        rows, cols = C.c_int32(), C.c_int32()
        self._check(L.ref_read_greens_bank(os.fsencode(path), C.byref(rows), C.byref(cols), *([None] * 6)))
        R, K = rows.value, cols.value
        out = dict(values=np.zeros((R, K)), obs_points=np.zeros((R, 3)), obs_axes=np.zeros(R, np.int32),
                   centers=np.zeros((K, 3)), directions=np.zeros(K, np.int32), radii=np.zeros(K))
        self._check(L.ref_read_greens_bank(os.fsencode(path), C.byref(rows), C.byref(cols), _p(out["obs_points"]),
                                           _p(out["obs_axes"]), _p(out["centers"]), _p(out["directions"]),
                                           _p(out["radii"]), _p(out["values"])))
        return out

    def write_mesh(self, m: MeshArrays, path) -> None:
        L = self._io()
        h = self._mesh(m)
        try:
            self._check(L.ref_write_mesh(h, os.fsencode(path)))
        finally:
            self._f("mesh_destroy")(h)

    def read_mesh(self, path) -> MeshArrays:
        L = self._io()
        h = C.c_void_p()
        self._check(L.ref_read_mesh(os.fsencode(path), C.byref(h)))
        try:
            return self._export(h)
        finally:
            self._f("mesh_destroy")(h)

    def write_dirichlet(self, m: MeshArrays, path) -> None:
        L = self._io()
        h = self._mesh(m)
        try:
            self._check(L.ref_write_dirichlet(h, os.fsencode(path)))
        finally:
            self._f("mesh_destroy")(h)

    def read_dirichlet(self, m: MeshArrays, path) -> MeshArrays:
        """read_dirichlet applied to a copy of m; returns the updated arrays."""
        L = self._io()
        h = self._mesh(m)
        try:
            self._check(L.ref_read_dirichlet(h, os.fsencode(path)))
            return self._export(h)
        finally:
            self._f("mesh_destroy")(h)

    def write_solution(self, path, u: np.ndarray) -> None:
        L = self._io()
        a = np.ascontiguousarray(u, np.float64)
        self._check(L.ref_write_solution(os.fsencode(path), _p(a), a.shape[0] // 3, a.shape[1]))

    def read_solution(self, path) -> np.ndarray:
        L = self._io()
        n, b = C.c_int32(), C.c_int32()
        self._check(L.ref_read_solution(os.fsencode(path), C.byref(n), C.byref(b), None))
        out = np.empty((3 * n.value, b.value), np.float64)
        self._check(L.ref_read_solution(os.fsencode(path), C.byref(n), C.byref(b), _p(out)))
        return out

    def hw_threads(self) -> int:
        return int(self.lib.ref_hw_threads()) if self.kind == "reference" else 1

    def time_ebe_apply(self, m: MeshArrays, order, lam, mu, use_mask, prec, workers, batch, reps, seed=12):
        assert self.kind == "reference"
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        sec, chk = C.c_double(), C.c_double()
        h = self._mesh(m)
        try:
            self._check(self.lib.ref_time_ebe_apply(h, order, len(lam), _p(lam), _p(mu), int(use_mask), prec,
                                                    workers, batch, reps, seed, C.byref(sec), C.byref(chk)))
        finally:
            self._f("mesh_destroy")(h)
        return sec.value, chk.value


class Levels:
    """SolverLevels built by the oracle; solve / solve_pcge against it."""

    def __init__(self, orc: Oracle, m: MeshArrays, lam, mu, cfg, workers):
        self.o = orc
        self.cfg = cfg
        lam = np.ascontiguousarray(lam, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        self.mesh_h = orc._mesh(m)
        t = C.c_double()
        self.h = orc._f("levels_create")(self.mesh_h, len(lam), _p(lam), _p(mu), C.byref(cfg), workers, C.byref(t))
        if not self.h:
            orc._f("mesh_destroy")(self.mesh_h)
            raise OracleError(1, orc._f("last_error")().decode())
        self.setup_s = t.value
        n0, n1, n2, nz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        orc._f("levels_sizes")(self.h, C.byref(n0), C.byref(n1), C.byref(n2), C.byref(nz))
        self.n0, self.n1, self.n2, self.nnzb2 = n0.value, n1.value, n2.value, nz.value

    def export(self):
        agg = np.zeros(self.n1, np.int32)
        rp = np.zeros(self.n2 + 1, np.int32)
        ci = np.zeros(self.nnzb2, np.int32)
        bl = np.zeros((self.nnzb2, 9), np.float32)
        m2k = np.zeros(3 * self.n2, np.uint8)
        m0 = np.zeros((self.n0, 9), np.float32)
        m1 = np.zeros((self.n1, 9), np.float32)
        m2 = np.zeros((self.n2, 9), np.float32)
        self.o._f("levels_export")(self.h, _p(agg), _p(rp), _p(ci), _p(bl), _p(m2k), _p(m0), _p(m1), _p(m2))
        return dict(agg=agg, row_ptr2=rp, col_idx2=ci, blocks2=bl, mask2=m2k, m0=m0, m1=m1, m2=m2)

    def outer_apply(self, u):
        u = np.ascontiguousarray(u, np.float64)
        f = np.zeros_like(u)
        self.o._check(self.o._f("levels_outer_apply")(self.h, _p(u), _p(f), u.shape[-1]))
        return f

    def solve(self, f, u0=None, cfg: SolverConfig | None = None, history: int = 0):
        cfg = cfg or self.cfg
        f = np.ascontiguousarray(f, np.float64)
        u0 = np.zeros_like(f) if u0 is None else np.ascontiguousarray(u0, np.float64)
        u = np.zeros_like(f)
        rep, bufs = make_report(f.shape[-1], history)
        rc = self.o._f("solve")(self.h, _p(f), _p(u0), _p(u), f.shape[-1], C.byref(cfg), C.byref(rep))
        if rc != 0:
            err = OracleError(rc, self.o._f("last_error")().decode())
            err.report = report_dict(rep, bufs)
            raise err
        return u, report_dict(rep, bufs)

    def solve_pcge(self, f, u0=None, tol=1e-8, max_iter=100000):
        f = np.ascontiguousarray(f, np.float64)
        u0 = np.zeros_like(f) if u0 is None else np.ascontiguousarray(u0, np.float64)
        u = np.zeros_like(f)
        rep, bufs = make_report(f.shape[-1], 0)
        rc = self.o._f("solve_pcge")(self.h, _p(f), _p(u0), _p(u), f.shape[-1], tol, max_iter, C.byref(rep))
        if rc != 0:
            err = OracleError(rc, self.o._f("last_error")().decode())
            err.report = report_dict(rep, bufs)
            raise err
        return u, report_dict(rep, bufs)

    def __del__(self):
        try:
            self.o._f("levels_destroy")(self.h)
            self.o._f("mesh_destroy")(self.mesh_h)
        except Exception:
            pass


def have_reference() -> bool:
    return os.path.exists(REF_SO)
