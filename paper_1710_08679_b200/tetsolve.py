"""Python mirror of the reference ``tetsolve`` solve-path interface over libtsgpu.

Names, argument meaning and error behaviour follow the reference C++ headers
(/root/reference/proj/include/tetsolve); each class cites the symbol it
mirrors. Vectors are ``[node][axis][case]`` (vector_batch.hpp:12-28): a
``VectorBatch`` here is a 2-D array of shape ``(3 * n_nodes, batch)`` — a
torch CUDA tensor for the device path, or a numpy array for the host path
(copies in/out inside the call, like the reference's host ``VectorBatch``).

Errors map to the reference's exception classes (errors.hpp:9-31):
``ValidationError``, ``SolverError`` and ``ConvergenceError`` (carrying the
report, solver_config.hpp:111-116).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import SolverConfig as _CConfig
from ._lib import SolveReportC as _CReport
from ._lib import lib

try:  # torch is plumbing for device memory and streams only
    import torch
except Exception:  # pragma: no cover
    torch = None


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """tetsolve::Error (errors.hpp:9-12)."""


class ValidationError(Error):
    """tetsolve::ValidationError (errors.hpp:15-18)."""


class ParseError(ValidationError):
    """tetsolve::ParseError (errors.hpp:21-25): message "file:line: msg"."""


class SolverError(Error):
    """tetsolve::SolverError (errors.hpp:27-30)."""


class ConvergenceError(SolverError):
    """tetsolve::ConvergenceError (solver_config.hpp:111-116); carries .report."""

    def __init__(self, msg, report):
        super().__init__(msg)
        self.report = report


class DeviceError(Error):
    """CUDA failure or no device: the product has no CPU fallback."""


def _raise(rc: int, report=None):
    msg = lib.ts_last_error().decode()
    if rc == _lib.TS_ERR_PARSE:
        raise ParseError(msg)
    if rc == _lib.TS_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == _lib.TS_ERR_NO_CONVERGENCE:
        raise ConvergenceError(msg, report)
    if rc in (_lib.TS_ERR_BREAKDOWN, _lib.TS_ERR_NONFINITE):
        raise SolverError(msg)
    raise DeviceError(msg)


def _ck(rc: int, report=None):
    if rc != 0:
        _raise(rc, report)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _device_vec(x, rows: int, dtype, what: str, batch: int | None = None):
    """A (rows, batch) CUDA tensor of `dtype` on the current device, C-contiguous
    (a strided view is copied). Anything else is the reference's ValidationError
    (ebe_operator.hpp:91-93): nothing mismatched ever reaches a kernel."""
    if not _is_torch(x) or not x.is_cuda or x.dtype != dtype or x.ndim != 2 or x.shape[0] != rows:
        raise ValidationError(f"{what}: dimension mismatch")
    if batch is not None and x.shape[1] != batch:
        raise ValidationError(f"{what}: dimension mismatch")
    if x.device.index != torch.cuda.current_device():
        raise ValidationError(f"{what}: tensor is on another device")
    return x if x.is_contiguous() else x.contiguous()


def _host_vec(x, rows: int, dtype, what: str, batch: int | None = None):
    """A (rows, batch) C-contiguous numpy array of `dtype` (converted copy if needed)."""
    if _is_torch(x):
        raise ValidationError(f"{what}: mixes host and device buffers")
    x = np.ascontiguousarray(x, dtype)
    if x.ndim != 2 or x.shape[0] != rows or (batch is not None and x.shape[1] != batch):
        raise ValidationError(f"{what}: dimension mismatch")
    return x


def _host_out(f, like):
    """`f` if it can receive the result in place (same shape/dtype, C-contiguous, writable), else a new array."""
    if (f is not None and not _is_torch(f) and isinstance(f, np.ndarray) and f.shape == like.shape
            and f.dtype == like.dtype and f.flags.c_contiguous and f.flags.writeable):
        return f
    return np.empty_like(like)


# ------------------------------------------------------------------ config
@dataclass
class InnerLoopConfig:
    """tetsolve::InnerLoopConfig (solver_config.hpp:16-19)."""

    tol: float = 0.1
    max_iter: int = 30


@dataclass
class SolverConfig:
    """tetsolve::SolverConfig (solver_config.hpp:21-48); defaults from Table 2."""

    outer_tol: float = 1e-8
    outer_max_iter: int = 5000
    level0: InnerLoopConfig = field(default_factory=lambda: InnerLoopConfig(0.1, 30))
    level1: InnerLoopConfig = field(default_factory=lambda: InnerLoopConfig(0.05, 300))
    level2: InnerLoopConfig = field(default_factory=lambda: InnerLoopConfig(0.025, 3000))
    batch_size: int = 16
    aggregate_target: int = 8
    residual_history_stride: int = 1

    def to_c(self) -> _CConfig:
        c = _CConfig()
        c.outer_tol = self.outer_tol
        c.outer_max_iter = self.outer_max_iter
        c.level_tol[:] = [self.level0.tol, self.level1.tol, self.level2.tol]
        c.level_max_iter[:] = [self.level0.max_iter, self.level1.max_iter, self.level2.max_iter]
        c.batch_size = self.batch_size
        c.aggregate_target = self.aggregate_target
        c.residual_history_stride = self.residual_history_stride
        return c

    def validate(self):
        """SolverConfig::validate (solver_config.hpp:31-47)."""
        c = self.to_c()
        _ck(lib.ts_config_validate(C.byref(c)))


@dataclass
class SolveReport:
    """tetsolve::SolveReport (solver_config.hpp:50-108)."""

    converged: bool = False
    residual_history_stride: int = 0
    outer_iterations: int = 0
    inner_iterations: list = field(default_factory=lambda: [0, 0, 0])
    final_rel_residual: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residual_history: list = field(default_factory=list)  # [(iter, per-column ndarray)]
    time_setup_s: float = 0.0
    time_outer_s: float = 0.0
    time_inner_s: list = field(default_factory=lambda: [0.0, 0.0, 0.0])
    time_total_s: float = 0.0
    batch_size: int = 0
    method: str = "amg"
    inner_precision: str = "float32"

    def max_final_residual(self) -> float:
        return float(self.final_rel_residual.max()) if len(self.final_rel_residual) else 0.0


class _ReportBuf:
    def __init__(self, batch: int, capacity: int):
        self.c = _CReport()
        self.final = np.zeros(batch, np.float64)
        self.hit = np.zeros(max(capacity, 1), np.int32)
        self.hist = np.zeros((max(capacity, 1), batch), np.float64)
        self.c.final_rel_residual = self.final.ctypes.data_as(C.POINTER(C.c_double))
        self.c.history_iter = self.hit.ctypes.data_as(C.POINTER(C.c_int32))
        self.c.history = self.hist.ctypes.data_as(C.POINTER(C.c_double))
        self.c.history_capacity = capacity

    def report(self, stride: int) -> SolveReport:
        c = self.c
        n = c.history_count
        return SolveReport(
            converged=bool(c.converged),
            residual_history_stride=stride,
            outer_iterations=int(c.outer_iterations),
            inner_iterations=[int(x) for x in c.inner_iterations],
            final_rel_residual=self.final.copy(),
            residual_history=[(int(self.hit[i]), self.hist[i].copy()) for i in range(n)],
            time_setup_s=float(c.time_setup_s),
            time_outer_s=float(c.time_outer_s),
            time_inner_s=[float(x) for x in c.time_inner_s],
            time_total_s=float(c.time_total_s),
            batch_size=int(c.batch_size),
            method="pcge" if c.method == 1 else "amg",
            inner_precision="float64" if c.inner_precision == 64 else "float32",
        )


# -------------------------------------------------------------- materials
@dataclass
class Material:
    """tetsolve::Material (material.hpp:14-20)."""

    vp: float = 0.0
    vs: float = 0.0
    rho: float = 0.0
    lam: float = 0.0
    mu: float = 0.0


def material_from_wavespeeds(vp: float, vs: float, rho: float) -> Material:
    """material_from_wavespeeds (material.hpp:22-34)."""
    lam, mu = C.c_double(), C.c_double()
    _ck(lib.ts_material_from_wavespeeds(vp, vs, rho, C.byref(lam), C.byref(mu)))
    return Material(vp, vs, rho, lam.value, mu.value)


def _lame(materials):
    lam = np.ascontiguousarray([m.lam for m in materials], np.float64)
    mu = np.ascontiguousarray([m.mu for m in materials], np.float64)
    return lam, mu


# ------------------------------------------------------------------- mesh
FIXED = {"none": 0, "bottom_and_sides": 1, "all_clamped": 2}


class Mesh:
    """tetsolve::Mesh (mesh.hpp:26-42), held by libtsgpu as a host container."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        nn, nv, ne, nbc = (C.c_int32() for _ in range(4))
        _ck(lib.ts_mesh_sizes(self._h, C.byref(nn), C.byref(nv), C.byref(ne), C.byref(nbc)))
        self._sizes = (nn.value, nv.value, ne.value, nbc.value)
        self._arrays = None

    @classmethod
    def from_arrays(cls, coords, tets10, material_id, vertex_count, bc_node=(), bc_axis=()):
        c = np.ascontiguousarray(coords, np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(tets10, np.int32).reshape(-1, 10)
        m = np.ascontiguousarray(material_id, np.int32)
        bn = np.ascontiguousarray(bc_node, np.int32)
        ba = np.ascontiguousarray(bc_axis, np.int8)
        h = C.c_void_p()
        _ck(lib.ts_mesh_from_arrays(c.shape[0], vertex_count, _p(c), t.shape[0], _p(t), _p(m),
                                    len(bn), _p(bn) if len(bn) else None, _p(ba) if len(ba) else None,
                                    C.byref(h)))
        return cls(h)

    def node_count(self) -> int:
        return self._sizes[0]

    @property
    def vertex_count(self) -> int:
        return self._sizes[1]

    def element_count(self) -> int:
        return self._sizes[2]

    def arrays(self):
        if self._arrays is None:
            nn, nv, ne, nbc = self._sizes
            coords = np.zeros((nn, 3), np.float64)
            tets = np.zeros((ne, 10), np.int32)
            mat = np.zeros(ne, np.int32)
            bn = np.zeros(max(nbc, 1), np.int32)
            ba = np.zeros(max(nbc, 1), np.int8)
            _ck(lib.ts_mesh_export(self._h, _p(coords), _p(tets), _p(mat), _p(bn), _p(ba)))
            self._arrays = dict(coords=coords, tets10=tets, material_id=mat, bc_node=bn[:nbc], bc_axis=ba[:nbc])
        return self._arrays

    @property
    def coords(self):
        return self.arrays()["coords"]

    @property
    def tets10(self):
        return self.arrays()["tets10"]

    @property
    def material_id(self):
        return self.arrays()["material_id"]

    def dirichlet_mask(self) -> np.ndarray:
        mask = np.zeros(3 * self.node_count(), np.uint8)
        _ck(lib.ts_mesh_dirichlet_mask(self._h, _p(mask)))
        return mask

    def __del__(self):
        try:
            lib.ts_mesh_destroy(self._h)
        except Exception:
            pass


def generate_box_mesh(extents, divisions, layer_interfaces=(), fixed_boundary="bottom_and_sides") -> Mesh:
    """generate_box_mesh (box_mesh.hpp:55-157), identical numbering."""
    ext = np.ascontiguousarray(extents, np.float64)
    div = np.ascontiguousarray(divisions, np.int32)
    ifs = np.ascontiguousarray(layer_interfaces, np.float64) if len(layer_interfaces) else None
    fb = FIXED[fixed_boundary] if isinstance(fixed_boundary, str) else int(fixed_boundary)
    h = C.c_void_p()
    _ck(lib.ts_box_mesh(_p(ext), _p(div), len(layer_interfaces), _p(ifs), fb, C.byref(h)))
    return Mesh(h)


def dirichlet_mask(mesh: Mesh) -> np.ndarray:
    """dirichlet_mask (mesh.hpp:150-154)."""
    return mesh.dirichlet_mask()


# ------------------------------------------------------------ file formats
def _path(p) -> bytes:
    import os

    return os.fsencode(p)


def write_mesh(mesh: Mesh, path) -> None:
    """write_mesh (mesh_io.hpp:20-36): TSMESH 1 text, byte-identical, atomic replace."""
    _ck(lib.ts_mesh_write_tsmesh(mesh._h, _path(path)))


def read_mesh(path) -> Mesh:
    """read_mesh (mesh_io.hpp:44-96): ParseError on a malformed line, then
    validate_mesh (ValidationError naming the first bad element). No Dirichlet
    entries (see read_dirichlet)."""
    h = C.c_void_p()
    _ck(lib.ts_mesh_read_tsmesh(_path(path), C.byref(h)))
    return Mesh(h)


def write_dirichlet(mesh: Mesh, path) -> None:
    """write_dirichlet (mesh_io.hpp:38-42): one "node axis" line per entry."""
    _ck(lib.ts_mesh_write_dirichlet(mesh._h, _path(path)))


def read_dirichlet(mesh: Mesh, path) -> None:
    """read_dirichlet (mesh_io.hpp:98-115): replaces the mesh's Dirichlet list in place."""
    _ck(lib.ts_mesh_read_dirichlet(mesh._h, _path(path)))
    mesh.__init__(mesh._h)


def write_mesh_binary(mesh: Mesh, path) -> None:
    """TSBMESH 1 (this library's binary mesh, Dirichlet list included)."""
    _ck(lib.ts_mesh_write_tsbmesh(mesh._h, _path(path)))


def read_mesh_binary(path) -> Mesh:
    """Read a TSBMESH 1 file; validated like read_mesh."""
    h = C.c_void_p()
    _ck(lib.ts_mesh_read_tsbmesh(_path(path), C.byref(h)))
    return Mesh(h)


def write_solution(u, path) -> None:
    """write_solution (solution_io.hpp:14-27) of a (3 * n_nodes, batch) fp64
    VectorBatch: numpy (host) or a CUDA tensor (streamed from the device)."""
    if _is_torch(u):
        if u.dtype != torch.float64 or u.dim() != 2 or u.shape[0] % 3 or not u.is_contiguous():
            raise ValidationError("write_solution: expected a contiguous float64 tensor of shape (3 * n_nodes, batch)")
        if u.is_cuda:
            torch.cuda.current_stream().synchronize()
            _ck(lib.ts_tsvec_write(_path(path), C.c_void_p(u.data_ptr()), u.shape[0] // 3, u.shape[1], 1))
            return
        u = u.numpy()
    a = np.ascontiguousarray(u, np.float64)
    if a.ndim != 2 or a.shape[0] % 3:
        raise ValidationError("write_solution: expected shape (3 * n_nodes, batch)")
    _ck(lib.ts_tsvec_write(_path(path), _p(a), a.shape[0] // 3, a.shape[1], 0))


def read_solution(path, device=None):
    """read_solution (solution_io.hpp:29-84) -> (3 * n_nodes, batch) fp64;
    numpy, or a CUDA tensor on ``device`` (streamed to the device)."""
    n, b = C.c_int64(), C.c_int32()
    _ck(lib.ts_tsvec_info(_path(path), C.byref(n), C.byref(b)))
    if device is not None:
        out = torch.empty((3 * n.value, b.value), dtype=torch.float64, device=device)
        _ck(lib.ts_tsvec_read(_path(path), C.c_void_p(out.data_ptr()), n.value, b.value, 1))
        return out
    out = np.empty((3 * n.value, b.value), np.float64)
    _ck(lib.ts_tsvec_read(_path(path), _p(out), n.value, b.value, 0))
    return out


# -------------------------------------------------------------- operators
def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class EbeOperator:
    """EbeOperator<T> (ebe_operator.hpp:29-226) on the device.

    ``prec`` is 32 (EbeOperator<float>) or 64 (EbeOperator<double>). ``workers``
    is accepted for signature compatibility and ignored (the device kernel is
    order-independent up to rounding).
    """

    def __init__(self, mesh: Mesh, order: int, materials, dof_mask=None, workers: int = 1, prec: int = 64,
                 _borrowed=None):
        self._own = _borrowed is None
        if _borrowed is not None:
            self._h = _borrowed if isinstance(_borrowed, C.c_void_p) else C.c_void_p(_borrowed)
        else:
            lam, mu = _lame(materials)
            mk = None if dof_mask is None or len(dof_mask) == 0 else np.ascontiguousarray(dof_mask, np.uint8)
            if mk is not None:
                nn = mesh.vertex_count if order == 1 else mesh.node_count()
                if len(mk) != 3 * nn:
                    raise ValidationError("ebe: dof mask length mismatch")
            self._h = C.c_void_p()
            _ck(lib.ts_ebe_create(mesh._h, order, len(lam), _p(lam), _p(mu), _p(mk), prec, C.byref(self._h)))
        nn, ne, od, pr = (C.c_int32() for _ in range(4))
        _ck(lib.ts_ebe_info(self._h, C.byref(nn), C.byref(ne), C.byref(od), C.byref(pr)))
        self._n, self._e, self._order, self.prec = nn.value, ne.value, od.value, pr.value
        self.dtype_np = np.float32 if self.prec == 32 else np.float64

    def n_nodes(self) -> int:
        return self._n

    def n_elements(self) -> int:
        return self._e

    def order(self) -> int:
        return self._order

    def nodes_per_element(self) -> int:
        return 4 if self._order == 1 else 10

    def apply(self, u, f=None):
        """f = A u for all batch columns (ebe_operator.hpp:90-134). Like the
        reference's apply, an `f` of the wrong shape is replaced (here: also a
        wrong dtype, device or a non-contiguous one), never written through."""
        if u.ndim != 2 or u.shape[0] != 3 * self._n:
            raise ValidationError("ebe apply: dimension mismatch")
        batch = int(u.shape[1])
        if _is_torch(u):
            want = torch.float32 if self.prec == 32 else torch.float64
            u = _device_vec(u, 3 * self._n, want, "ebe apply")
            if not (_is_torch(f) and f.shape == u.shape and f.dtype == u.dtype and f.device == u.device
                    and f.is_contiguous()):
                f = torch.empty_like(u)
            _ck(lib.ts_ebe_apply(self._h, C.c_void_p(u.data_ptr()), C.c_void_p(f.data_ptr()), batch, _stream()))
            return f
        u = _host_vec(u, 3 * self._n, self.dtype_np, "ebe apply")
        out = _host_out(f, u)
        _ck(lib.ts_ebe_apply_host(self._h, _p(u), _p(out), batch))
        return out

    def element_matrix(self, e: int) -> np.ndarray:
        """element_matrix (ebe_operator.hpp:78-87): fp64 K_e [3 npe, 3 npe] of element e."""
        n = 3 * self.nodes_per_element()
        k = np.zeros((n, n), np.float64)
        _ck(lib.ts_ebe_element_matrix(self._h, int(e), _p(k)))
        return k

    def set_deterministic(self, on: bool = True):
        """Colored, order-fixed sweep (bitwise reproducible, batch-independent bits)."""
        _ck(lib.ts_ebe_set_deterministic(self._h, 1 if on else 0))
        return self

    def launches_per_apply(self, batch: int) -> int:
        n = C.c_int32()
        _ck(lib.ts_ebe_launches_per_apply(self._h, int(batch), C.byref(n)))
        return n.value

    def unit_stats(self) -> dict:
        """The element sweep's unit plan (edge fans / face pairs / elements)."""
        k, u = C.c_int32(), C.c_int32()
        rpe, cf, epu = C.c_double(), C.c_double(), C.c_double()
        _ck(lib.ts_ebe_unit_stats(self._h, C.byref(k), C.byref(u), C.byref(rpe), C.byref(cf), C.byref(epu)))
        return {"kind": {2: "fans", 1: "pairs", 0: "elements"}[k.value], "units": u.value,
                "rows_per_element": rpe.value, "closed_fraction": cf.value, "elements_per_unit": epu.value}

    def host_stream_chunks(self) -> int:
        """Chunks of the pinned-host streaming schedule (0 = copy-apply-copy)."""
        n = C.c_int32()
        _ck(lib.ts_ebe_host_stream_chunks(self._h, C.byref(n)))
        return n.value

    def block_jacobi(self) -> np.ndarray:
        """extract_block_jacobi(EbeOperator) (ebe_operator.hpp:288-313): [n_nodes, 9]."""
        inv = np.zeros((self._n, 9), self.dtype_np)
        _ck(lib.ts_ebe_block_jacobi_host(self._h, _p(inv)))
        return inv

    def set_timing(self, enable: bool = True):
        _ck(lib.ts_ebe_set_timing(self._h, int(enable)))

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        _ck(lib.ts_ebe_last_kernel_ms(self._h, C.byref(ms)))
        return ms.value

    def __del__(self):
        if getattr(self, "_own", False):
            try:
                lib.ts_ebe_destroy(self._h)
            except Exception:
                pass


# ------------------------------------------------------------------ solver
def assemble_bcsr(op: EbeOperator) -> "BlockCsrMatrix":
    """assemble_bcsr (ebe_operator.hpp:230-284): identity rows at constrained dofs, constrained
    columns dropped, fp64 sums in element order rounded to the operator precision (device)."""
    nnzb = C.c_int64()
    _ck(lib.ts_ebe_assemble_bcsr(op._h, C.byref(nnzb), None, None, None))
    rp = np.zeros(op.n_nodes() + 1, np.int32)
    ci = np.zeros(nnzb.value, np.int32)
    bl = np.zeros((nnzb.value, 9), op.dtype_np)
    _ck(lib.ts_ebe_assemble_bcsr(op._h, C.byref(nnzb), _p(rp), _p(ci), _p(bl)))
    return BlockCsrMatrix(op.n_nodes(), rp, ci, bl)


class BlockCsrMatrix:
    """BlockCsrMatrix<T> (block_csr.hpp:16-70): 3x3-block CSR held on the device; apply =
    fp64 row accumulation in stored-block order rounded to T (bit-exact vs the reference)."""

    def __init__(self, n_block_rows: int, row_ptr, col_idx, blocks):
        self.n_block_rows = int(n_block_rows)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        bl = np.asarray(blocks)
        self.prec = 32 if bl.dtype == np.float32 else 64
        self.blocks = np.ascontiguousarray(bl, np.float32 if self.prec == 32 else np.float64).reshape(-1, 9)
        self._h = C.c_void_p()
        _ck(lib.ts_bcsr_create(self.n_block_rows, _p(self.row_ptr), _p(self.col_idx), _p(self.blocks), self.prec,
                               C.byref(self._h)))

    def apply(self, u, f=None):
        rows = 3 * self.n_block_rows
        if _is_torch(u):
            u = _device_vec(u, rows, torch.float32 if self.prec == 32 else torch.float64, "bcsr apply")
            f = torch.empty_like(u)
            _ck(lib.ts_bcsr_apply(self._h, C.c_void_p(u.data_ptr()), C.c_void_p(f.data_ptr()), int(u.shape[1]),
                                  _stream()))
            return f
        u = _host_vec(u, rows, np.float32 if self.prec == 32 else np.float64, "bcsr apply")
        out = _host_out(f, u)
        _ck(lib.ts_bcsr_apply_host(self._h, _p(u), _p(out), int(u.shape[1])))
        return out

    def block_jacobi(self) -> "BlockJacobi":
        """extract_block_jacobi(BlockCsrMatrix) (block_jacobi.hpp:72-85)."""
        inv = np.zeros((self.n_block_rows, 9), self.blocks.dtype)
        _ck(lib.ts_bcsr_block_jacobi_host(self._h, _p(inv)))
        return BlockJacobi(inv)

    def __del__(self):
        try:
            lib.ts_bcsr_destroy(self._h)
        except Exception:
            pass


class BlockJacobi:
    """BlockJacobi<T> (block_jacobi.hpp:15-39): z = M^-1 r, fp64 math rounded to T (device)."""

    def __init__(self, inv_blocks):
        inv = np.asarray(inv_blocks)
        self.prec = 32 if inv.dtype == np.float32 else 64
        self.inv_blocks = np.ascontiguousarray(inv, np.float32 if self.prec == 32 else np.float64).reshape(-1, 9)
        self._h = C.c_void_p()
        _ck(lib.ts_bj_create(len(self.inv_blocks), _p(self.inv_blocks), self.prec, C.byref(self._h)))

    def n_nodes(self) -> int:
        return len(self.inv_blocks)

    def apply(self, r, z=None):
        rows = 3 * self.n_nodes()
        if _is_torch(r):
            r = _device_vec(r, rows, torch.float32 if self.prec == 32 else torch.float64, "block jacobi apply")
            z = torch.empty_like(r)
            _ck(lib.ts_bj_apply(self._h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), int(r.shape[1]),
                                _stream()))
            return z
        r = _host_vec(r, rows, np.float32 if self.prec == 32 else np.float64, "block jacobi apply")
        out = _host_out(z, r)
        _ck(lib.ts_bj_apply_host(self._h, _p(r), _p(out), int(r.shape[1])))
        return out

    def __del__(self):
        try:
            lib.ts_bj_destroy(self._h)
        except Exception:
            pass


class Prolongation:
    """Prolongation (prolongation.hpp:13-62): per-fine-node CSR, the same weights on every
    axis; apply = P coarse, restrict_to_coarse = P^T fine (ascending fine rows), in T (device)."""

    def __init__(self, n_fine: int, n_coarse: int, row_ptr, cols, weights):
        self.n_fine_nodes, self.n_coarse_nodes = int(n_fine), int(n_coarse)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.cols = np.ascontiguousarray(cols, np.int32)
        self.weights = np.ascontiguousarray(weights, np.float64)
        self._h = C.c_void_p()
        _ck(lib.ts_prolong_create(self.n_fine_nodes, self.n_coarse_nodes, _p(self.row_ptr), _p(self.cols),
                                  _p(self.weights), C.byref(self._h)))

    def _run(self, x, restrict: bool):
        n_in, n_out = (self.n_fine_nodes, self.n_coarse_nodes) if restrict else (self.n_coarse_nodes,
                                                                                 self.n_fine_nodes)
        what = "prolongation restrict: fine" if restrict else "prolongation apply: coarse"
        if _is_torch(x):
            if x.dtype not in (torch.float32, torch.float64):
                raise ValidationError(f"{what} dimension mismatch")
            x = _device_vec(x, 3 * n_in, x.dtype, what)
            prec = 32 if x.dtype == torch.float32 else 64
            y = torch.empty((3 * n_out, x.shape[1]), dtype=x.dtype, device=x.device)
            fn = lib.ts_prolong_restrict if restrict else lib.ts_prolong_apply
            _ck(fn(self._h, prec, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), int(x.shape[1]), _stream()))
            return y
        x = np.asarray(x)
        dt = np.float32 if x.dtype == np.float32 else np.float64
        x = _host_vec(x, 3 * n_in, dt, what)
        y = np.empty((3 * n_out, x.shape[1]), dt)
        _ck(lib.ts_prolong_apply_host(self._h, 32 if dt == np.float32 else 64, 1 if restrict else 0, _p(x), _p(y),
                                      int(x.shape[1])))
        return y

    def apply(self, coarse):
        return self._run(coarse, False)

    def restrict_to_coarse(self, fine):
        return self._run(fine, True)

    def __del__(self):
        try:
            lib.ts_prolong_destroy(self._h)
        except Exception:
            pass


def build_geometric_prolongation(mesh: Mesh) -> Prolongation:
    """build_geometric_prolongation (prolongation.hpp:67-98)."""
    n, v = mesh.node_count(), mesh.vertex_count
    rp = np.zeros(n + 1, np.int32)
    cols = np.zeros(v + 2 * (n - v), np.int32)
    w = np.zeros(v + 2 * (n - v), np.float64)
    _ck(lib.ts_geometric_prolongation(mesh._h, _p(rp), _p(cols), _p(w)))
    return Prolongation(n, v, rp, cols, w)


class InnerStats:
    """InnerStats (pcg.hpp:15-18)."""

    def __init__(self, iterations: int, converged: bool):
        self.iterations, self.converged = iterations, converged


def inner_pcg(a, m: BlockJacobi, r, u, tol: float, max_iter: int) -> InnerStats:
    """inner_pcg (pcg.hpp:52-124) on an EbeOperator or a BlockCsrMatrix with the block-Jacobi
    preconditioner m; u (warm start) is updated in place. CUDA tensors or numpy arrays."""
    kind = 0 if isinstance(a, EbeOperator) else 1
    n = a.n_nodes() if kind == 0 else a.n_block_rows
    it, conv = C.c_int32(), C.c_int32()
    if _is_torch(r):
        dt = torch.float32 if a.prec == 32 else torch.float64
        r = _device_vec(r, 3 * n, dt, "inner_pcg")
        if not (_is_torch(u) and u.is_contiguous()):
            raise ValidationError("inner_pcg: u must be a contiguous CUDA tensor (updated in place)")
        _device_vec(u, 3 * n, dt, "inner_pcg", int(r.shape[1]))
        _ck(lib.ts_inner_pcg(kind, a._h, m._h, C.c_void_p(r.data_ptr()), C.c_void_p(u.data_ptr()), n,
                             int(r.shape[1]), float(tol), int(max_iter), C.byref(it), C.byref(conv), _stream()))
    else:
        dt = np.float32 if a.prec == 32 else np.float64
        r = _host_vec(r, 3 * n, dt, "inner_pcg")
        if not (isinstance(u, np.ndarray) and u.dtype == dt and u.flags.c_contiguous and u.shape == r.shape):
            raise ValidationError("inner_pcg: u must be a contiguous array of r's shape and dtype (updated in place)")
        _ck(lib.ts_inner_pcg_host(kind, a._h, m._h, _p(r), _p(u), n, int(r.shape[1]), float(tol), int(max_iter),
                                  C.byref(it), C.byref(conv)))
    return InnerStats(it.value, bool(conv.value))


class SolverLevels:
    """SolverLevels (adaptive_cg.hpp:27-37) built on the device by
    build_solver_levels (adaptive_cg.hpp:39-67)."""

    def __init__(self, handle, mesh: Mesh, owner=None):
        self._h = handle
        self.mesh = mesh
        self._owner = owner  # set: a level set owned by another object (e.g. a faulted model), not destroyed here
        n0, n1, n2, nz = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        _ck(lib.ts_levels_sizes(self._h, C.byref(n0), C.byref(n1), C.byref(n2), C.byref(nz)))
        self.n0, self.n1, self.n2, self.nnzb2 = n0.value, n1.value, n2.value, nz.value
        ops = []
        for which in range(3):
            h = C.c_void_p()
            _ck(lib.ts_levels_operator(self._h, which, C.byref(h)))
            ops.append(EbeOperator(None, 0, None, _borrowed=h))
        self.outer, self.level0, self.level1 = ops

    def apply(self, which: int, u, f=None):
        """The level operator the solve applies (CUDA tensors): 0 outer fp64, 1 level-0
        fp32 tet10, 2 level-1 fp32 tet4 (assembled K1 unless TSGPU_L1=ebe), 3 level-2 BCSR."""
        if which not in (0, 1, 2, 3):
            raise ValidationError("levels apply: operator index must be 0 (outer), 1 (level0), 2 (level1) or 3")
        rows = 3 * (self.n1 if which == 2 else self.n2 if which == 3 else self.n0)
        u = _device_vec(u, rows, torch.float64 if which == 0 else torch.float32, "levels apply")
        if not (_is_torch(f) and f.shape == u.shape and f.dtype == u.dtype and f.device == u.device
                and f.is_contiguous()):
            f = torch.empty_like(u)
        _ck(lib.ts_levels_apply(self._h, int(which), C.c_void_p(u.data_ptr()), C.c_void_p(f.data_ptr()),
                                int(u.shape[1]), _stream()))
        return f

    def transfer(self, which: int, x):
        """The solve's inter-grid transfers (fp32 CUDA tensors), each followed by zero_masked:
        0 u0 = P1 u1, 1 r1 = P1^T r0, 2 u1 = P2 u2, 3 r2 = P2^T r1."""
        n_in = {0: self.n1, 1: self.n0, 2: self.n2, 3: self.n1}[which]
        n_out = {0: self.n0, 1: self.n1, 2: self.n1, 3: self.n2}[which]
        x = _device_vec(x, 3 * n_in, torch.float32, "levels transfer")
        y = torch.empty((3 * n_out, x.shape[1]), dtype=torch.float32, device=x.device)
        _ck(lib.ts_levels_transfer(self._h, int(which), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                   int(x.shape[1]), _stream()))
        return y

    def export(self) -> dict:
        """Setup introspection: aggregation, level-2 Galerkin matrix, masks, M2."""
        agg = np.zeros(self.n1, np.int32)
        rp = np.zeros(self.n2 + 1, np.int32)
        ci = np.zeros(self.nnzb2, np.int32)
        bl = np.zeros((self.nnzb2, 9), np.float32)
        mk = np.zeros(3 * self.n2, np.uint8)
        m2 = np.zeros((self.n2, 9), np.float32)
        _ck(lib.ts_levels_export(self._h, _p(agg), _p(rp), _p(ci), _p(bl), _p(mk), _p(m2)))
        return dict(agg=agg, row_ptr2=rp, col_idx2=ci, blocks2=bl, mask2=mk, m2=m2)

    def __del__(self):
        if self._owner is not None:
            return
        try:
            # borrowed operators must not outlive the level set
            for op in (self.outer, self.level0, self.level1):
                op._own = False
            lib.ts_levels_destroy(self._h)
        except Exception:
            pass


def build_solver_levels(mesh: Mesh, materials, dof_mask=None, cfg: SolverConfig | None = None,
                        workers: int = 1) -> SolverLevels:
    """build_solver_levels (adaptive_cg.hpp:39-67); dof_mask None -> dirichlet_mask(mesh)."""
    cfg = cfg or SolverConfig()
    lam, mu = _lame(materials)
    mk = None if dof_mask is None else np.ascontiguousarray(dof_mask, np.uint8)
    c = cfg.to_c()
    h = C.c_void_p()
    _ck(lib.ts_levels_create(mesh._h, len(lam), _p(lam), _p(mu), _p(mk), C.byref(c), C.byref(h)))
    return SolverLevels(h, mesh)


@dataclass
class CrustModel:
    """CrustModel (model.hpp:14-19)."""

    mesh: Mesh
    materials: list
    mask: np.ndarray
    levels: SolverLevels


def build_crust_model(mesh: Mesh, materials, cfg: SolverConfig | None = None, workers: int = 1) -> CrustModel:
    """build_crust_model (model.hpp:21-29)."""
    mask = mesh.dirichlet_mask()
    return CrustModel(mesh, list(materials), mask, build_solver_levels(mesh, materials, mask, cfg, workers))


def solve(levels: SolverLevels, f, u0, cfg: SolverConfig | None = None, history: int = 4096, out=None):
    """solve (adaptive_cg.hpp:242-263). f, u0: (3N, batch) numpy (host path) or
    CUDA float64 tensors (device path); `out` optionally receives u (e.g. a
    pinned host array). Returns (u, SolveReport)."""
    cfg = cfg or SolverConfig()
    c = cfg.to_c()
    if f.ndim != 2:
        raise ValidationError("solve: dimension mismatch")
    batch = int(f.shape[1])
    rows = 3 * levels.n0
    rb = _ReportBuf(batch, history if cfg.residual_history_stride > 0 else 0)
    if _is_torch(f):
        f = _device_vec(f, rows, torch.float64, "solve")
        u0 = _device_vec(u0, rows, torch.float64, "solve: initial guess", batch)
        u = torch.empty_like(f)
        rc = lib.ts_solve_device(levels._h, C.c_void_p(f.data_ptr()), C.c_void_p(u0.data_ptr()),
                                 C.c_void_p(u.data_ptr()), levels.n0, batch, C.byref(c), C.byref(rb.c), _stream())
    else:
        f = _host_vec(f, rows, np.float64, "solve")
        u0 = _host_vec(u0, rows, np.float64, "solve: initial guess", batch)
        u = _host_out(out, f)
        rc = lib.ts_solve(levels._h, _p(f), _p(u0), _p(u), levels.n0, batch, C.byref(c), C.byref(rb.c))
    rep = rb.report(cfg.residual_history_stride)
    _ck(rc, rep)
    return u, rep


def solve_pcge(k: EbeOperator, f, u0, tol: float, max_iter: int):
    """solve_pcge (adaptive_cg.hpp:267-279): 64-bit CG + 3x3 block Jacobi."""
    if k.prec != 64:
        raise ValidationError("solve_pcge: needs the 64-bit second-order operator")
    f = _host_vec(f, 3 * k.n_nodes(), np.float64, "ebe apply")
    batch = int(f.shape[1])
    u0 = _host_vec(u0, 3 * k.n_nodes(), np.float64, "ebe apply", batch)
    rb = _ReportBuf(batch, 0)
    u = np.empty_like(f)
    rc = lib.ts_solve_pcge(k._h, _p(f), _p(u0), _p(u), k.n_nodes(), batch, tol, max_iter, C.byref(rb.c))
    rep = rb.report(0)
    _ck(rc, rep)
    return u, rep
