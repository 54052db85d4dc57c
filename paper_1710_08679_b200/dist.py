"""Partitioned (multi-GPU) solve path — Python mirror of include/tsgpu.h's
``ts_comm_* / ts_partition_rcb / ts_dist_*`` entries.

The reference has no distributed solve; this is the paper's: the mesh is cut
into element partitions (recursive coordinate bisection), one rank per GPU,
interface-node partial sums are exchanged inside every EBE product (NCCL
send/recv, overlapped with the interior elements) and dot products are
all-reduced. Vectors live in each rank's LOCAL node order; ``local_nodes()``
maps local -> global so callers scatter / gather with plain indexing.

Communicators:
  * ``Comm.nccl_from_torch()`` — one process per GPU under torchrun: rank 0
    creates the NCCL id, torch.distributed broadcasts it.
  * ``ThreadWorld`` + ``Comm.thread(...)`` — P ranks as P host threads of one
    process (any devices, including one shared GPU), used to exercise the
    partitioned solve on a single B200.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib
from .tetsolve import (Mesh, SolverConfig, _ck, _device_vec, _host_vec, _is_torch, _lame, _p, _ReportBuf,
                       _stream)


class ThreadWorld:
    """A group of in-process ranks (ts_thread_world)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _ck(lib.ts_thread_world_create(int(nranks), C.byref(h)))
        self._h, self.nranks = h, int(nranks)

    def __del__(self):
        try:
            lib.ts_thread_world_destroy(self._h)
        except Exception:
            pass


class Comm:
    """tsg::Comm handle (NCCL or in-process threads)."""

    def __init__(self, handle, keep=None):
        self._h, self._keep = handle, keep
        r, n, d = C.c_int32(), C.c_int32(), C.c_int32()
        _ck(lib.ts_comm_info(self._h, C.byref(r), C.byref(n), C.byref(d)))
        self.rank, self.size, self.device = r.value, n.value, d.value

    @classmethod
    def thread(cls, world: ThreadWorld, rank: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        _ck(lib.ts_comm_create_thread(world._h, int(rank), int(device), C.byref(h)))
        return cls(h, keep=world)

    def allreduce_sum(self, t):
        """In-place sum over the ranks of a CUDA float64 tensor (on the current stream)."""
        import torch

        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("allreduce_sum: expected a contiguous CUDA float64 tensor")
        _ck(lib.ts_comm_allreduce_sum(self._h, C.c_void_p(t.data_ptr()), t.numel(),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return t

    @staticmethod
    def nccl_available() -> tuple[bool, str]:
        buf = C.create_string_buffer(256)
        rc = lib.ts_comm_nccl_available(buf, 256)
        return rc == 0, buf.value.decode()

    @staticmethod
    def nccl_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _ck(lib.ts_comm_nccl_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, nranks: int, rank: int, uid: bytes, device: int) -> "Comm":
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _ck(lib.ts_comm_create_nccl(int(nranks), int(rank), buf, int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def nccl_from_torch(cls, device: int) -> "Comm":
        """NCCL communicator over the ranks of the default torch.distributed group."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.nccl(world, rank, obj[0], device)

    def __del__(self):
        try:
            lib.ts_comm_destroy(self._h)
        except Exception:
            pass


def partition_rcb(mesh: Mesh, nparts: int) -> np.ndarray:
    """Element parts [E] by recursive coordinate bisection of centroids."""
    part = np.zeros(mesh.element_count(), np.int32)
    _ck(lib.ts_partition_rcb(mesh._h, int(nparts), _p(part)))
    return part


def dist_plan(mesh: Mesh, part, nranks: int, rank: int, dof_mask=None) -> dict:
    """Host-only partition plan of one rank (no device needed)."""
    part = np.ascontiguousarray(part, np.int32)
    mk = None if dof_mask is None else np.ascontiguousarray(dof_mask, np.uint8)
    nl, nv, ne, nn = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    nh = C.c_int64()
    _ck(lib.ts_dist_plan_sizes(mesh._h, _p(mk), _p(part), int(nranks), int(rank), C.byref(nl), C.byref(nv),
                               C.byref(ne), C.byref(nn), C.byref(nh)))
    out = dict(l2g=np.zeros(nl.value, np.int32), owned=np.zeros(nl.value, np.uint8),
               elems=np.zeros(ne.value, np.int32), nbr=np.zeros(nn.value, np.int32),
               nbr_rows=np.zeros(nn.value, np.int32), halo_rows=np.zeros(nh.value, np.int32))
    _ck(lib.ts_dist_plan_export(mesh._h, _p(mk), _p(part), int(nranks), int(rank), _p(out["l2g"]), _p(out["owned"]),
                                _p(out["elems"]), _p(out["nbr"]), _p(out["nbr_rows"]), _p(out["halo_rows"])))
    out["n_local_vertices"] = nv.value
    rows, o = [], 0
    for k in range(nn.value):
        rows.append(out["halo_rows"][o:o + out["nbr_rows"][k]])
        o += out["nbr_rows"][k]
    out["rows"] = rows
    return out


class DistLevels:
    """build_solver_levels (adaptive_cg.hpp:39-67) on one rank's partition."""

    @classmethod
    def _view(cls, handle, comm: Comm, owner) -> "DistLevels":
        """A level set owned by another object (e.g. DistFaultedModel's base hierarchy)."""
        self = cls.__new__(cls)
        self._h, self.comm, self.mesh, self._owner = handle, comm, None, owner
        n0, n1, n2 = C.c_int32(), C.c_int32(), C.c_int32()
        _ck(lib.ts_dist_levels_sizes(self._h, C.byref(n0), C.byref(n1), C.byref(n2)))
        self.n_local, self.n_local_vertices, self.n2 = n0.value, n1.value, n2.value
        return self

    def __init__(self, mesh: Mesh, materials, part, comm: Comm, cfg: SolverConfig | None = None, dof_mask=None):
        cfg = cfg or SolverConfig()
        lam, mu = _lame(materials)
        part = np.ascontiguousarray(part, np.int32)
        mk = None if dof_mask is None else np.ascontiguousarray(dof_mask, np.uint8)
        c = cfg.to_c()
        h = C.c_void_p()
        _ck(lib.ts_dist_levels_create(mesh._h, len(lam), _p(lam), _p(mu), _p(mk), _p(part), C.byref(c), comm._h,
                                      C.byref(h)))
        self._h, self.comm, self.mesh, self._owner = h, comm, mesh, None
        n0, n1, n2 = C.c_int32(), C.c_int32(), C.c_int32()
        _ck(lib.ts_dist_levels_sizes(self._h, C.byref(n0), C.byref(n1), C.byref(n2)))
        self.n_local, self.n_local_vertices, self.n2 = n0.value, n1.value, n2.value

    def local_nodes(self) -> np.ndarray:
        l2g = np.zeros(self.n_local, np.int32)
        _ck(lib.ts_dist_local_nodes(self._h, _p(l2g)))
        return l2g

    def info(self) -> dict:
        """This rank's partition: elements, level-0 interface rows sent per product,
        neighbour ranks, setup wall time."""
        ne, nn = C.c_int32(), C.c_int32()
        hr, st = C.c_int64(), C.c_double()
        _ck(lib.ts_dist_levels_info(self._h, C.byref(ne), C.byref(hr), C.byref(nn), C.byref(st)))
        return {"elements": ne.value, "halo_rows0": hr.value, "neighbours": nn.value, "setup_s": st.value}

    def local_dofs(self) -> np.ndarray:
        """global dof index of every local dof row (3 per node)."""
        l2g = self.local_nodes().astype(np.int64)
        return (3 * l2g[:, None] + np.arange(3)[None, :]).reshape(-1)

    def solve(self, f, u0, cfg: SolverConfig | None = None, out=None):
        """solve (adaptive_cg.hpp:242-263) on local (3 n_local, batch) vectors; numpy
        (host entry) or CUDA float64 tensors (device entry). Returns (u, report). `out`
        (device entry): the solution buffer; it may be u0 itself (solved in place)."""
        cfg = cfg or SolverConfig()
        c = cfg.to_c()
        batch = int(f.shape[1])
        rb = _ReportBuf(batch, 0)
        rows = 3 * self.n_local
        if _is_torch(f):
            import torch
            f = _device_vec(f, rows, torch.float64, "solve")
            u0 = _device_vec(u0, rows, torch.float64, "solve: initial guess", batch)
            if out is not None:
                if not (_is_torch(out) and out.shape == f.shape and out.dtype == torch.float64 and out.is_cuda
                        and out.is_contiguous() and out.device == f.device):
                    raise ValueError("solve: out must be a contiguous CUDA float64 tensor shaped like f")
                u = out
            else:
                u = torch.empty_like(f)
            rc = lib.ts_dist_solve_device(self._h, C.c_void_p(f.data_ptr()), C.c_void_p(u0.data_ptr()),
                                          C.c_void_p(u.data_ptr()), self.n_local, batch, C.byref(c), C.byref(rb.c),
                                          _stream())
        else:
            f = _host_vec(f, rows, np.float64, "solve")
            u0 = _host_vec(u0, rows, np.float64, "solve: initial guess", batch)
            u = np.empty_like(f)
            rc = lib.ts_dist_solve(self._h, _p(f), _p(u0), _p(u), self.n_local, batch, C.byref(c), C.byref(rb.c))
        rep = rb.report(0)
        _ck(rc, rep)
        return u, rep

    def apply(self, which: int, u, f, stream=None):
        """One partitioned EBE product incl. the interface exchange (device tensors):
        which = 0 outer fp64 tet10, 1 level-0 fp32 tet10, 2 level-1 fp32 tet4."""
        st = _stream() if stream is None else stream
        _ck(lib.ts_dist_ebe_apply(self._h, int(which), C.c_void_p(u.data_ptr()), C.c_void_p(f.data_ptr()),
                                  int(u.shape[1]), st))
        return f

    def __del__(self):
        try:
            if getattr(self, "_owner", None) is None:
                lib.ts_dist_levels_destroy(self._h)
        except Exception:
            pass


class DistEbeOperator:
    """A partitioned EBE operator alone (ts_dist_ebe): this rank's elements of
    the global mesh, K u with the interface exchange inside (local node order)."""

    def __init__(self, mesh: Mesh, order: int, materials, part, comm: Comm, prec: int = 32, dof_mask=None):
        lam, mu = _lame(materials)
        part = np.ascontiguousarray(part, np.int32)
        mk = None if dof_mask is None else np.ascontiguousarray(dof_mask, np.uint8)
        h = C.c_void_p()
        _ck(lib.ts_dist_ebe_create(mesh._h, int(order), len(lam), _p(lam), _p(mu), _p(mk), _p(part), int(prec),
                                   comm._h, C.byref(h)))
        self._h, self.comm, self.prec, self.order = h, comm, int(prec), int(order)
        nl, ne, nn = C.c_int32(), C.c_int32(), C.c_int32()
        hr = C.c_int64()
        _ck(lib.ts_dist_ebe_info(self._h, C.byref(nl), C.byref(ne), C.byref(hr), C.byref(nn)))
        self.n_local, self.n_elements, self.halo_rows, self.n_neighbours = nl.value, ne.value, hr.value, nn.value

    def local_nodes(self) -> np.ndarray:
        l2g = np.zeros(self.n_local, np.int32)
        _ck(lib.ts_dist_ebe_local_nodes(self._h, _p(l2g)))
        return l2g

    def apply(self, u, f, stream=None):
        st = _stream() if stream is None else stream
        _ck(lib.ts_dist_ebe_op_apply(self._h, C.c_void_p(u.data_ptr()), C.c_void_p(f.data_ptr()), int(u.shape[1]),
                                     st))
        return f

    def __del__(self):
        try:
            lib.ts_dist_ebe_destroy(self._h)
        except Exception:
            pass


class DistFaultedModel:
    """build_faulted_model (model.hpp:41-51) on one rank's partition of the base mesh, for the
    partitioned Green's-function bank (ts_dist_faulted_*: BASELINE configs[4])."""

    def __init__(self, mesh: Mesh, materials, faces, part, comm: Comm, cfg: SolverConfig | None = None):
        cfg = cfg or SolverConfig()
        lam, mu = _lame(materials)
        faces = np.ascontiguousarray(faces, np.int32)
        part = np.ascontiguousarray(part, np.int32)
        c = cfg.to_c()
        h = C.c_void_p()
        _ck(lib.ts_dist_faulted_model_create(mesh._h, len(lam), _p(lam), _p(mu), _p(faces), len(faces), _p(part),
                                             C.byref(c), comm._h, C.byref(h)))
        self._h, self.comm = h, comm
        lv = C.c_void_p()
        _ck(lib.ts_dist_faulted_levels(self._h, C.byref(lv)))
        self.levels = DistLevels._view(lv, comm, owner=self)

    def slip_to_rhs(self, centers, directions, radii) -> np.ndarray:
        """This rank's rows [3 n_local, n_slips] of slip_to_rhs (fault.hpp:363-388)."""
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        directions = np.ascontiguousarray(directions, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        f = np.zeros((3 * self.levels.n_local, len(directions)), np.float64)
        _ck(lib.ts_dist_slip_to_rhs(self._h, len(directions), _p(centers), _p(directions), _p(radii), _p(f)))
        return f

    def greens_bank(self, centers, directions, radii, points, axes, cfg: SolverConfig | None = None):
        """compute_greens_bank (greens.hpp:114-145) over the partition: (bank [n_obs, n_slips] —
        the same on every rank —, solver_calls, outer_iterations)."""
        cfg = cfg or SolverConfig()
        c = cfg.to_c()
        centers = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        directions = np.ascontiguousarray(directions, np.int32)
        radii = np.ascontiguousarray(radii, np.float64)
        points = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        axes = np.ascontiguousarray(axes, np.int32)
        bank = np.zeros((len(axes), len(directions)), np.float64)
        calls, outer = C.c_int32(), C.c_int64()
        _ck(lib.ts_dist_greens_bank(self._h, len(directions), _p(centers), _p(directions), _p(radii), len(axes),
                                    _p(points), _p(axes), C.byref(c), _p(bank), C.byref(calls), C.byref(outer)))
        return bank, calls.value, outer.value

    def __del__(self):
        try:
            lib.ts_dist_faulted_model_destroy(self._h)
        except Exception:
            pass
