"""GPU parity of the partitioned (multi-GPU) solve path.

One B200 hosts P in-process ranks (ThreadWorld backend: the same SPMD device
code as the NCCL path, exchanging through device copies), so the partitioned
EBE products, the interface exchange with overlap, the owner-counted
all-reduced dots and the replicated level 2 are all exercised:

* a partitioned product equals the single-device product on the same global
  vector (1e-12 fp64 / 1e-5 fp32) and every copy of an interface row agrees
  bit for bit across ranks;
* a partitioned solve reproduces the single-device solve (displacement within
  1e-6, outer iterations within +-1, inner totals within +-2 %) and the
  reference's manufactured solution.
The NCCL backend is checked in its one-rank form (no second GPU here).
"""
import threading

import numpy as np
import pytest
from conftest import TWO_LAYER

import paper_1710_08679_b200 as ts
from paper_1710_08679_b200.dist import Comm, DistLevels, ThreadWorld, partition_rcb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPEC = ((16000.0, 20000.0, 10000.0), (8, 10, 5), (7000.0,), 1)


def mats():
    return [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]


def run_ranks(P, fn):
    """fn(rank, comm) on P threads of one process; returns the per-rank results."""
    world = ThreadWorld(P)
    comms = [Comm.thread(world, r, 0) for r in range(P)]
    out, err = [None] * P, [None] * P

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return out


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kernel", ["auto", "fan"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("overlap", ["1", "0"])
def test_partitioned_products_match_single_device(P, overlap, kernel, monkeypatch):
    """(kernel: the partitions' element sweeps as face pairs or edge fans; fans never cross the
    boundary / interior element groups the overlapped exchange relies on)"""
    monkeypatch.setenv("TSGPU_DIST_OVERLAP", overlap)
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    m = ts.generate_box_mesh(*SPEC)
    mask = m.dirichlet_mask()
    V = m.vertex_count
    part = partition_rcb(m, P)
    B = 4
    g = torch.Generator(device="cuda").manual_seed(5)
    ug = torch.rand(3 * m.node_count(), B, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
    want = {
        0: ts.EbeOperator(m, 2, mats(), mask, prec=64).apply(ug).cpu().numpy(),
        1: ts.EbeOperator(m, 2, mats(), mask, prec=32).apply(ug.float()).cpu().numpy(),
        2: ts.EbeOperator(m, 1, mats(), mask[: 3 * V], prec=32).apply(ug[: 3 * V].float().contiguous()).cpu().numpy(),
    }

    def fn(r, comm):
        dl = DistLevels(m, mats(), part, comm, ts.SolverConfig(batch_size=B))
        dofs = torch.from_numpy(dl.local_dofs()).cuda()
        res = {"dofs": dl.local_dofs()}
        for which in (0, 1, 2):
            n = dl.n_local if which < 2 else dl.n_local_vertices
            u = ug[dofs[: 3 * n]]
            u = u.float() if which else u
            f = torch.empty_like(u)
            dl.apply(which, u.contiguous(), f)
            torch.cuda.synchronize()
            res[which] = f.double().cpu().numpy()
        return res

    out = run_ranks(P, fn)
    tol = {0: 1e-12, 1: 1e-5, 2: 1e-5}
    for which in (0, 1, 2):
        glob = {}
        for r in range(P):
            d = out[r]["dofs"][: out[r][which].shape[0]]
            assert rel(out[r][which], want[which][d]) <= tol[which], (which, r)
            for i, dof in enumerate(d):
                if dof in glob:  # interface rows: every copy identical
                    assert np.array_equal(glob[dof], out[r][which][i]), (which, dof)
                else:
                    glob[dof] = out[r][which][i]
        assert len(glob) == want[which].shape[0]


def smooth(coords, ext, mask, B, seed):
    rng = np.random.default_rng(seed)
    x, y, z = (coords[:, k] / ext[k] for k in range(3))
    u = np.zeros((coords.shape[0], 3, B))
    for b in range(B):
        amp, ky = 0.05 * (1 + 0.2 * rng.uniform(-1, 1)), 1.0 + (rng.uniform() > 0.5)
        sz = np.sin(0.5 * np.pi * z)
        u[:, 0, b] = amp * np.sin(np.pi * x) * np.cos(ky * np.pi * y) * sz
        u[:, 1, b] = amp * np.cos(np.pi * x) * np.sin(ky * np.pi * y) * sz
        u[:, 2, b] = amp * np.cos(np.pi * x) * np.cos(ky * np.pi * y) * sz
    u = u.reshape(-1, B)
    u[mask == 1] = 0.0
    return u


@pytest.mark.parametrize("kernel", ["auto", "fan"])
@pytest.mark.parametrize("l2", ["replicated", "distributed"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_partitioned_solve_matches_single_device(P, l2, kernel, monkeypatch):
    """Level 2 either replicated on every rank or split by coarse rows with a gather halo in
    every product (TSGPU_DIST_L2), element sweeps as face pairs or edge fans: the same solution
    and iteration counts either way."""
    monkeypatch.setenv("TSGPU_DIST_L2", l2)
    monkeypatch.setenv("TSGPU_EBE_KERNEL", kernel)
    m = ts.generate_box_mesh(*SPEC)
    mask = m.dirichlet_mask()
    B = 3
    cfg = ts.SolverConfig(batch_size=B)
    model = ts.build_crust_model(m, mats(), cfg)
    us = smooth(np.asarray(m.coords).reshape(-1, 3), SPEC[0], mask, B, 31)
    f = model.levels.outer.apply(torch.from_numpy(us).cuda()).cpu().numpy()
    u1, rep1 = ts.solve(model.levels, f, np.zeros_like(f), cfg)
    part = partition_rcb(m, P)

    def fn(r, comm):
        dl = DistLevels(m, mats(), part, comm, cfg)
        d = dl.local_dofs()
        u, rep = dl.solve(f[d], np.zeros((len(d), B)), cfg)
        return d, u, rep

    out = run_ranks(P, fn)
    ug = np.zeros_like(f)
    for d, u, rep in out:
        ug[d] = u
        assert rep.converged
        assert abs(rep.outer_iterations - rep1.outer_iterations) <= 1
        for lvl in range(3):
            a, b = rep.inner_iterations[lvl], rep1.inner_iterations[lvl]
            assert abs(a - b) <= max(2, 0.02 * b), (lvl, a, b)
        assert rep.outer_iterations == out[0][2].outer_iterations  # identical control flow on every rank
    assert rel(ug, u1) <= 1e-6
    assert rel(ug, us) <= 1e-6


def test_nccl_single_rank_solve_matches_single_device():
    ok, why = Comm.nccl_available()
    if not ok:
        pytest.skip(f"nccl unavailable: {why}")
    m = ts.generate_box_mesh(*SPEC)
    B = 2
    cfg = ts.SolverConfig(batch_size=B)
    model = ts.build_crust_model(m, mats(), cfg)
    us = smooth(np.asarray(m.coords).reshape(-1, 3), SPEC[0], m.dirichlet_mask(), B, 7)
    f = model.levels.outer.apply(torch.from_numpy(us).cuda()).cpu().numpy()
    u1, rep1 = ts.solve(model.levels, f, np.zeros_like(f), cfg)
    comm = Comm.nccl(1, 0, Comm.nccl_id(), 0)
    dl = DistLevels(m, mats(), np.zeros(m.element_count(), np.int32), comm, cfg)
    d = dl.local_dofs()
    assert np.array_equal(d, np.arange(3 * m.node_count()))
    u, rep = dl.solve(f, np.zeros_like(f), cfg)
    assert rep.outer_iterations == rep1.outer_iterations
    assert rel(u, u1) <= 1e-9


@pytest.mark.parametrize("P", [1, 3])
def test_comm_allreduce_sum(P):
    """ts_comm_allreduce_sum (the partitioned solve's dot-product all-reduce) over in-process ranks,
    and over a one-rank NCCL communicator."""
    def fn(rank, comm):
        t = torch.arange(5, dtype=torch.float64, device="cuda") * (rank + 1)
        comm.allreduce_sum(t)
        torch.cuda.synchronize()
        return t.cpu().numpy()

    out = run_ranks(P, fn)
    want = np.arange(5, dtype=np.float64) * sum(range(1, P + 1))
    for o in out:
        assert np.array_equal(o, want)
    ok, _ = Comm.nccl_available()
    if ok and P == 1:
        comm = Comm.nccl(1, 0, Comm.nccl_id(), 0)
        t = torch.full((7,), 2.5, dtype=torch.float64, device="cuda")
        comm.allreduce_sum(t)
        assert torch.equal(t.cpu(), torch.full((7,), 2.5, dtype=torch.float64))


@pytest.mark.parametrize("P", [2, 3])
def test_partitioned_greens_bank_matches_single_device(P):
    """ts_dist_greens_bank (configs[4]'s sweep on a partitioned mesh) against the single-device
    bank (itself pinned to the reference in test_greens_gpu.py): this rank's slip_to_rhs rows
    equal the global right-hand side's (1e-12), the bank within 1e-6, the same solver calls and
    outer iterations within +-2 %, and every rank holds the same bank."""
    from paper_1710_08679_b200.dist import DistFaultedModel
    from paper_1710_08679_b200.greens import DIP, STRIKE, FaultedModel, find_plane_fault_faces
    ext, div, ifs = (8000.0, 8000.0, 6000.0), (8, 8, 6), (4500.0,)
    m = ts.generate_box_mesh(ext, div, ifs)
    faces = find_plane_fault_faces(m, 0, 4000.0, (4000.0, 2000.0, 1000.0), (4000.0, 6000.0, 5000.0))
    centers = np.array([[4000.0, 4000.0, 3000.0], [4000.0, 3000.0, 2500.0], [4000.0, 5000.0, 4000.0],
                        [4000.0, 4000.0, 3000.0], [4000.0, 3500.0, 2000.0]])
    dirs = np.array([DIP, DIP, STRIKE, STRIKE, DIP], np.int32)
    radii = np.array([1500.0, 1000.0, 1200.0, 1500.0, 900.0])
    obs = np.array([[1000.0, 2000.0, 6000.0], [3000.0, 4000.0, 6000.0], [5000.0, 4000.0, 6000.0],
                    [6500.0, 1500.0, 6000.0], [4000.0, 7000.0, 6000.0], [2500.0, 2500.0, 5500.0]])
    axes = np.array([0, 1, 2, 0, 2, 1], np.int32)
    cfg = ts.SolverConfig(batch_size=2)
    fm = FaultedModel(m, mats(), faces, cfg)
    want_f = fm.slip_to_rhs(centers, dirs, radii)
    want, wcalls, wouter = fm.greens_bank(centers, dirs, radii, obs, axes, cfg)
    part = partition_rcb(m, P)

    def fn(r, comm):
        dfm = DistFaultedModel(m, mats(), faces, part, comm, cfg)
        f = dfm.slip_to_rhs(centers, dirs, radii)
        bank, calls, outer = dfm.greens_bank(centers, dirs, radii, obs, axes, cfg)
        return dfm.levels.local_dofs(), f, bank, calls, outer

    out = run_ranks(P, fn)
    for dofs, f, bank, calls, outer in out:
        assert rel(f, want_f[dofs]) <= 1e-12
        assert calls == wcalls
        assert abs(outer - wouter) <= max(1, 0.02 * wouter)
        assert rel(bank, want) <= 1e-6
        assert np.array_equal(bank, out[0][2])
    assert np.abs(want).max() > 0
