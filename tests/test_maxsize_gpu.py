"""Maximum size: the configs[3] mesh (281 x 423 x 141 cells: 100.6M tet10, 135.0M nodes,
405M DOF; SURVEY.md §8 sizing) on ONE device, fp32, r = 8 load cases. At this size the
[node][axis][case] vectors hold 3.24G entries (13 GB), past every 32-bit element and byte
offset, so the sweep's 64-bit row addressing, the 28-bit node field of the connectivity
words (ebe.h) and the host setup's int64 loops are exercised where they matter.

Checks (north-star fp32 tolerance 1e-5):
* patch parity: for sample nodes (both ends of the numbering, the vertex/edge-node
  boundary, constrained and free rows, random interior nodes) the rows of K u equal the
  checker's product on the sub-mesh of the elements touching them — a row of K u depends
  only on those elements (ebe_operator.hpp:112-115);
* the host entry (pinned host u and f: H2D, sweep and D2H overlapped slab by slab) gives the
  device product (per case, to the rounding of the unordered scatter);
* symmetry of the constrained operator, (v, K u) = (u, K v) per case, a size-independent
  property of the whole sweep.
"""
import numpy as np
import pytest
from conftest import TWO_LAYER, lame

import paper_1710_08679_b200 as ts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EXT = (792e3, 1192e3, 400e3)
DIV = (281, 423, 141)
R = 8


def _fits():
    try:
        import psutil
        host = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        host = 0
    free, _ = torch.cuda.mem_get_info()
    return host >= 96 << 30 and free >= 100 << 30


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def chunked_dot(a, b, chunk=1 << 27):
    """Per-case fp64 dot of two [3N, R] device tensors without a full fp64 copy."""
    out = torch.zeros(a.shape[1], dtype=torch.float64, device=a.device)
    for i in range(0, a.shape[0], chunk):
        out += (a[i:i + chunk].double() * b[i:i + chunk].double()).sum(0)
    return out.cpu().numpy()


def test_configs3_mesh_on_one_device(checker):
    if not _fits():
        pytest.skip("needs >= 96 GB free host memory and >= 100 GB free device memory")
    mesh = ts.generate_box_mesh(EXT, DIV, (200e3,))
    N, V, E = mesh.node_count(), mesh.vertex_count, mesh.element_count()
    assert (N, V, E) == (134_951_663, 16_978_656, 100_558_098)
    mats = [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]
    mask = mesh.dirichlet_mask()
    op = ts.EbeOperator(mesh, 2, mats, mask, prec=32)
    assert 3 * N * R > 2**31

    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(3 * N, R, device="cuda", generator=g) * 2 - 1
    f = op.apply(u)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(f).all())

    # ---- patch parity at sample rows ---------------------------------------------
    a = mesh.arrays()
    tets = a["tets10"]
    rng = np.random.default_rng(11)
    samples = np.unique(np.concatenate([[0, 1, V - 1, V, N - 2, N - 1], rng.integers(0, N, 10)])).astype(np.int32)
    hit = np.isin(tets, samples, kind="table").any(axis=1)
    sub_t = tets[hit]
    nodes, inv = np.unique(sub_t, return_inverse=True)  # global order: vertices stay a prefix
    loc_t = inv.reshape(sub_t.shape).astype(np.int32)
    nv = int(np.searchsorted(nodes, V))
    from oracle import MeshArrays
    sub = MeshArrays(a["coords"][nodes], loc_t, a["material_id"][hit].astype(np.int32), nv,
                     np.zeros(0, np.int32), np.zeros(0, np.int8))
    dofs = (3 * nodes.astype(np.int64)[:, None] + np.arange(3)).ravel()
    u_loc = u[torch.from_numpy(dofs).cuda()].cpu().numpy()
    m_loc = mask[dofs]
    lam, mu = lame(TWO_LAYER)
    want = checker.ebe_apply(sub, 2, lam, mu, m_loc, 32, u_loc)
    pos = np.searchsorted(nodes, samples)
    rows_loc = (3 * pos[:, None] + np.arange(3)).ravel()
    rows_glb = (3 * samples.astype(np.int64)[:, None] + np.arange(3)).ravel()
    got = f[torch.from_numpy(rows_glb).cuda()].cpu().numpy()
    assert rel(got, want[rows_loc]) <= 1e-5
    assert np.array_equal(got[mask[rows_glb] == 1], u_loc[rows_loc][mask[rows_glb] == 1])
    assert mask[rows_glb].any() and not mask[rows_glb].all()

    # ---- the host entry (streamed H2D / sweep / D2H) at this size -------------------
    uh = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
    uh.copy_(u)
    fh = torch.empty(u.shape, dtype=u.dtype, pin_memory=True)
    op.apply(uh.numpy(), fh.numpy())
    del uh
    fd = fh.cuda()
    del fh
    num = torch.zeros(R, dtype=torch.float64, device="cuda")
    for i in range(0, f.shape[0], 1 << 27):
        d = (fd[i:i + (1 << 27)] - f[i:i + (1 << 27)]).double()
        num += (d * d).sum(0)
    del fd
    assert bool(torch.all(num.sqrt() <= 1e-6 * torch.from_numpy(np.sqrt(chunked_dot(f, f))).cuda()))

    # ---- symmetry: (v, K u) = (u, K v) per case ----------------------------------
    v = torch.rand(3 * N, R, device="cuda", generator=g) * 2 - 1
    kv = op.apply(v)
    vku, ukv = chunked_dot(v, f), chunked_dot(u, kv)
    scale = np.sqrt(chunked_dot(v, v) * chunked_dot(f, f))
    assert np.all(np.abs(vku - ukv) <= 1e-5 * scale)
