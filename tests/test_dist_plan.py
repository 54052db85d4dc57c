"""Host logic of the partitioned (multi-GPU) path on CPU.

* partition_rcb: balanced, complete, deterministic;
* per-rank plans: every node owned exactly once, halo rows symmetric between
  neighbours, local numbering keeps vertices first;
* the partitioned EBE product itself, world_size 2 and 3 over gloo: each rank
  applies the checker (oracle port) to its own partition's elements, exchanges
  interface partial rows with its neighbours (torch.distributed send/recv) and
  sums them in ascending rank order — exactly the device algorithm
  (dist_solver.cu k_halo_sum) — and the result must equal the global product.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import TWO_LAYER, lame

import paper_1710_08679_b200 as ts
from paper_1710_08679_b200.dist import dist_plan, partition_rcb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPEC = ((6000.0, 5000.0, 4000.0), (6, 5, 4), (3000.0,), 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
def test_partition_rcb_balanced_and_deterministic(nparts):
    m = ts.generate_box_mesh(*SPEC)
    p = partition_rcb(m, nparts)
    assert p.shape == (m.element_count(),)
    counts = np.bincount(p, minlength=nparts)
    assert counts.min() > 0 and counts.max() - counts.min() <= 1 + nparts
    assert np.array_equal(p, partition_rcb(m, nparts))


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_plans_consistent(nparts):
    m = ts.generate_box_mesh(*SPEC)
    part = partition_rcb(m, nparts)
    plans = [dist_plan(m, part, nparts, r) for r in range(nparts)]
    V = m.vertex_count
    own_count = np.zeros(m.node_count(), np.int32)
    seen_elems = []
    for r, pl in enumerate(plans):
        l2g = pl["l2g"]
        assert np.all(np.diff(l2g) > 0)                     # ascending global id
        nv = pl["n_local_vertices"]
        assert np.all(l2g[:nv] < V) and np.all(l2g[nv:] >= V)  # vertices first
        own_count[l2g[pl["owned"] == 1]] += 1
        seen_elems.append(pl["elems"])
        assert np.array_equal(np.sort(pl["elems"]), np.flatnonzero(part == r))
        for k, q in enumerate(pl["nbr"]):
            mine = l2g[pl["rows"][k]]
            other = plans[q]
            kk = list(other["nbr"]).index(r)
            theirs = other["l2g"][other["rows"][kk]]
            assert np.array_equal(mine, theirs)            # same interface rows, same order
    assert np.all(own_count == 1)                          # each node counted once in dots
    assert np.array_equal(np.sort(np.concatenate(seen_elems)), np.arange(m.element_count()))


def _local_arrays(om, pl):
    """The partition as oracle MeshArrays (local ids) and its local dof mask."""
    from oracle import MeshArrays
    g2l = -np.ones(om.n_nodes, np.int64)
    g2l[pl["l2g"]] = np.arange(len(pl["l2g"]))
    tets = g2l[om.tets10[pl["elems"]]].astype(np.int32)
    return MeshArrays(om.coords[pl["l2g"]].copy(), tets, om.material_id[pl["elems"]].copy(),
                      int(pl["n_local_vertices"]), np.zeros(0, np.int32), np.zeros(0, np.int8))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    orc = Oracle("port")
    m = ts.generate_box_mesh(*SPEC)
    om = orc.box_mesh(*SPEC)
    gmask = om.dirichlet_mask()
    lam, mu = lame(TWO_LAYER)
    part = partition_rcb(m, world)
    pl = dist_plan(m, part, world, rank)
    loc = _local_arrays(om, pl)
    ldofs = (3 * pl["l2g"][:, None].astype(np.int64) + np.arange(3)).reshape(-1)
    lmask = gmask[ldofs]
    B = 4
    ug = orc.rng_sym(77, 3 * om.n_nodes * B).reshape(-1, B)
    res = {}
    for prec in (64, 32):
        dt = np.float64 if prec == 64 else np.float32
        f = orc.ebe_apply(loc, 2, lam, mu, lmask, prec, ug[ldofs].astype(dt)).reshape(-1, 3 * B)
        # exchange interface partial rows with every neighbour (rows in ascending global id)
        recv = {}
        reqs = []
        for k, q in enumerate(pl["nbr"]):
            send = torch.from_numpy(np.ascontiguousarray(f[pl["rows"][k]]))
            buf = torch.empty_like(send)
            reqs.append(dist.isend(send, int(q)))
            reqs.append(dist.irecv(buf, int(q)))
            recv[int(q)] = (k, buf)
        for rq in reqs:
            rq.wait()
        g = f.copy()
        pos = {int(q): {int(i): j for j, i in enumerate(pl["rows"][k])} for k, q in enumerate(pl["nbr"])}
        shared = sorted({int(i) for rows in pl["rows"] for i in rows})
        for i in shared:
            srcs = sorted([rank] + [q for q in pos if i in pos[q]])
            acc = None
            for q in srcs:  # ascending rank order, own partial at its rank
                v = f[i] if q == rank else recv[q][1].numpy()[pos[q][i]]
                acc = v.copy() if acc is None else acc + v
            keep = lmask[3 * i:3 * i + 3].repeat(B).astype(bool)  # constrained dofs keep the identity row
            g[i] = np.where(keep, f[i], acc)
        want = orc.ebe_apply(om, 2, lam, mu, gmask, prec, ug.astype(dt))[ldofs].reshape(-1, 3 * B)
        res[prec] = float(np.linalg.norm(g - want) / np.linalg.norm(want))
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_ebe_product_over_gloo(world):
    mgr = mp.get_context("spawn").Manager()  # no fork of a process that holds OpenMP threads
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r][64] <= 1e-12, out[r]
        assert out[r][32] <= 1e-5, out[r]
