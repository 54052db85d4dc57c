#!/usr/bin/env python3
"""bench.py — B200 benchmark of the tetsolve solve path (arXiv 1710.08679).

Headline workload (BASELINE.json configs[1]): the multi-case EBE stiffness
matvec f = K u on the 10M-DOF layered-crust box (82 x 123 x 41 cells,
2.48M tet10 elements, 3.38M nodes), fp32 tier (the level-0 operator that
dominates the solve), r = 16 load cases. One step = one EbeOperator::apply
over the whole mesh. u and f (650 MB each) exceed the 126 MB L2, so no
explicit flush is needed between steps.

  value  : algorithmic GB/s (E*(40+14s) + 3N*(2rs+1) bytes per
           apply) of the device-resident step, summed over GPUs (replicas:
           each rank applies the operator to its own r cases — weak scaling).
  e2e    : same metric through the C ABI host-buffer entry (ts_ebe_apply_host:
           pinned H2D of u, apply, D2H of f, every step).
  roofline: the element-sweep kernel alone (CUDA events around it on its own
           stream, every timed step) against the measured HBM copy peak.
  cpu_baseline: the UNMODIFIED reference (oracle/_ref/libtsref.so) timing the
           same apply on this host's cores (rank 0, N = 1).
  --impl reference: the reference's own CPU implementation as the arm.
  northstar: BASELINE configs[3], the north-star run: the multigrid solve of r = 8
           cases on ONE layered-crust mesh partitioned over the N GPUs (RCB; NCCL
           halo exchange inside every product, all-reduced dots; level 2 built
           once and broadcast): time per case = the slowest rank's solve / r, the
           per-rank level-0 sweep roofline and interface bytes. N > 1: the 405M-DOF
           configs[3] mesh; N = 1: the configs[2] mesh on in-process ranks
           (--northstar-threads P; 1 by default) of the one GPU.
  greens_partitioned: BASELINE configs[4]: the Green's bank of unit slips batched
           r = 16 on the configs[3] mesh partitioned over the N GPUs (N > 1; 32 of
           the 368 cases by default, --greens-cases 368 for the whole sweep; the
           full-sweep time is projected from the per-case time). N = 1:
           --greens-partitioned P runs it on P in-process ranks.
  greens : the Green's-function bank (configs[4] workflow at one-GPU scale):
           48 unit slips on a vertical fault in the configs[1] box, batch 16,
           through ts_greens_bank; total sweep time and time per case.
  (N > 1: the configs[3] mesh and partition are built once for both partitioned legs;
           the configs[2] replica solves below run there only with --solve-replicas)
  solve  : BASELINE's other metric, time per case: the full multigrid solve
           (build_crust_model + solve, adaptive_cg.hpp:242-263) of configs[2]
           (50M-DOF 3-layer crust, 16 cases, mixed-precision PCG) through the
           host-buffer entry ts_solve; manufactured right-hand sides
           f = K u* (acceptance_main.cpp:82-102 fields). Beside it the
           reference's own solve() and ours on a bounded same-workload sample
           (16^3 cells, 16 cases) on this host's cores.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
       torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ebe_traffic.json")
TWO_LAYER = [(1600.0, 400.0, 1850.0), (5800.0, 3000.0, 2700.0)]  # Table 3
CELL_KM = 2.8  # config-4 cell size (792 x 1192 x 400 km / (281, 423, 141))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def hbm_peak():
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes(n_elems, n_nodes, r, s, npe=10):
    """conn int32 + 4 vertex xyz + (lambda, mu) per element,
    u read + f write + uint8 mask per dof."""
    return n_elems * (npe * 4 + 14 * s) + 3 * n_nodes * (2 * r * s + 1)


def mesh_spec(cells):
    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    return ext, tuple(cells), (0.75 * ext[2],)  # soft layer: top quarter (layer 0 on top)


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every ~5 ms) DURING the timed region."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.rows = []
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
                "hw_power_brake_slowdown": 0x80}

        def run():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, [k for k, v in bits.items() if rs & v]))
                except Exception:
                    pass
                self._stop.wait(self.period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self._max,
                "reasons": sorted({x for r in self.rows for x in r[1]}), "samples": len(self.rows)}


def max_over_ranks(vals, device="cpu"):
    """Max of each value over all ranks (the step time of a multi-GPU run is the
    slowest rank's). Identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in vals]
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def whole_job_gbps(world, alg_bytes_per_rank, step_ms):
    """value = bytes processed by ALL ranks / the (max-over-ranks) step time."""
    return world * alg_bytes_per_rank / (step_ms * 1e-3) / 1e9


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, have_reference

    cells = tuple(args.cells)
    ext, div, ifs = mesh_spec(cells)
    base = {"impl": "reference", "metric": METRIC, "unit": "GB/s", "higher_is_better": True,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup}
    if not have_reference():
        print(json.dumps({**base, "unavailable": "oracle/_ref/libtsref.so was not built (reference sources absent)"}))
        return
    ref = Oracle("reference")
    lam = [rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in TWO_LAYER]
    mu = [rho * vs * vs for vp, vs, rho in TWO_LAYER]
    cores = ref.hw_threads()
    r, prec = args.cases, args.prec
    steps = max(1, min(args.steps, 20))  # bounded CPU sample (~1.3 s per apply)
    sec, _ = ref.time_ebe_apply_box(ext, div, ifs, 1, 2, lam, mu, prec, cores, r, steps)
    E = 6 * cells[0] * cells[1] * cells[2]
    N = (2 * cells[0] + 1) * (2 * cells[1] + 1) * (2 * cells[2] + 1)
    B = alg_bytes(E, N, r, prec // 8)
    val = B / sec / 1e9
    sample = (f"reference EbeOperator<{'float' if prec == 32 else 'double'}>::apply, order 2, r={r}, "
              f"{cells} cells ({E} tet10, {N} nodes), workers={cores} (colored std::thread path), "
              f"1 warm-up + {steps} timed applies")
    print(json.dumps({**base, "value": round(val, 4), "ms_per_step": round(sec * 1e3, 2),
                      "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                                       "cpu_model": cpu_model(), "sample": sample},
                      "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                      "dtype": "f32" if prec == 32 else "f64", "data": "synthetic",
                      "config": config_dict(cells, r, prec, world, E, N)}))


METRIC = "EBE matvec HBM GB/s (tet10 K u, r load cases, 10M-DOF layered crust)"


def precision_tier(prec):
    if prec == 32:
        return ("fp32 (level-0 operator): element arithmetic in fp32 on fp32-rounded geometry and Lame values, "
                "fp32 accumulation; the reference's EbeOperator<float> forms K_e and the local product in fp64 "
                "and accumulates in fp32 (SURVEY A6); matvec parity 1e-5 relative")
    return "fp64 (outer operator): fp64 element arithmetic and accumulation; matvec parity 1e-12 relative"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(cells, r, prec, world, E, N):
    return {"workload": "configs[1]: EBE matvec microbench, 10M-DOF layered-crust tet10 box",
            "cells": list(cells), "elements": E, "nodes": N, "dof": 3 * N, "cases_r": r,
            "precision_tier": precision_tier(prec), "parallelism": f"replicas x{world} (cases batched across GPUs)",
            "l2_policy": "inputs larger than L2 (u, f = 650 MB each vs 126 MB L2); no flush"}


# ---------------------------------------------------------------- solve leg
THREE_LAYER = TWO_LAYER + [(6800.0, 3900.0, 2900.0)]  # 3rd layer invented (vp^2 > 2 vs^2)


def manufactured(mesh, ext, mask, batch, seed, torch):
    """acceptance_main.cpp:82-102 smooth fields, per-column amplitude / ky (device)."""
    import numpy as np
    N = mesh.node_count()
    xyz = torch.from_numpy(np.asarray(mesh.coords).reshape(-1, 3)).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    amp = 0.05 * (1 + 0.2 * (torch.rand(batch, device="cuda", dtype=torch.float64, generator=g) * 2 - 1))
    ky = 1.0 + (torch.rand(batch, device="cuda", dtype=torch.float64, generator=g) > 0.5).double()
    X, Y, Z = [xyz[:, k:k + 1] / ext[k] for k in range(3)]
    sz = torch.sin(0.5 * torch.pi * Z)
    us = torch.stack([amp * torch.sin(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz,
                      amp * torch.cos(torch.pi * X) * torch.sin(ky * torch.pi * Y) * sz,
                      amp * torch.cos(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz], 1)
    us = us.reshape(3 * N, batch).contiguous()
    us[torch.from_numpy(mask).cuda().bool()] = 0
    return us


def gpu_solve(ts, torch, cells, table, batch, seed):
    """build_crust_model + solve on (3N, batch) host buffers (ts_solve: H2D f/u0, solve, D2H u).
    Returns a dict of times and iteration counts."""
    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    ifs = (0.75 * ext[2],) if len(table) == 2 else (0.4 * ext[2], 0.75 * ext[2])
    t0 = time.perf_counter()
    mesh = ts.generate_box_mesh(ext, cells, ifs)
    mats = [ts.material_from_wavespeeds(*t) for t in table]
    cfg = ts.SolverConfig(batch_size=batch)
    model = ts.build_crust_model(mesh, mats, cfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    us = manufactured(mesh, ext, model.mask, batch, seed, torch)
    fd = model.levels.outer.apply(us)
    # device-resident solve (ts_solve_device)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ud, rep_d = ts.solve(model.levels, fd, torch.zeros_like(fd), cfg, history=0)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t1
    # end to end through the host entry ts_solve from pinned host buffers (H2D f, u0; D2H u)
    fh = torch.empty(fd.shape, dtype=fd.dtype, pin_memory=True)
    fh.copy_(fd)
    u0h = torch.zeros(fd.shape, dtype=fd.dtype, pin_memory=True)
    uh = torch.empty(fd.shape, dtype=fd.dtype, pin_memory=True)
    f, u0 = fh.numpy(), u0h.numpy()
    t1 = time.perf_counter()
    u, rep = ts.solve(model.levels, f, u0, cfg, history=0, out=uh.numpy())
    t_solve = time.perf_counter() - t1
    err = float((uh.cuda() - us).norm() / us.norm())
    assert rep.outer_iterations == rep_d.outer_iterations
    return {"cells": list(cells), "dof": 3 * mesh.node_count(), "elements": mesh.element_count(), "cases": batch,
            "setup_s": round(t_setup, 3), "solve_s": round(t_solve, 4), "s_per_case": t_solve / batch,
            "device_solve_s": round(t_dev, 4), "device_s_per_case": round(t_dev / batch, 5),
            "outer_iterations": rep.outer_iterations, "inner_iterations": list(rep.inner_iterations),
            "time_inner_s": [round(x, 4) for x in rep.time_inner_s], "time_outer_s": round(rep.time_outer_s, 4),
            "max_final_rel_residual": rep.max_final_residual(), "rel_err_vs_manufactured": err,
            "h2d_bytes_per_solve": int(2 * f.nbytes), "d2h_bytes_per_solve": int(u.nbytes)}


def solve_leg(args, ts, torch, world, rank, local):
    """BASELINE metric 'time per case (s)': configs[2] solve per rank (replicas:
    each rank its own cases), max over ranks; plus the CPU reference on a
    bounded same-workload sample (rank 0, N = 1)."""
    cells, r = tuple(args.solve_cells), args.solve_cases
    with ClockSampler(local) as clk:
        g = gpu_solve(ts, torch, cells, THREE_LAYER, r, 31 + rank)
    solve_s = max_over_ranks([g["solve_s"]], "cuda")[0]
    out = {"metric": "time per case (s)", "higher_is_better": False,
           "workload": f"configs[2]: {g['dof'] / 1e6:.1f}M-DOF 3-layer crust box {list(cells)}, {r} cases per GPU, "
                       "mixed-precision multigrid PCG (fp32 inner, fp64 outer), manufactured RHS",
           "value": round(solve_s / (r * world), 5), "unit": "s", "n_gpus": world,
           "entry": "ts_solve (pinned host f/u0/u; H2D + solve + D2H timed); device_* = ts_solve_device",
           **g, "clocks": clk.summary()}
    out["s_per_case"] = round(g["s_per_case"], 5)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            from oracle import Oracle, SolverConfig as OCfg, have_reference
            if have_reference():
                ref = Oracle("reference")
                cores = ref.hw_threads()
                sc = tuple(args.cpu_solve_cells)
                gpu_solve(ts, torch, sc, THREE_LAYER, r, 31)  # warm (setup caches, clocks)
                gs = gpu_solve(ts, torch, sc, THREE_LAYER, r, 31)
                ext = tuple(c * CELL_KM * 1e3 for c in sc)
                om = ref.box_mesh(ext, sc, (0.4 * ext[2], 0.75 * ext[2]), 1)
                lam = [rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in THREE_LAYER]
                mu = [rho * vs * vs for vp, vs, rho in THREE_LAYER]
                t0 = time.perf_counter()
                olv = ref.levels(om, lam, mu, OCfg.default(batch_size=r), workers=cores)
                t_set = time.perf_counter() - t0
                mesh = ts.generate_box_mesh(ext, sc, (0.4 * ext[2], 0.75 * ext[2]))
                us = manufactured(mesh, ext, mesh.dirichlet_mask(), r, 31, torch).cpu().numpy()
                fo = olv.outer_apply(us)
                t0 = time.perf_counter()
                uo, ro = olv.solve(fo)
                t_ref = time.perf_counter() - t0
                out["cpu_reference_sample"] = {
                    "kind": "reference", "cores": cores,
                    "sample": f"reference solve() on {list(sc)} cells ({3 * mesh.node_count()} DOF), {r} cases, "
                              f"workers={cores}; same mesh/RHS solved here on the GPU through ts_solve",
                    "reference_s_per_case": round(t_ref / r, 4), "reference_setup_s": round(t_set, 3),
                    "reference_outer_iterations": ro["outer_iterations"],
                    "reference_inner_iterations": list(ro["inner_iterations"]),
                    "gpu_s_per_case": round(gs["s_per_case"], 5), "gpu_device_s_per_case": gs["device_s_per_case"],
                    "gpu_outer_iterations": gs["outer_iterations"],
                    "gpu_inner_iterations": gs["inner_iterations"]}
        except Exception as exc:  # reported, never fatal
            out["cpu_reference_sample"] = {"failed": str(exc)}
        try:
            out["configs0"] = configs0_leg(ts, torch)
        except Exception as exc:  # reported, never fatal
            out["configs0"] = {"failed": str(exc)}
    out["cpu_reference_extrapolation"] = config2_cpu_extrapolation(g)
    return out


def configs0_leg(ts, torch):
    """BASELINE configs[0] (the cube the CPU reference solves in full: 8^3 cells, extents 8,
    one interface at 4, two layers, r = 4): the reference's own solve() and solve_pcge() on
    this host's cores beside ours through the host entries, same manufactured right-hand sides
    (BASELINE.md §3 config 1)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, SolverConfig as OCfg, have_reference
    if not have_reference():
        return {"failed": "oracle/_ref not built on this box"}
    ref = Oracle("reference")
    cores = ref.hw_threads()
    ext, cells, ifs, r = (8.0, 8.0, 8.0), (8, 8, 8), (4.0,), 4
    lam = [rho * (vp * vp - 2 * vs * vs) for vp, vs, rho in TWO_LAYER]
    mu = [rho * vs * vs for vp, vs, rho in TWO_LAYER]
    om = ref.box_mesh(ext, cells, ifs, 1)
    t0 = time.perf_counter()
    olv = ref.levels(om, lam, mu, OCfg.default(batch_size=r), workers=cores)
    ref_setup = time.perf_counter() - t0
    mesh = ts.generate_box_mesh(ext, cells, ifs)
    us = manufactured(mesh, ext, mesh.dirichlet_mask(), r, 31, torch).cpu().numpy()
    f = olv.outer_apply(us)
    t0 = time.perf_counter()
    uo, ro = olv.solve(f)
    ref_solve = time.perf_counter() - t0
    t0 = time.perf_counter()
    up, rp = olv.solve_pcge(f)
    ref_pcge = time.perf_counter() - t0
    cfg = ts.SolverConfig(batch_size=r)
    t0 = time.perf_counter()
    model = ts.build_crust_model(mesh, [ts.material_from_wavespeeds(*t) for t in TWO_LAYER], cfg)
    torch.cuda.synchronize()
    our_setup = time.perf_counter() - t0
    ts.solve(model.levels, f, np.zeros_like(f), cfg)  # warm-up (workspaces)
    t0 = time.perf_counter()
    u, rep = ts.solve(model.levels, f, np.zeros_like(f), cfg)
    our_solve = time.perf_counter() - t0
    t0 = time.perf_counter()
    u2, rep2 = ts.solve_pcge(model.levels.outer, f, np.zeros_like(f), 1e-8, 100000)
    our_pcge = time.perf_counter() - t0
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    return {"workload": f"configs[0]: {list(cells)} cells, {3 * mesh.node_count()} DOF, r={r}, two layers",
            "cores": cores, "cpu_model": cpu_model(),
            "reference": {"setup_s": round(ref_setup, 4), "solve_s": round(ref_solve, 4), "pcge_s": round(ref_pcge, 4),
                          "outer": ro["outer_iterations"], "inner": list(ro["inner_iterations"]),
                          "pcge_iterations": rp["outer_iterations"]},
            "ours": {"setup_s": round(our_setup, 4), "solve_s": round(our_solve, 4), "pcge_s": round(our_pcge, 4),
                     "outer": rep.outer_iterations, "inner": list(rep.inner_iterations),
                     "pcge_iterations": rep2.outer_iterations, "entry": "ts_solve / ts_solve_pcge (host buffers)"},
            "u_rel_diff_solve": rel(u, uo), "u_rel_diff_pcge": rel(u2, up)}


def config2_cpu_extrapolation(g):
    """a full CPU solve of configs[2] takes about a day, so the reference
    was run capped at one outer iteration (tests/golden/make_config2_capped.py, the UNMODIFIED
    reference, r = 4, in the build container); the LABELLED extrapolation scales its time per
    outer iteration by the outer iterations this GPU solve needed and by r (per-case linearity)."""
    path = os.path.join(ROOT, "tests", "golden", "config2_outer1_reference.json")
    try:
        with open(path) as fh:
            cap = json.load(fh)
    except OSError:
        return None
    per_outer = cap["seconds"]["report_total"] / max(1, cap["outer_iterations"])
    scale_r = g["cases"] / cap["batch"]
    est = cap["seconds"]["levels_setup"] + per_outer * g["outer_iterations"] * scale_r
    return {"label": "EXTRAPOLATED, not measured: reference solve() at configs[2] capped at outer_max_iter=1 "
                     f"(r={cap['batch']}, {cap['host']['workers']} threads, {cap['host']['cpu_model']}, build "
                     f"container) x {g['outer_iterations']} outer iterations x {scale_r:g} (r={g['cases']} / "
                     f"r={cap['batch']}, assumed linear in r) + its level setup",
            "reference_capped_solve_s": cap["seconds"]["report_total"], "reference_setup_s":
                cap["seconds"]["levels_setup"], "reference_first_outer_inner": cap["inner_iterations"],
            "estimated_full_solve_s": round(est, 1), "estimated_s_per_case": round(est / g["cases"], 1),
            "gpu_s_per_case": round(g["s_per_case"], 5),
            "source": "tests/golden/config2_outer1_reference.json"}


class stdout_to_stderr:
    """Route the process's C-level stdout (fd 1) to stderr for the block."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


# -------------------------------------------------- N > 1: partitioned matvec
def main_partitioned(args, world, rank, local):
    """N GPUs: ONE mesh of N configs[1] slabs (82 x 123N x 41 cells) split by
    recursive coordinate bisection, one partition per rank; every step is the
    partitioned EBE product with its interface exchange (NCCL send/recv of the
    interface partial sums, overlapped with the interior elements). Weak
    scaling: per-GPU work is one configs[1] box."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1710_08679_b200 as ts
    from paper_1710_08679_b200.dist import Comm, DistEbeOperator, partition_rcb

    # our own NCCL communicator over the torch.distributed ranks; a failure is fatal (no silent
    # fallback to replicas: the partitioned path is what N > 1 measures)
    with stdout_to_stderr():  # NCCL prints its version banner on stdout; the JSON line must be alone there
        comm = Comm.nccl_from_torch(local)
    probe = comm.allreduce_sum(torch.ones(4, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    if not bool((probe == world).all()):
        raise RuntimeError(f"NCCL all-reduce self-test returned {probe.tolist()} on rank {rank}")

    cells = (args.cells[0], args.cells[1] * world, args.cells[2])
    ext, div, ifs = mesh_spec(cells)
    t0 = time.time()
    mesh = ts.generate_box_mesh(ext, div, ifs)
    mats = [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]
    part = partition_rcb(mesh, world)
    op = DistEbeOperator(mesh, 2, mats, part, comm, prec=args.prec)
    del mesh
    E, N = op.n_elements, op.n_local
    log(f"[rank {rank}] partition of {cells}: {E} tet10, {N} local nodes, {op.n_neighbours} neighbours, "
        f"{op.halo_rows} interface rows, setup {time.time() - t0:.1f}s")
    r, s = args.cases, args.prec // 8
    B_loc = alg_bytes(E, N, r, s)
    dt = torch.float32 if args.prec == 32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    u = torch.rand(3 * N, r, device="cuda", dtype=dt, generator=g) * 2 - 1
    f = torch.empty_like(u)
    stream = torch.cuda.current_stream()

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        op.apply(u, f)
    barrier()
    with ClockSampler(local) as clk:
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            op.apply(u, f)
        ev1.record(stream)
        barrier()
    step_ms = max_over_ranks([ev0.elapsed_time(ev1) / args.steps], "cuda")[0]
    tot = torch.tensor([float(B_loc)], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot)
    total_bytes = float(tot.item())
    value = total_bytes / (step_ms * 1e-3) / 1e9
    # e2e through the public partitioned operator with pinned host buffers
    uh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    uh.copy_(u.cpu())
    fh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    ud, fd = torch.empty_like(u), torch.empty_like(u)
    barrier()
    e2e_steps = max(3, args.steps // 4)
    te = time.perf_counter()
    for _ in range(e2e_steps):
        ud.copy_(uh, non_blocking=True)
        op.apply(ud, fd)
        fh.copy_(fd, non_blocking=True)
        torch.cuda.synchronize()
    e2e_ms = max_over_ranks([(time.perf_counter() - te) * 1e3 / e2e_steps], "cuda")[0]
    io_bytes = int(u.numel() * u.element_size())
    peak, peak_kind = hbm_peak()
    halo_bytes = int(op.halo_rows) * 3 * r * s
    del u, f, ud, fd, uh, fh, op
    torch.cuda.empty_cache()
    def sync():
        torch.cuda.synchronize()
        dist.barrier()

    cells_ns = (tuple(args.northstar_cells) if args.northstar_cells
                else NORTHSTAR_CELLS if world > 1 else tuple(args.solve_cells))
    cells_g = (tuple(args.greens_cells) if args.greens_cells
               else NORTHSTAR_CELLS if world > 1 else tuple(args.cells))
    # a leg whose per-rank footprint exceeds the device is reported as skipped on every rank
    # (e.g. the configs[4] sweep at r = 16 on 2 GPUs: SURVEY §8e) instead of failing the run
    need_ns = rank_bytes_needed(cells_ns, world, args.northstar_cases)
    need_g = rank_bytes_needed(cells_g, world, 16, greens=True)
    run_ns, free_ns = fits_on_ranks(torch, need_ns) if not args.no_northstar else (False, 0)
    run_g, free_g = fits_on_ranks(torch, need_g) if not args.no_greens_partitioned else (False, 0)
    # the configs[3] mesh and its partition are built once for both legs when they share it
    shared = (crust_mesh(ts, cells_ns, world) if run_ns and run_g and cells_ns == cells_g else None)
    northstar = None
    if not args.no_northstar and not run_ns:
        northstar = {"skipped": f"needs ~{need_ns / 1e9:.0f} GB per rank at r = {args.northstar_cases}, "
                                f"{free_ns / 1e9:.0f} GB free", "cells": list(cells_ns), "ranks": world}
    if run_ns:  # BASELINE configs[3]: the partitioned 400M-DOF solve, r = 8, on these N GPUs
        mine = northstar_rank(ts, torch, cells_ns, args.northstar_cases, comm, rank, world, sync, args.steps,
                              prebuilt=shared)
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        northstar = northstar_summary(allr, cells_ns, args.northstar_cases, world, f"NCCL x{world}", hbm_peak()[0])
        torch.cuda.empty_cache()
    greens_part = None
    if not args.no_greens_partitioned and not run_g:
        greens_part = {"skipped": f"needs ~{need_g / 1e9:.0f} GB per rank at r = 16, {free_g / 1e9:.0f} GB free",
                       "cells": list(cells_g), "ranks": world}
    if run_g:  # BASELINE configs[4]: the sweep on the partitioned configs[3] mesh
        mine = greens_dist_rank(ts, torch, cells_g, comm, rank, world, sync, args.greens_cases, 16, prebuilt=shared)
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        greens_part = greens_dist_summary(allr, cells_g, world, f"NCCL x{world}", 16, 368)
        torch.cuda.empty_cache()
    del shared
    solve = None
    if not args.no_solve and args.solve_replicas:  # configs[2] replicas (cases batched across the GPUs)
        solve = solve_leg(args, ts, torch, world, rank, local)
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.prec == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"configs[1] x {world}: one {list(cells)}-cell layered-crust tet10 mesh "
                                   f"partitioned over {world} GPUs (RCB), halo exchange every matvec",
                       "cells": list(cells), "elements_per_rank_rank0": E, "nodes_per_rank_rank0": N, "cases_r": r,
                       "precision_tier": precision_tier(args.prec),
                       "parallelism": f"mesh partition x{world} (NCCL send/recv interface halo, overlapped)",
                       "l2_policy": "inputs larger than L2; no flush",
                       "interface_bytes_per_step_rank0": halo_bytes},
            "e2e": {"value": round(total_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
                    "entry": "ts_dist_ebe_op_apply (pinned H2D u, partitioned apply, D2H f)"},
            "roofline": {"bound": "hbm", "achieved": round(B_loc / step_ms / 1e6, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(B_loc / step_ms / 1e6 / peak, 4), "traffic": None, "peak_kind": peak_kind,
                         "kernel": "partitioned apply per rank (boundary sweep; interior sweep || halo exchange)",
                         "kernel_ms": round(step_ms, 4), "alg_bytes_per_launch": int(B_loc)},
            "cpu_baseline": None,
            "clocks": clk.summary(),
            "gpu_launches": 5 * args.steps,
            "northstar": northstar,
            "greens_partitioned": greens_part,
            "solve": solve,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    del comm
    dist.destroy_process_group()


# ------------------------------------------------------------ Green's sweep leg
def greens_leg(args, ts, torch, world, rank, local):
    """configs[4]-style workload at one-GPU scale: the Green's-function bank
    (compute_greens_bank, greens.hpp:114-145) of n unit slips (dip + strike on a
    grid of centres on a vertical fault) on the configs[1] layered box, batched
    r = 16 per solve; total wall time and time per case (setup and a one-batch
    warm-up reported apart).
    Replicas for N > 1 (each rank its own sweep)."""
    import numpy as np
    from paper_1710_08679_b200.greens import DIP, STRIKE, FaultedModel, find_plane_fault_faces

    cells = tuple(args.cells)
    ext, div, ifs = mesh_spec(cells)
    h = CELL_KM * 1e3
    xm = (cells[0] // 2) * h
    t0 = time.perf_counter()
    mesh = ts.generate_box_mesh(ext, div, ifs)
    lo = (xm, 4 * h, 4 * h)
    hi = (xm, (cells[1] - 4) * h, (cells[2] - 8) * h)
    faces = find_plane_fault_faces(mesh, 0, xm, lo, hi)
    cfg = ts.SolverConfig(batch_size=16)
    fm = FaultedModel(mesh, [ts.material_from_wavespeeds(*t) for t in TWO_LAYER], faces, cfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    ny, nz = 6, 4
    ys = np.linspace(lo[1] + 0.15 * (hi[1] - lo[1]), hi[1] - 0.15 * (hi[1] - lo[1]), ny)
    zs = np.linspace(lo[2] + 0.2 * (hi[2] - lo[2]), hi[2] - 0.2 * (hi[2] - lo[2]), nz)
    centers = np.array([[xm, y, z] for y in ys for z in zs for _ in (DIP, STRIKE)])
    dirs = np.array([d for _ in ys for _ in zs for d in (DIP, STRIKE)], np.int32)
    radii = np.full(len(dirs), 0.6 * (hi[1] - lo[1]) / ny)
    gx, gy = np.meshgrid(np.linspace(0.1, 0.9, 10) * ext[0], np.linspace(0.1, 0.9, 10) * ext[1])
    pts = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, ext[2])], 1)
    axes = (np.arange(len(pts)) % 3).astype(np.int32)
    # warm-up: one batch (first-call workspace allocation and module load stay out of the timed sweep)
    fm.greens_bank(centers[:16], dirs[:16], radii[:16], pts, axes, cfg)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        bank, calls, outer = fm.greens_bank(centers, dirs, radii, pts, axes, cfg)
        t_sweep = time.perf_counter() - t1
    t_sweep = max_over_ranks([t_sweep], "cuda")[0]
    n = len(dirs)
    return {"metric": "Green's sweep time per case (s)", "higher_is_better": False,
            "workload": f"configs[4] at one-GPU scale: {n} unit slips (dip+strike, {ny}x{nz} centres) on a vertical "
                        f"fault ({len(faces)} faces, {fm.n_split_nodes} split nodes) in the configs[1] box "
                        f"{list(cells)}, batch 16, {len(pts)} surface observations",
            "value": round(t_sweep / (n * world), 5), "unit": "s", "n_gpus": world, "cases_per_rank": n,
            "sweep_s": round(t_sweep, 3), "setup_s": round(t_setup, 3), "solver_calls": calls,
            "outer_iterations": outer, "bank_shape": list(bank.shape), "bank_finite": bool(np.isfinite(bank).all()),
            "entry": "ts_greens_bank (slip_to_rhs + solve + sampling per batch, host bank out)",
            "clocks": clk.summary()}


# ------------------------------------------------- north star: partitioned solve
FOUR_LAYER = THREE_LAYER + [(8000.0, 4500.0, 3300.0)]  # configs[3]: layered crust over mantle (synthetic)
NORTHSTAR_CELLS = (281, 423, 141)  # configs[3]: 405M DOF (2.8 km cells over 792 x 1192 x 400 km)


# Device bytes per DOF of one rank's partitioned solve at r cases (fp64 outer batches, fp32 level
# vectors, operators, halo and level-2 workspaces): 852 B/DOF measured at r = 8
# (profiles/r02_northstar_half_configs3_one_gpu.json: 173.1 GB for 203.1M DOF); the Green's sweep
# at r = 16 measured 1,697 B/DOF (84.9 GB for 50.0M DOF, one rank: split-mesh fault band, RHS
# batches), 1.03x the model.
def rank_bytes_needed(cells, nranks, r, greens=False):
    nodes = (2 * cells[0] + 1) * (2 * cells[1] + 1) * (2 * cells[2] + 1)
    dof_rank = 3.0 * nodes / nranks * 1.03  # RCB parts are balanced; halo copies a few percent
    return dof_rank * (55.0 + 100.0 * r) * (1.03 if greens else 1.0)


def fits_on_ranks(torch, need, margin=3e9):
    """Whether `need` bytes fit every rank's free device memory (decided together, so that no
    rank starts a leg whose collectives another rank skips)."""
    import torch.distributed as dist
    free, _ = torch.cuda.mem_get_info()
    ok = torch.tensor([1.0 if need + margin <= free else 0.0], device="cuda", dtype=torch.float64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(ok.item() > 0.5), free


def crust_mesh(ts, cells, nranks):
    """The configs[3]-style 4-layer crust box and its RCB partition (every rank builds the same)."""
    from paper_1710_08679_b200.dist import partition_rcb
    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    t0 = time.perf_counter()
    mesh = ts.generate_box_mesh(ext, cells, (0.2 * ext[2], 0.45 * ext[2], 0.8 * ext[2]))
    return mesh, partition_rcb(mesh, nranks), time.perf_counter() - t0


def northstar_rank(ts, torch, cells, r, comm, rank, nranks, sync, steps, prebuilt=None):
    """One rank of the configs[3] workload: build_solver_levels on this rank's RCB
    partition of the global layered-crust mesh (DistLevels: level 2 built once on
    rank 0 and broadcast), manufactured fields (acceptance_main.cpp:82-102) ->
    f = K u* through the partitioned fp64 operator, then ONE timed solve of r cases
    (fp64 outer, fp32 inner, halo exchange inside every product, all-reduced dots).
    `sync()` is a barrier over the ranks. Returns this rank's numbers."""
    import numpy as np
    from paper_1710_08679_b200.dist import DistLevels

    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    t0 = time.perf_counter()
    prebuilt_given = prebuilt is not None
    mesh, part, t_mesh = prebuilt if prebuilt_given else crust_mesh(ts, cells, nranks)
    cfg = ts.SolverConfig(batch_size=r)
    mats = [ts.material_from_wavespeeds(*t) for t in FOUR_LAYER]
    dl = DistLevels(mesh, mats, part, comm, cfg)
    info = dl.info()
    l2g = dl.local_nodes().astype(np.int64)
    xyz = torch.from_numpy(np.asarray(mesh.coords).reshape(-1, 3)[l2g]).cuda()
    mask = torch.from_numpy(mesh.dirichlet_mask().reshape(-1, 3)[l2g].reshape(-1).copy()).cuda().bool()
    n_glob, e_glob = mesh.node_count(), mesh.element_count()
    dl.mesh = None
    del mesh, part, prebuilt
    sync()
    t_setup = time.perf_counter() - t0 + (t_mesh if prebuilt_given else 0.0)
    n = dl.n_local

    g = torch.Generator(device="cuda").manual_seed(31)  # the same cases on every rank
    amp = 0.05 * (1 + 0.2 * (torch.rand(r, device="cuda", dtype=torch.float64, generator=g) * 2 - 1))
    ky = 1.0 + (torch.rand(r, device="cuda", dtype=torch.float64, generator=g) > 0.5).double()

    def manufactured_rows(lo, hi):  # acceptance_main.cpp:82-102 fields at local nodes [lo, hi) -> [3(hi-lo), r]
        X, Y, Z = [xyz[lo:hi, k:k + 1] / ext[k] for k in range(3)]
        sz = torch.sin(0.5 * torch.pi * Z)
        v = torch.stack([amp * torch.sin(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz,
                         amp * torch.cos(torch.pi * X) * torch.sin(ky * torch.pi * Y) * sz,
                         amp * torch.cos(torch.pi * X) * torch.cos(ky * torch.pi * Y) * sz], 1).reshape(3 * (hi - lo), r)
        v[mask[3 * lo:3 * hi]] = 0
        return v

    chunk = 1 << 22  # nodes per piece: the fields are built / checked piecewise (no full-size temporaries)

    def manufactured_local():
        v = torch.empty(3 * n, r, device="cuda", dtype=torch.float64)
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            v[3 * lo:3 * hi] = manufactured_rows(lo, hi)
        return v

    us = manufactured_local()
    f = torch.empty_like(us)
    dl.apply(0, us, f)
    # the partitioned level-0 sweep (fp32, halo exchange overlapped with the interior elements)
    u32 = us.float()
    del us  # regenerated after the solve (device memory: at configs[3] / 2 ranks every fp64 batch is 13 GB)
    f32 = torch.empty_like(u32)
    for _ in range(3):
        dl.apply(1, u32, f32)
    sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        dl.apply(1, u32, f32)
    b.record()
    sync()
    l0_ms = a.elapsed_time(b) / steps
    del u32, f32
    torch.cuda.empty_cache()  # torch's cached blocks back to the driver: the solver allocates its own
    u = torch.zeros_like(f)   # initial guess, solved in place (u0 = out)
    # warm-up: one capped outer iteration allocates the solver workspaces
    try:
        dl.solve(f, u, ts.SolverConfig(batch_size=r, outer_max_iter=1), out=u)
    except ts.ConvergenceError:
        pass
    u.zero_()
    sync()
    a.record()
    u, rep = dl.solve(f, u, cfg, out=u)
    b.record()
    sync()
    solve_s = a.elapsed_time(b) / 1e3
    free, total = torch.cuda.mem_get_info()
    del f
    torch.cuda.empty_cache()
    e2 = n2 = 0.0
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        ref = manufactured_rows(lo, hi)
        e2 += float(((u[3 * lo:3 * hi] - ref) ** 2).sum())
        n2 += float((ref ** 2).sum())
    err2 = torch.tensor([e2, n2], dtype=torch.float64)
    return {"rank": rank, "n_local": n, "elements": info["elements"], "halo_rows0": info["halo_rows0"],
            "neighbours": info["neighbours"], "n2": dl.n2, "levels_setup_s": info["setup_s"], "mesh_s": t_mesh,
            "setup_s": t_setup, "l0_ms": l0_ms, "solve_s": solve_s, "outer": rep.outer_iterations,
            "inner": list(rep.inner_iterations), "time_inner_s": list(rep.time_inner_s),
            "max_final_rel_residual": rep.max_final_residual(), "err2": err2.tolist(),
            "device_used_gb": (total - free) / 1e9, "n_global": n_glob, "e_global": e_glob}


def northstar_summary(per_rank, cells, r, nranks, backend, peak):
    """BASELINE metric 'time per case (s)' of the partitioned solve: the slowest rank's
    solve time / r; the per-rank level-0 sweep roofline (algorithmic bytes / time)."""
    solve_s = max(x["solve_s"] for x in per_rank)
    l0 = []
    for x in per_rank:
        B = alg_bytes(x["elements"], x["n_local"], r, 4)
        l0.append({"rank": x["rank"], "ms": round(x["l0_ms"], 4), "GBps": round(B / x["l0_ms"] / 1e6, 1),
                   "frac": round(B / x["l0_ms"] / 1e6 / peak, 4), "interface_rows": x["halo_rows0"],
                   "interface_bytes": int(x["halo_rows0"]) * 3 * r * 4, "neighbours": x["neighbours"]})
    e2 = sum(x["err2"][0] for x in per_rank)
    n2 = sum(x["err2"][1] for x in per_rank)
    x0 = per_rank[0]
    return {"metric": "time per case (s)", "higher_is_better": False,
            "workload": f"configs[3]-shaped partitioned solve: {list(cells)} cells, {3 * x0['n_global']} DOF, "
                        f"{x0['e_global']} tet10, 4-layer crust, {r} cases, RCB over {nranks} ranks",
            "value": round(solve_s / r, 5), "unit": "s", "ranks": nranks, "backend": backend, "cases": r,
            "solve_s": round(solve_s, 4), "setup_s": round(max(x["setup_s"] for x in per_rank), 2),
            "levels_setup_s": round(max(x["levels_setup_s"] for x in per_rank), 2),
            "mesh_s": round(max(x["mesh_s"] for x in per_rank), 2),
            "outer_iterations": x0["outer"], "inner_iterations": x0["inner"],
            "time_inner_s_rank0": [round(t, 3) for t in x0["time_inner_s"]],
            "max_final_rel_residual": max(x["max_final_rel_residual"] for x in per_rank),
            "rel_err_vs_manufactured": (e2 / max(n2, 1e-300)) ** 0.5, "n2": x0["n2"],
            "l0_sweep_per_rank": l0, "device_used_gb_max": round(max(x["device_used_gb"] for x in per_rank), 1),
            "level2": (os.environ.get("TSGPU_DIST_L2", "auto") if os.environ.get("TSGPU_DIST_L2", "auto") != "auto"
                       else ("distributed" if nranks >= 4 else "replicated")),
            "level2_share_of_solve": round(max(x["time_inner_s"][2] for x in per_rank) / max(solve_s, 1e-9), 4),
            "entry": "ts_dist_levels_create + ts_dist_solve_device (device-resident f / u per rank)"}


def northstar_threads(args, ts, torch, cells, r, P):
    """The north-star leg with P in-process ranks on ONE GPU (ThreadWorld: the same SPMD
    device code as NCCL ranks, halo / all-reduce through device copies)."""
    import threading
    from paper_1710_08679_b200.dist import Comm, ThreadWorld
    world = ThreadWorld(P)
    comms = [Comm.thread(world, k, 0) for k in range(P)]
    bar = threading.Barrier(P)
    out, err = [None] * P, [None] * P

    def body(k):
        try:
            torch.cuda.set_device(0)

            def sync():
                torch.cuda.synchronize()
                bar.wait()
            with torch.cuda.stream(torch.cuda.Stream()):  # each rank its own stream, as on its own GPU
                out[k] = northstar_rank(ts, torch, cells, r, comms[k], k, P, sync, args.steps)
        except BaseException as e:  # noqa: BLE001
            err[k] = e
            bar.abort()
    th = [threading.Thread(target=body, args=(k,)) for k in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    real = [e for e in err if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if real:  # the first rank's own failure, not a peer's "a peer rank failed"
        real.sort(key=lambda e: "peer rank failed" in str(e))
        raise real[0]
    return northstar_summary(out, cells, r, P, f"threads x{P} on one GPU", hbm_peak()[0])


# --------------------------------------- configs[4]: Green's sweep on the partitioned mesh
def greens_dist_rank(ts, torch, cells, comm, rank, nranks, sync, n_cases, batch, prebuilt=None):
    """One rank of the configs[4] workload: compute_greens_bank (greens.hpp:114-145) of
    n_cases unit slips (dip + strike on a grid of centres on a vertical fault) on the
    partitioned layered-crust mesh, batch r = `batch` per solve (ts_dist_greens_bank:
    slip lifting on the fault band per rank, partitioned solve, owner-rank sampling,
    one all-reduce of the bank). One warm-up batch first; returns this rank's numbers."""
    import numpy as np
    from paper_1710_08679_b200.dist import DistFaultedModel
    from paper_1710_08679_b200.greens import DIP, STRIKE, find_plane_fault_faces

    ext = tuple(c * CELL_KM * 1e3 for c in cells)
    h = CELL_KM * 1e3
    xm = (cells[0] // 2) * h
    t0 = time.perf_counter()
    prebuilt_given = prebuilt is not None
    mesh, part, t_mesh = prebuilt if prebuilt_given else crust_mesh(ts, cells, nranks)
    lo = (xm, 4 * h, 4 * h)
    hi = (xm, (cells[1] - 4) * h, (cells[2] - 8) * h)
    faces = find_plane_fault_faces(mesh, 0, xm, lo, hi)
    cfg = ts.SolverConfig(batch_size=batch)
    dfm = DistFaultedModel(mesh, [ts.material_from_wavespeeds(*t) for t in FOUR_LAYER], faces, part, comm, cfg)
    del mesh, part, prebuilt
    sync()
    t_setup = time.perf_counter() - t0 + (t_mesh if prebuilt_given else 0.0)
    nc = n_cases // 2
    ny = max(1, int(round((nc * (hi[1] - lo[1]) / (hi[2] - lo[2])) ** 0.5)))
    nz = max(1, -(-nc // ny))
    ys = np.linspace(lo[1] + 0.1 * (hi[1] - lo[1]), hi[1] - 0.1 * (hi[1] - lo[1]), ny)
    zs = np.linspace(lo[2] + 0.1 * (hi[2] - lo[2]), hi[2] - 0.1 * (hi[2] - lo[2]), nz)
    centers = np.array([[xm, y, z] for y in ys for z in zs for _ in (DIP, STRIKE)])[:n_cases]
    dirs = np.array([d for _ in ys for _ in zs for d in (DIP, STRIKE)], np.int32)[:n_cases]
    radii = np.full(len(dirs), 1.5 * (hi[1] - lo[1]) / ny)
    gx, gy = np.meshgrid(np.linspace(0.1, 0.9, 10) * ext[0], np.linspace(0.1, 0.9, 10) * ext[1])
    pts = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, ext[2])], 1)
    axes = (np.arange(len(pts)) % 3).astype(np.int32)
    dfm.greens_bank(centers[:batch], dirs[:batch], radii[:batch], pts, axes, cfg)  # warm-up batch
    sync()
    t1 = time.perf_counter()
    bank, calls, outer = dfm.greens_bank(centers, dirs, radii, pts, axes, cfg)
    sync()
    free, total = torch.cuda.mem_get_info()
    return {"rank": rank, "sweep_s": time.perf_counter() - t1, "setup_s": t_setup, "calls": calls, "outer": outer,
            "device_used_gb": (total - free) / 1e9,
            "faces": int(len(faces)), "cases": int(len(dirs)), "bank_finite": bool(np.isfinite(bank).all()),
            "bank_absmax": float(np.abs(bank).max()), "bank_sum": float(bank.sum())}


def greens_dist_summary(per_rank, cells, nranks, backend, batch, full_cases):
    sweep = max(x["sweep_s"] for x in per_rank)
    x0 = per_rank[0]
    n = x0["cases"]
    return {"metric": "Green's sweep time per case (s)", "higher_is_better": False,
            "workload": f"configs[4]-shaped sweep: {n} unit slips (of the configuration's {full_cases}) on a "
                        f"vertical fault ({x0['faces']} faces) in the {list(cells)}-cell 4-layer crust, batch {batch}, "
                        f"mesh partitioned over {nranks} ranks (RCB), 100 surface observations",
            "value": round(sweep / n, 5), "unit": "s", "ranks": nranks, "backend": backend, "cases": n,
            "sweep_s": round(sweep, 3), "projected_full_sweep_s": round(sweep / n * full_cases, 1),
            "setup_s": round(max(x["setup_s"] for x in per_rank), 2), "solver_calls": x0["calls"],
            "device_used_gb_max": round(max(x.get("device_used_gb", 0.0) for x in per_rank), 1),
            "outer_iterations": x0["outer"], "bank_finite": all(x["bank_finite"] for x in per_rank),
            "bank_identical_on_ranks": len({(x["bank_absmax"], x["bank_sum"]) for x in per_rank}) == 1,
            "entry": "ts_dist_faulted_model_create + ts_dist_greens_bank"}


def greens_dist_threads(ts, torch, cells, P, n_cases, batch, full_cases):
    import threading
    from paper_1710_08679_b200.dist import Comm, ThreadWorld
    world = ThreadWorld(P)
    comms = [Comm.thread(world, k, 0) for k in range(P)]
    bar = threading.Barrier(P)
    out, err = [None] * P, [None] * P

    def body(k):
        try:
            torch.cuda.set_device(0)

            def sync():
                torch.cuda.synchronize()
                bar.wait()
            with torch.cuda.stream(torch.cuda.Stream()):
                out[k] = greens_dist_rank(ts, torch, cells, comms[k], k, P, sync, n_cases, batch)
        except BaseException as e:  # noqa: BLE001
            err[k] = e
            bar.abort()
    th = [threading.Thread(target=body, args=(k,)) for k in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    real = [e for e in err if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if real:
        real.sort(key=lambda e: "peer rank failed" in str(e))
        raise real[0]
    return greens_dist_summary(out, cells, P, f"threads x{P} on one GPU", batch, full_cases)


# --------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, nargs=3, default=[82, 123, 41])
    ap.add_argument("--cases", type=int, default=16, help="load cases r per GPU")
    ap.add_argument("--prec", type=int, default=32, choices=[32, 64])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-single", action="store_true", help="skip the workers=1 reference timing")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=2)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-greens", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of the partitioned mesh")
    ap.add_argument("--partitioned", action="store_true", help="N=1: run the partitioned (N>1) path with one rank")
    ap.add_argument("--solve-cells", type=int, nargs=3, default=[140, 210, 70], help="configs[2]: 50M DOF")
    ap.add_argument("--solve-cases", type=int, default=16)
    ap.add_argument("--cpu-solve-cells", type=int, nargs=3, default=[16, 16, 16])
    ap.add_argument("--no-northstar", action="store_true", help="skip the partitioned-solve (configs[3]) leg")
    ap.add_argument("--northstar-cells", type=int, nargs=3, default=None,
                    help="mesh of the partitioned solve (default: configs[3] at N > 1, configs[2] at N = 1)")
    ap.add_argument("--northstar-cases", type=int, default=8)
    ap.add_argument("--northstar-l2", default="auto", choices=["auto", "replicated", "distributed"],
                    help="level 2 of the partitioned solve: replicated on every rank, split by coarse rows, "
                         "or auto (split from 4 ranks on)")
    ap.add_argument("--solve-replicas", action="store_true",
                    help="N > 1: also run configs[2] solves as independent replicas (one per GPU)")
    ap.add_argument("--no-greens-partitioned", action="store_true",
                    help="N > 1: skip the configs[4] Green's sweep on the partitioned mesh")
    ap.add_argument("--greens-partitioned", type=int, default=0,
                    help="N = 1: run the partitioned Green's sweep on this many in-process ranks")
    ap.add_argument("--greens-cases", type=int, default=32,
                    help="unit slips of the partitioned sweep (configs[4]: 368 = 23 batches of 16)")
    ap.add_argument("--greens-cells", type=int, nargs=3, default=None,
                    help="mesh of the partitioned sweep (default: configs[3] at N > 1, configs[1] at N = 1)")
    ap.add_argument("--northstar-threads", type=int, default=1,
                    help="N = 1: in-process ranks of the partitioned solve on the one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    os.environ["TSGPU_DIST_L2"] = args.northstar_l2  # read by ts_dist_levels_create
    world, rank, local = dist_setup()

    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo", init_method="env://")
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    if world > 1 and "OMP_NUM_THREADS" not in os.environ:  # ranks share the host cores (setup)
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or world) // world))
    import numpy as np
    import torch

    import paper_1710_08679_b200 as ts

    torch.cuda.set_device(local)
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        if world == 1:  # one-rank partitioned run (exercises the N>1 code path on one GPU)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        with stdout_to_stderr():
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
        if not args.replicas:
            return main_partitioned(args, world, rank, local)

    cells = tuple(args.cells)
    ext, div, ifs = mesh_spec(cells)
    t0 = time.time()
    mesh = ts.generate_box_mesh(ext, div, ifs)
    mats = [ts.material_from_wavespeeds(*t) for t in TWO_LAYER]
    mask = mesh.dirichlet_mask()
    op = ts.EbeOperator(mesh, 2, mats, mask, prec=args.prec)
    op.set_timing(True)
    E, N = op.n_elements(), op.n_nodes()
    log(f"[rank {rank}] mesh {cells}: {E} tet10, {N} nodes ({3 * N} dof), setup {time.time() - t0:.1f}s")
    r, s = args.cases, args.prec // 8
    B = alg_bytes(E, N, r, s)
    dt = torch.float32 if args.prec == 32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    u = torch.rand(3 * N, r, device="cuda", dtype=dt, generator=g) * 2 - 1
    f = torch.empty_like(u)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        op.apply(u, f)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region
    kernel_ms = []
    with ClockSampler(local) as clk:
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            op.apply(u, f)
            kernel_ms.append(op.last_kernel_ms())
        ev1.record(stream)
        barrier()
    step_ms, kms = max_over_ranks([ev0.elapsed_time(ev1) / args.steps, float(np.mean(kernel_ms))], "cuda")
    value = whole_job_gbps(world, B, step_ms)

    # ---- end to end through the C ABI with pinned host buffers
    uh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    uh.copy_(u.cpu())
    fh = torch.empty(u.shape, dtype=dt, pin_memory=True)
    uh_np, fh_np = uh.numpy(), fh.numpy()
    for _ in range(2):
        op.apply(uh_np, fh_np)
    barrier()
    e2e_steps = max(3, args.steps // 2)
    te = time.perf_counter()
    for _ in range(e2e_steps):
        op.apply(uh_np, fh_np)  # ts_ebe_apply_host: H2D u, apply, D2H f
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks([(time.perf_counter() - te) * 1e3 / e2e_steps], "cuda")[0]
    e2e_val = whole_job_gbps(world, B, e2e_ms)
    fd = torch.from_numpy(fh_np).cuda().double()
    ok = bool(torch.isfinite(fd).all()) and float((fd - f.double()).norm() / f.double().norm()) < 1e-5

    peak, peak_kind = hbm_peak()
    traffic = None
    try:
        with open(TRAFFIC_FILE) as fh_:
            tj = json.load(fh_)
        key = f"fp{args.prec}_r{r}_{'x'.join(map(str, cells))}"
        traffic = tj.get(key)
    except Exception:
        pass

    # ---- r sweep (configs[1]: r = 1/4/8/16), fp32 and fp64, kernel + apply time
    sweep = {}
    if not args.no_sweep:
        for prec in (32, 64):
            opp = op if prec == args.prec else ts.EbeOperator(mesh, 2, mats, mask, prec=prec)
            opp.set_timing(True)
            dtp = torch.float32 if prec == 32 else torch.float64
            for rr in (1, 4, 8, 16):
                uu = torch.rand(3 * N, rr, device="cuda", dtype=dtp, generator=g)
                ff = torch.empty_like(uu)
                for _ in range(3):
                    opp.apply(uu, ff)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ks = []
                a.record(stream)
                for _ in range(5):
                    opp.apply(uu, ff)
                    ks.append(opp.last_kernel_ms())
                b.record(stream)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / 5
                bb = alg_bytes(E, N, rr, prec // 8)
                sweep[f"fp{prec}_r{rr}"] = {"apply_ms": round(ms, 4), "kernel_ms": round(float(np.mean(ks)), 4),
                                            "GBps": round(bb / ms / 1e6, 1),
                                            "kernel_frac": round(bb / float(np.mean(ks)) / 1e6 / peak, 4)}
                del uu, ff
            if opp is not op:
                del opp
        # the edge-fan sweep (opt-in kernel 8: 4.5 node rows per element instead of 7) beside it
        os.environ["TSGPU_EBE_KERNEL"] = "fan"
        try:
            opf = ts.EbeOperator(mesh, 2, mats, mask, prec=32)
        finally:
            del os.environ["TSGPU_EBE_KERNEL"]
        opf.set_timing(True)
        for rr in (1, 4, 8, 16):
            uu = torch.rand(3 * N, rr, device="cuda", dtype=torch.float32, generator=g)
            ff = torch.empty_like(uu)
            for _ in range(3):
                opf.apply(uu, ff)
            torch.cuda.synchronize()
            ks = []
            for _ in range(5):
                opf.apply(uu, ff)
                ks.append(opf.last_kernel_ms())
            bb = alg_bytes(E, N, rr, 4)
            sweep[f"fp32_r{rr}_fan"] = {"kernel_ms": round(float(np.mean(ks)), 4),
                                        "kernel_frac": round(bb / float(np.mean(ks)) / 1e6 / peak, 4),
                                        "unit_stats": opf.unit_stats()}
            del uu, ff
        del opf

    # ---- CPU baseline: the reference itself on this host (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            from oracle import Oracle, have_reference
            if have_reference():
                ref = Oracle("reference")
                cores = ref.hw_threads()
                lam = [m.lam for m in mats]
                mu = [m.mu for m in mats]
                sec, _ = ref.time_ebe_apply_box(ext, div, ifs, 1, 2, lam, mu, args.prec, cores, r, args.cpu_reps)
                cpu = {"value": round(B / sec / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                       "cpu_model": cpu_model(),
                       "sample": f"reference EbeOperator<{'float' if args.prec == 32 else 'double'}>::apply on the same "
                                 f"{cells} mesh, r={r}, workers={cores}, 1 warm-up + {args.cpu_reps} timed "
                                 f"({sec:.2f} s/apply)"}
                if not args.no_cpu_single:  # also workers = 1 (the reference's serial path)
                    sec1, _ = ref.time_ebe_apply_box(ext, div, ifs, 1, 2, lam, mu, args.prec, 1, r, 1)
                    cpu["workers1"] = {"value": round(B / sec1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                                       "s_per_apply": round(sec1, 2), "sample": "1 warm-up + 1 timed apply, workers=1"}
            else:
                cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                       "sample": "oracle/_ref not built on this box"}
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"failed: {exc}"}

    # ---- time per case: the full solve (configs[2]) through the host entry
    solve = None
    io_bytes = int(u.numel() * u.element_size())
    if not args.no_solve:
        del u, f, uh, fh, fd
        torch.cuda.empty_cache()
        solve = solve_leg(args, ts, torch, world, rank, local)
    greens = None
    if not args.no_greens:
        torch.cuda.empty_cache()
        greens = greens_leg(args, ts, torch, world, rank, local)
    northstar = None
    if world == 1 and not args.no_northstar:  # the partitioned path on this one GPU (in-process ranks)
        torch.cuda.empty_cache()
        cells_ns = tuple(args.northstar_cells) if args.northstar_cells else tuple(args.solve_cells)
        northstar = northstar_threads(args, ts, torch, cells_ns, args.northstar_cases, args.northstar_threads)
    greens_part = None
    if world == 1 and args.greens_partitioned > 0:
        torch.cuda.empty_cache()
        cells_g = tuple(args.greens_cells) if args.greens_cells else tuple(args.cells)
        greens_part = greens_dist_threads(ts, torch, cells_g, args.greens_partitioned, args.greens_cases, 16, 368)

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.prec == 32 else "f64", "data": "synthetic",
            "config": config_dict(cells, r, args.prec, world, E, N),
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes, "entry": "ts_ebe_apply_host"},
            "roofline": {"bound": "hbm", "achieved": round(B / kms / 1e6, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(B / kms / 1e6 / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": (f"k_ebe_pair<{'float,float2' if args.prec == 32 else 'double,double'},10,{r}>"
                                    if r in (1, 2, 4, 8, 16) else
                                    f"k_ebe_fast<{'float,float2' if args.prec == 32 else 'double,double'},10,12,{r}>"),
                         "kernel_ms": round(kms, 4), "alg_bytes_per_launch": int(B)},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps,
            "r_sweep": sweep,
            "e2e_result_matches_device": ok,
            "solve": solve,
            "greens": greens,
            "northstar": northstar,
            "greens_partitioned": greens_part,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
