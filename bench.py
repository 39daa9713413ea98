"""Benchmark: FP64 Neo-Hookean Q2 matrix-free Jacobian apply (BASELINE.json
metric, configs[1]: Q2 hex cube 64^3 elements per GPU), GDoF/s.

One step = one Jacobian apply y = J x over the whole mesh (operator.hpp:184,
the reference perf-harness unit, study.hpp:203-212), linearised at u = 0 with
Dirichlet lifting on -x like the harness (study.hpp:198-201), x_i = 1e-3
sin(0.7 i).  N GPUs: weak scaling, the box is split into N slabs along x
(64^3 elements each) and the shared interface planes are summed over NCCL
after every apply (the halo exchange of SURVEY.md §8(e)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement): value is the
device-timed whole-job GDoF/s; e2e is the same metric through the C-ABI
host-buffer entry point (hxg_op_apply_jacobian_host: H2D of x, apply, D2H of
y); roofline / cpu_baseline / clocks as documented in DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 Q2 Neo-Hookean matrix-free Jacobian apply throughput"
UNIT = "GDoF/s"
ORDER, CELLS = 2, 64


def peak_gbs():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    except Exception:
        return 6650.0


def algorithmic_bytes(num_elements, q, ndof):
    """Reference byte model (operator.hpp:137-141 = PAPER.md:476):
    8 (17 E q^3 + 2 N_dof) per Jacobian apply."""
    return 8.0 * (17.0 * num_elements * q**3 + 2.0 * ndof)


# --------------------------------------------------------------------------
# clocks (NVML sampled DURING the timed region)
# --------------------------------------------------------------------------
_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, device_index=0, period=0.005):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for b, n in _REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# --------------------------------------------------------------------------
# CPU baseline / reference arm: the unmodified reference compiled into
# oracle/_ref (kind "reference"), else the numpy port (kind "port").
# --------------------------------------------------------------------------
def cpu_reference_time(order, cells, applies, threads, warmup=1, one_thread_applies=0):
    """Seconds for `applies` Jacobian applies after `warmup`, reference perf
    harness method (study.hpp:196-212); with one_thread_applies > 0 the
    same operator is also timed on one thread (report
    1-thread and all-core), returned as a 5th value."""
    import numpy as np
    from oracle import ref_lib as R
    if R.available():
        rp = R.RefProblem(extents=(1.0, 1.0, 1.0), cells=(cells,) * 3, order=order,
                          fixed=("-x",), threads=threads)
        rp.set_threads(threads)
        u = rp.impose_dirichlet(np.zeros(rp.n))
        rp.apply_residual(u)
        x = 1e-3 * np.sin(0.7 * np.arange(rp.n))
        sec = rp.time_jacobian(x, warmup=warmup, repeats=applies)
        if one_thread_applies > 0:
            rp.set_threads(1)
            sec1 = rp.time_jacobian(x, warmup=0, repeats=one_thread_applies)
            return rp.n, sec, "reference", threads, sec1
        return rp.n, sec, "reference", threads
    from oracle import hexmg_np as H
    P = H.make_problem((1.0, 1.0, 1.0), (cells,) * 3, order)
    P.op.apply_residual(np.zeros(P.op.size))
    x = 1e-3 * np.sin(0.7 * np.arange(P.op.size))
    for _ in range(warmup):
        P.op.apply_jacobian(x)
    t0 = time.perf_counter()
    for _ in range(applies):
        P.op.apply_jacobian(x)
    return P.op.size, time.perf_counter() - t0, "port", 1


# SURVEY.md §8(d) "CPU p-MG solve baseline sizes": the reference's simplicial
# coarse Cholesky (coarse_solver.hpp:44) limits the CPU solve to small cubes
# (Q2 32^3 alone spends ~5 min in the single-threaded coarse factorisation),
# so the default sample is Q2 20^3, Q3 21^3, Q4 16^3 (--cpu-pmg-sizes).
CPU_PMG_SIZES = "2:20,3:21,4:16"


def cpu_pmg_baseline(cases, threads):
    """The compiled reference's p-MG solve on the host cores (study.hpp:83-107
    timing method: setup_numeric and PCG to 1e-8 timed separately): cube,
    fixed -x, traction (0,0,-0.02) on +x, linearised at u = 0."""
    import numpy as np
    from oracle import ref_lib as R
    out = []
    for order, n in cases:
        ref = R.RefProblem(extents=(1, 1, 1), cells=(n,) * 3, order=order, fixed=("-x",),
                           traction_face="+x", traction=(0, 0, -0.02), threads=threads)
        b = -ref.apply_residual(np.zeros(ref.n))
        t0 = time.perf_counter()
        ref.mg_setup()
        t1 = time.perf_counter()
        r = ref.cg(b, precond="mg", rtol=1e-8)
        t2 = time.perf_counter()
        out.append({"order": order, "cells": n, "dofs": ref.n, "setup_numeric_s": t1 - t0,
                    "pcg_rtol1e-8_s": t2 - t1, "pcg_rtol1e-8_iterations": r["iterations"],
                    "condition": r["eig_max"] / r["eig_min"]})
        del ref
    return out


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    t_start = time.perf_counter()
    # each step is one full apply (~0.3-0.5 s on the host cores); at most 100
    # timed and 3 warm-up applies so any --steps K finishes within minutes
    applies, warm = min(args.steps, 100), min(args.warmup, 3)
    ndof, sec, kind, cores = cpu_reference_time(ORDER, CELLS, applies, threads, warmup=warm)
    value = ndof * applies / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec / applies * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (u = 0 linearisation, x_i = 1e-3 sin(0.7 i))",
        "config": {"workload": f"Q{ORDER} Neo-Hookean cube {CELLS}^3 elements, Jacobian apply",
                   "order": ORDER, "cells": [CELLS] * 3, "dofs": ndof},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{applies} Jacobian applies (after {warm} warm-up) of the full "
                                   f"{CELLS}^3 Q{ORDER} problem, {cores} threads "
                                   "(MatrixFreeOperator::set_threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_start,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def make_comm(rank, world, dist, backend):
    """The library's communicator: built-in NCCL, or gloo callbacks (the
    shared-GPU multi-rank test mode)."""
    from paper_2204_01722_b200.distributed import Communicator
    return Communicator(rank, world, dist, backend="nccl" if backend == "nccl" else "gloo")


def run_distributed_pmg(rank, world, dist, stream, comm, mode="auto"):
    """Strong scaling of the cfg4 beam: the partitioned p-MG of the C++
    library (hxg_mg_create_partitioned), slabs along x.  mode "auto": the
    exact coarse solve (global Q1 matrix replicated); "hmg": the inexact
    coarse mode, its h-levels distributed with the slabs."""
    import torch

    from paper_2204_01722_b200.distributed import PartitionedProblem

    cells, order, ext = (96, 48, 48), 2, (2.0, 1.0, 1.0)
    pp = PartitionedProblem(comm, cells, (world, 1, 1), order=order, extents=ext,
                            fixed_faces=("-x",), traction_face="+x", traction=(-0.02, 0.0, 0.0),
                            geometry="box")
    pp.set_coarse_mode(mode)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    f = pp.residual(torch.zeros(pp.size(), dtype=torch.float64, device="cuda"))
    b = -f
    ev[1].record(stream)
    pp.setup_numeric()  # symbolic (global coarse pattern, analysis) + numeric
    pp.cg_solve(b, rtol=1e-3)  # warm-up
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev[2].record(stream)
    pp.setup_numeric()
    ev[3].record(stream)
    rep = pp.cg_solve(b, rtol=1e-8)
    ev[4].record(stream)
    torch.cuda.synchronize()
    # full Newton solve (1 load step, line search) on the slabs
    en = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    en[0].record(stream)
    nrep = pp.solve(load_steps=1)
    en[1].record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3]),
                      ev[3].elapsed_time(ev[4]), en[0].elapsed_time(en[1])], dtype=torch.float64,
                     device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"config": f"Q{order} beam {cells} cells, extents {ext}, fixed -x, traction "
                     f"(-0.02,0,0) on +x, {world} slab(s) along x",
           "dofs": 3 * (order * cells[0] + 1) * (order * cells[1] + 1) * (order * cells[2] + 1),
           "residual_ms": t[0].item(), "setup_numeric_ms": t[1].item(),
           "pcg_rtol1e-8_ms": t[2].item(), "pcg_rtol1e-8_iterations": rep["iterations"],
           "condition": rep["eig_max"] / rep["eig_min"],
           "newton_solve_ms": t[3].item(), "newton_iterations": nrep["newton_iterations"],
           "newton_cg_iterations": nrep["cg_iterations"], "newton_final_fnorm": nrep["final_fnorm"],
           "path": "hxg_mg_create_partitioned (C++ library: interface sums, owned dots, "
                   "partitioned transfers, Newton) over the library's communicator",
           "coarse": "exact: global Q1 matrix summed over the blocks (one all-reduce per setup), "
                     "replicated device Cholesky" if mode == "auto" else
                     "inexact: one Galerkin h-multigrid V-cycle, h-levels distributed with the "
                     "slabs (interface sums, owned dots), replicated dense bottom",
           "timing": "device events, max over ranks"}
    del pp
    torch.cuda.empty_cache()
    return out


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2204_01722_b200.hexmg import FemProblem

    # --dist-backend gloo: every rank may share one GPU (multi-rank test mode)
    torch.cuda.set_device(local_rank % torch.cuda.device_count())
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    # Slab `rank` of a (64 N) x 64 x 64 box (weak scaling), only the global
    # -x face fixed; N > 1: the library's partitioned operator (local fused
    # apply + interface sums over its NCCL communicator).
    from paper_2204_01722_b200.distributed import PartitionedProblem
    comm = make_comm(rank, world, dist, args.dist_backend)
    pp = PartitionedProblem(comm, (CELLS * world, CELLS, CELLS), (world, 1, 1), order=ORDER,
                            extents=(float(world), 1.0, 1.0), fixed_faces=("-x",), geometry=True)
    prob = pp.prob
    op = prob.op
    fixed = ("-x",) if rank == 0 else ()
    N = prob.size()
    u = torch.zeros(N, dtype=torch.float64, device="cuda")
    op.apply_residual(u)  # linearisation state at u = 0 (study.hpp:198-201)
    gidx = torch.arange(N, dtype=torch.float64, device="cuda") + rank * N
    x = 1e-3 * torch.sin(0.7 * gidx)
    y = torch.empty_like(x)
    ndof_job = N * world  # per-rank DoF incl. the shared planes, as study.hpp:196 counts
    stream = torch.cuda.current_stream()

    def step():
        pp.apply(x, y)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local_rank)
    with sampler:
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    value = ndof_job / (ms_per_step * 1e-3) / 1e9

    # Dominant kernel: the apply itself (one fused kernel), timed per launch
    # with events on the launching stream.
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(20)]
    for a, b in ev:
        a.record(stream)
        op.apply_jacobian(x, y)
        b.record(stream)
    torch.cuda.synchronize()
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    alg_bytes = algorithmic_bytes(prob.num_elements, prob.q, N)
    # the two launches of one apply split by an event between them (library
    # instrumentation, events on the operator's stream)
    brick_ms, fixup_ms = op.time_jacobian_parts(x, y, 3, 20)
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_apply_summary.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass

    # BASELINE.json configs[4] scale: Q2 160^3 elements per GPU (99.2 M DoF,
    # ~1e8 DoF per GPU), geometry built on the device; same slab weak scaling.
    cfg5 = None
    if not args.no_cfg5:
        c5 = 160
        # cfg5 weak scaling: one 160^3 block per GPU in a px x py x pz
        # arrangement (2 x 2 x 2 at 8 GPUs), interface sums
        # through faces, edges and corners (the library's partitioned operator)
        dims5 = {2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(world, (world, 1, 1))
        pp5 = PartitionedProblem(comm, tuple(c5 * d for d in dims5), dims5, order=ORDER,
                                 extents=tuple(float(d) for d in dims5), fixed_faces=("-x",),
                                 traction_face="+x", traction=(0.0, 0.0, -0.02), geometry="box")
        prob5 = pp5.prob
        n5 = prob5.size()
        prob5.op.apply_residual(torch.zeros(n5, dtype=torch.float64, device="cuda"))
        x5 = 1e-3 * torch.sin(0.7 * (torch.arange(n5, dtype=torch.float64, device="cuda") + rank * n5))
        y5 = torch.empty_like(x5)

        def step5():
            pp5.apply(x5, y5)

        for _ in range(3):
            step5()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e5 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps5 = 20
        e5[0].record(stream)
        for _ in range(reps5):
            step5()
        e5[1].record(stream)
        torch.cuda.synchronize()
        ms5 = e5[0].elapsed_time(e5[1]) / reps5
        if dist is not None:
            t5 = torch.tensor([ms5], dtype=torch.float64, device="cuda")
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
            ms5 = t5.item()
        b5 = algorithmic_bytes(prob5.num_elements, prob5.q, n5)
        cfg5 = {"config": f"Q2 {c5}^3 elements per GPU, Jacobian apply (BASELINE configs[4] per-GPU "
                          "size), device-built box geometry", "dofs_per_gpu": n5,
                "partition": "x".join(str(d) for d in dims5),
                "ms_per_apply": ms5, "GDoF_s": n5 * world / (ms5 * 1e-3) / 1e9,
                "algorithmic_GB_s_per_gpu": b5 / (ms5 * 1e-3) / 1e9,
                "roofline_frac": b5 / (ms5 * 1e-3) / 1e9 / peak_gbs()}
        if args.cfg5_pmg:
            # the configs[4] p-MG solve at ~1e8 DoF per GPU: only the inexact
            # coarse mode is feasible (an exact factorization of the 12.5 M-DoF
            # Q1 level per GPU is not, SURVEY.md §7.2 hard part 3)
            pp5.set_coarse_mode("hmg")
            z5 = torch.zeros(n5, dtype=torch.float64, device="cuda")
            f5 = pp5.residual(z5)
            pp5.setup_numeric()  # symbolic (patterns) + first numeric
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            e[0].record(stream)
            f5 = pp5.residual(z5)
            e[1].record(stream)
            pp5.setup_numeric()
            e[2].record(stream)
            r5 = pp5.cg_solve(-f5, rtol=1e-8)
            e[3].record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]),
                               e[2].elapsed_time(e[3])], dtype=torch.float64, device="cuda")
            if dist is not None:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            cfg5["pmg_inexact"] = {"residual_ms": tt[0].item(), "setup_numeric_ms": tt[1].item(),
                                   "pcg_rtol1e-8_ms": tt[2].item(),
                                   "pcg_rtol1e-8_iterations": r5["iterations"],
                                   "condition": r5["eig_max"] / r5["eig_min"],
                                   "coarse": "one Galerkin h-multigrid V-cycle (h-levels on the blocks)"}
            del z5, f5, r5
        del pp5, prob5, x5, y5
        torch.cuda.empty_cache()

    # JacobianStorage variants (paper Table III, material.hpp:66-78) on the
    # headline Q2 64^3 problem: bytes per DoF from each variant's state and
    # the measured apply (fused brick kernel for every storage).  Rank 0,
    # N = 1 only.
    storage_table = None
    if world == 1 and not args.no_newton:
        storage_table = []
        for sname in ("current", "initial-native", "initial-tuned", "initial-ad"):
            ps = FemProblem(extents=(1.0, 1.0, 1.0), cells=(CELLS,) * 3, order=ORDER,
                            fixed_faces=fixed, geometry="box", storage=sname)
            ns = ps.size()
            ps.op.apply_residual(torch.zeros(ns, dtype=torch.float64, device="cuda"))
            xs = 1e-3 * torch.sin(0.7 * torch.arange(ns, dtype=torch.float64, device="cuda"))
            ys = torch.empty_like(xs)
            for _ in range(3):
                ps.op.apply_jacobian(xs, ys)
            es = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            es[0].record(stream)
            for _ in range(20):
                ps.op.apply_jacobian(xs, ys)
            es[1].record(stream)
            torch.cuda.synchronize()
            mss = es[0].elapsed_time(es[1]) / 20
            bpd = ps.op.stored_bytes_per_dof()
            storage_table.append({"storage": sname, "bytes_per_dof": bpd, "ms_per_apply": mss,
                                  "GDoF_s": ns / (mss * 1e-3) / 1e9,
                                  "roofline_frac": bpd * ns / (mss * 1e-3) / 1e9 / peak_gbs(),
                                  "path": "fused brick kernel"})
            del ps, xs, ys
            torch.cuda.empty_cache()

    # End-to-end through the C-ABI host-buffer entry point (pinned host x/y).
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xh_np, yh_np = xh.numpy(), yh.numpy()
    for _ in range(2):
        op.apply_jacobian_host(xh_np, yh_np)
    torch.cuda.synchronize()
    e2e_steps = max(5, min(args.steps, 50))
    xd, yd = torch.empty_like(x), torch.empty_like(x)
    e2e_rounds = []
    for _ in range(3):  # the median of three rounds (host-side PCIe / page noise)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            if dist is None:
                op.apply_jacobian_host(xh_np, yh_np)
            else:  # host x -> device, partitioned apply (interface sums), -> host y
                xd.copy_(xh)
                pp.apply(xd, yd)
                yh.copy_(yd)
        e2e_rounds.append((time.perf_counter() - t0) / e2e_steps)
    e2e_s = sorted(e2e_rounds)[1]
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    e2e_value = ndof_job / e2e_s / 1e9

    # p-MG Newton-Krylov step on the same problem (BASELINE.json configs[1]:
    # "single Jacobian apply + Newton-Krylov step"): residual (state), p-MG
    # numeric setup (diagonals, Chebyshev lambda_max, coarse assembly +
    # nested-dissection Cholesky), PCG to the reference's linear_rtol = 1e-3
    # (nonlinear.hpp:20), device-timed.
    newton = newton_inexact = None
    pmg, pmg_inexact = [], []
    if world == 1 and not args.no_newton:
        from paper_2204_01722_b200.hexmg import cg_solve

        def pmg_case(order, cells, newton_step, mode="auto"):
            """p-MG on the cube (fixed -x, traction (0,0,-0.02) on +x, u = 0):
            residual (state), setup_numeric (diagonals, Chebyshev lambda_max,
            coarse assembly + coarse factorization), PCG; device-timed.
            mode "auto": the reference's exact coarse solve (nested-dissection
            Cholesky); "hmg": the inexact coarse mode (one Galerkin h-multigrid
            V-cycle on the p = 1 level, a documented deviation)."""
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            prob_n = FemProblem(extents=(1.0, 1.0, 1.0), cells=(cells,) * 3, order=order,
                                fixed_faces=("-x",), traction_face="+x",
                                traction=(0.0, 0.0, -0.02), geometry="box")
            un = torch.zeros(prob_n.size(), dtype=torch.float64, device="cuda")
            mg = prob_n.hierarchy
            mg.set_coarse_mode(mode)
            prob_n.op.apply_residual(un)
            # warm-up pass of the timed sequence: symbolic analysis, library
            # workspaces and the torch allocations of these calls
            fw = prob_n.op.apply_residual(un)
            mg.setup_numeric()
            cg_solve(prob_n.op, -fw, rtol=1e-3, precond="mg", mg=mg)
            cg_solve(prob_n.op, -fw, rtol=1e-8, precond="mg", mg=mg)
            mg.v_cycle(-fw)
            del fw
            torch.cuda.synchronize()
            evs[0].record(stream)
            fn = prob_n.op.apply_residual(un)
            evs[1].record(stream)
            mg.setup_numeric()
            evs[2].record(stream)
            rep = cg_solve(prob_n.op, -fn, rtol=1e-3, precond="mg", mg=mg)
            evs[3].record(stream)
            rep8 = cg_solve(prob_n.op, -fn, rtol=1e-8, precond="mg", mg=mg)
            evs[3 + 1].record(stream)
            torch.cuda.synchronize()
            # the same solve again (host-synchronous iterations pick up host
            # jitter): report the faster of the two
            ev8 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev8[0].record(stream)
            cg_solve(prob_n.op, -fn, rtol=1e-8, precond="mg", mg=mg)
            ev8[1].record(stream)
            torch.cuda.synchronize()
            # V-cycle alone: mean of 5 on preallocated vectors
            nb = -fn
            xv = torch.zeros_like(nb)
            torch.cuda.synchronize()
            ev_v = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev_v[0].record(stream)
            for _ in range(5):
                mg.v_cycle(nb, xv)
            ev_v[1].record(stream)
            torch.cuda.synchronize()
            if newton_step:
                un += rep["x"]
            out = {"config": f"Q{order} {cells}^3, levels {[mg.level_size(k) for k in range(mg.num_levels())]} DoF",
                   "residual_ms": evs[0].elapsed_time(evs[1]),
                   "setup_numeric_ms": evs[1].elapsed_time(evs[2]),
                   "pcg_rtol1e-3_ms": evs[2].elapsed_time(evs[3]),
                   "pcg_rtol1e-3_iterations": rep["iterations"],
                   "pcg_rtol1e-8_ms": min(evs[3].elapsed_time(evs[4]), ev8[0].elapsed_time(ev8[1])),
                   "pcg_rtol1e-8_iterations": rep8["iterations"],
                   "vcycle_ms": ev_v[0].elapsed_time(ev_v[1]) / 5,
                   "condition": rep8["eig_max"] / rep8["eig_min"],
                   "coarse_mode": "exact (nested-dissection Cholesky)" if mode == "auto"
                   else "inexact (one Galerkin h-multigrid V-cycle)"}
            del prob_n, mg
            torch.cuda.empty_cache()
            return out

        # BASELINE.json configs[1]: single Newton-Krylov step at Q2 64^3
        # (linear_rtol = 1e-3, nonlinear.hpp:20); configs[2]: Q3 / Q4 p-MG.
        def nk_step(nk, solver):
            return {"config": nk["config"] + ", fixed -x, traction (0,0,-0.02) on +x, u = 0",
                    "step_ms": nk["residual_ms"] + nk["setup_numeric_ms"] + nk["pcg_rtol1e-3_ms"],
                    "residual_ms": nk["residual_ms"], "setup_numeric_ms": nk["setup_numeric_ms"],
                    "pcg_ms": nk["pcg_rtol1e-3_ms"], "cg_iterations": nk["pcg_rtol1e-3_iterations"],
                    "linear_rtol": 1e-3, "coarse_solver": solver}

        nk = pmg_case(ORDER, CELLS, True)
        newton = nk_step(nk, "exact: nested-dissection multifrontal Cholesky (device, "
                             "inverse-panel solve)")
        pmg = [nk] + [pmg_case(o, c, False) for o, c in ((3, 43), (4, 32))]
        # the inexact coarse mode beside the exact one (SURVEY.md §7.2 hard
        # part 3): same problems, coarse level = one h-multigrid V-cycle
        nki = pmg_case(ORDER, CELLS, True, "hmg")
        newton_inexact = nk_step(nki, "inexact: one Galerkin h-multigrid V-cycle on the p = 1 "
                                      "level (Chebyshev-Jacobi, dense-inverse bottom)")
        pmg_inexact = [nki] + [pmg_case(o, c, False, "hmg") for o, c in ((3, 43), (4, 32))]

    # Full Newton solve of the compressed beam (BASELINE.json configs[3] on one
    # GPU): FemProblem::solve with load continuation (1 step), critical-point
    # line search, p-MG rebuilt at every Newton iterate; device-timed.
    newton_full = None
    if world == 1 and not args.no_newton:
        prob_b = FemProblem(extents=(2.0, 1.0, 1.0), cells=(96, 48, 48), order=2,
                            fixed_faces=("-x",), traction_face="+x", traction=(-0.02, 0.0, 0.0),
                            geometry="box")
        eb = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        eb[0].record(stream)
        rep_b = prob_b.solve(load_steps=1)
        eb[1].record(stream)
        torch.cuda.synchronize()
        newton_full = {"config": "Q2 beam (96, 48, 48) cells, extents (2,1,1), fixed -x, traction "
                                 "(-0.02,0,0) on +x, 1 load step, critical-point line search",
                       "dofs": prob_b.size(), "solve_ms": eb[0].elapsed_time(eb[1]),
                       "newton_iterations": rep_b["newton_iterations"],
                       "cg_iterations": rep_b["cg_iterations"],
                       "final_fnorm": rep_b["final_fnorm"], "converged": rep_b["converged"],
                       "note": "includes the symbolic (first) p-MG setup"}
        del prob_b, rep_b
        torch.cuda.empty_cache()
        # the same solve with the inexact coarse mode
        prob_b = FemProblem(extents=(2.0, 1.0, 1.0), cells=(96, 48, 48), order=2,
                            fixed_faces=("-x",), traction_face="+x", traction=(-0.02, 0.0, 0.0),
                            geometry="box")
        prob_b.hierarchy.set_coarse_mode("hmg")
        torch.cuda.synchronize()
        eb[0].record(stream)
        rep_b = prob_b.solve(load_steps=1)
        eb[1].record(stream)
        torch.cuda.synchronize()
        newton_full["inexact_coarse"] = {
            "solve_ms": eb[0].elapsed_time(eb[1]), "newton_iterations": rep_b["newton_iterations"],
            "cg_iterations": rep_b["cg_iterations"], "final_fnorm": rep_b["final_fnorm"],
            "converged": rep_b["converged"],
            "coarse_solver": "one Galerkin h-multigrid V-cycle on the p = 1 level"}
        del prob_b, rep_b
        torch.cuda.empty_cache()

    # Slab-partitioned p-MG PCG on the compressed beam (BASELINE.json
    # configs[3]: Q2, 96 x 48 x 48 cells over N GPUs, strong scaling; halo
    # exchange over NCCL), device-timed, max over ranks: exact coarse mode
    # (replicated Cholesky) and the inexact mode (distributed h-levels).
    pmg_dist = pmg_dist_inexact = None
    if not args.no_newton:
        pmg_dist = run_distributed_pmg(rank, world, dist, stream, comm)
        pmg_dist_inexact = run_distributed_pmg(rank, world, dist, stream, comm, "hmg")

    # CPU baseline: the reference on the host cores, rank 0, N = 1 only.
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            res = cpu_reference_time(ORDER, CELLS, args.cpu_applies, threads, one_thread_applies=2)
            ndof_c, sec, kind, cores = res[:4]
            cpu = {"value": ndof_c * args.cpu_applies / sec / 1e9, "unit": UNIT, "cores": cores,
                   "kind": kind,
                   "sample": f"{args.cpu_applies} Jacobian applies of the same {CELLS}^3 "
                             f"Q{ORDER} problem after 1 warm-up, {cores} threads"}
            if len(res) > 4:
                cpu["one_thread"] = {"value": ndof_c * 2 / res[4] / 1e9, "unit": UNIT,
                                     "sample": "2 applies of the same operator on 1 thread"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"failed: {exc}"}

    # CPU p-MG solve baseline beside the GPU at the same sizes (rank 0, N = 1).
    cpu_pmg = None
    if (rank == 0 and world == 1 and not args.no_cpu_baseline and not args.no_newton
            and args.cpu_pmg_sizes):
        cases = [tuple(int(v) for v in c.split(":")) for c in args.cpu_pmg_sizes.split(",")]
        threads = os.cpu_count() or 1
        try:
            rows = cpu_pmg_baseline(cases, threads)
            for row in rows:
                g = pmg_case(row["order"], row["cells"], False)
                row["gpu"] = {"setup_numeric_s": g["setup_numeric_ms"] * 1e-3,
                              "pcg_rtol1e-8_s": g["pcg_rtol1e-8_ms"] * 1e-3,
                              "pcg_rtol1e-8_iterations": g["pcg_rtol1e-8_iterations"]}
                row["iterations_within_1"] = abs(g["pcg_rtol1e-8_iterations"]
                                                 - row["pcg_rtol1e-8_iterations"]) <= 1
                row["speedup_setup"] = row["setup_numeric_s"] / row["gpu"]["setup_numeric_s"]
                row["speedup_pcg"] = row["pcg_rtol1e-8_s"] / row["gpu"]["pcg_rtol1e-8_s"]
            cpu_pmg = {"kind": "reference", "cores": threads, "cases": rows,
                       "note": "compiled reference (oracle/_ref, Eigen-API shim for the Lanczos "
                               "eigensolve and SimplicialLLT: a restatement, single-threaded) vs "
                               "this library on cuda:0; wall seconds (CPU) / device events (GPU)"}
        except Exception as exc:  # noqa: BLE001
            cpu_pmg = {"kind": "reference", "cores": threads, "failed": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (u = 0 linearisation, x_i = 1e-3 sin(0.7 i))",
            "config": {"workload": f"Q{ORDER} Neo-Hookean cube {CELLS}^3 elements per GPU, "
                                   "Jacobian apply", "order": ORDER, "q": prob.q,
                       "cells_per_gpu": [CELLS] * 3, "dofs_per_gpu": N,
                       "parallelism": f"slab x{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (state 963 MB/GPU)",
                       "bytes_per_dof_model": alg_bytes / N},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel_ms": kern_ms, "algorithmic_bytes": alg_bytes,
                         "scope": "whole apply (brick kernel + boundary fix-up kernel)",
                         "kernels": {"fused_jacobian_kernel": {"ms": brick_ms, "share": brick_ms / (brick_ms + fixup_ms),
                                                               "alg_bytes_over_ms_GBs": alg_bytes / (brick_ms * 1e-3) / 1e9},
                                     "fused_fixup_kernel": {"ms": fixup_ms, "share": fixup_ms / (brick_ms + fixup_ms)}},
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                    "d2h_bytes_per_step": 8 * N, "ms_per_step": e2e_s * 1e3,
                    "rounds_ms": [round(t * 1e3, 3) for t in e2e_rounds],
                    "path": "hxg_op_apply_jacobian_host (pinned host buffers)"},
            "gpu_launches": args.steps * op.kernel_launches(),
            "clocks": sampler.summary(),
            "cpu_baseline": cpu,
            "cpu_pmg": cpu_pmg,
            "newton_krylov_step": newton,
            "newton_krylov_step_inexact": newton_inexact,
            "pmg_solves": pmg,
            "pmg_solves_inexact": pmg_inexact,
            "pmg_distributed": pmg_dist,
            "pmg_distributed_inexact": pmg_dist_inexact,
            "newton_solve": newton_full,
            "apply_cfg5": cfg5,
            "storage_variants": storage_table,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 1000 for our arm, 50 for the reference arm)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-applies", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-pmg-sizes", default=CPU_PMG_SIZES,
                    help="order:cells,... of the CPU p-MG solve baseline ('' to skip)")
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--cfg5-pmg", action="store_true",
                    help="also run the configs[4] p-MG solve (inexact coarse mode) at Q2 160^3 per GPU")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the N > 1 path with every rank on one GPU")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 50 if args.impl == "reference" else 1000
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        print(json.dumps({"error": "launch N>1 under torch.distributed.run"}))
        return
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
