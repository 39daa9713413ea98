"""Study harness (study.hpp): the accuracy-per-DoF study and the operator
throughput study with the reference's CSV schemas, so their outputs diff
against the reference's byte for byte in every deterministic column.

  * format_double / csv_row            study.hpp:19-33
  * accuracy_csv_header / _row         study.hpp:50-64
  * run_accuracy_study                 study.hpp:66-141
  * performance_csv_header / _row      study.hpp:157-168
  * run_performance_study              study.hpp:170-233

Times are host steady-clock seconds around device-synchronised work, as in
the reference; setup_seconds covers problem construction on the device."""
from __future__ import annotations

import math
import time

import torch

from .config import ConfigError, ProblemConfig, StudyCase, build_problem, newton_overrides


def format_double(v: float) -> str:
    """'%.17g' (round-trip exact)."""
    return "%.17g" % v


def csv_row(cells) -> str:
    return ",".join(cells)


def accuracy_csv_header() -> str:
    return ("case_id,order,refinement,dofs,strain_energy,rel_energy_error,newton_iterations,"
            "cg_iterations,condition_max,bytes_per_dof,setup_seconds,solve_seconds,"
            "dofs_per_second")


def accuracy_csv_row(r: dict) -> str:
    return csv_row([r["case_id"], str(r["order"]), str(r["refinement"]), str(r["dofs"]),
                    format_double(r["energy"]), format_double(r["rel_error"]),
                    str(r["newton_iterations"]), str(r["cg_iterations"]),
                    format_double(r["condition_max"]), format_double(r["bytes_per_dof"]),
                    format_double(r["setup_seconds"]), format_double(r["solve_seconds"]),
                    format_double(r["dofs_per_second"])])


def performance_csv_header() -> str:
    return ("case_id,representation,order,cells,dofs,nnz,bytes_per_dof,applies,status,seconds,"
            "dofs_per_second")


def performance_csv_row(r: dict) -> str:
    return csv_row([r["case_id"], r["representation"], str(r["order"]), str(r["cells"]),
                    str(r["dofs"]), str(r["nnz"]), format_double(r["bytes_per_dof"]),
                    str(r["applies"]), r["status"], format_double(r["seconds"]),
                    format_double(r["dofs_per_second"])])


def case_config(base: ProblemConfig, c: StudyCase) -> ProblemConfig:
    """detail::case_config (study.hpp:68-75)."""
    return base.copy(case_id=c.id(), order=c.order,
                     cells=[n * c.refinement for n in base.cells], study_cases=[])


def run_case(cfg: ProblemConfig, c: StudyCase, reference_line_search_quirk=False):
    """detail::run_case (study.hpp:82-110): build, solve with load
    continuation, strain energy of the solution."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = build_problem(cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = prob.solve(**newton_overrides(cfg, reference_line_search_quirk))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    energy = prob.op.total_strain_energy(rep["u"])
    cond = max([it["condition_estimate"] for it in rep.get("records", [])] or [0.0])
    r = {"case_id": c.id(), "order": c.order, "refinement": c.refinement, "dofs": prob.size(),
         "energy": energy, "rel_error": 0.0, "newton_iterations": rep["newton_iterations"],
         "cg_iterations": rep["cg_iterations"], "condition_max": cond,
         "bytes_per_dof": prob.op.stored_bytes_per_dof(), "setup_seconds": t1 - t0,
         "solve_seconds": t2 - t1}
    r["dofs_per_second"] = r["dofs"] / r["solve_seconds"] if r["solve_seconds"] > 0 else 0.0
    return r


def run_accuracy_study(base: ProblemConfig, csv, log=None, reference_line_search_quirk=False):
    """run_accuracy_study (study.hpp:114-141): the overkill reference case
    first, then every case with its relative strain-energy error."""
    if not base.study_cases:
        raise ConfigError("study_cases must list at least one case")
    seen = set()
    for c in base.study_cases:
        if c.id() in seen:
            raise ConfigError(f"duplicate study case '{c.id()}'")
        seen.add(c.id())
    if base.study_reference.id() in seen:
        raise ConfigError("reference case duplicates a study case")
    if log:
        log.write(f"reference case {base.study_reference.id()}\n")
    ref = run_case(case_config(base, base.study_reference), base.study_reference,
                   reference_line_search_quirk)
    if ref["energy"] == 0.0:
        raise RuntimeError("reference case produced zero energy")
    records = []
    csv.write(accuracy_csv_header() + "\n")
    for c in base.study_cases:
        if log:
            log.write(f"case {c.id()}\n")
        r = run_case(case_config(base, c), c, reference_line_search_quirk)
        r["rel_error"] = abs(r["energy"] - ref["energy"]) / abs(ref["energy"])
        csv.write(accuracy_csv_row(r) + "\n")
        records.append(r)
    return records


def perf_cells(target: int, order: int) -> int:
    """Cube with ~target DoFs: 3 (p n + 1)^3 ~= target (study.hpp:180-181)."""
    return max(1, int(_lround((math.cbrt(target / 3.0) - 1.0) / order)))


def _lround(x):
    return math.floor(x + 0.5) if x >= 0 else math.ceil(x - 0.5)


def run_performance_study(base: ProblemConfig, csv, log=None):
    """run_performance_study (study.hpp:170-233): repeated Jacobian applies
    at the zero linearization state after 3 discarded warm-ups, for the
    matrix-free and assembled representations; out-of-memory cases become
    failed rows."""
    from .hexmg import AssembledOperator
    records = []
    csv.write(performance_csv_header() + "\n")
    for order in base.perf_orders:
        for target in base.perf_target_dofs:
            n = perf_cells(target, order)
            for repr_ in base.perf_representations:
                rec = {"case_id": f"p{order}n{n}_{repr_}", "representation": repr_,
                       "order": order, "cells": n, "dofs": 0, "nnz": 0, "bytes_per_dof": 0.0,
                       "applies": 0, "status": "ok", "seconds": 0.0, "dofs_per_second": 0.0}
                if log:
                    log.write(f"perf case {rec['case_id']}\n")
                try:
                    cfg = base.copy(order=order, cells=[n, n, n], extents=[1.0, 1.0, 1.0])
                    prob = build_problem(cfg)
                    N = prob.size()
                    rec["dofs"] = N
                    u = torch.zeros(N, dtype=torch.float64, device="cuda")
                    prob.op.apply_residual(u)  # populate the linearization state
                    x = 1e-3 * torch.sin(0.7 * torch.arange(N, dtype=torch.float64, device="cuda"))
                    y = torch.empty_like(x)
                    if repr_ == "matrix-free":
                        rec["bytes_per_dof"] = prob.op.stored_bytes_per_dof()

                        def apply():
                            prob.op.apply_jacobian(x, y)
                    else:
                        A = AssembledOperator(prob.op)
                        A.numeric()
                        rec["nnz"] = A.nnz
                        rec["bytes_per_dof"] = (A.nnz * (8 + 4) + (N + 1) * 4 + 2.0 * N * 8) / N

                        def apply():
                            A.matvec(x, y)
                    for _ in range(3):
                        apply()
                    torch.cuda.synchronize()  # steady clock around the applies, as the reference
                    t0 = time.perf_counter()
                    for _ in range(base.perf_repeats):
                        apply()
                    torch.cuda.synchronize()
                    rec["seconds"] = time.perf_counter() - t0
                    rec["applies"] = base.perf_repeats
                    if rec["seconds"] > 0:
                        rec["dofs_per_second"] = N * rec["applies"] / rec["seconds"]
                except torch.cuda.OutOfMemoryError:
                    rec["status"] = "out-of-memory"
                except RuntimeError as exc:
                    # device allocation failures and CSR index spaces beyond
                    # int32 (the reference's bad_alloc range) become failed rows
                    msg = str(exc).lower()
                    if "out of memory" not in msg and "exceeds int32" not in msg:
                        raise
                    rec["status"] = "out-of-memory"
                csv.write(performance_csv_row(rec) + "\n")
                records.append(rec)
    return records


if __name__ == "__main__":
    import sys
    from .config import load_problem_config
    if len(sys.argv) != 3 or sys.argv[2] not in ("accuracy", "performance"):
        sys.exit("usage: python -m paper_2204_01722_b200.study <config> accuracy|performance")
    cfg = load_problem_config(sys.argv[1])
    run = run_accuracy_study if sys.argv[2] == "accuracy" else run_performance_study
    run(cfg, sys.stdout, sys.stderr)
