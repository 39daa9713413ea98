"""Reproduce bench.py's pmg_case timing sequence (dev helper)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve
stream = torch.cuda.current_stream()
for order, cells in ((2, 64), (4, 32), (2, 64)):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    p = FemProblem(extents=(1.0, 1.0, 1.0), cells=(cells,) * 3, order=order, fixed_faces=("-x",),
                   traction_face="+x", traction=(0.0, 0.0, -0.02))
    un = torch.zeros(p.size(), dtype=torch.float64, device="cuda")
    mg = p.hierarchy
    p.op.apply_residual(un)
    mg.setup_numeric()
    cg_solve(p.op, torch.ones_like(un), rtol=1e-1, precond="mg", mg=mg)
    torch.cuda.synchronize()
    evs[0].record(stream); fn = p.op.apply_residual(un); evs[1].record(stream)
    mg.setup_numeric(); evs[2].record(stream)
    r3 = cg_solve(p.op, -fn, rtol=1e-3, precond="mg", mg=mg); evs[3].record(stream)
    r8 = cg_solve(p.op, -fn, rtol=1e-8, precond="mg", mg=mg); evs[4].record(stream)
    mg.v_cycle(-fn); evs[5].record(stream)
    mg.v_cycle(-fn); evs[6].record(stream)
    torch.cuda.synchronize()
    free, tot = torch.cuda.mem_get_info()
    print(json.dumps({"case": f"Q{order} {cells}", "setup": evs[1].elapsed_time(evs[2]), "pcg3": evs[2].elapsed_time(evs[3]),
                      "pcg8": evs[3].elapsed_time(evs[4]), "vc1": evs[4].elapsed_time(evs[5]), "vc2": evs[5].elapsed_time(evs[6]),
                      "free_gb": free / 1e9}), flush=True)
    del p, mg, fn, un
    torch.cuda.empty_cache()
