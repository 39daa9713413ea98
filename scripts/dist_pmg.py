"""Slab-partitioned p-MG PCG on the compressed beam (BASELINE configs[3]):
python -m torch.distributed.run --nproc-per-node N scripts/dist_pmg.py [cx cy cz] (or plain python for N = 1)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.distributed import DistributedHierarchy, SlabBackend, SlabComm, distributed_pcg
from paper_2204_01722_b200.hexmg import FemProblem, constraint_mask, cg_solve
from paper_2204_01722_b200.partition import slab_partition

cells = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (96, 48, 48)
order = 2
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
ext = (2.0, 1.0, 1.0)
slab = slab_partition(cells, world, rank, order)
h = ext[0] / cells[0]
fixed = ("-x",) if rank == 0 else ()
prob = FemProblem(extents=(h * slab.cells[0], ext[1], ext[2]), cells=slab.cells, order=order,
                  fixed_faces=fixed, traction_face="+x" if rank == world - 1 else None,
                  traction=(-0.02, 0.0, 0.0))
comm = SlabComm(rank, world, dist)
f = prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
comm.exchange(f, slab.npd)
b = -f
t0 = time.perf_counter()
hier = DistributedHierarchy(SlabBackend(prob, fixed), comm, cells, slab.x0,
                            lambda p: constraint_mask(cells, p, ("-x",))[0])
hier.setup_numeric(); torch.cuda.synchronize(); t1 = time.perf_counter()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record(); hier.setup_numeric(); ev[1].record()
r3 = distributed_pcg(hier, b, rtol=1e-3); ev[2].record()
r8 = distributed_pcg(hier, b, rtol=1e-8); ev[3].record(); torch.cuda.synchronize()
res = {"rank": rank, "world": world, "cells": cells, "first_setup_s": t1 - t0,
       "setup_ms": ev[0].elapsed_time(ev[1]), "pcg1e-3_ms": ev[1].elapsed_time(ev[2]),
       "its1e-3": r3["iterations"], "pcg1e-8_ms": ev[2].elapsed_time(ev[3]), "its1e-8": r8["iterations"],
       "lambda_max": hier.lambda_max[1:]}
if world == 1:
    mg = prob.hierarchy
    mg.setup_numeric()
    rep = cg_solve(prob.op, b, rtol=1e-8, precond="mg", mg=mg)
    res["local_its1e-8"] = rep["iterations"]
    res["rel_diff_vs_local"] = float(torch.linalg.norm(rep["x"] - r8["x"]) / torch.linalg.norm(rep["x"]))
    res["local_lambda_max"] = [mg.lambda_max(k) for k in range(1, mg.num_levels())]
print(json.dumps(res), flush=True)
if dist is not None:
    dist.destroy_process_group()
