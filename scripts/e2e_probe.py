"""Host-buffer apply timing vs chunk count and raw PCIe copy rates (dev helper)."""
import os, sys, time, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2204_01722_b200.hexmg import FemProblem
    prob = FemProblem(extents=(1, 1, 1), cells=(64, 64, 64), order=2, fixed_faces=("-x",))
    N = prob.size()
    prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
    xh = (1e-3 * torch.sin(0.7 * torch.arange(N, dtype=torch.float64))).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    for _ in range(3): prob.op.apply_jacobian_host(xh.numpy(), yh.numpy())
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(30): prob.op.apply_jacobian_host(xh.numpy(), yh.numpy())
    dt = (time.perf_counter() - t0) / 30
    print(json.dumps({"chunks": os.environ.get("HXG_HOST_CHUNKS"), "ms": dt * 1e3, "gdofs": N / dt / 1e9}))
    sys.exit(0)
n = 6440067
a = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty_like(d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, f in [("h2d", lambda: d.copy_(a, non_blocking=True)), ("d2h", lambda: b.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
    print(name, f"{n*8/dt/1e9:.1f} GB/s", flush=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1): d.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
print("both", f"{2*n*8/dt/1e9:.1f} GB/s aggregate, {dt*1e3:.3f} ms per pair", flush=True)
for c in (8, 16):
    for extra in ({}, {"HXG_HOST_NOCOMPUTE": "1"}):
        out = subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, HXG_HOST_CHUNKS=str(c), **extra), capture_output=True, text=True)
        print(extra, out.stdout.strip() or out.stderr[-500:], flush=True)
