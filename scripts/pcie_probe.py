"""Raw chunked H2D -> D2H pipeline over torch streams (dev helper): what the
host-buffer apply can reach without compute."""
import time, torch
n = 6440067
xh = torch.empty(n, dtype=torch.float64).pin_memory(); yh = torch.empty_like(xh).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda"); yd = torch.empty_like(xd)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
def run(C, mode):
    bounds = [n * i // C for i in range(C + 1)]
    evs = [torch.cuda.Event() for _ in range(C)]
    for i in range(C):
        a, b = bounds[i], bounds[i + 1]
        with torch.cuda.stream(s_in):
            xd[a:b].copy_(xh[a:b], non_blocking=True); evs[i].record(s_in)
        if mode == "interleave":
            with torch.cuda.stream(s_out):
                s_out.wait_event(evs[i]); yh[a:b].copy_(xd[a:b], non_blocking=True)
    if mode == "after":
        for i in range(C):
            a, b = bounds[i], bounds[i + 1]
            with torch.cuda.stream(s_out):
                s_out.wait_event(evs[i]); yh[a:b].copy_(xd[a:b], non_blocking=True)
    s_out.synchronize()
for mode in ("interleave", "after"):
    for C in (2, 4, 8, 16, 32):
        run(C, mode); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20): run(C, mode)
        dt = (time.perf_counter() - t0) / 20
        print(mode, C, f"{dt*1e3:.3f} ms", flush=True)
