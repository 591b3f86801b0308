"""Pinned host <-> device copy bandwidth on the GPU box (the e2e transfer ceiling)."""
import torch, time, numpy as np
torch.cuda.init()
n = 140_000_000 // 8 * 8
a = np.random.rand(n // 8 * 1)  # ~140MB? n doubles = 1.1 GB; use smaller
a = np.ones(17_500_000)  # 140 MB
d = torch.empty(a.size, dtype=torch.float64, device="cuda")
t = torch.from_numpy(a)
for name, src in [("pageable", t), ("pinned", t.pin_memory())]:
    d.copy_(src); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): d.copy_(src)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(name, "H2D GB/s", a.nbytes / dt / 1e9)
t0 = time.perf_counter(); p = t.pin_memory(); print("pin_memory copy s", time.perf_counter() - t0)
cr = torch.cuda.cudart()
t0 = time.perf_counter(); r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0); print("register s", time.perf_counter() - t0, r)
t0 = time.perf_counter(); d.copy_(torch.from_numpy(a), non_blocking=True); torch.cuda.synchronize(); print("registered copy GB/s", a.nbytes / (time.perf_counter() - t0) / 1e9)
h = torch.empty(a.size, dtype=torch.float64)
t0 = time.perf_counter(); h.copy_(d); print("D2H pageable GB/s", a.nbytes / (time.perf_counter() - t0) / 1e9)
import os; print("cpus", os.cpu_count())
