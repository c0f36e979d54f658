import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2205_05982_b200 as vx
from paper_2205_05982_b200 import workloads
x, kt, desc = workloads.make("c2-u32-asc")
pinned = torch.empty(x.shape, dtype=torch.uint32).pin_memory(); h = pinned.numpy(); h[...] = x
d = torch.empty_like(pinned, device="cuda")
for _ in range(2): d.copy_(pinned, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(pinned, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
pinned.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
print("H2D GB/s", round(4e8 / (t1 - t0) / 1e9, 1), "D2H GB/s", round(4e8 / (t2 - t1) / 1e9, 1))
for i in range(4):
    h[...] = x
    t0 = time.perf_counter(); vx.sort(h); t1 = time.perf_counter()
    print("e2e ms", round((t1 - t0) * 1e3, 2))
