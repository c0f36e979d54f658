"""Host-pointer path timing: raw PCIe bandwidth, then vxs_sort_host with the
pipeline off (VXSORT_HOST_CHUNKS=1) and with several chunk/slice settings,
pinned and pageable sources.  Checks every result against np.sort.
    python tools/e2e_probe.py [--workload c2-u32-asc]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2205_05982_b200 as vx  # noqa: E402
from paper_2205_05982_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2-u32-asc")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--settings", default="1x2,8x16,8x32,16x32,16x64")
a = ap.parse_args()
x, kt, desc = workloads.make(a.workload)
tdt = {np.dtype(np.uint32): torch.uint32, np.dtype(np.uint64): torch.uint64,
       np.dtype(np.float32): torch.float32}[x.dtype]
pinned = torch.empty(x.shape, dtype=tdt).pin_memory()
h = pinned.numpy()
h[...] = x
d = torch.empty_like(pinned, device="cuda")
for _ in range(2):
    d.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(pinned, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
pinned.copy_(d, non_blocking=True)
torch.cuda.synchronize()
t2 = time.perf_counter()
print("H2D GB/s", round(x.nbytes / (t1 - t0) / 1e9, 1), "D2H GB/s", round(x.nbytes / (t2 - t1) / 1e9, 1),
      "serial floor ms", round((t2 - t0) * 1e3, 2))
ref = np.sort(x) if not desc else np.sort(x)[::-1]
cfg = vx.SortConfig(order=vx.Order(int(desc)), seed=1)
pageable = np.empty_like(x)
for setting in a.settings.split(","):
    c, s = setting.split("x")
    os.environ["VXSORT_HOST_CHUNKS"] = c
    os.environ["VXSORT_HOST_SLICES"] = s
    for name, buf in (("pinned", h), ("pageable", pageable)):
        ts = []
        for _ in range(a.reps + 1):
            buf[...] = x
            t0 = time.perf_counter()
            vx.sort(buf, cfg)
            ts.append(time.perf_counter() - t0)
        ok = np.array_equal(buf.view(np.uint8), ref.view(np.uint8)) if x.dtype != np.float32 else \
            np.array_equal(buf.view(np.uint32), np.ascontiguousarray(ref).view(np.uint32))
        best = min(ts[1:])
        print(f"chunks={c:>2} slices={s:>2} {name:8s} ms {best * 1e3:7.2f}  {x.shape[0] / best / 1e9:.2f} Gkeys/s  "
              f"equal_np={ok}")
os.environ.pop("VXSORT_HOST_CHUNKS")
os.environ.pop("VXSORT_HOST_SLICES")
