"""f32 normal keys with / without the 0.1% special values (experiments)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_05982_b200 as vx
from paper_2205_05982_b200 import workloads
x, kt, desc = workloads.make("c2-f32-asc")
spec = ~np.isfinite(x) | (x == 0)
y = x.copy()
y[spec] = np.float32(1.5)  # replace the specials by one ordinary value -> still 1e5 duplicates
z = x.copy()
rng = np.random.default_rng(3)
z[spec] = (rng.standard_normal(int(spec.sum())) * 1e3).astype(np.float32)  # no duplicates at all
for name, arr in (("with-specials", x), ("dups-of-1.5", y), ("no-dups", z)):
    src = torch.from_numpy(arr).cuda(); buf = torch.empty_like(src)
    ws = torch.empty(vx.workspace_bytes(arr.shape[0], kt), dtype=torch.uint8, device="cuda")
    cfg = vx.SortConfig(order=vx.Order(0), seed=1)
    for _ in range(2):
        buf.copy_(src); vx.sort(buf, cfg, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        buf.copy_(src); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); vx.sort(buf, cfg, workspace=ws); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    vx.profile_reset(); vx.profile_enable(True)
    buf.copy_(src); vx.sort(buf, cfg, workspace=ws); torch.cuda.synchronize()
    prof = vx.profile_read(); vx.profile_enable(False)
    print(name, "ms", round(min(ts), 4), {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:9]})
