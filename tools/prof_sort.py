"""Small driver for ncu captures: sorts one workload a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_05982_b200 as vx  # noqa: E402
from paper_2205_05982_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2-u32-asc")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
x, kt, desc = workloads.make(a.workload, n=a.n)
src = torch.from_numpy(x).cuda()
buf = torch.empty_like(src)
ws = torch.empty(vx.workspace_bytes(x.shape[0], kt), dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    buf.copy_(src)
    st = vx.sort(buf, vx.SortConfig(order=vx.Order(int(desc)), seed=1),
                 key_type=kt if kt in ("k128", "kv64") else None, workspace=ws)
torch.cuda.synchronize()
print("ok", st.as_dict())
