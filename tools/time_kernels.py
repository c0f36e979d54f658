"""Per-kernel device times of one workload (no validation; for experiments).
    python tools/time_kernels.py --workload c2-u32-asc --reps 5"""
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
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--op", default="sort", choices=["sort", "argsort", "pairs", "nth", "topk1000"])
a = ap.parse_args()
x, kt, desc = workloads.make(a.workload, n=a.n)
src = torch.from_numpy(x).cuda()
buf = torch.empty_like(src)
ws = torch.empty(vx.workspace_bytes(x.shape[0], kt), dtype=torch.uint8, device="cuda")
cfg = vx.SortConfig(order=vx.Order(int(desc)), seed=1)
ktarg = kt if kt in ("k128", "kv64") else None
vals = torch.empty(x.shape[0], dtype=torch.int32, device="cuda") if a.op == "pairs" else None


def run_op():
    if a.op == "sort":
        vx.sort(buf, cfg, key_type=ktarg, workspace=ws)
    elif a.op == "argsort":
        vx.argsort(buf, cfg.order, key_type=ktarg)
    elif a.op == "pairs":
        vx.sort_pairs(buf, vals, cfg, key_type=ktarg)
    elif a.op == "nth":
        vx.nth_element(buf, x.shape[0] // 3, cfg, key_type=ktarg, workspace=ws)
    else:
        vx.partial_sort(buf, 1000, cfg, key_type=ktarg, workspace=ws)


for _ in range(2):
    buf.copy_(src)
    run_op()
torch.cuda.synchronize()
plain = []
for _ in range(a.reps):  # unprofiled (no per-launch events)
    buf.copy_(src)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run_op()
    e.record()
    torch.cuda.synchronize()
    plain.append(s.elapsed_time(e))
vx.profile_reset()
vx.profile_enable(True)
ev = []
for _ in range(a.reps):
    buf.copy_(src)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run_op()
    e.record()
    torch.cuda.synchronize()
    ev.append(s.elapsed_time(e))
prof = vx.profile_read()
print(a.workload, a.op, "ms/op", round(sum(plain) / len(plain), 4), "profiled", round(sum(ev) / len(ev), 4),
      {k: round(v[1] / a.reps, 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])})
