"""Small-size parity subset for compute-sanitizer (memcheck / racecheck /
synccheck): every key width, both orders, one and two levels, the counting
sort and its network fallback, argsort, partition, select, graph capture.
Each result is checked against the oracle.  Usage:
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2205_05982_b200 as vx  # noqa: E402

rng = np.random.default_rng(3)
cases = [("u32", 200_000, False), ("u64", 150_000, True), ("f32", 120_000, False), ("i16", 70_000, True),
         ("k128", 60_000, False), ("u64", 3_000, False), ("u32", 1_500_000, False),
         # two levels: known-bounds digits below a radix parent, weighted CTA ranges, tile prefixes
         ("u32", 3_000_000, True), ("u64", 3_000_000, False), ("f32", 3_000_000, True)]
ok = True
for kt, n, desc in cases:
    if kt == "k128":
        x = rng.integers(0, 2**64, (n, 2), dtype=np.uint64)
        x[:, 1] >>= np.uint64(52)
    elif kt == "f32":
        x = (rng.standard_normal(n) * 1e3).astype(np.float32)
        x[::101] = np.nan
        x[1::89] = -0.0
    else:
        dt = {"u32": np.uint32, "u64": np.uint64, "i16": np.int16}[kt]
        info = np.iinfo(dt)
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    d = torch.from_numpy(x.copy()).cuda()
    vx.sort(d, vx.SortConfig(order=vx.Order(int(desc)), seed=1), key_type=kt if kt == "k128" else None)
    want, _ = oracle.sort(x, kt, descending=desc)
    good = d.cpu().numpy().tobytes() == want.tobytes()
    ok &= good
    print(kt, n, desc, "ok" if good else "MISMATCH", flush=True)
# power-law keys: piecewise radix over log units, then known-bounds / clamped digits below it
u = rng.random(3_000_000)
x = np.minimum(np.floor(np.ldexp(u ** 4, 64)), float(2**64 - 2**11)).astype(np.uint64)
d = torch.from_numpy(x.copy()).cuda()
vx.sort(d, vx.SortConfig(seed=1))
good = d.cpu().numpy().tobytes() == oracle.sort(x, "u64")[0].tobytes()
ok &= good
print("u64 skew", "ok" if good else "MISMATCH", flush=True)
# clustered keys -> counting-sort rejection -> network fallback
x = (rng.integers(0, 50, 100_000, dtype=np.uint64) << np.uint64(40)) | rng.integers(0, 3, 100_000, dtype=np.uint64)
d = torch.from_numpy(x.copy()).cuda()
vx.sort(d, vx.SortConfig(seed=1))
ok &= d.cpu().numpy().tobytes() == oracle.sort(x, "u64")[0].tobytes()
# argsort, partition, select
x = rng.integers(0, 2**32, 90_000, dtype=np.uint32)
idx = vx.argsort(torch.from_numpy(x).cuda()).cpu().numpy()
ok &= np.array_equal(idx, oracle.canonical_argsort(x, "u32", False))
src = torch.from_numpy(x).cuda()
spl = torch.from_numpy(np.sort(rng.integers(0, 2**32, 15, dtype=np.uint32))).cuda()
out, counts = vx.partition(src, spl)
ok &= int(counts.sum()) == len(x)
d = torch.from_numpy(x.copy()).cuda()
vx.nth_element(d, 12345)
ok &= int(d[12345]) == int(np.sort(x)[12345])
# graph capture
d = torch.from_numpy(x.copy()).cuda()
ws = torch.empty(vx.workspace_bytes(len(x), "u32"), dtype=torch.uint8, device="cuda")
vx.sort(d, vx.SortConfig(seed=1), workspace=ws)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    vx.sort(d, vx.SortConfig(seed=1), workspace=ws)
d.copy_(torch.from_numpy(x))
g.replay()
torch.cuda.synchronize()
ok &= d.cpu().numpy().tobytes() == np.sort(x).tobytes()
print("ALL OK" if ok else "FAILED", flush=True)
sys.exit(0 if ok else 1)
