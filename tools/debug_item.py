import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_05982_b200 as vx
rng = np.random.default_rng(1)
fails = 0
for n in (600, 1500, 3000, 5000, 8000):
    for kind in ("two_clusters", "one_outlier", "dense_low", "many_dups"):
        if kind == "two_clusters":
            x = rng.integers(0, 1 << 10, n, dtype=np.uint64) + (np.uint64(1) << np.uint64(50)) * rng.integers(0, 2, n, dtype=np.uint64)
        elif kind == "one_outlier":
            x = rng.integers(0, 1 << 20, n, dtype=np.uint64); x[0] = np.uint64(2**63 + 5)
        elif kind == "dense_low":
            x = rng.integers(0, 2**64, n, dtype=np.uint64); x[: n * 9 // 10] &= np.uint64((1 << 43) - 1)
        else:
            x = rng.integers(0, 40, n, dtype=np.uint64) * np.uint64(1 << 40)
        t = torch.from_numpy(x.copy()).cuda()
        vx.sort(t, vx.SortConfig(seed=1))
        ok = t.cpu().numpy().tobytes() == np.sort(x).tobytes()
        if not ok:
            fails += 1
            print("FAIL", n, kind)
print("fails", fails)
