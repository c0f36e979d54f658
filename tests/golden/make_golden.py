"""Generate golden vectors from the REAL reference (oracle/_ref, compiled from
/root/reference/proj sources).  Run in the authoring container:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz with, per case, the input bytes, the
reference's sorted output bytes and its SortStats (seeded).  The reference
has no golden files of its own (its tests compare with std::sort at run
time, test_util.hpp:64-80); these fixtures freeze that comparison so the
GPU box (which has no /root/reference) can check against them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

TYPES = ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64", "k128"]
SIZES = [0, 1, 2, 3, 17, 255, 256, 257, 1000, 3000]


def main():
    out = {}
    meta = []
    for kt in TYPES:
        for dist in oracle.DISTS:
            for n in SIZES:
                if dist != "uniform" and n not in (257, 3000):
                    continue
                x = oracle.ref_generate(kt, dist, n, seed=1)
                for desc in (False, True):
                    y, st = oracle.ref_sort(x, kt, descending=desc, seed=3)
                    key = f"{kt}|{dist}|{n}|{int(desc)}"
                    out["in|" + key] = x
                    out["out|" + key] = y
                    out["stats|" + key] = np.array([st["max_depth"], st["partition_calls"],
                                                    st["base_case_calls"], st["keys_partitioned"],
                                                    st["fallback_triggered"]], dtype=np.int64)
                    meta.append(key)
    # float specials (NaN-free: the reference rejects NaN, driver.hpp:176-180)
    rng = np.random.default_rng(2205)
    for kt, dt in (("f32", np.float32), ("f64", np.float64)):
        x = (rng.standard_normal(2000) * 1e3).astype(dt)
        x[::50] = 0.0
        x[1::50] = -0.0
        x[2::97] = np.inf
        x[3::97] = -np.inf
        for desc in (False, True):
            y, st = oracle.ref_sort(x, kt, descending=desc, seed=3)
            key = f"{kt}|specials|2000|{int(desc)}"
            out["in|" + key] = x
            out["out|" + key] = y
            out["stats|" + key] = np.array([st["max_depth"], st["partition_calls"], st["base_case_calls"],
                                            st["keys_partitioned"], st["fallback_triggered"]], dtype=np.int64)
            meta.append(key)
    # the reference's driver known-answer inputs (test_driver.cpp:20-34, 169-185)
    n = 8192
    for kt, dt in (("u16", np.uint16), ("u32", np.uint32)):
        x = np.full(n, np.iinfo(dt).max, dtype=dt)
        stride = n // 72
        x[np.arange(72) * stride] = np.arange(1, 73, dtype=dt)
        y, st = oracle.ref_sort(x, kt, seed=42)
        key = f"{kt}|adversarial|{n}|0"
        out["in|" + key] = x
        out["out|" + key] = y
        out["stats|" + key] = np.array([st["max_depth"], st["partition_calls"], st["base_case_calls"],
                                        st["keys_partitioned"], st["fallback_triggered"]], dtype=np.int64)
        meta.append(key)
    out["meta"] = np.array(meta)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(meta)} cases to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
