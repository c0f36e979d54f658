"""Parity of the B200 sort against the oracle (and the reference's frozen
golden vectors), through the C ABI.  Bit-exact for every key type."""
import numpy as np
import pytest

import oracle
import paper_2205_05982_b200 as vx

pytestmark = pytest.mark.gpu

TYPES = ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64", "k128"]
NP = {"i16": np.int16, "u16": np.uint16, "i32": np.int32, "u32": np.uint32, "f32": np.float32,
      "i64": np.int64, "u64": np.uint64, "f64": np.float64}


def rand_keys(kt, n, rng, specials=True):
    if kt in ("k128", "kv64"):
        return rng.integers(0, 2**64, size=(n, 2), dtype=np.uint64)
    if kt in ("f32", "f64"):
        x = (rng.standard_normal(n) * 1e3).astype(NP[kt])
        if specials and n:
            vals = np.array([-0.0, 0.0, -np.inf, np.inf, np.nan], dtype=NP[kt])
            pos = rng.integers(0, n, size=max(1, n // 50))
            x[pos] = vals[np.arange(len(pos)) % 5]
        return x
    info = np.iinfo(NP[kt])
    return rng.integers(info.min, info.max, size=n, dtype=NP[kt], endpoint=True)


def gpu_sort(x, kt, desc, seed=1):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x).copy()).cuda()
    st = vx.sort(t, vx.SortConfig(order=vx.Order(int(desc)), seed=seed),
                 key_type=kt if kt in ("k128", "kv64") else None)
    torch.cuda.synchronize()
    return t.cpu().numpy(), st


def oracle_kt(kt):
    return "k128" if kt == "kv64" else kt


def check(x, kt, desc, seed=1):
    got, st = gpu_sort(x, kt, desc, seed)
    want, _ = oracle.sort(x, oracle_kt(kt), descending=desc, seed=1)
    assert got.tobytes() == want.tobytes(), (kt, desc, len(x))
    return st


SIZES = [0, 1, 2, 3, 31, 32, 33, 64, 255, 256, 257, 1000, 1024, 2047, 2049, 4095, 4096, 4097,
         8191, 8192, 8193, 12345, 100_000]


@pytest.mark.parametrize("kt", TYPES)
def test_sizes_all_types_both_orders(cuda, kt):
    rng = np.random.default_rng(hash(kt) & 0xFFFF)
    for n in SIZES:
        x = rand_keys(kt, n, rng)
        for desc in (False, True):
            check(x, kt, desc)


def test_golden_vectors(cuda):
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    for key in g["meta"]:
        kt, dist, n, desc = key.split("|")
        x = g["in|" + key]
        want = g["out|" + key]
        got, _ = gpu_sort(x, kt, bool(int(desc)))
        if kt in ("f32", "f64") and dist == "specials":
            # harness rule (harness.cpp:286-298): +-0 may differ from vexsort
            bad = got.view(np.uint8).reshape(len(got), -1) != want.view(np.uint8).reshape(len(want), -1)
            bad = bad.any(axis=1)
            assert np.all((got[bad] == 0) & (want[bad] == 0)), key
            assert got.tobytes() == oracle.canonical_sorted(x, kt, bool(int(desc))).tobytes(), key
        else:
            assert got.tobytes() == want.tobytes(), key


@pytest.mark.parametrize("dist", ["uniform", "equal", "lowentropy", "asc", "desc", "twovalue"])
def test_harness_distributions(cuda, dist):
    for kt in ("u32", "u64", "f32", "k128", "i16"):
        for n in (5000, 300_000):
            x = oracle.generate(kt, dist, n, seed=1)
            for desc in (False, True):
                check(x, kt, desc)


def test_low_entropy_and_presorted_u64(cuda):
    rng = np.random.default_rng(3)
    n = 2_000_000
    cases = {
        "0..7": rng.integers(0, 8, n, dtype=np.uint64),
        "allequal": np.full(n, 0x2A, np.uint64),
        "ramp": np.arange(n, dtype=np.uint64),
        "desc": np.arange(n, dtype=np.uint64)[::-1].copy(),
        "organ": np.concatenate([np.arange(n // 2), np.arange(n - n // 2)[::-1]]).astype(np.uint64),
    }
    r = np.arange(n, dtype=np.uint64)
    sw = rng.integers(0, n, size=(n // 200, 2))
    for a, b in sw:
        r[a], r[b] = r[b], r[a]
    cases["ramp+swaps"] = r
    for name, x in cases.items():
        for desc in (False, True):
            st = check(x, "u64", desc)
            assert not st.fallback_triggered, name


def test_float_specials_canonical_order(cuda):
    x = np.array([np.nan, 1.0, -0.0, 0.0, -np.inf, np.inf, -1.0, np.nan] * 700, dtype=np.float32)
    x.view(np.uint32)[::16] = 0xFFC00000  # negative NaN
    x.view(np.uint32)[3::16] = 0x7F800001  # signalling NaN payload
    for desc in (False, True):
        check(x, "f32", desc)
        check(x.astype(np.float64), "f64", desc)


def test_k128_hi_ties_and_kv64(cuda):
    rng = np.random.default_rng(5)
    n = 500_000
    k = np.empty((n, 2), np.uint64)
    k[:, 0] = rng.integers(0, 2**64, n, dtype=np.uint64)
    k[:, 1] = rng.integers(0, 2**64, n, dtype=np.uint64) >> np.uint64(44)
    for desc in (False, True):
        check(k, "k128", desc)
    kv = np.empty((n, 2), np.uint64)
    kv[:, 0] = np.arange(n, dtype=np.uint64)  # payload = original index
    kv[:, 1] = rng.integers(0, 2**64, n, dtype=np.uint64) & np.uint64(0xFFFF)  # many equal keys
    got, _ = gpu_sort(kv, "kv64", False)
    order = np.argsort(kv[:, 1], kind="stable")  # key-only STABLE sort
    assert got.tobytes() == kv[order].tobytes()


def test_adversarial_driver_inputs(cuda):
    # test_driver.cpp:20-34 adversarial keys and :169-185 maximal pivot
    for kt, dt in (("u16", np.uint16), ("u32", np.uint32)):
        n = 8192
        x = np.full(n, np.iinfo(dt).max, dtype=dt)
        x[np.arange(72) * (n // 72)] = np.arange(1, 73, dtype=dt)
        check(x, kt, False)
    x = np.full(4096, 0xFFFFFFFF, np.uint32)
    x[[100, 2000, 3000]] = [5, 6, 7]
    check(x, "u32", False)
    for n in (300, 5000, 100_000):
        x = np.full(n, 1234567, np.uint32)
        st = check(x, "u32", False)
        assert st.max_depth <= 2


def test_host_api_and_seed_independence(cuda):
    rng = np.random.default_rng(9)
    x = rng.integers(0, 2**64, 1_000_000, dtype=np.uint64)
    want = np.sort(x)
    for seed in (None, 0, 3, 2**63 + 5):
        y = x.copy()
        st = vx.sort(y, vx.SortConfig(seed=seed))
        assert y.tobytes() == want.tobytes()
        assert st.partition_calls >= 1 and st.base_case_calls >= 1
        assert st.keys_partitioned >= len(x)


def test_workspace_reuse_and_stream(cuda):
    import torch
    n = 300_000
    ws = torch.empty(vx.workspace_bytes(n, "u64"), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    rng = np.random.default_rng(1)
    for it in range(4):
        x = rng.integers(0, 2**64, n, dtype=np.uint64)
        t = torch.from_numpy(x).cuda()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            vx.sort(t, vx.SortConfig(order=vx.Order(it % 2)), workspace=ws, stream=s)
        s.synchronize()
        want = np.sort(x)
        assert t.cpu().numpy().tobytes() == (want if it % 2 == 0 else want[::-1]).tobytes()
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        vx.sort(torch.zeros(100_000, dtype=torch.int64, device="cuda"), workspace=small)


def test_clustered_keys_outside_sample_range(cuda):
    """Regression: 64/128-bit keys far above a bucket's sampled range must
    classify monotonically (saturating cell/digit maps)."""
    rng = np.random.default_rng(11)
    n = 4_000_000
    for frac in (0.5, 0.9, 0.99):
        x = rng.integers(0, 2**64, n, dtype=np.uint64)
        k = int(n * frac)
        x[:k] &= np.uint64((1 << 43) - 1)
        rng.shuffle(x)
        for desc in (False, True):
            check(x, "u64", desc)
        check(x.view(np.int64), "i64", False)
        f = rng.standard_normal(n) * 1e-3
        f[: n // 10] *= 1e300
        check(f, "f64", False)
    k128 = np.empty((n // 2, 2), np.uint64)
    k128[:, 0] = rng.integers(0, 2**64, n // 2, dtype=np.uint64)
    k128[:, 1] = rng.integers(0, 2**64, n // 2, dtype=np.uint64)
    k128[: n // 4, 1] &= np.uint64(0xFF)
    check(k128, "k128", False)


def test_skewed_keys_log_units(cuda):
    # power-law keys (C5's u^4 skew; also u^8 and log-uniform): the piecewise
    # radix over log units (fine_unit_log) must stay bit-exact for every word
    rng = np.random.default_rng(11)
    n = 3_000_000
    u = rng.random(n)
    for name, f in (("u4", u ** 4), ("u8", u ** 8), ("logu", np.exp2(-40.0 * u))):
        x64 = np.minimum(np.floor(np.ldexp(f, 64)), float(2**64 - 2**11)).astype(np.uint64)
        for desc in (False, True):
            check(x64, "u64", desc)
            check((x64 >> np.uint64(32)).astype(np.uint32), "u32", desc)
            check((x64 >> np.uint64(1)).astype(np.int64) - np.int64(2**40), "i64", desc)
        k = np.empty((n // 4, 2), np.uint64)
        k[:, 1] = x64[: n // 4]
        k[:, 0] = rng.integers(0, 2**64, n // 4, dtype=np.uint64)
        check(k, "k128", False)
        check((x64 >> np.uint64(48)).astype(np.uint16), "u16", False)


@pytest.mark.parametrize("kt", ["i32", "u32", "f32", "i64", "u64", "f64", "k128", "i16"])
def test_two_levels_every_word_vs_oracle(cuda, kt):
    # 5e6 keys: two levels (known-bounds radix below a radix parent, weighted
    # CTA tile ranges, per-tile prefixes), bit-exact against the oracle
    rng = np.random.default_rng(hash(kt) & 0xFFF)
    n = 5_000_000
    x = rand_keys(kt, n, rng)
    for desc in (False, True):
        st = check(x, kt, desc)
        if kt != "i16":  # (65536 distinct values end in equality buckets after one level)
            assert st.max_depth >= 2
    if kt in ("u32", "u64", "i64"):  # a narrow range off the word boundaries: clamped digits at the root
        lo = 123456789
        y = (rand_keys("u32", n, rng).astype(np.uint64) % np.uint64(3_000_000_000) + np.uint64(lo)).astype(NP[kt])
        check(y, kt, False)
