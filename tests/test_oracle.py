"""Pins the oracle (test infrastructure) against the real reference and its
known-answer tests, before the oracle is trusted as the GPU checker."""
import numpy as np
import pytest

import oracle

GOLDEN = None


def golden():
    global GOLDEN
    if GOLDEN is None:
        import os
        GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    return GOLDEN


def harness_equal(a, b, kt):
    """harness.cpp:286-298: bit-exact, except -0.0/+0.0 may differ."""
    if a.tobytes() == b.tobytes():
        return True
    if kt not in ("f32", "f64"):
        return False
    diff = a.view(np.uint8).reshape(len(a), -1) != b.view(np.uint8).reshape(len(b), -1)
    bad = diff.any(axis=1)
    return bool(np.all((a[bad] == 0) & (b[bad] == 0)))


def test_depth_budget_known_answers():
    # test_driver.cpp:55-60
    lib = oracle.lib()
    assert lib.vxo_depth_budget(1) == 4
    assert lib.vxo_depth_budget(2) == 6
    assert lib.vxo_depth_budget(1024) == 24
    assert lib.vxo_depth_budget(1_000_000) == 44


def test_sfc64_determinism_and_divergence():
    # test_pivot.cpp:46-61
    a = oracle.sfc64_stream(42, 100)
    assert (a == oracle.sfc64_stream(42, 100)).all()
    assert (oracle.sfc64_stream(42, 4) != oracle.sfc64_stream(43, 4)).any()


def test_bounded_offset_range():
    # test_pivot.cpp:75-83
    lib = oracle.lib()
    r = oracle.sfc64_stream(9, 20000)
    for i in range(0, 20000, 2):
        assert lib.vxo_bounded_offset(int(r[i]), 1) == 0
        bound = 1 + int(r[i + 1] % 1000)
        assert lib.vxo_bounded_offset(int(r[i]), bound) < bound


def test_five_draws_in_range():
    # test_pivot.cpp:97-108
    import ctypes
    idx = np.zeros(9, dtype=np.uint32)
    oracle.lib().vxo_five_draws(21, 17, 9, idx.ctypes.data)
    assert (idx < 17).all()
    oracle.lib().vxo_five_draws(23, 1, 9, idx.ctypes.data)
    assert (idx == 0).all()


def test_golden_vectors_reproduced_by_oracle():
    g = golden()
    n_cases = 0
    for key in g["meta"]:
        kt, dist, n, desc = key.split("|")
        x = g["in|" + key]
        want = g["out|" + key]
        got, st = oracle.sort(x, kt, descending=bool(int(desc)), seed=3)
        assert harness_equal(got, want, kt), key
        if not (kt in ("f32", "f64") and dist == "specials"):
            assert got.tobytes() == want.tobytes(), key
        # canonical order restated independently in numpy
        assert got.tobytes() == oracle.canonical_sorted(x, kt, bool(int(desc))).tobytes(), key
        n_cases += 1
    assert n_cases > 300


def test_golden_adversarial_stats():
    # test_driver.cpp:187-203: the reference's adversarial input exhausts the
    # depth budget and falls back to heapsort; the frozen stats say so.
    g = golden()
    for kt in ("u16", "u32"):
        st = g[f"stats|{kt}|adversarial|8192|0"]
        assert st[4] == 1 and st[0] == oracle.lib().vxo_depth_budget(8192)
        got, ost = oracle.sort(g[f"in|{kt}|adversarial|8192|0"], kt, seed=42)
        assert got.tobytes() == g[f"out|{kt}|adversarial|8192|0"].tobytes()


def test_oracle_driver_known_answers():
    # test_driver.cpp:116-167
    st = oracle.sort(np.zeros(0, np.uint32), "u32")[1]
    assert st["max_depth"] == 0 and st["partition_calls"] == 0
    for n in (300, 5000, 100_000):
        x = np.full(n, 1234567, dtype=np.uint32)
        y, st = oracle.sort(x, "u32", seed=5)
        assert (y == 1234567).all() and not st["fallback_triggered"] and st["max_depth"] <= 2
    rng = np.random.default_rng(73)
    for n in (1000, 30000, 200000):
        x = rng.integers(0, 2, n).astype(np.uint16)
        y, st = oracle.sort(x, "u16", seed=11)
        assert (y == np.sort(x)).all() and not st["fallback_triggered"]
    x = rng.integers(0, 2**64, 1_000_000, dtype=np.uint64)
    y, st = oracle.sort(x, "u64", seed=3)
    assert (y == np.sort(x)).all()
    assert not st["fallback_triggered"]
    assert st["max_depth"] <= oracle.lib().vxo_depth_budget(len(x))


def test_oracle_heap_sort_matches_sort():
    rng = np.random.default_rng(67)
    x = rng.integers(0, 2**64, size=(500, 2), dtype=np.uint64)
    y = x.copy()
    oracle.lib().vxo_heap_sort(y.ctypes.data, 500, oracle.KEY_CODE["k128"], 0)
    assert y.tobytes() == oracle.canonical_sorted(x, "k128").tobytes()


def test_canonical_float_order_nan_and_zero():
    x = np.array([np.nan, 1.0, -0.0, 0.0, -np.inf, np.inf, -1.0, np.nan], dtype=np.float32)
    x[0] = np.frombuffer(np.uint32(0xFFC00000).tobytes(), np.float32)[0]  # negative qNaN
    asc, _ = oracle.sort(x, "f32")
    bits = asc.view(np.uint32)
    assert list(bits[:6]) == [0xFF800000, 0xBF800000, 0x80000000, 0x00000000, 0x3F800000, 0x7F800000]
    assert list(bits[6:]) == [0x7FC00000, 0xFFC00000]  # NaN last, raw bits ascending
    desc, _ = oracle.sort(x, "f32", descending=True)
    bits = desc.view(np.uint32)
    assert list(bits[:6]) == [0x7F800000, 0x3F800000, 0x00000000, 0x80000000, 0xBF800000, 0xFF800000]
    assert list(bits[6:]) == [0x7FC00000, 0xFFC00000]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
class TestAgainstRealReference:
    def test_generators_match_reference_harness(self):
        for kt in oracle.KEY_TYPES:
            for d in oracle.DISTS:
                a = oracle.generate(kt, d, 3000, seed=5)
                b = oracle.ref_generate(kt, d, 3000, seed=5)
                assert a.tobytes() == b.tobytes(), (kt, d)

    def test_sfc64_matches(self):
        assert (oracle.sfc64_stream(7, 1000) == oracle.sfc64_stream(7, 1000, use_ref=True)).all()

    def test_pivot_matches_reference(self):
        # same sampled pivot as PivotSampler<ScalarTag>::choose_pivot for u64
        import ctypes
        rng = np.random.default_rng(5)
        lib = oracle.ref()
        for it in range(50):
            n = int(rng.integers(300, 5000))
            x = rng.integers(0, 2**64, n, dtype=np.uint64)
            for desc in (0, 1):
                want = lib.ref_choose_pivot_u64(x.ctypes.data, n, 1000 + it, desc)
                got = oracle.lib().vxo_choose_pivot_u64(x.ctypes.data, n, 1000 + it, desc)
                assert got == want

    def test_scratch_bytes_match_reference(self):
        import paper_2205_05982_b200 as vx
        for kt in oracle.KEY_TYPES:
            assert vx.scratch_bytes(kt) == oracle.ref().ref_scratch_bytes(oracle.KEY_CODE[kt]), kt

    def test_random_sorts_match_reference(self):
        rng = np.random.default_rng(11)
        for kt in oracle.KEY_TYPES:
            for desc in (False, True):
                for n in (0, 1, 5, 256, 257, 777, 20000):
                    if kt == "k128":
                        x = rng.integers(0, 2**64, size=(n, 2), dtype=np.uint64)
                    elif kt in ("f32", "f64"):
                        x = (rng.standard_normal(n) * 100).astype(oracle.NP_DTYPE[kt])
                    else:
                        info = np.iinfo(oracle.NP_DTYPE[kt])
                        x = rng.integers(info.min, info.max, n, dtype=oracle.NP_DTYPE[kt], endpoint=True)
                    a, _ = oracle.sort(x, kt, desc)
                    b, _ = oracle.ref_sort(x, kt, desc, seed=9)
                    assert harness_equal(a, b, kt), (kt, desc, n)

    def test_reference_rejects_nan_and_small_scratch(self):
        # test_driver.cpp:240-255
        with pytest.raises(ValueError, match="NaN"):
            oracle.ref_sort(np.array([1.0, np.nan, 2.0], np.float32), "f32")
        x = np.ones(10, np.uint64)
        assert oracle.ref().ref_sort_with_scratch(x.ctypes.data, 10, oracle.KEY_CODE["u64"], 16) == 1
        assert oracle.ref().ref_scratch_bytes(oracle.KEY_CODE["u64"]) == 2048


@pytest.mark.parametrize("kt", ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64"])
def test_canonical_argsort_consistent_with_canonical_sort(kt):
    """The stable-argsort oracle (§8 f2) permutes keys into exactly the
    canonical sorted order, and is stable (ties by ascending index)."""
    rng = np.random.default_rng(3)
    dt = {"i16": np.int16, "u16": np.uint16, "i32": np.int32, "u32": np.uint32, "f32": np.float32,
          "i64": np.int64, "u64": np.uint64, "f64": np.float64}[kt]
    if kt in ("f32", "f64"):
        x = (rng.standard_normal(5000) * 10).round().astype(dt)
        x[::7] = np.array([-0.0, 0.0, np.inf, -np.inf, np.nan], dt)[np.arange(len(x[::7])) % 5]
    else:
        x = rng.integers(0, 50, 5000).astype(dt)
    for desc in (False, True):
        o = oracle.canonical_argsort(x, kt, desc)
        assert x[o].tobytes() == oracle.canonical_sorted(x, kt, desc).tobytes()
        same = x[o][1:].view(np.uint8).reshape(len(x) - 1, -1) == x[o][:-1].view(np.uint8).reshape(len(x) - 1, -1)
        ties = same.all(axis=1)
        assert np.all(o[1:][ties] > o[:-1][ties])
