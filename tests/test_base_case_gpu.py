"""Counting-sort base case (block_sort.cuh bin_sort_item): the paths a
uniform workload never takes.  Inputs of <= Cap keys are one base-case item,
so each case below drives one item through a specific branch:
  * clustered keys (sum c^2 over the bins too large) -> rejected, sorted by
    the full-width network fallback kernel (k_final_fallback);
  * a bin holding > 64 keys -> rejected on the round limit;
  * a bin of exactly 64 distinct keys -> 64 odd-even rounds;
  * distinct keys crowded into one bin that straddles a warp boundary of the
    item's sorted order -> the smem insertion repair;
  * ties spread over many bins, descending, every class size.
All bit-exact against the oracle."""
import numpy as np
import pytest

import oracle
from test_sort_gpu import NP, check, rand_keys

pytestmark = pytest.mark.gpu

WIDE = ["u16", "u32", "i32", "f32", "u64", "i64", "f64", "k128"]
CLASS_SIZES = [300, 1000, 1900, 2048, 3000, 4096, 6000, 8192]


def _cast(kt, v):
    if kt == "k128":
        out = np.zeros((len(v), 2), dtype=np.uint64)
        out[:, 1] = v.astype(np.uint64)
        out[:, 0] = np.arange(len(v), dtype=np.uint64)[::-1]
        return out
    if kt in ("f32", "f64"):
        return v.astype(NP[kt])
    info = np.iinfo(NP[kt])
    return np.clip(v, info.min, info.max).astype(NP[kt])


@pytest.mark.parametrize("kt", WIDE)
def test_clustered_item_rejected(cuda, kt):
    rng = np.random.default_rng(11)
    for n in CLASS_SIZES:
        v = rng.integers(0, 100, size=n).astype(np.float64)
        v[rng.integers(0, n, size=5)] = 30000.0  # outliers stretch [lo, hi]
        for desc in (False, True):
            check(_cast(kt, v), kt, desc)


@pytest.mark.parametrize("kt", ["u32", "u64", "f32", "k128"])
def test_bin_round_limit(cuda, kt):
    rng = np.random.default_rng(12)
    for n in (2048, 4096, 8192):
        width = 2 * n  # one key per two bins ...
        v = rng.permutation(width)[:n].astype(np.float64) * 16
        v[:63] = v[0] + np.arange(63)      # ... except 64 distinct keys in one bin
        check(_cast(kt, v), kt, False)
        v[:70] = v[0]                      # 70 equal keys: over the round limit
        check(_cast(kt, v), kt, True)


@pytest.mark.parametrize("kt", ["u32", "u64", "i64", "f64", "k128"])
def test_bin_straddles_warp_boundary(cuda, kt):
    rng = np.random.default_rng(13)
    for n, items in ((2048, 16), (4096, 16), (8192, 16), (1024, 16)):
        span = 1 << 20
        v = np.sort(rng.integers(0, span, size=n)).astype(np.float64)
        warp_keys = 32 * items
        for b in range(warp_keys, n, warp_keys):
            # 24 distinct keys packed into a quarter of one bin around the
            # sorted position of the warp boundary b
            base = v[b - 12]
            v[b - 12:b + 12] = base + rng.permutation(24)
        v = rng.permutation(v)
        for desc in (False, True):
            check(_cast(kt, v), kt, desc)


@pytest.mark.parametrize("kt", WIDE)
def test_ties_all_classes(cuda, kt):
    rng = np.random.default_rng(14)
    for n in CLASS_SIZES + [257, 1025, 2049, 4097, 8191]:
        v = rng.integers(0, max(2, n // 3), size=n).astype(np.float64) * 977
        for desc in (False, True):
            check(_cast(kt, v), kt, desc)


def test_uniform_items_many_sizes(cuda):
    rng = np.random.default_rng(15)
    for kt in ("u32", "u64", "f32", "k128", "u16"):
        for n in list(range(257, 8193, 479)):
            x = rand_keys(kt, n, rng)
            check(x, kt, bool(n & 1))


@pytest.mark.parametrize("kt", ["u64", "i64", "f64", "k128"])
def test_item_straddling_high_word(cuda, kt):
    """64-bit items whose keys cross a 2^32 (high-word) boundary with a tiny
    range: the high-word bounds are coarse (the item is rejected and sorted by
    the fallback) and still exact; also items inside one high word."""
    rng = np.random.default_rng(16)
    for n, base in ((3000, 2**32 - 1500), (8000, 7 * 2**32 - 10), (2048, 5 * 2**32 + 1000),
                    (200_000, 2**40 - 100_000)):
        v = (base + rng.integers(0, 3000 if n < 100_000 else 200_000, n)).astype(np.uint64)
        if kt == "k128":
            x = np.zeros((n, 2), dtype=np.uint64)
            x[:, 0] = v
            x[:, 1] = rng.integers(0, 3, n).astype(np.uint64)
        elif kt == "f64":
            x = v.astype(np.float64)
        else:
            x = v.view(np.int64) if kt == "i64" else v
        for desc in (False, True):
            check(x, kt, desc)
