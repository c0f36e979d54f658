"""Partial sort / selection (vxs_sort_range, nth_element,
partial_sort, top-k) against the canonical sorted order: keys[lo:hi] bit-exact,
keys[:lo] and keys[hi:] equal (as multisets) to the oracle's prefix/suffix."""
import numpy as np
import pytest

import oracle
import paper_2205_05982_b200 as vx

from test_sort_gpu import oracle_kt, rand_keys

pytestmark = pytest.mark.gpu


def check_range(x, kt, desc, lo, hi):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x).copy()).cuda()
    vx.sort_range(t, lo, hi, vx.SortConfig(order=vx.Order(int(desc))),
                  key_type=kt if kt in ("k128", "kv64") else None)
    got = t.cpu().numpy()
    want = oracle.canonical_sorted(x, oracle_kt(kt), desc)
    assert got[lo:hi].tobytes() == want[lo:hi].tobytes(), (kt, desc, len(x), lo, hi)
    okt = oracle_kt(kt)
    assert oracle.canonical_sorted(got[:lo], okt, desc).tobytes() == want[:lo].tobytes()
    assert oracle.canonical_sorted(got[hi:], okt, desc).tobytes() == want[hi:].tobytes()


@pytest.mark.parametrize("kt", ["i16", "u32", "f32", "i64", "u64", "f64", "k128"])
def test_sort_range_types(cuda, kt):
    rng = np.random.default_rng(hash(kt) & 0xFFFF)
    for n in (1000, 9000, 300_000, 3_000_000):
        x = rand_keys(kt, n, rng)
        for desc in (False, True):
            for lo, hi in ((0, 1), (n - 1, n), (n // 2, n // 2 + 1), (0, min(n, 100)), (n // 3, n // 3 + 5000),
                           (0, n)):
                hi = min(hi, n)
                check_range(x, kt, desc, lo, hi)


def test_sort_range_low_entropy_and_presorted(cuda):
    rng = np.random.default_rng(2)
    n = 2_000_000
    cases = [rng.integers(0, 8, n, dtype=np.uint64), np.full(n, 7, np.uint64), np.arange(n, dtype=np.uint64),
             np.arange(n, 0, -1, dtype=np.uint64), ((rng.random(n) ** 4) * 2.0**64).astype(np.uint64)]
    for x in cases:
        for lo, hi in ((0, 10), (n // 2, n // 2 + 1), (n - 1000, n)):
            check_range(x, "u64", False, lo, hi)


def test_nth_element_partial_sort_topk(cuda):
    import torch
    rng = np.random.default_rng(4)
    n = 50_000_000
    x = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    want = np.sort(x)
    t = torch.from_numpy(x.copy()).cuda()
    k = 12_345_678
    vx.nth_element(t, k)
    assert int(t[k].item()) == int(want[k])
    t = torch.from_numpy(x.copy()).cuda()
    st = vx.partial_sort(t, 1000)
    assert np.array_equal(t[:1000].cpu().numpy(), want[:1000])
    assert st.base_case_calls < 50  # only the buckets holding ranks < 1000 were sorted
    top = vx.topk(torch.from_numpy(x).cuda(), 777)
    assert np.array_equal(top.cpu().numpy(), want[::-1][:777])
    with pytest.raises(ValueError):
        vx.sort_range(t, 10, 5)
    with pytest.raises(ValueError):
        vx.sort_range(t, 0, n + 1)
