"""Stable argsort / key+value sort against the canonical
stable order (oracle.canonical_argsort): indices bit-exact, sorted keys equal
to the sort's output, values permuted alongside."""
import numpy as np
import pytest

import oracle
import paper_2205_05982_b200 as vx

from test_sort_gpu import rand_keys

pytestmark = pytest.mark.gpu

TYPES = ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64"]
SIZES = [0, 1, 2, 31, 257, 2049, 8193, 100_003, 1_000_000]


def _dups(kt, n, rng):
    """Heavy duplicates so stability is visible."""
    x = rand_keys(kt, n, rng)
    if n:
        x = x[rng.integers(0, max(1, n // 20), n)]
    return x


@pytest.mark.parametrize("kt", TYPES)
def test_argsort_parity(cuda, kt):
    import torch
    rng = np.random.default_rng(hash(kt) & 0xFFFF)
    for n in SIZES:
        for gen in (rand_keys, _dups):
            x = gen(kt, n, rng)
            t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
            for desc in (False, True):
                out = torch.empty_like(t)
                idx = vx.argsort(t, vx.Order(int(desc)), sorted_keys=out)
                want = oracle.canonical_argsort(x, kt, desc)
                assert np.array_equal(idx.cpu().numpy(), want), (kt, n, desc, gen.__name__)
                assert out.cpu().numpy().tobytes() == x[want].tobytes()
                assert t.cpu().numpy().tobytes() == x.tobytes()  # input untouched


@pytest.mark.parametrize("vb", [1, 2, 4, 8, 16])
def test_sort_pairs_values(cuda, vb):
    import torch
    rng = np.random.default_rng(vb)
    n = 300_001
    for kt in ("u32", "i64", "f32", "u16"):
        x = _dups(kt, n, rng)
        vals = rng.integers(0, 256, size=(n, vb), dtype=np.uint8)
        for desc in (False, True):
            k = torch.from_numpy(np.ascontiguousarray(x)).cuda()
            v = torch.from_numpy(vals.copy()).cuda()
            vx.sort_pairs(k, v, vx.SortConfig(order=vx.Order(int(desc))))
            want = oracle.canonical_argsort(x, kt, desc)
            assert k.cpu().numpy().tobytes() == x[want].tobytes()
            assert np.array_equal(v.cpu().numpy(), vals[want])


def test_argsort_large_and_workspace(cuda):
    import torch
    rng = np.random.default_rng(5)
    n = 20_000_000
    x = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    t = torch.from_numpy(x).cuda()
    ws = torch.empty(vx.argsort_workspace_bytes(n, "u32"), dtype=torch.uint8, device="cuda")
    idx = vx.argsort(t, workspace=ws)
    assert np.array_equal(idx.cpu().numpy(), np.argsort(x, kind="stable"))
    y = rng.integers(0, 2**64, 5_000_000, dtype=np.uint64)
    ty = torch.from_numpy(y).cuda()
    idy = vx.argsort(ty, vx.Order.kDescending)
    assert np.array_equal(idy.cpu().numpy(), oracle.canonical_argsort(y, "u64", True))
    with pytest.raises(ValueError):
        vx.argsort(t, workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        vx.argsort(torch.zeros((10, 2), dtype=torch.uint64, device="cuda"), key_type="k128")
