"""Very large inputs: C5's per-GPU shape (2^30 u64 = 8 GiB, uniform and
u^4-skewed) and an input of more than 2^32 keys (64-bit positions)."""
import numpy as np
import pytest
import torch

import paper_2205_05982_b200 as vx
from test_baseline_sizes_gpu import check_sorted, fingerprint

pytestmark = pytest.mark.gpu


def _device_uniform(n, dtype, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    if dtype == torch.int64:
        return torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    return torch.randint(-2**15, 2**15 - 1, (n,), dtype=torch.int16, device="cuda", generator=g)


@pytest.mark.parametrize("skew", [False, True])
def test_c5_shape_2pow30_u64(cuda, skew):
    n = 1 << 30
    x = _device_uniform(n, torch.int64, 5)
    if skew:  # floor(2^64 * u^4) computed on the device in float64 (mantissa-limited, still skewed)
        u = (x.view(torch.int64) >> 11).to(torch.float64) * (2.0 ** -53) + 0.5
        x = torch.clamp(torch.ldexp(u ** 4, torch.tensor(64, device="cuda")), max=2.0 ** 64 - 4096)
        x = x.to(torch.float64)
        hi = torch.floor(x / 2.0 ** 32)
        lo = x - hi * 2.0 ** 32
        x = (hi.to(torch.int64) << 32) | lo.to(torch.int64)
        del hi, lo, u
    x = x.view(torch.uint64)
    fp = fingerprint(x, 8)
    st = vx.sort(x, vx.SortConfig(seed=3))
    torch.cuda.synchronize()
    assert check_sorted(x, "u64", False)
    assert fingerprint(x, 8) == fp
    assert st.max_depth <= 4


def test_more_than_2pow32_keys_i16(cuda):
    """> 2^32 keys: 64-bit positions everywhere.  Checks are chunked (torch
    reductions are limited to < 2^31 elements)."""
    n = (1 << 32) + 12345
    x = _device_uniform(n, torch.int16, 7)
    chunk = 1 << 30

    def hist(t):
        h = torch.zeros(65536, dtype=torch.int64, device="cuda")
        for s in range(0, n, chunk):
            h += torch.bincount(t[s:s + chunk].to(torch.int32) + 32768, minlength=65536)
        return h

    before = hist(x)
    vx.sort(x, vx.SortConfig(order=vx.Order.kDescending, seed=1))
    torch.cuda.synchronize()
    for s in range(0, n - 1, chunk):
        e = min(n, s + chunk + 1)
        assert bool((x[s + 1:e] <= x[s:e - 1]).all())
    assert torch.equal(hist(x), before)
