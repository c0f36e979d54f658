"""Host-pointer pipeline: chunked H2D + per-chunk sorts +
per-slice merges + D2H inside vxs_sort_host.  Forced on at small sizes with
VXSORT_HOST_CHUNKS / VXSORT_HOST_SLICES and compared bit-exactly with the
oracle, for every key type and order, pinned and pageable sources, and the
distributions that stress the slicing (duplicates, presorted, all equal)."""
import os

import numpy as np
import pytest

import oracle
import paper_2205_05982_b200 as vx

from test_sort_gpu import TYPES, oracle_kt, rand_keys

pytestmark = pytest.mark.gpu


@pytest.fixture
def pipeline(request):
    old = {k: os.environ.get(k) for k in ("VXSORT_HOST_CHUNKS", "VXSORT_HOST_SLICES")}

    def set_(chunks, slices):
        os.environ["VXSORT_HOST_CHUNKS"] = str(chunks)
        os.environ["VXSORT_HOST_SLICES"] = str(slices)

    yield set_
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def host_check(x, kt, desc, pinned=False):
    import torch
    y = np.ascontiguousarray(x).copy()
    if pinned:
        t = torch.from_numpy(y.view(np.uint8).reshape(-1)).pin_memory()
        buf = t.numpy().view(y.dtype).reshape(y.shape)
    else:
        buf = y
    st = vx.sort(buf, vx.SortConfig(order=vx.Order(int(desc)), seed=5),
                 key_type=kt if kt in ("k128", "kv64") else None)
    want, _ = oracle.sort(x, oracle_kt(kt), descending=desc, seed=1)
    assert buf.tobytes() == want.tobytes(), (kt, desc, len(x), pinned)
    return st


@pytest.mark.parametrize("kt", TYPES + ["kv64"])
def test_pipeline_all_types(cuda, pipeline, kt):
    rng = np.random.default_rng(hash(kt) & 0xFFFF)
    pipeline(5, 16)
    for n in (5 * 4096, 200_003):
        x = rand_keys(kt, n, rng)
        for desc in (False, True):
            st = host_check(x, kt, desc, pinned=desc)
            assert st.max_depth >= 1  # chunk sorts + slice merge stage


@pytest.mark.parametrize("chunks,slices", [(2, 2), (3, 4), (8, 16), (16, 64)])
def test_pipeline_shapes(cuda, pipeline, chunks, slices):
    rng = np.random.default_rng(chunks * 100 + slices)
    pipeline(chunks, slices)
    x = rng.integers(0, 2**32, 1_000_003, dtype=np.uint64).astype(np.uint32)
    host_check(x, "u32", False)
    host_check(x, "u32", True, pinned=True)


def test_pipeline_distributions(cuda, pipeline):
    pipeline(8, 32)
    n = 2_000_000
    rng = np.random.default_rng(7)
    cases = {
        "equal": np.full(n, 42, np.uint64),
        "two": (rng.integers(0, 2, n, dtype=np.uint64) * 7),
        "small8": rng.integers(0, 8, n, dtype=np.uint64),
        "sorted": np.arange(n, dtype=np.uint64),
        "reverse": np.arange(n, 0, -1, dtype=np.uint64),
        "organ": np.concatenate([np.arange(n // 2), np.arange(n - n // 2, 0, -1)]).astype(np.uint64),
        "skew": ((rng.random(n) ** 4) * 2.0**64).astype(np.uint64),
    }
    for name, x in cases.items():
        for desc in (False, True):
            host_check(x, "u64", desc, pinned=name in ("sorted", "skew"))
    f = (rng.standard_normal(n) * 1e3).astype(np.float32)
    f[rng.integers(0, n, 5000)] = np.array([-0.0, 0.0, -np.inf, np.inf, np.nan], np.float32)[np.arange(5000) % 5]
    for desc in (False, True):
        host_check(f, "f32", desc)


def test_pipeline_default_large(cuda):
    """Default dimensions (pipeline on above 64 MB): 5e7 u32 pageable, 2.5e7
    u64 pinned; compared with np.sort."""
    import torch
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2**32, 50_000_000, dtype=np.uint64).astype(np.uint32)
    y = x.copy()
    st = vx.sort(y)
    assert st.max_depth >= 2
    assert np.array_equal(y, np.sort(x))
    x = rng.integers(0, 2**64, 25_000_000, dtype=np.uint64)
    t = torch.from_numpy(x.copy()).pin_memory()
    vx.sort(t.numpy(), vx.SortConfig(order=vx.Order.kDescending))
    assert np.array_equal(t.numpy(), np.sort(x)[::-1])
