"""The distributed sort's device building blocks on one GPU: vxs_sample and
vxs_partition (the classify+scatter kernels with caller splitters), and
dist_sort's world_size==1 path through torch.distributed."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2205_05982_b200 as vx

pytestmark = pytest.mark.gpu


def enc(a, kt, desc):
    u = {"u32": np.uint32, "i32": np.uint32, "u64": np.uint64, "i64": np.uint64}[kt]
    w = a.view(u).copy()
    if kt[0] == "i":
        w ^= u(1) << u(8 * a.itemsize - 1)
    return ~w if desc else w


@pytest.mark.parametrize("kt,desc", [("u64", False), ("i32", True), ("u32", False), ("i64", True)])
def test_partition_matches_searchsorted(cuda, kt, desc):
    rng = np.random.default_rng(3)
    dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[kt]
    info = np.iinfo(dt)
    for n, nspl in ((100_000, 7), (1_000_003, 1), (2_000_000, 255), (5000, 3)):
        x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        smp = np.sort(enc(x[rng.integers(0, n, 4096)], kt, desc))
        spl = smp[np.linspace(0, 4095, nspl + 2).astype(int)[1:-1]]
        spl[0] = spl[min(1, nspl - 1)]  # duplicate splitters are legal
        d = torch.from_numpy(x).cuda()
        out, counts = vx.partition(d, torch.from_numpy(spl).cuda(), order=vx.Order(int(desc)))
        torch.cuda.synchronize()
        seg = np.searchsorted(spl, enc(x, kt, desc), side="left")
        want_counts = np.bincount(seg, minlength=nspl + 1)
        assert (counts.cpu().numpy() == want_counts).all()
        o = out.cpu().numpy()
        off = np.concatenate([[0], np.cumsum(want_counts)])
        for i in range(nspl + 1):
            got = np.sort(o[off[i]:off[i + 1]])
            exp = np.sort(x[seg == i])
            assert got.tobytes() == exp.tobytes()


def test_sample_is_order_transformed_subset(cuda):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(300_000).astype(np.float32)
    d = torch.from_numpy(x).cuda()
    s = vx.sample(d, 2048, order=vx.Order.kDescending, seed=9).cpu().numpy()
    w = torch.from_numpy(x.copy()).cuda()
    vx.transform(w, vx.Order.kDescending)
    allw = set(w.cpu().numpy().view(np.uint32).tolist())
    assert all(v in allw for v in s.tolist())


def test_dist_sort_world1_nccl(cuda):
    import torch.distributed as dist
    from paper_2205_05982_b200.dist import dist_sort
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(1)
        x = rng.integers(0, 2**64, 1_000_000, dtype=np.uint64)
        out = dist_sort(torch.from_numpy(x).cuda())
        assert out.cpu().numpy().tobytes() == np.sort(x).tobytes()
    finally:
        dist.destroy_process_group()
