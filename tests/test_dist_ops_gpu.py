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


@pytest.mark.parametrize("kt,desc,world", [("u64", False, 3), ("i32", True, 4), ("u32", False, 2),
                                           ("i64", True, 8), ("f32", False, 3), ("k128", False, 3)])
def test_fused_exchange_virtual_ranks(cuda, kt, desc, world):
    """vxs_partition_counts + vxs_partition_exchange with `world` ranks
    emulated in one process (B200_PROFILING: with fewer GPUs than
    ranks, run the ranks' kernels on one GPU -- none of them waits on
    another).  Each rank's scatter stores straight into the other ranks'
    receive buffers at the offsets dist.exchange_offsets computes; the
    concatenated, locally sorted buffers must equal the oracle's sort."""
    from paper_2205_05982_b200.dist import choose_splitters, exchange_offsets
    rng = np.random.default_rng(17 + world)
    kb = vx.KEY_BYTES[kt]
    locs = []
    for r in range(world):
        n = 300_000 + 7919 * r if r != 1 else 0  # rank 1 holds no keys
        if kt == "k128":
            x = rng.integers(0, 2**64, (n, 2), dtype=np.uint64)
            x[:, 1] >>= 44  # many hi ties
        elif kt == "f32":
            x = (rng.standard_normal(n) * 1e3).astype(np.float32)
        else:
            dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[kt]
            info = np.iinfo(dt)
            x = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
        locs.append(x)
    order = vx.Order(int(desc))
    ktarg = kt if kt == "k128" else None
    dev = [torch.from_numpy(x).cuda() for x in locs]
    s = 256 * world
    smp = [vx.sample(d, s, order=order, seed=r + 1, key_type=ktarg) for r, d in enumerate(dev) if d.shape[0]]
    words = torch.cat(smp)
    vx.sort(words, vx.SortConfig(seed=1), key_type={2: "u16", 4: "u32", 8: "u64", 16: "k128"}[kb])
    spl = choose_splitters(words, world, words.shape[0] // world)
    ws = [torch.empty(vx.workspace_bytes(max(1, d.shape[0]), kt), dtype=torch.uint8, device="cuda") for d in dev]
    counts = [vx.partition_counts(d, spl, w, order=order, key_type=ktarg) if d.shape[0]
              else torch.zeros(world, dtype=torch.int64, device="cuda") for d, w in zip(dev, ws)]
    m = torch.stack(counts).cpu().tolist()
    recv = [sum(m[s_][r] for s_ in range(world)) for r in range(world)]
    bufs = [torch.empty((recv[r], 2) if kb == 16 else (recv[r],), dtype=dev[0].dtype, device="cuda")
            for r in range(world)]
    addrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    for r in range(world):
        offs, got_recv, _ = exchange_offsets(m, r)
        assert got_recv == recv[r]
        if dev[r].shape[0]:
            vx.partition_exchange(dev[r], world - 1, addrs, torch.tensor(offs, dtype=torch.int64, device="cuda"),
                                  ws[r], order=order, key_type=ktarg)
    for b in bufs:
        if b.shape[0] > 1:
            vx.sort(b, vx.SortConfig(order=order, seed=1), key_type=ktarg)
    got = np.concatenate([b.cpu().numpy() for b in bufs])
    want, _ = oracle.sort(np.concatenate(locs), kt, descending=desc)
    assert got.tobytes() == want.tobytes()
    if kt in ("u64", "u32", "i32", "i64"):
        assert max(recv) < 1.5 * sum(recv) / world  # sampled splitters balance the ranks


def _ipc_child(handle, nbytes, q):
    import torch
    import paper_2205_05982_b200 as vx2
    torch.cuda.set_device(0)
    try:
        blk = vx2.DeviceBlock.open(handle, nbytes)
        t = blk.tensor()
        q.put(int(t[:4096].view(torch.int32).sum().item()))
        t[:4096].view(torch.int32).fill_(7)  # write through the mapping
        torch.cuda.synchronize()
        blk.close()
        q.put("ok")
    except Exception as e:  # noqa: BLE001
        q.put(repr(e))


def test_device_block_ipc(cuda):
    """The fused exchange's symmetric window plumbing: an IPC-exported block
    (vxs_device_alloc / vxs_ipc_handle), viewed as a tensor through
    __cuda_array_interface__, mapped by another process (vxs_ipc_open) that
    reads and writes it -- no kernel waits on another process."""
    import torch.multiprocessing as mp
    nbytes = 1 << 20
    blk = vx.DeviceBlock(nbytes)
    t = blk.tensor()
    assert t.numel() == nbytes and t.device.type == "cuda" and t.data_ptr() == blk.ptr
    t.view(torch.int32)[:1024].fill_(3)
    t.view(torch.int32)[1024:].zero_()
    torch.cuda.synchronize()
    h = blk.handle()
    assert isinstance(h, bytes) and len(h) == 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(h, nbytes, q))
    p.start()
    got = q.get(timeout=120)
    status = q.get(timeout=120)
    p.join(timeout=60)
    assert status == "ok", status
    assert got == 3 * 1024
    assert int(t[:4096].view(torch.int32).sum().item()) == 7 * 1024
    blk.close()
