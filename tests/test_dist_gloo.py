"""World-size-2 (and 3) CPU runs of the distributed sample sort's host logic
over the gloo backend, for both exchanges (NCCL-style all-to-all and the
fused partition+exchange, whose peer stores are emulated here).  The three device kernels are replaced, in this test
only, by CPU stand-ins built on the oracle; the collectives, splitter choice,
split sizes and segment ordering are the product code in dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2205_05982_b200 import Order
from paper_2205_05982_b200.dist import dist_sort

SIGN = {"i32": np.uint32(1 << 31), "i64": np.uint64(1 << 63)}
UNS = {"u32": np.uint32, "i32": np.uint32, "u64": np.uint64, "i64": np.uint64}


def enc(a: np.ndarray, kt, desc):
    """Transformed words (keys.cuh enc) for integer types."""
    w = a.view(UNS[kt]).copy()
    if kt in SIGN:
        w ^= SIGN[kt]
    if desc:
        w = ~w
    return w


class CpuOps:
    def __init__(self, kt):
        self.kt = kt

    def sample(self, keys, s, order, key_type, seed):
        a = keys.numpy()
        rng = np.random.default_rng(seed & 0xFFFFFFFF)
        idx = (np.arange(s) * len(a)) // s + rng.integers(0, max(1, len(a) // s), s)
        idx = np.minimum(idx, len(a) - 1)
        return torch.from_numpy(enc(a[idx], key_type, bool(order)))

    def sort_words(self, words, kb):
        w = words.numpy()
        return torch.from_numpy(np.sort(w))

    def partition(self, keys, spl, order, key_type):
        a = keys.numpy()
        seg = np.searchsorted(spl.numpy(), enc(a, key_type, bool(order)), side="left")
        o = np.argsort(seg, kind="stable")
        counts = np.bincount(seg, minlength=len(spl) + 1).astype(np.int64)
        return torch.from_numpy(a[o].copy()), torch.from_numpy(counts)

    def sort(self, keys, order, key_type):
        out, _ = oracle.sort(keys.numpy(), key_type, descending=bool(order))
        keys.copy_(torch.from_numpy(out))  # in place, like the device sort
        return keys

    # fused exchange stand-ins: the "window" is a host tensor and the fused
    # kernel's peer stores are emulated by a gloo all-to-all that carries the
    # SENDER's offsets, so the product's offset/capacity logic is what places
    # every segment
    def workspace(self, keys, key_type):
        return None

    def partition_counts(self, keys, spl, order, key_type, ws):
        return self.partition(keys, spl, order, key_type)[1]

    def window(self, group):
        return self._win

    def exchange(self, keys, nspl, window, offsets, order, key_type, ws, group=None):
        world = nspl + 1
        kb = {"u32": 4, "i32": 4, "u64": 8, "i64": 8}[key_type]
        if keys is not None and keys.shape[0] > 0:
            parted, counts = self.partition(keys, self._spl, order, key_type)
        else:
            parted, counts = torch.zeros(0, dtype=torch.uint8), torch.zeros(world, dtype=torch.int64)
        hdr = torch.tensor(list(offsets), dtype=torch.int64)
        rhdr = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rhdr, hdr, group=group)
        rcnt = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rcnt, counts, group=group)
        send = parted.contiguous().view(torch.uint8).reshape(-1)
        recv = torch.empty(int(rcnt.sum()) * kb, dtype=torch.uint8)
        dist.all_to_all_single(recv, send, output_split_sizes=[int(c) * kb for c in rcnt.tolist()],
                               input_split_sizes=[int(c) * kb for c in counts.tolist()], group=group)
        loc = window.local()
        pos = 0
        for src in range(world):
            nb = int(rcnt[src]) * kb
            o = int(rhdr[src]) * kb
            loc[o:o + nb] = recv[pos:pos + nb]
            pos += nb


class CpuWindow:
    def __init__(self):
        self.buf = torch.zeros(0, dtype=torch.uint8)

    def ensure(self, nbytes, group, device):
        if nbytes > self.buf.numel():
            self.buf = torch.zeros(nbytes, dtype=torch.uint8)

    def local(self):
        return self.buf


class CpuOpsFused(CpuOps):
    """Remembers the splitters the product passes to partition_counts (the
    fused kernel keeps them in its workspace)."""

    def __init__(self, kt):
        super().__init__(kt)
        self._win = CpuWindow()

    def partition_counts(self, keys, spl, order, key_type, ws):
        self._spl = spl
        return super().partition_counts(keys, spl, order, key_type, ws)

    def exchange(self, keys, nspl, window, offsets, order, key_type, ws, group=None):
        if not hasattr(self, "_spl"):
            self._spl = None
        return super().exchange(keys, nspl, window, offsets, order, key_type, ws, group)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [("u64", False, "uniform"), ("i32", True, "uniform"), ("u32", False, "equal"),
         ("i64", False, "few"), ("u64", True, "skew"), ("u32", False, "empty_rank")]


def _make(rank, kt, dist_name, n_per):
    rng = np.random.default_rng(100 + rank)
    dt = {"u32": np.uint32, "i32": np.int32, "u64": np.uint64, "i64": np.int64}[kt]
    n = n_per + rank * 137
    if dist_name == "uniform":
        info = np.iinfo(dt)
        return rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    if dist_name == "equal":
        return np.full(n, 42, dtype=dt)
    if dist_name == "few":
        return rng.integers(0, 5, n).astype(dt)
    if dist_name == "empty_rank":
        return rng.integers(0, 1000, 0 if rank == 0 else n).astype(dt)
    return (rng.random(n) ** 4 * 1e9).astype(dt)  # skewed


def _worker(rank, world, port, q, exchange):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    for ci, (kt, desc, dist_name) in enumerate(CASES):
        x = _make(rank, kt, dist_name, 20000)
        ops = CpuOpsFused(kt) if exchange == "fused" else CpuOps(kt)
        out = dist_sort(torch.from_numpy(x), order=Order(int(desc)), key_type=kt, ops=ops, oversample=16,
                        exchange=exchange)
        q.put((ci, rank, x, out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,exchange", [(2, "nccl"), (3, "nccl"), (2, "fused"), (3, "fused")])
def test_dist_sort_gloo(world, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world * len(CASES)):
        ci, r, x, out = q.get(timeout=300)
        res[(ci, r)] = (x, out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (kt, desc, dist_name) in enumerate(CASES):
        allin = np.concatenate([res[(ci, r)][0] for r in range(world)])
        got = np.concatenate([res[(ci, r)][1] for r in range(world)])
        want, _ = oracle.sort(allin, kt, descending=desc)
        assert got.tobytes() == want.tobytes(), (kt, desc, dist_name)
        if dist_name == "uniform":
            sizes = [len(res[(ci, r)][1]) for r in range(world)]
            assert max(sizes) < 1.5 * (len(allin) / world)  # sampled splitters balance


def test_exchange_offsets():
    from paper_2205_05982_b200.dist import exchange_offsets
    m = [[3, 1, 0], [2, 5, 4], [0, 7, 1]]  # row s: rank s's counts per destination
    offs, recv, need = exchange_offsets(m, 1)
    assert offs == [3, 1, 0] and recv == 13 and need == 13
    offs, recv, need = exchange_offsets(m, 2)
    assert offs == [5, 6, 4] and recv == 5
    offs, recv, _ = exchange_offsets(m, 0)
    assert offs == [0, 0, 0] and recv == 5
