"""Distributed sample sort across GPUs (new work -- the
reference is single-threaded).

One process per GPU; ``torch.distributed`` (NCCL over NVLink/NVSwitch) is the
plumbing for the two real exchange steps of a sample sort:

  1. local splitter sampling on the device (vxs_sample: s stratified keys,
     order-transformed so they compare as unsigned words);
  2. all-gather of the G*s samples; every rank sorts them with the B200 sort
     and picks the same G-1 global splitters (quantiles);
  3. local multiway partition by those splitters (vxs_partition: the same
     classify+scatter kernels as one sort level) into G contiguous segments;
  4. all-to-all of the segment counts, then of the keys (NCCL grouped
     send/recv under ``all_to_all_single``);
  5. local B200 sort of the received keys.

Rank r ends with the r-th key range, sorted; concatenation over ranks in rank
order equals the single-array sort.  Host-side logic (splitter choice, split
sizes, offsets) is plain Python so the world_size>1 path is tested on CPU
with the gloo backend (tests/test_dist_gloo.py), where ``ops`` supplies CPU
stand-ins for the three device kernels.  The product path always uses the
CUDA ops (``CudaOps``) and fails loudly without them.

Exchange (step 4) comes in two forms:
  * ``exchange="fused"`` (default): the partition is split in
    two -- ``vxs_partition_counts`` (read-only classify + per-CTA offsets),
    an all-gather of the tiny G x G count matrix, then
    ``vxs_partition_exchange``, whose scatter stores every segment straight
    into its owner's receive buffer (a symmetric window: one IPC-exported
    block per rank, mapped by every peer over NVLink) at this rank's offset
    there.  The all-to-all rides on the scatter's own stores: no local
    partitioned copy, no NCCL data movement; one small all-reduce orders the
    peers' stores before the local sort.
  * ``exchange="nccl"``: partition into a local buffer, then NCCL
    ``all_to_all_single`` of counts and keys (the baseline).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch
import torch.distributed as dist

from . import (KEY_BYTES, KEY_CODE, DeviceBlock, Order, SortConfig, SortStats, _check, _device_of, _nkeys,
               _stream_ptr, infer_key_type, lib, partition, partition_counts, partition_exchange, sample, sort,
               workspace_bytes)


class SymmetricWindow:
    """Per-group receive buffers of the fused exchange: one IPC-exportable
    device block per rank, each mapped by every peer (P2P over NVLink /
    NVSwitch).  Capacity only grows, collectively (every rank computes the
    same required size from the same all-gathered count matrix)."""

    def __init__(self):
        self.nbytes = 0
        self.mine = None
        self.peers = []   # DeviceBlock per rank (rank's own = self.mine)
        self.addrs = None  # int64 device tensor of the ranks' base addresses

    def ensure(self, nbytes: int, group, device):
        if nbytes <= self.nbytes:
            return
        nbytes = max(nbytes, int(self.nbytes * 1.25))
        nbytes = (nbytes + (1 << 21) - 1) & ~((1 << 21) - 1)
        torch.cuda.synchronize(device)
        self.close(group)
        self.mine = DeviceBlock(nbytes)
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, self.mine.handle(), group=group)
        me = dist.get_rank(group)
        self.peers = [self.mine if r == me else DeviceBlock.open(h, nbytes) for r, h in enumerate(handles)]
        self.addrs = torch.tensor([b.ptr for b in self.peers], dtype=torch.int64, device=device)
        self.nbytes = nbytes

    def local(self):
        return self.mine.tensor()

    def close(self, group=None):
        # every rank unmaps its peers' blocks before any owner frees its own
        # (freeing an exported block that is still mapped elsewhere is undefined)
        for b in self.peers:
            if b is not self.mine:
                b.close()
        if self.mine is not None:
            if dist.is_initialized():
                dist.barrier(group=group)
            self.mine.close()
        self.peers, self.mine, self.nbytes = [], None, 0


_WINDOWS = {}


def _window(group) -> SymmetricWindow:
    return _WINDOWS.setdefault(id(group), SymmetricWindow())


class CudaOps:
    """The device kernels a rank runs (libvxsort_b200.so)."""

    def sample(self, keys, s, order, key_type, seed):
        return sample(keys, s, order=order, seed=seed, key_type=key_type)

    def sort_words(self, words, key_bytes):
        """Sort transformed-domain words ascending (unsigned)."""
        kt = {2: "u16", 4: "u32", 8: "u64", 16: "k128"}[key_bytes]
        sort(words, SortConfig(seed=1), key_type=kt)
        return words

    def partition(self, keys, splitters, order, key_type):
        return partition(keys, splitters, order=order, key_type=key_type)

    def sort(self, keys, order, key_type):
        sort(keys, SortConfig(order=order, seed=1), key_type=key_type if key_type in ("k128", "kv64") else None)
        return keys

    # fused exchange
    def workspace(self, keys, key_type):
        return torch.empty(workspace_bytes(max(1, keys.shape[0]), key_type), dtype=torch.uint8, device=keys.device)

    def partition_counts(self, keys, splitters, order, key_type, ws):
        return partition_counts(keys, splitters, ws, order=order, key_type=key_type)

    def window(self, group):
        return _window(group)

    def exchange(self, keys, nspl, window, offsets, order, key_type, ws, group=None):
        dev = window.addrs.device
        if keys is not None and keys.shape[0] > 0:
            offs = torch.as_tensor(offsets, dtype=torch.int64).to(dev, non_blocking=True)
            partition_exchange(keys, nspl, window.addrs, offs, ws, order=order, key_type=key_type)
        # order every peer's stores before anyone reads its window: a stream-
        # ordered collective after the exchange kernel on every rank
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        dist.all_reduce(flag, group=group)


def _bytes(t: torch.Tensor) -> torch.Tensor:
    if t.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=t.device)
    return t.contiguous().view(torch.uint8).reshape(-1)


def choose_splitters(gathered_sorted: torch.Tensor, world: int, per_rank: int) -> torch.Tensor:
    """G-1 equidistant global splitters from the sorted G*s sample (every rank
    computes the same ones from the same all-gathered bytes)."""
    idx = torch.arange(1, world, device=gathered_sorted.device) * per_rank - 1
    # (CUDA indexing has no unsigned kernels: gather the same bits as signed)
    signed = {torch.uint64: torch.int64, torch.uint32: torch.int32, torch.uint16: torch.int16}
    t = gathered_sorted
    if t.dtype in signed:
        return t.view(signed[t.dtype])[idx].contiguous().view(t.dtype)
    return t[idx].contiguous()


def exchange_offsets(all_counts, rank: int):
    """From the G x G count matrix (row s = rank s's per-destination counts):
    this rank's element offset inside every destination's receive buffer
    (senders land in rank order) and how many keys this rank receives."""
    world = len(all_counts)
    offs = [sum(all_counts[s][r] for s in range(rank)) for r in range(world)]
    recv = sum(all_counts[s][rank] for s in range(world))
    need = max(sum(all_counts[s][r] for s in range(world)) for r in range(world))
    return offs, recv, need


def dist_sort(local: torch.Tensor, order: Order = Order.kAscending, key_type: Optional[str] = None,
              group=None, oversample: int = 256, seed: int = 1, ops=None, timings: Optional[dict] = None,
              exchange: str = "fused", copy_out: bool = True):
    """Sort the union of every rank's ``local`` keys; returns this rank's
    sorted slice of the global order (a new tensor; with exchange="fused" and
    copy_out=False, a view of the group's receive window that the next
    dist_sort on the group overwrites)."""
    ops = ops or CudaOps()
    kt = infer_key_type(local, key_type)
    kb = KEY_BYTES[kt]
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        out = local.clone()
        return ops.sort(out, order, kt)
    n = int(local.shape[0])
    s = oversample * world
    # 1. local samples (transformed words); empty ranks contribute max words
    if n > 0:
        smp = ops.sample(local, s, order, kt, seed ^ (rank * 0x9E3779B97F4A7C15 & (2**64 - 1)))
    else:
        shape = (s, 2) if kb == 16 else (s,)
        smp = torch.full(shape, -1, dtype={2: torch.int16, 4: torch.int32, 8: torch.int64, 16: torch.int64}[kb],
                         device=local.device).view({2: torch.uint16, 4: torch.uint32, 8: torch.uint64,
                                                    16: torch.uint64}[kb])
    # 2. all-gather, identical sort + splitter choice on every rank
    sb = _bytes(smp)
    gathered = torch.empty(world * sb.numel(), dtype=torch.uint8, device=local.device)
    dist.all_gather_into_tensor(gathered, sb, group=group)
    words = gathered.view(smp.dtype).reshape((world * s, 2) if kb == 16 else (world * s,)).clone()
    words = ops.sort_words(words, kb)
    spl = choose_splitters(words, world, s)
    if exchange == "fused":
        return _fused_tail(local, n, kt, kb, spl, order, group, world, rank, ops, timings, copy_out)
    # 3. local multiway partition into `world` segments
    if n > 0:
        parted, seg_counts = ops.partition(local, spl, order, kt)
    else:
        parted, seg_counts = local, torch.zeros(world, dtype=torch.int64, device=local.device)
    # 4. exchange counts, then keys
    recv_counts = torch.empty_like(seg_counts)
    dist.all_to_all_single(recv_counts, seg_counts, group=group)
    send_sizes = [int(c) * kb for c in seg_counts.tolist()]
    recv_sizes = [int(c) * kb for c in recv_counts.tolist()]
    recv = torch.empty(sum(recv_sizes), dtype=torch.uint8, device=local.device)
    dist.all_to_all_single(recv, _bytes(parted), output_split_sizes=recv_sizes,
                           input_split_sizes=send_sizes, group=group)
    shape = (sum(recv_sizes) // kb, 2) if kb == 16 else (sum(recv_sizes) // kb,)
    out = recv.view(local.dtype).reshape(shape)
    # 5. local sort of this rank's key range
    if out.shape[0] > 1:
        out = ops.sort(out, order, kt)
    if timings is not None:
        timings["recv_keys"] = int(out.shape[0])
        timings["send_counts"] = seg_counts.tolist()
    return out


def _fused_tail(local, n, kt, kb, spl, order, group, world, rank, ops, timings, copy_out):
    """Steps 3-5 with the fused exchange (module docstring)."""
    ws = ops.workspace(local, kt)
    if n > 0:
        counts = ops.partition_counts(local, spl, order, kt, ws)
    else:
        counts = torch.zeros(world, dtype=torch.int64, device=local.device)
    allc = torch.empty(world * world, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(allc, counts, group=group)
    m = allc.view(world, world).tolist()
    offs, recv, need = exchange_offsets(m, rank)
    win = ops.window(group)
    win.ensure(need * kb, group, local.device)
    ops.exchange(local if n > 0 else None, world - 1, win, offs, order, kt, ws, group)
    buf = win.local()[: recv * kb]
    shape = (recv, 2) if kb == 16 else (recv,)
    out = buf.view(local.dtype).reshape(shape)
    if recv > 1:
        out = ops.sort(out, order, kt)
    if timings is not None:
        timings["recv_keys"] = int(recv)
        timings["send_counts"] = m[rank]
    return out.clone() if copy_out else out


# ---- the C-ABI distributed sort (vxs_dist_*, include/vxsort_b200.h) ----------
_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)


class _DistGroup(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_comm", ctypes.c_void_p),
                ("allgather", _ALLGATHER_FN), ("allgather_ctx", ctypes.c_void_p)]


class NativeDist:
    """Python handle on the C++ distributed sort (``vxs_dist_sort``): the
    whole sample sort -- sampling, splitters, exchange, local sort -- runs in
    the library; Python only supplies the process group.

    ``comm="nccl"``: a native NCCL communicator (bootstrapped over the torch
    group), the small collectives on the device.  ``comm="host"``: the
    library's host all-gather callback over a CPU (gloo) group -- works when
    ranks share a GPU, which NCCL refuses.  Collective: every rank of the
    group constructs, sorts and closes together."""

    def __init__(self, group=None, comm: str = "host"):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.comm = None
        self._cpu_group = None
        self._cb = _ALLGATHER_FN(0)
        if comm == "nccl":
            idb = ctypes.create_string_buffer(128)
            if self.rank == 0:
                _check(lib().vxs_nccl_unique_id(idb))
            obj = [idb.raw]
            dist.broadcast_object_list(obj, src=0, group=group)
            idb = ctypes.create_string_buffer(obj[0], 128)
            out = ctypes.c_void_p()
            _check(lib().vxs_nccl_comm_create(idb, self.world, self.rank, ctypes.byref(out)))
            self.comm = out.value
        elif self.world > 1:
            backend = dist.get_backend(group)
            self._cpu_group = group if backend == "gloo" else dist.new_group(backend="gloo")
            self._cb = _ALLGATHER_FN(self._allgather)
        g = _DistGroup(self.rank, self.world, self.comm, self._cb, None)
        out = ctypes.c_void_p()
        _check(lib().vxs_dist_create(ctypes.byref(g), ctypes.byref(out)))
        self.ctx = out.value

    def _allgather(self, _ctx, send, recv, nbytes):
        try:
            src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8)
            dst = torch.empty(self.world * nbytes, dtype=torch.uint8)
            dist.all_gather_into_tensor(dst, src, group=self._cpu_group)
            ctypes.memmove(recv, dst.data_ptr(), self.world * nbytes)
            return 0
        except Exception:  # noqa: BLE001  (reported to the library as a failed collective)
            return 1

    def sort(self, keys: torch.Tensor, order: Order = Order.kAscending, key_type: Optional[str] = None,
             seed: int = 1, exchange: str = "fused", stream=None):
        """This rank's sorted slice of the union of every rank's ``keys`` --
        a view of the context's receive window, valid until the next sort or
        close.  Returns (tensor, SortStats)."""
        kt = infer_key_type(keys, key_type)
        if not keys.is_cuda or not keys.is_contiguous():
            raise ValueError("keys must be a contiguous CUDA tensor")
        n = _nkeys(keys, kt)
        d_out = ctypes.c_void_p()
        n_out = ctypes.c_size_t()
        st = SortStats()
        with _device_of(keys):
            _check(lib().vxs_dist_sort(self.ctx, keys.data_ptr() if n else None, n, KEY_CODE[kt], int(order),
                                       int(seed) & (2**64 - 1), 0 if exchange == "fused" else 1,
                                       ctypes.byref(d_out), ctypes.byref(n_out), _stream_ptr(stream),
                                       ctypes.byref(st)))
        kb = KEY_BYTES[kt]
        m = int(n_out.value)
        blk = DeviceBlock(max(m * kb, 1), ptr=d_out.value, owned=False)
        raw = torch.as_tensor(blk, device=keys.device)[: m * kb]
        shape = (m, 2) if kb == 16 else (m,)
        return raw.view(keys.dtype).reshape(shape), st

    def last_counts(self):
        """(keys received per rank, this rank's keys sent per destination)."""
        r = (ctypes.c_uint64 * self.world)()
        s_ = (ctypes.c_uint64 * self.world)()
        _check(lib().vxs_dist_last_counts(self.ctx, r, s_))
        return list(r), list(s_)

    def close(self):
        if self.ctx:
            _check(lib().vxs_dist_destroy(self.ctx))
            self.ctx = None
        if self.comm:
            _check(lib().vxs_nccl_comm_destroy(self.comm))
            self.comm = None
