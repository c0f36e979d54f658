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
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import KEY_BYTES, Order, SortConfig, infer_key_type, partition, sample, sort


class CudaOps:
    """The three device kernels a rank runs (libvxsort_b200.so)."""

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


def _bytes(t: torch.Tensor) -> torch.Tensor:
    if t.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=t.device)
    return t.contiguous().view(torch.uint8).reshape(-1)


def choose_splitters(gathered_sorted: torch.Tensor, world: int, per_rank: int) -> torch.Tensor:
    """G-1 equidistant global splitters from the sorted G*s sample (every rank
    computes the same ones from the same all-gathered bytes)."""
    idx = torch.arange(1, world, device=gathered_sorted.device) * per_rank - 1
    return gathered_sorted[idx].contiguous()


def dist_sort(local: torch.Tensor, order: Order = Order.kAscending, key_type: Optional[str] = None,
              group=None, oversample: int = 256, seed: int = 1, ops=None, timings: Optional[dict] = None):
    """Sort the union of every rank's ``local`` keys; returns this rank's
    sorted slice of the global order (a new tensor)."""
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
