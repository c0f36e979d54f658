"""paper_2205_05982_b200 -- B200-native in-memory key sort behind the vexsort surface.

Python host mirror of the reference API (``/root/reference/proj/core/include/
vexsort/vexsort.hpp:31-132``):

    stats = sort(keys, SortConfig(order=Order.kDescending, seed=3))

``keys`` is sorted IN PLACE and may be a numpy array (host memory: the
reference's ``std::span`` semantics, copied through the device) or a torch
CUDA tensor (device memory, stream-ordered on torch's current stream).  Key
types: the reference's nine (int16, uint16, int32, uint32, float32, int64,
uint64, float64, K128 as an (n, 2) uint64 array of {lo, hi}) plus KV64
(K128 layout {lo=payload, hi=key}).

Everything computes in ``lib/libvxsort_b200.so`` (hand-written sm_100a
kernels behind the C ABI of ``include/vxsort_b200.h``).  There is no CPU
fallback: if the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# VXSORT_LIB=checked loads the checked build (device-side bounds and
# consistency checks, `make checked`); the default is the product build.
LIB_PATH = os.path.join(_HERE, "lib", "libvxsort_b200_checked.so" if os.environ.get("VXSORT_LIB") == "checked"
                        else "libvxsort_b200.so")

KEY_TYPES = ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64", "k128", "kv64"]
KEY_CODE = {k: i for i, k in enumerate(KEY_TYPES)}
KEY_BYTES = {"i16": 2, "u16": 2, "i32": 4, "u32": 4, "f32": 4, "i64": 8, "u64": 8, "f64": 8,
             "k128": 16, "kv64": 16}
_NP_TO_KEY = {np.dtype(np.int16): "i16", np.dtype(np.uint16): "u16", np.dtype(np.int32): "i32",
              np.dtype(np.uint32): "u32", np.dtype(np.float32): "f32", np.dtype(np.int64): "i64",
              np.dtype(np.uint64): "u64", np.dtype(np.float64): "f64"}


class Order(enum.IntEnum):
    """vexsort::Order (vexsort.hpp:31)."""
    kAscending = 0
    kDescending = 1


class Backend(enum.IntEnum):
    """vexsort::Backend (vexsort.hpp:36).  Accepted for source compatibility;
    every backend value runs the B200 kernels (there is no CPU path)."""
    kAuto = 0
    kScalar = 1
    kWide = 2


class VxsError(RuntimeError):
    """CUDA / internal failure (the reference has no analogue; C++ wrapper
    maps it to std::runtime_error)."""


class SortStats(ctypes.Structure):
    """vexsort::SortStats (driver.hpp:26-32) + device extras (vxs_stats)."""
    _fields_ = [
        ("max_depth", ctypes.c_size_t),
        ("partition_calls", ctypes.c_size_t),
        ("base_case_calls", ctypes.c_size_t),
        ("keys_partitioned", ctypes.c_size_t),
        ("fallback_triggered", ctypes.c_int),
        ("kernel_launches", ctypes.c_int),
        ("workspace_bytes", ctypes.c_size_t),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


@dataclasses.dataclass
class SortConfig:
    """vexsort::SortConfig (vexsort.hpp:112-119)."""
    order: Order = Order.kAscending
    backend: Backend = Backend.kAuto
    seed: Optional[int] = None
    scratch: Optional["SortScratch"] = None


# Reference scratch sizes (vexsort.hpp:58-66), reproduced so that the
# reference's "too-small scratch -> std::invalid_argument" behaviour
# (vexsort.cpp:19-31) carries over unchanged.  The B200 path needs O(n)
# DEVICE workspace instead (workspace_bytes()).
_REF_SCRATCH_BYTES = {"i16": 512, "u16": 512, "i32": 1024, "u32": 1024, "f32": 1024,
                      "i64": 2048, "u64": 2048, "f64": 2048, "k128": 4096, "kv64": 4096}


def scratch_bytes(key_type: str) -> int:
    return _REF_SCRATCH_BYTES[key_type]


class SortScratch:
    """vexsort::SortScratch (vexsort.hpp:69-110): a host buffer of a given size."""

    def __init__(self, nbytes: int = 0):
        self._buf = bytearray(nbytes)

    @classmethod
    def for_key(cls, key_type: str) -> "SortScratch":
        return cls(scratch_bytes(key_type))

    def size(self) -> int:
        return len(self._buf)


_lib = None


def lib():
    """Load the CUDA library; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise VxsError(f"libvxsort_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, u64, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int
        L.vxs_sort.argtypes = [vp, sz, i, i, u64, i, vp, sz, vp, ctypes.POINTER(SortStats)]
        L.vxs_sort_host.argtypes = [vp, sz, i, i, u64, i, ctypes.POINTER(SortStats)]
        L.vxs_sort_workspace_bytes.argtypes = [sz, i, ctypes.POINTER(ctypes.c_size_t)]
        L.vxs_sample.argtypes = [vp, sz, i, i, u64, vp, i, vp]
        L.vxs_partition.argtypes = [vp, sz, i, i, vp, i, vp, vp, vp, sz, vp]
        L.vxs_transform.argtypes = [vp, sz, i, i, i, vp]
        L.vxs_last_error.restype = ctypes.c_char_p
        L.vxs_version.restype = ctypes.c_char_p
        L.vxs_key_bytes.argtypes = [i]
        L.vxs_key_bytes.restype = sz
        L.vxs_base_case_capacity.argtypes = [i]
        L.vxs_base_case_capacity.restype = sz
        L.vxs_profile_enable.argtypes = [i]
        L.vxs_profile_read.argtypes = [ctypes.c_void_p, i]
        L.vxs_profile_read.restype = i
        L.vxs_sort_range.argtypes = [vp, sz, i, i, sz, sz, u64, i, vp, sz, vp, ctypes.POINTER(SortStats)]
        L.vxs_sort_range.restype = ctypes.c_int
        L.vxs_argsort_workspace_bytes.argtypes = [sz, i, sz, ctypes.POINTER(ctypes.c_size_t)]
        L.vxs_argsort.argtypes = [vp, sz, i, i, vp, vp, u64, i, vp, sz, vp, ctypes.POINTER(SortStats)]
        L.vxs_sort_pairs.argtypes = [vp, vp, sz, sz, i, i, u64, i, vp, sz, vp, ctypes.POINTER(SortStats)]
        L.vxs_partition_counts.argtypes = [vp, sz, i, i, vp, i, vp, vp, sz, vp]
        L.vxs_partition_exchange.argtypes = [vp, sz, i, i, i, vp, vp, vp, sz, vp]
        L.vxs_device_alloc.argtypes = [sz, ctypes.POINTER(ctypes.c_void_p)]
        L.vxs_device_free.argtypes = [vp]
        L.vxs_ipc_handle.argtypes = [vp, vp]
        L.vxs_ipc_open.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
        L.vxs_ipc_close.argtypes = [vp]
        L.vxs_workspace_status.argtypes = [vp, sz, i, vp, ctypes.POINTER(SortStats)]
        L.vxs_workspace_status.restype = ctypes.c_int
        L.vxs_dist_create.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
        L.vxs_dist_destroy.argtypes = [vp]
        L.vxs_dist_sort.argtypes = [vp, vp, sz, i, i, u64, i, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_size_t), vp, ctypes.POINTER(SortStats)]
        L.vxs_dist_last_counts.argtypes = [vp, vp, vp]
        L.vxs_nccl_unique_id.argtypes = [vp]
        L.vxs_nccl_comm_create.argtypes = [vp, i, i, ctypes.POINTER(ctypes.c_void_p)]
        L.vxs_nccl_comm_destroy.argtypes = [vp]
        for fn in ("vxs_dist_create", "vxs_dist_destroy", "vxs_dist_sort", "vxs_dist_last_counts",
                   "vxs_nccl_unique_id", "vxs_nccl_comm_create", "vxs_nccl_comm_destroy"):
            getattr(L, fn).restype = ctypes.c_int
        for fn in ("vxs_sort", "vxs_sort_host", "vxs_sort_workspace_bytes", "vxs_sample",
                   "vxs_partition", "vxs_transform", "vxs_argsort_workspace_bytes", "vxs_argsort",
                   "vxs_sort_pairs", "vxs_partition_counts", "vxs_partition_exchange", "vxs_device_alloc",
                   "vxs_device_free", "vxs_ipc_handle", "vxs_ipc_open", "vxs_ipc_close"):
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTED_SYMBOLS = ["vxs_sort_workspace_bytes", "vxs_sort", "vxs_sort_host", "vxs_sample",
                    "vxs_partition", "vxs_transform", "vxs_argsort_workspace_bytes", "vxs_argsort",
                    "vxs_sort_pairs", "vxs_sort_range", "vxs_last_error", "vxs_key_bytes",
                    "vxs_base_case_capacity", "vxs_version", "vxs_profile_enable",
                    "vxs_profile_reset", "vxs_profile_read", "vxs_partition_counts",
                    "vxs_partition_exchange", "vxs_device_alloc", "vxs_device_free", "vxs_ipc_handle",
                    "vxs_ipc_open", "vxs_ipc_close", "vxs_dist_create", "vxs_dist_destroy", "vxs_dist_sort",
                    "vxs_dist_last_counts", "vxs_nccl_unique_id", "vxs_nccl_comm_create", "vxs_nccl_comm_destroy",
                    "vxs_workspace_status"]


class KernelProfile(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_longlong), ("total_ms", ctypes.c_double)]


def profile_enable(on: bool = True):
    lib().vxs_profile_enable(int(bool(on)))


def profile_reset():
    lib().vxs_profile_reset()


def profile_read():
    """{kernel name: (launches, total device ms)} since the last reset."""
    arr = (KernelProfile * 32)()
    k = lib().vxs_profile_read(arr, 32)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(k)}


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().vxs_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    raise VxsError(f"status {rc}: {msg}")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def infer_key_type(keys, key_type: Optional[str] = None) -> str:
    if key_type is not None:
        if key_type not in KEY_CODE:
            raise ValueError(f"unknown key type {key_type}")
        return key_type
    if _is_torch(keys):
        import torch
        m = {torch.int16: "i16", torch.int32: "i32", torch.float32: "f32", torch.int64: "i64",
             torch.float64: "f64", torch.uint16: "u16", torch.uint32: "u32", torch.uint64: "u64"}
        if keys.dtype not in m:
            raise ValueError(f"unsupported dtype {keys.dtype}")
        if keys.dim() == 2 and keys.shape[1] == 2 and keys.dtype in (torch.int64, torch.uint64):
            raise ValueError("2-D 64-bit tensor: pass key_type='k128' or 'kv64'")
        return m[keys.dtype]
    dt = np.asarray(keys).dtype
    if dt not in _NP_TO_KEY:
        raise ValueError(f"unsupported dtype {dt}")
    if np.asarray(keys).ndim == 2:
        raise ValueError("2-D array: pass key_type='k128' or 'kv64'")
    return _NP_TO_KEY[dt]


def _nkeys(keys, key_type):
    if key_type in ("k128", "kv64"):
        if keys.ndim != 2 or tuple(keys.shape[1:]) != (2,):
            raise ValueError("K128/KV64 keys must have shape (n, 2) of 64-bit words {lo, hi}")
        return int(keys.shape[0])
    if keys.ndim != 1:
        raise ValueError(f"{key_type} keys must be a 1-D array (got shape {tuple(keys.shape)})")
    return int(keys.shape[0])


def _device_of(t):
    """torch.cuda.device context for a CUDA tensor: kernels launch on the
    tensor's device and that device's current stream."""
    import torch
    return torch.cuda.device(t.device)


def _check_cuda(t, what="keys"):
    if not (_is_torch(t) and t.is_cuda):
        raise ValueError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


def workspace_bytes(n: int, key_type: str) -> int:
    out = ctypes.c_size_t()
    _check(lib().vxs_sort_workspace_bytes(n, KEY_CODE[key_type], ctypes.byref(out)))
    return out.value


def _ws_args(workspace, keys):
    if workspace is None:
        return None, 0
    _check_cuda(workspace, "workspace")
    if workspace.device != keys.device:
        raise ValueError("workspace must live on the keys' device")
    return workspace.data_ptr(), workspace.numel() * workspace.element_size()


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def sort(keys, config: Optional[SortConfig] = None, key_type: Optional[str] = None,
         workspace=None, stream=None) -> SortStats:
    """vexsort::sort (vexsort.hpp:121-129): sort ``keys`` in place."""
    cfg = config or SortConfig()
    kt = infer_key_type(keys, key_type)
    if cfg.scratch is not None and cfg.scratch.size() < scratch_bytes(kt):
        raise ValueError("vexsort: provided scratch is too small")  # vexsort.cpp:23-25
    n = _nkeys(keys, kt)
    seed = 0 if cfg.seed is None else int(cfg.seed) & (2**64 - 1)
    has_seed = 0 if cfg.seed is None else 1
    st = SortStats()
    if _is_torch(keys):
        if not keys.is_cuda:
            raise ValueError("torch tensors must live on a CUDA device (use numpy for host arrays)")
        if not keys.is_contiguous():
            raise ValueError("keys must be contiguous")
        ws_ptr, ws_n = _ws_args(workspace, keys)
        with _device_of(keys):
            _check(lib().vxs_sort(keys.data_ptr(), n, KEY_CODE[kt], int(cfg.order), seed, has_seed,
                                  ws_ptr, ws_n, _stream_ptr(stream), ctypes.byref(st)))
        return st
    arr = keys
    if not isinstance(arr, np.ndarray) or not arr.flags.c_contiguous or not arr.flags.writeable:
        raise ValueError("host keys must be a writeable C-contiguous numpy array")
    _check(lib().vxs_sort_host(arr.ctypes.data, n, KEY_CODE[kt], int(cfg.order), seed, has_seed,
                               ctypes.byref(st)))
    return st


def sort_range(keys, lo: int, hi: int, config: Optional[SortConfig] = None, key_type: Optional[str] = None,
               workspace=None, stream=None) -> SortStats:
    """Partial sort of device keys (vxs_sort_range): afterwards
    keys[lo:hi] is sorted and holds exactly the keys of sorted ranks lo..hi-1,
    keys[:lo] precede them and keys[hi:] follow them (unordered)."""
    cfg = config or SortConfig()
    kt = infer_key_type(keys, key_type)
    _check_cuda(keys)
    n = _nkeys(keys, kt)
    ws_ptr, ws_n = _ws_args(workspace, keys)
    sd, has = _seed_args(cfg.seed)
    st = SortStats()
    with _device_of(keys):
        _check(lib().vxs_sort_range(keys.data_ptr(), n, KEY_CODE[kt], int(cfg.order), int(lo), int(hi), sd, has,
                                    ws_ptr, ws_n, _stream_ptr(stream), ctypes.byref(st)))
    return st


def nth_element(keys, k: int, config: Optional[SortConfig] = None, key_type: Optional[str] = None, **kw):
    """std::nth_element: keys[k] becomes the key of sorted rank k, smaller
    ranks before it, larger after.  Returns the stats."""
    return sort_range(keys, k, k + 1, config, key_type, **kw)


def partial_sort(keys, k: int, config: Optional[SortConfig] = None, key_type: Optional[str] = None, **kw):
    """std::partial_sort: keys[:k] becomes the k first keys in sorted order."""
    return sort_range(keys, 0, k, config, key_type, **kw)


def topk(keys, k: int, largest: bool = True, key_type: Optional[str] = None):
    """The k largest (or smallest) keys, sorted from the extreme inwards, as a
    new tensor; ``keys`` is not modified."""
    work = keys.clone()
    order = Order.kDescending if largest else Order.kAscending
    partial_sort(work, k, SortConfig(order=order), key_type)
    return work[:k].clone()


def _seed_args(seed):
    return (0, 0) if seed is None else (int(seed) & (2**64 - 1), 1)


def argsort_workspace_bytes(n: int, key_type: str, value_bytes: int = 0) -> int:
    out = ctypes.c_size_t()
    _check(lib().vxs_argsort_workspace_bytes(n, KEY_CODE[key_type], value_bytes, ctypes.byref(out)))
    return out.value


def argsort(keys, order: Order = Order.kAscending, key_type: Optional[str] = None, sorted_keys=None,
            workspace=None, stream=None, seed: Optional[int] = None):
    """Stable argsort of device keys: int64 indices such that
    keys[idx] is sorted; ties keep ascending index in both orders.  Optionally
    writes the sorted keys into ``sorted_keys``.  ``keys`` is not modified."""
    import torch
    kt = infer_key_type(keys, key_type)
    _check_cuda(keys)
    n = _nkeys(keys, kt)
    if sorted_keys is not None:
        _check_cuda(sorted_keys, "sorted_keys")
        if (sorted_keys.dtype != keys.dtype or sorted_keys.numel() != keys.numel()
                or sorted_keys.device != keys.device):
            raise ValueError("sorted_keys must match keys in dtype, size and device")
    idx = torch.empty(n, dtype=torch.int64, device=keys.device)
    ws_ptr, ws_n = _ws_args(workspace, keys)
    sd, has = _seed_args(seed)
    st = SortStats()
    with _device_of(keys):
        _check(lib().vxs_argsort(keys.data_ptr(), n, KEY_CODE[kt], int(order), idx.data_ptr(),
                                 None if sorted_keys is None else sorted_keys.data_ptr(), sd, has, ws_ptr, ws_n,
                                 _stream_ptr(stream), ctypes.byref(st)))
    return idx


def sort_pairs(keys, values, config: Optional[SortConfig] = None, key_type: Optional[str] = None,
               workspace=None, stream=None) -> SortStats:
    """Sort device keys in place and permute ``values`` (same length, any
    element size of 1/2/4/8/16 bytes per key) alongside, stably (§8 f2)."""
    cfg = config or SortConfig()
    kt = infer_key_type(keys, key_type)
    _check_cuda(keys)
    _check_cuda(values, "values")
    if values.device != keys.device:
        raise ValueError("values must live on the keys' device")
    n = _nkeys(keys, kt)
    if values.ndim == 0 or values.shape[0] != n:
        raise ValueError("values must have one row per key")
    vb = values.numel() * values.element_size() // max(n, 1) if n else values.element_size()
    ws_ptr, ws_n = _ws_args(workspace, keys)
    sd, has = _seed_args(cfg.seed)
    st = SortStats()
    with _device_of(keys):
        _check(lib().vxs_sort_pairs(keys.data_ptr(), values.data_ptr(), vb, n, KEY_CODE[kt], int(cfg.order), sd,
                                    has, ws_ptr, ws_n, _stream_ptr(stream), ctypes.byref(st)))
    return st


def sample(keys, s: int, order: Order = Order.kAscending, seed: int = 1, key_type=None, stream=None):
    """s stratified samples of device keys, as order-transformed unsigned words."""
    import torch
    kt = infer_key_type(keys, key_type)
    n = _nkeys(keys, kt)
    shape = (s, 2) if KEY_BYTES[kt] == 16 else (s,)
    wdt = {2: torch.uint16, 4: torch.uint32, 8: torch.uint64, 16: torch.uint64}[KEY_BYTES[kt]]
    out = torch.empty(shape, dtype=wdt, device=keys.device)
    with _device_of(keys):
        _check(lib().vxs_sample(keys.data_ptr(), n, KEY_CODE[kt], int(order), seed, out.data_ptr(), s,
                                _stream_ptr(stream)))
    return out


def partition(keys, splitters, order: Order = Order.kAscending, key_type=None, out=None, stream=None):
    """Multiway partition of device keys by sorted transformed-domain splitters.
    Returns (out, seg_counts[int64 tensor of nspl+1])."""
    import torch
    kt = infer_key_type(keys, key_type)
    n = _nkeys(keys, kt)
    nspl = int(splitters.shape[0])
    if out is None:
        out = torch.empty_like(keys)
    counts = torch.zeros(nspl + 1, dtype=torch.int64, device=keys.device)
    with _device_of(keys):
        _check(lib().vxs_partition(keys.data_ptr(), n, KEY_CODE[kt], int(order),
                                   splitters.data_ptr() if nspl else None, nspl, out.data_ptr(),
                                   counts.data_ptr(), None, 0, _stream_ptr(stream)))
    return out, counts


def partition_counts(keys, splitters, workspace, order: Order = Order.kAscending, key_type=None, stream=None):
    """Fused-exchange phase 1 (vxs_partition_counts): per-segment counts
    (int64 tensor of nspl+1); `workspace` (uint8 device tensor of
    workspace_bytes(n, key_type)) keeps the offsets for phase 2."""
    import torch
    kt = infer_key_type(keys, key_type)
    n = _nkeys(keys, kt)
    nspl = int(splitters.shape[0])
    counts = torch.zeros(nspl + 1, dtype=torch.int64, device=keys.device)
    with _device_of(keys):
        _check(lib().vxs_partition_counts(keys.data_ptr(), n, KEY_CODE[kt], int(order),
                                          splitters.data_ptr() if nspl else None, nspl, counts.data_ptr(),
                                          workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))
    return counts


def partition_exchange(keys, nspl: int, dst_addrs, dst_offsets, workspace, order: Order = Order.kAscending,
                       key_type=None, stream=None):
    """Fused-exchange phase 2 (vxs_partition_exchange): segment i's keys are
    stored at element dst_offsets[i] of the buffer at address dst_addrs[i]
    (int64 device tensors of nspl+1 entries; peers' receive buffers)."""
    kt = infer_key_type(keys, key_type)
    with _device_of(keys):
        _check(lib().vxs_partition_exchange(keys.data_ptr(), _nkeys(keys, kt), KEY_CODE[kt], int(order),
                                            int(nspl), dst_addrs.data_ptr(), dst_offsets.data_ptr(),
                                            workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))


class DeviceBlock:
    """An IPC-exportable device allocation (vxs_device_alloc) viewed as a
    torch tensor through __cuda_array_interface__; `handle()` is its 64-byte
    CUDA IPC handle, `DeviceBlock.open(handle, ...)` maps a peer's block."""

    def __init__(self, nbytes: int, ptr: Optional[int] = None, owned: bool = True):
        self.nbytes = int(nbytes)
        self.owned = owned
        if ptr is None:
            out = ctypes.c_void_p()
            _check(lib().vxs_device_alloc(max(self.nbytes, 16), ctypes.byref(out)))
            ptr = out.value
        self.ptr = int(ptr)

    @classmethod
    def open(cls, handle: bytes, nbytes: int) -> "DeviceBlock":
        out = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(handle), 64)
        _check(lib().vxs_ipc_open(buf, ctypes.byref(out)))
        return cls(nbytes, ptr=out.value, owned=False)

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(lib().vxs_ipc_handle(ctypes.c_void_p(self.ptr), buf))
        return buf.raw

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def tensor(self):
        import torch
        return torch.as_tensor(self, device="cuda")

    def close(self):
        if self.ptr:
            _check(lib().vxs_device_free(ctypes.c_void_p(self.ptr)) if self.owned
                   else lib().vxs_ipc_close(ctypes.c_void_p(self.ptr)))
            self.ptr = 0


def transform(keys, order: Order = Order.kAscending, inverse=False, key_type=None, stream=None):
    """Apply the order-preserving key transform in place (device keys)."""
    kt = infer_key_type(keys, key_type)
    _check_cuda(keys)
    with _device_of(keys):
        _check(lib().vxs_transform(keys.data_ptr(), _nkeys(keys, kt), KEY_CODE[kt], int(order),
                                   int(bool(inverse)), _stream_ptr(stream)))


def workspace_status(workspace, n: int, key_type: str, stream=None) -> SortStats:
    """Stats of the last sort that ran in ``workspace`` (e.g. a replayed CUDA
    graph, whose captured call could not report them); raises if the device
    scheduler flagged an error (vxs_workspace_status)."""
    st = SortStats()
    with _device_of(workspace):
        _check(lib().vxs_workspace_status(workspace.data_ptr(), n, KEY_CODE[key_type], _stream_ptr(stream),
                                          ctypes.byref(st)))
    return st


def base_case_capacity(key_type: str) -> int:
    return int(lib().vxs_base_case_capacity(KEY_CODE[key_type]))


def wide_backend_is_simd() -> bool:
    """vexsort::wide_backend_is_simd (vexsort.hpp:132): the B200 path is the
    only backend and it is data-parallel, so always True."""
    return True
