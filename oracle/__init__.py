"""TEST INFRASTRUCTURE ONLY -- the checker for the B200 sort, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps two C libraries
built by ``oracle/Makefile``:

* ``liboracle.so`` -- this repo's plain-C restatement of the reference sort
  path (``vexsort_oracle.c``; every function cites the reference file:line it
  follows).  It orders floats by the canonical total order.
* ``_ref/libvexsort_ref.so`` -- the unmodified reference (``/root/reference/
  proj``) compiled from its own sources plus a C shim (``ref_shim.cpp``).  It
  is built in the authoring container and travels prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# Key-type codes (same numbering as include/vxsort_b200.h).
KEY_TYPES = ["i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64", "k128"]
KEY_CODE = {k: i for i, k in enumerate(KEY_TYPES)}
NP_DTYPE = {
    "i16": np.int16, "u16": np.uint16, "i32": np.int32, "u32": np.uint32,
    "f32": np.float32, "i64": np.int64, "u64": np.uint64, "f64": np.float64,
    # K128 keys are (lo, hi) uint64 pairs: shape (n, 2).
    "k128": np.uint64,
}
# vexbench::Dist (harness.hpp:22-29)
DISTS = ["uniform", "equal", "lowentropy", "asc", "desc", "twovalue"]


class Stats(ctypes.Structure):
    """vexsort::SortStats (driver.hpp:26-32)."""

    _fields_ = [
        ("max_depth", ctypes.c_size_t),
        ("partition_calls", ctypes.c_size_t),
        ("base_case_calls", ctypes.c_size_t),
        ("keys_partitioned", ctypes.c_size_t),
        ("fallback_triggered", ctypes.c_int),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load(path):
    if not os.path.exists(path):
        raise RuntimeError(f"oracle library missing: {path} (run `make -C oracle`)")
    return ctypes.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load(os.path.join(_HERE, "liboracle.so"))
        _lib.vxo_sort.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_uint64, ctypes.POINTER(Stats)]
        _lib.vxo_generate.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_uint64]
        _lib.vxo_precedes.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        _lib.vxo_heap_sort.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
        _lib.vxo_sfc64_stream.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t]
        _lib.vxo_bounded_offset.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        _lib.vxo_bounded_offset.restype = ctypes.c_uint32
        _lib.vxo_five_draws.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p]
        _lib.vxo_depth_budget.argtypes = [ctypes.c_size_t]
        _lib.vxo_depth_budget.restype = ctypes.c_size_t
        _lib.vxo_default_seed.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        _lib.vxo_default_seed.restype = ctypes.c_uint64
        _lib.vxo_choose_pivot_u64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int]
        _lib.vxo_choose_pivot_u64.restype = ctypes.c_uint64
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libvexsort_ref.so"))


def host_has_avx512vl_dq() -> bool:
    """The reference's ISA probe (CMakeLists.txt:34-65): AVX-512VL + DQ."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return all(f" {f}" in flags for f in ("avx512f", "avx512vl", "avx512dq"))


def ref_path() -> str:
    """The reference build this host would get from its own CMake: the
    AVX-512VL/DQ variant when the CPU has it, else the AVX2 build."""
    wide = os.path.join(_HERE, "_ref", "libvexsort_ref_avx512.so")
    if os.environ.get("VXSORT_REF_ISA", "auto") != "avx2" and os.path.exists(wide) and host_has_avx512vl_dq():
        return wide
    return os.path.join(_HERE, "_ref", "libvexsort_ref.so")


def ref():
    """The real reference (compiled from /root/reference sources)."""
    global _ref
    if _ref is None:
        _ref = _load(ref_path())
        _ref.ref_isa.restype = ctypes.c_char_p
        _ref.ref_partition_bench.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64,
                                             ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double),
                                             ctypes.c_int]
        _ref.ref_sort.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Stats)]
        _ref.ref_sort_instances.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        _ref.ref_sort_with_scratch.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t]
        _ref.ref_scratch_bytes.argtypes = [ctypes.c_int]
        _ref.ref_scratch_bytes.restype = ctypes.c_size_t
        _ref.ref_depth_budget.argtypes = [ctypes.c_size_t]
        _ref.ref_depth_budget.restype = ctypes.c_size_t
        _ref.ref_sfc64_stream.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t]
        _ref.ref_five_draws.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_void_p]
        _ref.ref_choose_pivot_u64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int]
        _ref.ref_choose_pivot_u64.restype = ctypes.c_uint64
        _ref.ref_heap_sort.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
        _ref.ref_generate.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        _ref.ref_last_error.restype = ctypes.c_char_p
    return _ref


def empty_keys(key_type: str, n: int) -> np.ndarray:
    if key_type == "k128":
        return np.zeros((n, 2), dtype=np.uint64)
    return np.zeros(n, dtype=NP_DTYPE[key_type])


def n_keys(a: np.ndarray, key_type: str) -> int:
    return a.shape[0]


def sort(keys: np.ndarray, key_type: str, descending: bool = False, seed: int = 1):
    """Oracle sort (C restatement), returns (sorted copy, stats dict)."""
    out = np.ascontiguousarray(keys).copy()
    st = Stats()
    rc = lib().vxo_sort(out.ctypes.data, n_keys(out, key_type), KEY_CODE[key_type],
                        int(descending), seed, ctypes.byref(st))
    if rc != 0:
        raise ValueError(f"oracle: bad key type {key_type}")
    return out, st.as_dict()


def ref_sort(keys: np.ndarray, key_type: str, descending: bool = False, seed=None, backend=0):
    """The REAL reference's vexsort::sort on a copy; raises like the reference."""
    out = np.ascontiguousarray(keys).copy()
    st = Stats()
    rc = ref().ref_sort(out.ctypes.data, n_keys(out, key_type), KEY_CODE[key_type], int(descending),
                        0 if seed is None else seed, 0 if seed is None else 1, backend, ctypes.byref(st))
    if rc == 1:
        raise ValueError(ref().ref_last_error().decode())
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out, st.as_dict()


def generate(key_type: str, dist: str, n: int, seed: int = 1) -> np.ndarray:
    """vexbench::generate<T> restated in C (harness.cpp:179-219)."""
    out = empty_keys(key_type, n)
    rc = lib().vxo_generate(out.ctypes.data, n, KEY_CODE[key_type], DISTS.index(dist), seed)
    if rc != 0:
        raise ValueError("bad generate args")
    return out


def ref_generate(key_type: str, dist: str, n: int, seed: int = 1) -> np.ndarray:
    out = empty_keys(key_type, n)
    ref().ref_generate(out.ctypes.data, n, KEY_CODE[key_type], DISTS.index(dist), seed)
    return out


def sfc64_stream(seed: int, n: int, use_ref=False) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    (ref().ref_sfc64_stream if use_ref else lib().vxo_sfc64_stream)(seed, out.ctypes.data, n)
    return out


def canonical_sorted(keys: np.ndarray, key_type: str, descending: bool = False) -> np.ndarray:
    """Canonical order via numpy (an independent second restatement used to pin
    the C oracle): integers by value, K128 by (hi, lo), floats by the canonical
    total order of SURVEY.md §8c."""
    a = np.ascontiguousarray(keys)
    if key_type == "k128":
        idx = np.lexsort((a[:, 0], a[:, 1]))
        if descending:
            idx = idx[::-1]
        return a[idx]
    if key_type in ("f32", "f64"):
        ut = np.uint32 if key_type == "f32" else np.uint64
        bits = a.view(ut)
        nan = np.isnan(a)
        body = a[~nan]
        bb = body.view(ut)
        sign = (bb >> ut(8 * a.itemsize - 1)).astype(bool)
        # IEEE totalOrder key on non-NaN, then NaNs by raw bits.
        tkey = np.where(sign, ~bb, bb | (ut(1) << ut(8 * a.itemsize - 1)))
        o = np.argsort(tkey, kind="stable")
        if descending:
            o = o[::-1]
        nanbits = np.sort(bits[nan])
        return np.concatenate([bb[o], nanbits]).view(a.dtype)
    s = np.sort(a, kind="stable")
    return s[::-1].copy() if descending else s


def canonical_argsort(keys: np.ndarray, key_type: str, descending: bool = False) -> np.ndarray:
    """Stable argsort in the canonical order (test oracle for vxs_argsort /
    vxs_sort_pairs, SURVEY §8 f2 + §8c.3): keys by the canonical total order
    (floats: IEEE totalOrder on non-NaN, NaN last in both orders, NaNs by raw
    bits), ties by ascending original index in both orders -- i.e. the
    order of the packed (key, row id) words of PAPER.md:907-910."""
    a = np.ascontiguousarray(keys)
    n = a.shape[0]
    idx = np.arange(n, dtype=np.int64)
    nbits = 8 * a.itemsize
    ut = {2: np.uint16, 4: np.uint32, 8: np.uint64}[a.itemsize]
    u = a.view(ut)
    top = ut(1) << ut(nbits - 1)
    if key_type in ("f32", "f64"):
        isnan = np.isnan(a)
        sign = (u & top) != 0
        tk = np.where(sign, ~u, u | top).astype(ut)
        prim = np.where(isnan, u, ~tk if descending else tk).astype(ut)
        return np.lexsort((idx, prim, isnan.astype(np.uint8)))
    if key_type in ("i16", "i32", "i64"):
        u = (u ^ top).astype(ut)
    prim = ~u if descending else u
    return np.lexsort((idx, prim))
