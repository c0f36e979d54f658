"""Synthetic inputs with BASELINE.json's shapes.

No public dataset is involved; every config is a seeded synthetic array.  A
counter-based SplitMix64 stream (vectorised numpy) replaces the reference
harness's sequential Sfc64 (harness.cpp:179-219) so 1e8-key inputs generate
in about a second; the distributions are the ones BASELINE.json names:

  c1      u64, n=1e6, uniform full range, ascending
  c2      u32 / f32, n=1e8, asc and desc; u32 uniform full range; f32 = 1e3*N(0,1)
          with 0.1% of entries replaced cyclically by -0.0, +0.0, -inf, +inf, qNaN
  c3a-f   u64, n=1e8: [0,7] / all equal / ramp / reversed ramp / organ pipe /
          ramp with 1% of positions swapped
  c4a     K128 {lo uniform, hi uniform in [0, 2^20)}, n=5e7
  c4b     KV64 {lo = original index, hi = uniform key}, n=5e7
  c5      u64 uniform / skewed floor(2^64 * u^4), n=2^30 per rank
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, start: int, n: int) -> np.ndarray:
    """Counter-based stream: x_i = mix(seed + (start+i+1)*golden)."""
    with np.errstate(over="ignore"):
        z = (np.arange(start + 1, start + n + 1, dtype=np.uint64) * _G) + np.uint64(seed & (2**64 - 1))
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _chunked(seed, n, fn, dtype, chunk=1 << 24):
    out = np.empty(n, dtype=dtype)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        out[s:e] = fn(splitmix64(seed, s, e - s))
    return out


def uniform_u64(n, seed=1):
    return _chunked(seed, n, lambda r: r, np.uint64)


def uniform_u32(n, seed=1):
    return _chunked(seed, n, lambda r: (r >> np.uint64(32)).astype(np.uint32), np.uint32)


def normal_f32_specials(n, seed=1):
    """1e3 * N(0,1) via Box-Muller on 53-bit uniforms; 0.1% specials."""
    def gen(r):
        u = ((r >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
        v = ((r * _G >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
        return (1e3 * np.sqrt(-2.0 * np.log(u)) * np.cos(2 * np.pi * v)).astype(np.float32)
    x = _chunked(seed, n, gen, np.float32)
    k = n // 1000
    if k:
        pos = (splitmix64(seed ^ 0x5EC1A15, 0, k) % np.uint64(n)).astype(np.int64)
        specials = np.array([-0.0, 0.0, -np.inf, np.inf, np.nan], dtype=np.float32)
        x[pos] = specials[np.arange(k) % 5]
    return x


def c3(variant: str, n=100_000_000, seed=1):
    if variant == "a":
        return _chunked(seed, n, lambda r: r & np.uint64(7), np.uint64)
    if variant == "b":
        return np.full(n, 0x2A, dtype=np.uint64)
    if variant == "c":
        return np.arange(n, dtype=np.uint64)
    if variant == "d":
        return np.arange(n - 1, -1, -1, dtype=np.int64).astype(np.uint64)
    if variant == "e":
        i = np.arange(n, dtype=np.int64)
        return np.where(i < n // 2, i, n - 1 - i).astype(np.uint64)
    if variant == "f":
        # n/200 disjoint random pairs swapped (~1% of positions), a permutation
        x = np.arange(n, dtype=np.uint64)
        m = n // 200
        r = splitmix64(seed, 0, 4 * m + 16) % np.uint64(n)
        _, first = np.unique(r, return_index=True)
        pos = r[np.sort(first)][: 2 * m].astype(np.int64)
        a, b = pos[0::2], pos[1::2]
        t = x[a].copy()
        x[a] = x[b]
        x[b] = t
        return x
    raise ValueError(variant)


def c4(variant: str, n=50_000_000, seed=1):
    k = np.empty((n, 2), dtype=np.uint64)
    if variant == "a":
        k[:, 0] = uniform_u64(n, seed)
        k[:, 1] = uniform_u64(n, seed ^ 0xABCDEF) >> np.uint64(44)
    elif variant == "b":
        k[:, 0] = np.arange(n, dtype=np.uint64)
        k[:, 1] = uniform_u64(n, seed)
    else:
        raise ValueError(variant)
    return k


def c5(n, rank=0, skewed=False, seed=1):
    s = seed ^ ((rank * 0x9E3779B97F4A7C15) & (2**64 - 1)) ^ 0x6A09E667F3BCC909
    if not skewed:
        return uniform_u64(n, s)

    def gen(r):
        u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        u2 = u * u
        v = (u2 * u2) * 2.0 ** 64  # explicit products: bit-identical on the device
        v = np.minimum(v, 2.0 ** 64 - 2.0 ** 11)
        return v.astype(np.uint64)
    return _chunked(s, n, gen, np.uint64)


def make(name: str, n=None, seed=1, rank=0):
    """(keys, key_type, descending) for a named workload."""
    if name == "c1":
        return uniform_u64(n or 1_000_000, seed), "u64", False
    if name in ("c2-u32-asc", "c2-u32-desc"):
        return uniform_u32(n or 100_000_000, seed), "u32", name.endswith("desc")
    if name.startswith("f32-normal"):  # (diagnostics) C2's f32 distribution, specials replaced / kept by kind
        x = normal_f32_specials(n or 100_000_000, seed)
        r = normal_f32_specials(1 << 20, seed + 99)
        keep = name.split("-")[2] if name.count("-") == 2 else ""
        bad = ~np.isfinite(x) | (x == 0)
        if keep == "nan":
            bad &= ~np.isnan(x)
        elif keep == "zero":
            bad &= x != 0
        elif keep == "inf":
            bad &= ~np.isinf(x)
        r = r[np.isfinite(r) & (r != 0)]
        x[bad] = r[: int(bad.sum())]
        return x, "f32", False
    if name in ("c2-f32-asc", "c2-f32-desc"):
        return normal_f32_specials(n or 100_000_000, seed), "f32", name.endswith("desc")
    if name.startswith("c3") and len(name) == 3:
        return c3(name[2], n or 100_000_000, seed), "u64", False
    if name == "u64-uniform":
        return uniform_u64(n or 100_000_000, seed), "u64", False
    if name == "c4a":
        return c4("a", n or 50_000_000, seed), "k128", False
    if name == "c4b":
        return c4("b", n or 50_000_000, seed), "kv64", False
    if name in ("c5", "c5-skew"):
        return c5(n or (1 << 30), rank, name == "c5-skew", seed), "u64", False
    raise ValueError(name)


# ---- device-side generation (bench only: 2^30-key configs) -----------------
# The same counter-based SplitMix64 stream computed with torch int64 ops on
# the GPU (wrapping multiplies; logical shifts via masks), so an 8 GB C5 input
# appears in milliseconds instead of a minute of numpy + an 8 GB H2D copy.
# Bit-identical to splitmix64() above.

def _i64(v: int) -> int:
    v &= 2**64 - 1
    return v - 2**64 if v >= 2**63 else v


def _shr(z, k: int):
    import torch
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64_device(seed: int, start: int, n: int, device):
    import torch
    z = torch.arange(start + 1, start + n + 1, dtype=torch.int64, device=device)
    z = z * _i64(0x9E3779B97F4A7C15) + _i64(seed)
    z = (z ^ _shr(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _shr(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _shr(z, 31)


def make_device(name: str, n=None, seed=1, rank=0, device="cuda"):
    """(device keys, key_type, descending) for the uniform / C5 workloads
    (same bits as make() for the uniform streams; the skewed stream maps the
    same uniforms through floor(2^64 * u^4) in float64 on the device)."""
    import torch
    if name == "u64-uniform":
        n = n or 100_000_000
        return splitmix64_device(seed, 0, n, device).view(torch.uint64), "u64", False
    if name in ("c5", "c5-skew"):
        n = n or (1 << 30)
        s = seed ^ ((rank * 0x9E3779B97F4A7C15) & (2**64 - 1)) ^ 0x6A09E667F3BCC909
        out = torch.empty(n, dtype=torch.int64, device=device)
        step = 1 << 26
        for b in range(0, n, step):
            e = min(n, b + step)
            r = splitmix64_device(s, b, e - b, device)
            if name == "c5-skew":
                u = _shr(r, 11).to(torch.float64) * (2.0 ** -53)
                u2 = u * u
                v = torch.clamp((u2 * u2) * 2.0 ** 64, max=2.0 ** 64 - 2.0 ** 11)
                # float64 -> uint64 through two int64 halves (v may exceed 2^63)
                hi = torch.floor(v / 2.0 ** 32)
                lo = v - hi * 2.0 ** 32
                r = (hi.to(torch.int64) << 32) | lo.to(torch.int64)
            out[b:e] = r
        return out.view(torch.uint64), "u64", False
    raise ValueError(f"no device generator for {name}")
