// keys.cuh -- key words and the order-preserving key transforms.
//
// Every supported key type is sorted as an unsigned word of the same width
// ("transformed domain") in which plain unsigned ascending order IS the
// requested order.  The transform is fused into the first kernel that reads
// the caller's keys and its inverse into the last kernel that writes them, so
// it costs no extra HBM pass.
//
// Orders reproduced (reference /root/reference/proj):
//   integers: a<b (asc) / b<a (desc)                  traits.hpp:58-64
//   K128 {lo, hi}: hi then lo, little-endian layout   traits.hpp:24-31, 163-170
//   floats: the reference uses IEEE '<' and rejects NaN (driver.hpp:176-180);
//           we commit to the canonical total order of SURVEY.md §8c:
//           asc  -inf < ... < -0 < +0 < ... < +inf < NaN (NaNs by raw bits)
//           desc +inf > ... > +0 > -0 > ... > -inf, then NaN (raw bits asc)
//           realised as a BIJECTION onto [0, 2^W) so no key information is
//           lost and the inverse restores the exact input bits.
#pragma once
#include <cstdint>
#include <cstdio>

// Checked build (make checked -> lib/libvxsort_b200_checked.so, -DVXS_CHECKS):
// device-side bounds and consistency checks on every index the kernels
// compute (the analogue of the reference's bounds-checked scalar backend,
// vec.hpp:85-120 / config.hpp:42-52).  A failed check prints where and traps
// (the launch fails with a CUDA error).  Compiled out of the product build.
#ifdef VXS_CHECKS
#define VXS_DCHECK(cond, what)                                                                        \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("vxsort check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,        \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define VXS_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

namespace vxs {

struct U128 {  // same memory layout as vexsort::K128 {lo, hi}
  unsigned long long lo, hi;
};

// Transform codes (runtime, warp-uniform).
enum Xform : int {
  XF_NONE = 0,       // unsigned ascending; K128 ascending
  XF_NOT = 1,        // unsigned descending; K128 descending
  XF_SIGN = 2,       // signed ascending
  XF_SIGN_NOT = 3,   // signed descending
  XF_FLT_ASC = 4,    // float ascending (canonical total order)
  XF_FLT_DESC = 5,   // float descending (canonical total order)
};

template <typename W>
struct WordTraits;

template <>
struct WordTraits<uint16_t> {
  static constexpr int kBits = 16;
  static constexpr int kMant = 0;
};
template <>
struct WordTraits<uint32_t> {
  static constexpr int kBits = 32;
  static constexpr int kMant = 23;
};
template <>
struct WordTraits<unsigned long long> {
  static constexpr int kBits = 64;
  static constexpr int kMant = 52;
};
template <>
struct WordTraits<U128> {
  static constexpr int kBits = 128;
  static constexpr int kMant = 0;
};

// ---- comparisons in the transformed domain -------------------------------
__host__ __device__ __forceinline__ bool key_lt(uint16_t a, uint16_t b) { return a < b; }
__host__ __device__ __forceinline__ bool key_lt(uint32_t a, uint32_t b) { return a < b; }
__host__ __device__ __forceinline__ bool key_lt(unsigned long long a, unsigned long long b) { return a < b; }
__host__ __device__ __forceinline__ bool key_lt(const U128& a, const U128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__host__ __device__ __forceinline__ bool key_eq(uint16_t a, uint16_t b) { return a == b; }
__host__ __device__ __forceinline__ bool key_eq(uint32_t a, uint32_t b) { return a == b; }
__host__ __device__ __forceinline__ bool key_eq(unsigned long long a, unsigned long long b) { return a == b; }
__host__ __device__ __forceinline__ bool key_eq(const U128& a, const U128& b) {
  return a.hi == b.hi && a.lo == b.lo;
}

template <typename W>
__host__ __device__ __forceinline__ W key_max();
template <>
__host__ __device__ __forceinline__ uint16_t key_max<uint16_t>() { return 0xFFFFu; }
template <>
__host__ __device__ __forceinline__ uint32_t key_max<uint32_t>() { return 0xFFFFFFFFu; }
template <>
__host__ __device__ __forceinline__ unsigned long long key_max<unsigned long long>() { return ~0ull; }
template <>
__host__ __device__ __forceinline__ U128 key_max<U128>() { return U128{~0ull, ~0ull}; }

// ---- arithmetic used by the splitter lookup table --------------------------
__host__ __device__ __forceinline__ uint16_t key_sub(uint16_t a, uint16_t b) { return uint16_t(a - b); }
__host__ __device__ __forceinline__ uint32_t key_sub(uint32_t a, uint32_t b) { return a - b; }
__host__ __device__ __forceinline__ unsigned long long key_sub(unsigned long long a, unsigned long long b) {
  return a - b;
}
__host__ __device__ __forceinline__ U128 key_sub(const U128& a, const U128& b) {
  const unsigned long long lo = a.lo - b.lo;
  return U128{lo, a.hi - b.hi - (a.lo < b.lo ? 1ull : 0ull)};
}
// (d >> s) saturated to 32 bits (0xFFFFFFFF if it does not fit); s may
// exceed the word width (returns 0).  Saturation keeps every cell / digit
// map monotone for keys far above a bucket's sampled range.
__device__ __forceinline__ unsigned key_shr32(uint16_t d, int s) { return s >= 16 ? 0u : (unsigned)(d >> s); }
__device__ __forceinline__ unsigned key_shr32(uint32_t d, int s) { return s >= 32 ? 0u : (d >> s); }
__device__ __forceinline__ unsigned key_shr32(unsigned long long d, int s) {
  if (s >= 64) return 0u;
  const unsigned long long q = d >> s;
  return q > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)q;
}
__device__ __forceinline__ unsigned key_shr32(const U128& d, int s) {
  if (s >= 128) return 0u;
  unsigned long long qlo, qhi;
  if (s >= 64) {
    qlo = d.hi >> (s - 64);
    qhi = 0;
  } else if (s == 0) {
    qlo = d.lo;
    qhi = d.hi;
  } else {
    qlo = (d.lo >> s) | (d.hi << (64 - s));
    qhi = d.hi >> s;
  }
  return (qhi != 0 || qlo > 0xFFFFFFFFull) ? 0xFFFFFFFFu : (unsigned)qlo;
}
// Number of significant bits.
__device__ __forceinline__ int key_bitlen(uint16_t d) { return 32 - __clz((unsigned)d); }
__device__ __forceinline__ int key_bitlen(uint32_t d) { return 32 - __clz(d); }
__device__ __forceinline__ int key_bitlen(unsigned long long d) { return 64 - __clzll(d); }
__device__ __forceinline__ int key_bitlen(const U128& d) {
  return d.hi ? 128 - __clzll(d.hi) : 64 - __clzll(d.lo);
}
// lo + (c << s), saturating: returns false if it exceeds `hi`.
template <typename W>
__device__ __forceinline__ bool cell_start(const W& lo, const W& hi, unsigned c, int s, W& out);
template <>
__device__ __forceinline__ bool cell_start<uint16_t>(const uint16_t& lo, const uint16_t& hi, unsigned c, int s,
                                                     uint16_t& out) {
  const unsigned long long off = (unsigned long long)c << s;
  if (off > (unsigned long long)(uint16_t)(hi - lo)) return false;
  out = uint16_t(lo + off);
  return true;
}
template <>
__device__ __forceinline__ bool cell_start<uint32_t>(const uint32_t& lo, const uint32_t& hi, unsigned c, int s,
                                                     uint32_t& out) {
  const unsigned long long off = (unsigned long long)c << s;
  if (off > (unsigned long long)(hi - lo)) return false;
  out = uint32_t(lo + off);
  return true;
}
template <>
__device__ __forceinline__ bool cell_start<unsigned long long>(const unsigned long long& lo,
                                                               const unsigned long long& hi, unsigned c, int s,
                                                               unsigned long long& out) {
  const unsigned long long r = hi - lo;
  if (c == 0) {
    out = lo;
    return true;
  }
  const int cb = 32 - __clz(c);
  if (s + cb > 64) return false;
  const unsigned long long off = (unsigned long long)c << s;
  if (off > r) return false;
  out = lo + off;
  return true;
}
template <>
__device__ __forceinline__ bool cell_start<U128>(const U128& lo, const U128& hi, unsigned c, int s, U128& out) {
  const U128 r = key_sub(hi, lo);
  U128 off{0, 0};
  if (c != 0) {
    const int cb = 32 - __clz(c);
    if (s + cb > 128) return false;
    if (s >= 64) off = U128{0, (unsigned long long)c << (s - 64)};
    else if (s == 0) off = U128{c, 0};
    else off = U128{(unsigned long long)c << s, (unsigned long long)c >> (64 - s)};
    if (key_lt(r, off)) return false;
  }
  const unsigned long long l = lo.lo + off.lo;
  out = U128{l, lo.hi + off.hi + (l < lo.lo ? 1ull : 0ull)};
  return true;
}

// Conditional swap so that a <= b afterwards (a compare-exchange).
template <typename W>
__device__ __forceinline__ void cas(W& a, W& b) {
  const bool s = key_lt(b, a);
  const W lo = s ? b : a;
  const W hi = s ? a : b;
  a = lo;
  b = hi;
}

// Half-cleaner step against a partner value: keep the smaller key when
// take_min, else the larger.  For 32/16-bit words this is one predicated
// integer min/max (VIMNMX with a lane-dependent predicate), not a compare +
// select.
template <typename W>
__device__ __forceinline__ W keep_minmax(const W& k, const W& other, bool take_min) {
  const bool lt = key_lt(other, k);
  return (take_min ? lt : !lt) ? other : k;
}
template <>
__device__ __forceinline__ uint32_t keep_minmax<uint32_t>(const uint32_t& k, const uint32_t& other, bool take_min) {
  return take_min ? umin(k, other) : umax(k, other);
}
template <>
__device__ __forceinline__ uint16_t keep_minmax<uint16_t>(const uint16_t& k, const uint16_t& other, bool take_min) {
  return (uint16_t)(take_min ? umin((unsigned)k, (unsigned)other) : umax((unsigned)k, (unsigned)other));
}

// ---- transforms -----------------------------------------------------------
template <typename W>
__host__ __device__ __forceinline__ W flt_enc(W b, bool desc) {
  constexpr int B = WordTraits<W>::kBits;
  constexpr int M = WordTraits<W>::kMant;
  const W sign = W(1) << (B - 1);
  const W expm = ((W(1) << (B - 1 - M)) - 1) << M;  // exponent mask
  const W mant = (W(1) << M) - 1;                    // NaN payloads per sign
  const W nn = W(0) - W(2) * mant;                   // # non-NaN values (mod 2^B)
  // IEEE totalOrder key, shifted down by the negative-NaN slots: non-NaN keys
  // land on [0, nn), positive NaNs (raw bits ascending) on [nn, nn + mant);
  // negative NaNs keep their raw bits, which are exactly [nn + mant, 2^B) in
  // raw order.  So NaNs follow every non-NaN key, ordered by raw bits, and
  // only the non-NaN keys are reversed for descending order.  Branch-free:
  // a handful of ALU ops per key on the first read of a level.
  const W to = (b & sign) ? W(~b) : W(b ^ sign);
  const W t = b > (expm | sign) ? b : W(to - mant);
  if (!desc) return t;
  const bool is_nan = W(b & ~sign) > expm;
  return is_nan ? t : W(nn - W(1) - t);
}

template <typename W>
__host__ __device__ __forceinline__ W flt_dec(W t, bool desc) {
  constexpr int B = WordTraits<W>::kBits;
  constexpr int M = WordTraits<W>::kMant;
  const W sign = W(1) << (B - 1);
  const W expm = ((W(1) << (B - 1 - M)) - 1) << M;
  const W mant = (W(1) << M) - 1;
  const W nn = W(0) - W(2) * mant;
  if (desc && t < nn) t = W(nn - W(1) - t);  // (NaN words are not reversed)
  if (t > (expm | sign)) return t;           // negative NaNs: raw bits
  const W to = t + mant;                     // positive NaNs decode like the rest
  return (to & sign) ? W(to ^ sign) : W(~to);
}

// Integer transforms are one XOR with a per-call constant.
template <typename W>
__host__ __device__ __forceinline__ W xf_mask(int xf) {
  constexpr int B = WordTraits<W>::kBits;
  const W sign = W(1) << (B - 1);
  return xf == XF_NOT ? W(~W(0)) : xf == XF_SIGN ? sign : xf == XF_SIGN_NOT ? W(~sign) : W(0);
}

template <typename W>
__host__ __device__ __forceinline__ W enc(W b, int xf) {
  if (xf >= XF_FLT_ASC) return flt_enc<W>(b, xf == XF_FLT_DESC);
  return W(b ^ xf_mask<W>(xf));
}

template <typename W>
__host__ __device__ __forceinline__ W dec(W t, int xf) {
  if (xf >= XF_FLT_ASC) return flt_dec<W>(t, xf == XF_FLT_DESC);
  return W(t ^ xf_mask<W>(xf));
}

// A transform resolved once per kernel/tile: `flt` 0 = integer XOR with
// `mask`, 1 = float ascending, 2 = float descending.  Hot loops branch on
// `flt` OUTSIDE the loop (see with_xf) so the per-key cost is one XOR.
template <typename W>
struct Xf {
  W mask;
  int flt;
};
template <typename W>
__host__ __device__ __forceinline__ Xf<W> make_xf(int xf) {
  Xf<W> x;
  x.flt = xf == XF_FLT_ASC ? 1 : (xf == XF_FLT_DESC ? 2 : 0);
  x.mask = xf_mask<W>(xf);
  return x;
}
template <bool FLT, typename W>
__host__ __device__ __forceinline__ W enc_x(W b, const Xf<W>& x) {
  if constexpr (FLT) return flt_enc<W>(b, x.flt == 2);
  else return W(b ^ x.mask);
}
template <bool FLT, typename W>
__host__ __device__ __forceinline__ W dec_x(W t, const Xf<W>& x) {
  if constexpr (FLT) return flt_dec<W>(t, x.flt == 2);
  else return W(t ^ x.mask);
}

// 16-bit: no float type; only integer transforms.
template <>
__host__ __device__ __forceinline__ uint16_t enc<uint16_t>(uint16_t b, int xf) {
  switch (xf) {
    case XF_NOT: return uint16_t(~b);
    case XF_SIGN: return uint16_t(b ^ 0x8000u);
    case XF_SIGN_NOT: return uint16_t(~(b ^ 0x8000u));
    default: return b;
  }
}
template <>
__host__ __device__ __forceinline__ uint16_t dec<uint16_t>(uint16_t t, int xf) {
  switch (xf) {
    case XF_NOT: return uint16_t(~t);
    case XF_SIGN: return uint16_t(t ^ 0x8000u);
    case XF_SIGN_NOT: return uint16_t((~t) ^ 0x8000u);
    default: return t;
  }
}
template <>
__host__ __device__ __forceinline__ uint16_t flt_enc<uint16_t>(uint16_t b, bool) { return b; }
template <>
__host__ __device__ __forceinline__ uint16_t flt_dec<uint16_t>(uint16_t t, bool) { return t; }
template <>
__host__ __device__ __forceinline__ U128 flt_enc<U128>(U128 b, bool) { return b; }
template <>
__host__ __device__ __forceinline__ U128 flt_dec<U128>(U128 t, bool) { return t; }
template <>
__host__ __device__ __forceinline__ U128 xf_mask<U128>(int xf) {
  return xf == XF_NOT ? U128{~0ull, ~0ull} : U128{0, 0};
}
__host__ __device__ __forceinline__ U128 operator^(const U128& a, const U128& b) { return U128{a.lo ^ b.lo, a.hi ^ b.hi}; }
template <>
__host__ __device__ __forceinline__ U128 enc<U128>(U128 b, int xf) {
  return xf == XF_NOT ? U128{~b.lo, ~b.hi} : b;
}
template <>
__host__ __device__ __forceinline__ U128 dec<U128>(U128 t, int xf) {
  return xf == XF_NOT ? U128{~t.lo, ~t.hi} : t;
}

// ---- global memory access -------------------------------------------------
template <typename W>
__device__ __forceinline__ W ldg(const W* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ U128 ldg<U128>(const U128* p) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p);
  return U128{__ldg(q), __ldg(q + 1)};
}
template <typename W>
__device__ __forceinline__ W ldcs(const W* p) {
  return __ldcs(p);
}
template <>
__device__ __forceinline__ uint16_t ldcs<uint16_t>(const uint16_t* p) {
  return __ldcs(reinterpret_cast<const unsigned short*>(p));
}
template <>
__device__ __forceinline__ U128 ldcs<U128>(const U128* p) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p);
  return U128{__ldcs(q), __ldcs(q + 1)};
}

// Warp shuffle for every word type.
template <typename W>
__device__ __forceinline__ W shfl_xor(W v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
template <>
__device__ __forceinline__ uint16_t shfl_xor<uint16_t>(uint16_t v, int m) {
  return (uint16_t)__shfl_xor_sync(0xffffffffu, (unsigned)v, m);
}
template <>
__device__ __forceinline__ U128 shfl_xor<U128>(U128 v, int m) {
  return U128{__shfl_xor_sync(0xffffffffu, v.lo, m), __shfl_xor_sync(0xffffffffu, v.hi, m)};
}
// Value of lane + 1 (shfl_next) / lane - 1 (shfl_prev); the edge lanes get their own.
template <typename W>
__device__ __forceinline__ W shfl_next(W v) {
  if constexpr (sizeof(W) == 16) return W{__shfl_down_sync(0xffffffffu, v.lo, 1), __shfl_down_sync(0xffffffffu, v.hi, 1)};
  else if constexpr (sizeof(W) == 2) return (W)__shfl_down_sync(0xffffffffu, (unsigned)v, 1);
  else return __shfl_down_sync(0xffffffffu, v, 1);
}
template <typename W>
__device__ __forceinline__ W shfl_prev(W v) {
  if constexpr (sizeof(W) == 16) return W{__shfl_up_sync(0xffffffffu, v.lo, 1), __shfl_up_sync(0xffffffffu, v.hi, 1)};
  else if constexpr (sizeof(W) == 2) return (W)__shfl_up_sync(0xffffffffu, (unsigned)v, 1);
  else return __shfl_up_sync(0xffffffffu, v, 1);
}

}  // namespace vxs
