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

// Conditional swap so that a <= b afterwards (a compare-exchange).
template <typename W>
__device__ __forceinline__ void cas(W& a, W& b) {
  const bool s = key_lt(b, a);
  const W lo = s ? b : a;
  const W hi = s ? a : b;
  a = lo;
  b = hi;
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
  const bool is_nan = ((b & expm) == expm) && (b & mant) != 0;
  if (is_nan) {
    // Positive NaNs (raw bits ascending) then negative NaNs, after all
    // non-NaN keys, in both orders.
    const bool neg = (b & sign) != 0;
    const W base = neg ? (expm | sign) + 1 : expm + 1;
    return nn + (neg ? mant : W(0)) + (b - base);
  }
  const W to = (b & sign) ? W(~b) : W(b ^ sign);  // IEEE totalOrder key
  const W t = to - mant;                          // shift out the negative NaNs
  return desc ? W(nn - W(1) - t) : t;
}

template <typename W>
__host__ __device__ __forceinline__ W flt_dec(W t, bool desc) {
  constexpr int B = WordTraits<W>::kBits;
  constexpr int M = WordTraits<W>::kMant;
  const W sign = W(1) << (B - 1);
  const W expm = ((W(1) << (B - 1 - M)) - 1) << M;
  const W mant = (W(1) << M) - 1;
  const W nn = W(0) - W(2) * mant;
  if (t >= nn) {
    const W idx = t - nn;
    return idx < mant ? W(expm + 1 + idx) : W((expm | sign) + 1 + (idx - mant));
  }
  const W u = desc ? W(nn - W(1) - t) : t;
  const W to = u + mant;
  return (to & sign) ? W(to ^ sign) : W(~to);
}

template <typename W>
__host__ __device__ __forceinline__ W enc(W b, int xf) {
  constexpr int B = WordTraits<W>::kBits;
  const W sign = W(1) << (B - 1);
  switch (xf) {
    case XF_NOT: return W(~b);
    case XF_SIGN: return W(b ^ sign);
    case XF_SIGN_NOT: return W(~(b ^ sign));
    case XF_FLT_ASC: return flt_enc<W>(b, false);
    case XF_FLT_DESC: return flt_enc<W>(b, true);
    default: return b;
  }
}

template <typename W>
__host__ __device__ __forceinline__ W dec(W t, int xf) {
  constexpr int B = WordTraits<W>::kBits;
  const W sign = W(1) << (B - 1);
  switch (xf) {
    case XF_NOT: return W(~t);
    case XF_SIGN: return W(t ^ sign);
    case XF_SIGN_NOT: return W((~t) ^ sign);
    case XF_FLT_ASC: return flt_dec<W>(t, false);
    case XF_FLT_DESC: return flt_dec<W>(t, true);
    default: return t;
  }
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

}  // namespace vxs
