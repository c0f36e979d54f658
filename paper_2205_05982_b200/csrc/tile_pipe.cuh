// tile_pipe.cuh -- TMA bulk-copy (cp.async.bulk) tile pipeline for the
// streaming kernels.
//
// One elected thread issues `cp.async.bulk.shared::cluster.global` for the
// NEXT tile of keys into a shared-memory stage while the CTA classifies the
// current one; completion is tracked by a transaction-count mbarrier per
// stage.  The copy covers the 16-byte-aligned middle of the tile's byte
// range; the few keys in the unaligned head/tail (< 16 bytes each side) are
// read straight from global memory by the consumer.
#pragma once
#include <cstdint>
#include <cstring>

#include "keys.cuh"

namespace vxs {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Byte geometry of one tile [addr, addr + bytes) in global memory.
struct TileSpan {
  unsigned long long base;  // addr rounded down to 16
  unsigned long long a0;    // first 16-aligned byte inside the tile
  unsigned long long a1;    // end of the last full 16-byte chunk inside the tile
};

__device__ __forceinline__ TileSpan tile_span(const void* p, unsigned long long bytes) {
  const unsigned long long addr = reinterpret_cast<unsigned long long>(p);
  TileSpan s;
  s.base = addr & ~15ull;
  s.a0 = (addr + 15) & ~15ull;
  s.a1 = (addr + bytes) & ~15ull;
  if (s.a1 < s.a0) s.a1 = s.a0;
  return s;
}

// Thread 0 only: start copying the aligned middle of the tile into `stage`
// (stage byte 0 == global byte s.base).  Always arrives on the barrier, so
// a tile with no aligned middle completes immediately.
__device__ __forceinline__ void tile_issue(const void* p, unsigned long long bytes, unsigned char* stage,
                                           unsigned long long* bar) {
  const TileSpan s = tile_span(p, bytes);
  const unsigned n = (unsigned)(s.a1 - s.a0);
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, n);
  if (n) bulk_g2s(stage + (s.a0 - s.base), reinterpret_cast<const void*>(s.a0), n, bar);
}

// Consumer read of key j of a tile whose first key is at global `g`.
template <typename W>
__device__ __forceinline__ W tile_key(const W* g, int j, const TileSpan& s, const unsigned char* stage) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(g + j);
  if (a >= s.a0 && a + sizeof(W) <= s.a1) return *reinterpret_cast<const W*>(stage + (a - s.base));
  return ldcs(g + j);
}

}  // namespace vxs

namespace vxs {

// Shared-memory key access at byte pointer p (K128 may be only 8-aligned).
template <typename W>
__device__ __forceinline__ W lds_key(const unsigned char* p, int j) {
  return reinterpret_cast<const W*>(p)[j];
}
template <>
__device__ __forceinline__ U128 lds_key<U128>(const unsigned char* p, int j) {
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(p) + 2 * j;
  return U128{q[0], q[1]};
}
template <typename W>
__device__ __forceinline__ void sts_key(unsigned char* p, int j, const W& v) {
  reinterpret_cast<W*>(p)[j] = v;
}
template <>
__device__ __forceinline__ void sts_key<U128>(unsigned char* p, int j, const U128& v) {
  unsigned long long* q = reinterpret_cast<unsigned long long*>(p) + 2 * j;
  q[0] = v.lo;
  q[1] = v.hi;
}

// After the stage's barrier completed: load the (< 16 bytes each side) head
// and tail keys the bulk copy did not cover, so the whole tile is in smem.
// Returns the smem address of key 0.  Caller must __syncthreads() before
// reading keys written by other threads.
template <typename W, int THREADS>
__device__ __forceinline__ unsigned char* tile_fixup(const W* g, int cnt, const TileSpan& s, unsigned char* stage) {
  const unsigned long long addr = reinterpret_cast<unsigned long long>(g);
  unsigned char* k0 = stage + (addr - s.base);
  long long h = (long long)((s.a0 - addr + sizeof(W) - 1) / sizeof(W));
  if (h > cnt) h = cnt;
  long long tl = s.a1 > addr ? (long long)((s.a1 - addr) / sizeof(W)) : 0;
  if (tl < h) tl = h;
  for (int j = threadIdx.x; j < h; j += THREADS) sts_key<W>(k0, j, ldcs(g + j));
  for (long long j = tl + threadIdx.x; j < cnt; j += THREADS) sts_key<W>(k0, (int)j, ldcs(g + j));
  return k0;
}

// Full-tile key access in 16-byte chunks (LDS.128): the tile's aligned middle
// [a0, a1) is nch chunks of KPC keys, thread t owning chunks q*THREADS + t
// (consecutive threads read consecutive 16 bytes: conflict-free).  A tile
// that starts off a 16-byte boundary has one chunk fewer; its head and tail
// keys (KPC in all) fill the last chunk slot of the last thread.  Item i of
// a thread is key e = i % KPC of its chunk slot q = i / KPC.  Word types of
// <= 8 bytes only (a 16-byte key need not be 16-byte aligned).
template <typename W, int THREADS>
struct TileVec {
  static constexpr int KPC = 16 / (int)sizeof(W);
  const W* g;        // key 0 of the tile in global memory (head / tail keys are read from there,
                     // so a full tile needs no tile_fixup and no barrier after the mbarrier wait)
  const uint4* mid;  // first aligned chunk = keys [h, h + nch*KPC)
  int h, nch;
  __device__ __forceinline__ TileVec(const W* g_, const TileSpan& s, const unsigned char* stage)
      : g(g_), mid(reinterpret_cast<const uint4*>(stage + (s.a0 - s.base))),
        h((int)((s.a0 - reinterpret_cast<unsigned long long>(g_)) / sizeof(W))), nch((int)((s.a1 - s.a0) >> 4)) {}
  // tile-relative key index of item i of this thread
  __device__ __forceinline__ int index(int i) const {
    const int c = (i / KPC) * THREADS + (int)threadIdx.x, e = i % KPC;
    return c < nch ? h + c * KPC + e : (e < h ? e : nch * KPC + e);
  }
  // Chunk slot q from the aligned middle only (false, out[] untouched, when
  // the slot falls past it -- only a thread's LAST slot can; `last` is a
  // compile-time value so the other slots carry no test).  The caller handles
  // the KPC head / tail keys of an unaligned tile itself (extra_index).
  __device__ __forceinline__ bool load_mid(int q, W (&out)[KPC], bool last) const {
    const int c = q * THREADS + (int)threadIdx.x;
    if (last && c >= nch) return false;
    const uint4 v = mid[c];
    memcpy(out, &v, 16);
    return true;
  }
  __device__ __forceinline__ bool unaligned() const { return h != 0; }
  // tile-relative index of head / tail key e (e < KPC) of an unaligned tile
  __device__ __forceinline__ int extra_index(int e) const { return e < h ? e : nch * KPC + e; }
  // `last`: q is the thread's last chunk slot -- the only one that can fall
  // past the aligned middle (pass a compile-time value: the other slots then
  // carry no test and no global-load path)
  __device__ __forceinline__ void load(int q, W (&out)[KPC], bool last) const {
    const int c = q * THREADS + (int)threadIdx.x;
    if (!last || c < nch) {
      const uint4 v = mid[c];
      memcpy(out, &v, 16);
    } else {
#pragma unroll
      for (int e = 0; e < KPC; ++e) out[e] = ldcs(g + (e < h ? e : nch * KPC + e));
    }
  }
};

}  // namespace vxs
