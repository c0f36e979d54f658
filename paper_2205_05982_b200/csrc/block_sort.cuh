// block_sort.cuh -- the base case: sorting one bucket of <= CAP keys per CTA.
//
// Replaces the reference's 16-row Green network + bitonic merge base case
// (network.hpp:291-404, <= 256 keys) with a B200 design sized for a CTA:
//   1. thread level: ITEMS keys per thread sorted by a bitonic network fully
//      unrolled over registers (compare-exchange = min/max on the key word);
//   2. warp level:  bitonic merge across lanes with __shfl_xor_sync, each lane
//      keeping its register rows (lanes hold "columns" of the warp's run);
//   3. block level: merge-path merges of the sorted warp runs staged in shared
//      memory, ITEMS outputs per thread per round.
// Padding uses the transformed-domain maximum, the analogue of
// TR::last_value() padding in network.hpp:300-315: padded slots sort behind
// every real key and are never written back.
#pragma once
#include "keys.cuh"

namespace vxs {

// In-register bitonic sort of N (power of two) keys, ascending.
template <typename W, int N>
__device__ __forceinline__ void thread_sort(W (&k)[N]) {
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          if ((i & size) == 0) cas(k[i], k[j]);
          else cas(k[j], k[i]);
        }
      }
    }
  }
}

// Warp-level bitonic sort of 32*N keys held as k[N] per lane, where the
// logical key index is lane*N + i (blocked).  Precondition: each lane's row
// is sorted ascending.  Merges runs of N, 2N, ... up to 32N with
// __shfl_xor_sync for the cross-lane strides and register CAS for the rest.
template <typename W, int N>
__device__ __forceinline__ void warp_bitonic_merge(W (&k)[N], int lane) {
#pragma unroll
  for (int size = 2 * N; size <= 32 * N; size <<= 1) {
    // Flip step: the second half of each size-run is compared reversed so
    // both halves can stay ascending (bitonic "merge of two sorted runs").
    {
      // Element (lane, i) pairs with its mirror in the run: lane ^ lane_mask,
      // register N-1-i.  All partners are read before any register changes.
      const int lane_mask = (size / N) - 1;
      const bool lower = (lane & ((size / N) >> 1)) == 0;
      W other[N];
#pragma unroll
      for (int i = 0; i < N; ++i) other[i] = shfl_xor(k[N - 1 - i], lane_mask);
#pragma unroll
      for (int i = 0; i < N; ++i) k[i] = keep_minmax(k[i], other[i], lower);
    }
    // Half-cleaner steps with strides size/4 ... 1 (in keys).
#pragma unroll
    for (int stride = size >> 2; stride > 0; stride >>= 1) {
      if (stride >= N) {
        const int lx = stride / N;
#pragma unroll
        const bool lower = (lane & lx) == 0;
#pragma unroll
        for (int i = 0; i < N; ++i) k[i] = keep_minmax(k[i], shfl_xor(k[i], lx), lower);
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const int j = i ^ stride;
          if (j > i) cas(k[i], k[j]);
        }
      }
    }
  }
}

// Shared-memory index padding: one spare slot per 128 bytes, so blocked
// accesses (lane stride ITEMS) and merge-path windows hit distinct banks.
template <typename W>
__host__ __device__ constexpr int pad_idx(int i) {
  return (int)((unsigned)i + (unsigned)i / (128u / (unsigned)sizeof(W)));  // i >= 0: shift, no sign fixup
}
template <typename W>
__host__ __device__ constexpr int padded_size(int n) {
  return n + n / (128 / (int)sizeof(W)) + 1;
}

// Merge-path partition: number of elements taken from A among the first
// `diag` outputs of merge(A[0..la), B[0..lb)), ties taken from A.  A and B
// are offsets into the padded smem array S.
template <typename W>
__device__ __forceinline__ int merge_path(const W* S, int a0, int la, int b0, int lb, int diag) {
  int lo = diag > lb ? diag - lb : 0;
  int hi = diag < la ? diag : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (!key_lt(S[pad_idx<W>(b0 + diag - 1 - mid)], S[pad_idx<W>(a0 + mid)])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sort THREADS*ITEMS keys.  On entry k[] holds this thread's keys (any
// arrangement); on exit k[] holds keys blocked and sorted: thread t owns
// sorted positions [t*ITEMS, (t+1)*ITEMS).  `smem` must hold
// padded_size<W>(THREADS*ITEMS) W; element i lives at smem[pad_idx<W>(i)].
// WARP_NET: merge the first 5 levels (runs up to 32*ITEMS) with the
// __shfl_xor_sync bitonic network instead of shared-memory merge path (used
// for the smallest class, where one or two warps hold the whole bucket).
template <typename W, int THREADS, int ITEMS, bool WARP_NET = false>
__device__ __forceinline__ void block_sort(W (&k)[ITEMS], W* smem) {
  const int tid = threadIdx.x;
  thread_sort<W, ITEMS>(k);
  int first_run = ITEMS;
  if constexpr (WARP_NET) {
    warp_bitonic_merge<W, ITEMS>(k, tid & 31);
    first_run = 32 * ITEMS;
  }
  constexpr int TOTAL = THREADS * ITEMS;
#pragma unroll 1
  for (int run = first_run; run < TOTAL; run <<= 1) {
    // stage blocked
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) smem[pad_idx<W>(tid * ITEMS + i)] = k[i];
    __syncthreads();
    const int group_threads = (2 * run) / ITEMS;
    const int g = tid / group_threads;
    const int r = tid - g * group_threads;
    const int a0 = g * 2 * run;
    const int b0 = a0 + run;
    const int diag = r * ITEMS;
    const int a = merge_path(smem, a0, run, b0, run, diag);
    // Branch-free serial merge: one smem load per output refills the side
    // just consumed; exhausted sides read as the maximum key.
    int ai = a, bi = diag - a;
    W va = ai < run ? smem[pad_idx<W>(a0 + ai)] : key_max<W>();
    W vb = bi < run ? smem[pad_idx<W>(b0 + bi)] : key_max<W>();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool take_a = (bi >= run) || (ai < run && !key_lt(vb, va));
      k[i] = take_a ? va : vb;
      ai += take_a ? 1 : 0;
      bi += take_a ? 0 : 1;
      if (i + 1 < ITEMS) {
        const int nidx = take_a ? ai : bi;
        const int base = take_a ? a0 : b0;
        const W nv = nidx < run ? smem[pad_idx<W>(base + nidx)] : key_max<W>();
        va = take_a ? nv : va;
        vb = take_a ? vb : nv;
      }
    }
    __syncthreads();
  }
}

}  // namespace vxs
