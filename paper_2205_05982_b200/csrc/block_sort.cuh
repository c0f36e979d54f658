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
      for (int i = 0; i < N; ++i) {
        const bool lt = key_lt(other[i], k[i]);
        if (lower ? lt : !lt) k[i] = other[i];
      }
    }
    // Half-cleaner steps with strides size/4 ... 1 (in keys).
#pragma unroll
    for (int stride = size >> 2; stride > 0; stride >>= 1) {
      if (stride >= N) {
        const int lx = stride / N;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          W other = shfl_xor(k[i], lx);
          const bool lower = (lane & lx) == 0;
          const bool lt = key_lt(other, k[i]);
          if (lower ? lt : !lt) k[i] = other;
        }
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

// Merge-path partition: number of elements taken from A among the first
// `diag` outputs of merge(A[0..la), B[0..lb)), ties taken from A.
template <typename W>
__device__ __forceinline__ int merge_path(const W* A, int la, const W* B, int lb, int diag) {
  int lo = diag > lb ? diag - lb : 0;
  int hi = diag < la ? diag : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (!key_lt(B[diag - 1 - mid], A[mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Sort THREADS*ITEMS keys.  On entry k[] holds this thread's keys (any
// arrangement); on exit k[] holds keys blocked and sorted: thread t owns
// sorted positions [t*ITEMS, (t+1)*ITEMS).  `smem` must hold THREADS*ITEMS W.
template <typename W, int THREADS, int ITEMS>
__device__ __forceinline__ void block_sort(W (&k)[ITEMS], W* smem) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  thread_sort<W, ITEMS>(k);
  // Warp level via shuffles: runs of 32*ITEMS keys.
  warp_bitonic_merge<W, ITEMS>(k, lane);
  constexpr int WARP_RUN = 32 * ITEMS;
  constexpr int TOTAL = THREADS * ITEMS;
#pragma unroll 1
  for (int run = WARP_RUN; run < TOTAL; run <<= 1) {
    // stage blocked
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) smem[tid * ITEMS + i] = k[i];
    __syncthreads();
    const int group_threads = (2 * run) / ITEMS;
    const int g = tid / group_threads;
    const int r = tid - g * group_threads;
    const W* A = smem + g * 2 * run;
    const W* B = A + run;
    const int diag = r * ITEMS;
    const int a = merge_path(A, run, B, run, diag);
    int ai = a, bi = diag - a;
    W va = ai < run ? A[ai] : key_max<W>();
    W vb = bi < run ? B[bi] : key_max<W>();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool take_a = (bi >= run) || (ai < run && !key_lt(vb, va));
      if (take_a) {
        k[i] = va;
        ++ai;
        va = ai < run ? A[ai] : key_max<W>();
      } else {
        k[i] = vb;
        ++bi;
        vb = bi < run ? B[bi] : key_max<W>();
      }
    }
    __syncthreads();
  }
}

}  // namespace vxs
