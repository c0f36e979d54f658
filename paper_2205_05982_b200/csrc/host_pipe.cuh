// host_pipe.cuh -- device kernels of the host-pointer pipeline.
//
// The reference sorts a host std::span in place (vexsort.hpp:121-129,
// sort_typed vexsort.cpp:11-49).  On the GPU that call is dominated by PCIe,
// so vxs_sort_host streams it:
//   1. the input arrives in C chunks (H2D on its own stream); each chunk is
//      sorted on the device while the next one is in flight;
//   2. k_pick_splitters draws a regular sample of the C sorted chunks and
//      picks S-1 global splitters; k_slice_bounds binary-searches each
//      splitter in each chunk -> per-(chunk, slice) bounds;
//   3. slice s = the C sub-runs between splitters s-1 and s, gathered and
//      sorted (a C-run merge), then copied back to the host (D2H on its own
//      stream) while slice s+1 is being merged.
// Only the last chunk's sort and the first slice's merge are exposed; the rest
// hides under the two PCIe transfers.  Comparisons use the same
// order-preserving transform as the sort (keys.cuh), so every key type and
// order (NaN last, -0 < +0 ascending) merges exactly as it sorts.
#pragma once
#include "block_sort.cuh"
#include "keys.cuh"

namespace vxs {

constexpr int kPipeMaxChunks = 16;
constexpr int kPipeMaxSlices = 64;
constexpr int kPipeCand = 4096;  // splitter candidates (512 threads x 8)

struct ChunkSet {
  unsigned long long off[kPipeMaxChunks + 1];  // chunk c = [off[c], off[c+1])
  int C;
};

// One CTA: kPipeCand regular samples of the concatenated sorted chunks (one
// at the centre of each of kPipeCand equal strata of the whole array, so each
// chunk is sampled in proportion to its length), block-sorted in the
// transformed domain; the S-1 splitters are the candidates at ranks
// s * kPipeCand / S.
template <typename W>
__global__ void __launch_bounds__(512) k_pick_splitters(const W* keys, ChunkSet cs, int xf, int S, W* spl) {
  constexpr int ITEMS = kPipeCand / 512;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  const unsigned long long n = cs.off[cs.C];
  W k[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const unsigned long long j = threadIdx.x * ITEMS + i;
    const unsigned long long pos = (n * (2ull * j + 1)) / (2ull * kPipeCand);
    k[i] = pos < n ? enc<W>(keys[pos], xf) : key_max<W>();
  }
  block_sort<W, 512, ITEMS>(k, sm);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = threadIdx.x * ITEMS + i;
    // splitter s (1..S-1) = candidate at rank s * kPipeCand / S
    if (j % (kPipeCand / S) == 0 && j > 0) spl[j / (kPipeCand / S) - 1] = k[i];
  }
}

// bounds[c * (S + 1) + s] = number of keys of sorted chunk c that precede
// splitter s-1 (lower bound in the transformed order); s = 0 -> 0, s = S ->
// chunk length.
template <typename W>
__global__ void k_slice_bounds(const W* keys, ChunkSet cs, int xf, int S, const W* spl,
                               unsigned long long* bounds) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cs.C * (S + 1)) return;
  const int c = t / (S + 1);
  const int s = t - c * (S + 1);
  const unsigned long long len = cs.off[c + 1] - cs.off[c];
  unsigned long long r;
  if (s == 0) {
    r = 0;
  } else if (s == S) {
    r = len;
  } else {
    const W v = spl[s - 1];
    const W* a = keys + cs.off[c];
    unsigned long long lo = 0, hi = len;
    while (lo < hi) {
      const unsigned long long mid = (lo + hi) >> 1;
      if (key_lt(enc<W>(a[mid], xf), v)) lo = mid + 1;
      else hi = mid;
    }
    r = lo;
  }
  bounds[t] = r;
}

// ---- pairwise merge rounds (slice = C sorted sub-runs) ----------------------

struct Runs {
  unsigned long long src[kPipeMaxChunks];  // run r = in[src[r], src[r] + len[r])
  unsigned long long len[kPipeMaxChunks];
  int m;                                   // number of runs
};

// Merge-path split of pair (a[0..la), b[0..lb)) at output diagonal d: the
// number of outputs taken from a (ties from a).  One warp, 32-ary search:
// each step tests 31 evenly spaced candidates with one load per lane.
template <typename W>
__device__ __forceinline__ unsigned long long merge_split_warp(const W* a, unsigned long long la, const W* b,
                                                               unsigned long long lb, unsigned long long d, int xf) {
  const int lane = threadIdx.x & 31;
  unsigned long long lo = d > lb ? d - lb : 0ull;     // answer in [lo, hi]
  unsigned long long hi = d < la ? d : la;
  while (hi > lo) {
    // predicate p(i) = a[i] <= b[d-1-i] ("a[i] is taken before the split"),
    // true on a prefix of [lo, hi); find the first false
    const unsigned long long span = hi - lo;
    const unsigned long long i = lo + (span * (unsigned long long)lane) / 32ull;
    const bool p = !key_lt(enc<W>(b[d - 1 - i], xf), enc<W>(a[i], xf));
    const unsigned bal = __ballot_sync(0xffffffffu, p);
    // candidates are non-decreasing in lane; p is monotone -> bal is a prefix
    const int t = __popc(bal);  // lanes 0..t-1 true
    if (t == 0) {
      hi = lo;  // p(lo) false -> answer lo
    } else {
      const unsigned long long last_true = lo + (span * (unsigned long long)(t - 1)) / 32ull;
      const unsigned long long first_false = t < 32 ? lo + (span * (unsigned long long)t) / 32ull : hi;
      lo = last_true + 1;
      hi = first_false;
    }
  }
  return lo;
}

// One round of pairwise merges: runs (2j, 2j+1) -> one run, written
// contiguously to out (run j's output starts at the sum of the lengths of
// runs < 2j).  An odd last run is copied.  CTA = one output tile of
// THREADS*ITEMS keys; pairs intersecting the tile are merged in turn.
template <typename W, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_merge_pairs(const W* in, Runs R, W* out, int xf) {
  constexpr int T = THREADS * ITEMS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);                 // inputs, padded
  __shared__ unsigned long long s_split[2];
  unsigned long long total = 0;
  for (int r = 0; r < R.m; ++r) total += R.len[r];
  const unsigned long long g0 = (unsigned long long)blockIdx.x * T;
  if (g0 >= total) return;
  const unsigned long long g1 = g0 + T < total ? g0 + T : total;
  unsigned long long pstart = 0;
  for (int j = 0; 2 * j < R.m; ++j) {
    const unsigned long long la = R.len[2 * j];
    const unsigned long long lb = 2 * j + 1 < R.m ? R.len[2 * j + 1] : 0ull;
    const unsigned long long pend = pstart + la + lb;
    if (pend > g0 && pstart < g1) {
      const unsigned long long d0 = (g0 > pstart ? g0 : pstart) - pstart;
      const unsigned long long d1 = (g1 < pend ? g1 : pend) - pstart;
      const W* a = in + R.src[2 * j];
      const W* b = lb ? in + R.src[2 * j + 1] : a;
      const int warp = threadIdx.x >> 5;
      if (warp < 2) {
        const unsigned long long d = warp ? d1 : d0;
        const unsigned long long sp = merge_split_warp<W>(a, la, b, lb, d, xf);
        if ((threadIdx.x & 31) == 0) s_split[warp] = sp;
      }
      __syncthreads();
      const unsigned long long a0 = s_split[0], a1 = s_split[1];
      const unsigned long long b0 = d0 - a0, b1 = d1 - a1;
      const int na = (int)(a1 - a0), nb = (int)(b1 - b0);
      for (int i = threadIdx.x; i < na; i += THREADS) sm[pad_idx<W>(i)] = enc<W>(a[a0 + i], xf);
      for (int i = threadIdx.x; i < nb; i += THREADS) sm[pad_idx<W>(na + i)] = enc<W>(b[b0 + i], xf);
      __syncthreads();
      // per thread: ITEMS outputs from local diagonal tid*ITEMS
      const int nout = na + nb;
      const int diag = threadIdx.x * ITEMS;
      W k[ITEMS];
      if (diag < nout) {
        const int ai0 = merge_path(sm, 0, na, na, nb, diag);
        int ai = ai0, bi = diag - ai0;
        W va = ai < na ? sm[pad_idx<W>(ai)] : key_max<W>();
        W vb = bi < nb ? sm[pad_idx<W>(na + bi)] : key_max<W>();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const bool take_a = (bi >= nb) || (ai < na && !key_lt(vb, va));
          k[i] = take_a ? va : vb;
          ai += take_a ? 1 : 0;
          bi += take_a ? 0 : 1;
          const int nidx = take_a ? ai : bi;
          const int lim = take_a ? na : nb;
          const int base = take_a ? 0 : na;
          const W nv = nidx < lim ? sm[pad_idx<W>(base + nidx)] : key_max<W>();
          va = take_a ? nv : va;
          vb = take_a ? vb : nv;
        }
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (diag + i < nout) sm[pad_idx<W>(diag + i)] = k[i];
      __syncthreads();
      W* o = out + pstart + d0;
      for (int i = threadIdx.x; i < nout; i += THREADS) o[i] = dec<W>(sm[pad_idx<W>(i)], xf);
      __syncthreads();
    }
    pstart = pend;
  }
}

}  // namespace vxs
