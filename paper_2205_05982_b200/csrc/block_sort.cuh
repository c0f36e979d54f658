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

// ---- counting-sort base case ------------------------------------------------
// Keys of a final bucket are (close to) uniform over the bucket's range
// [lo, hi]: the level above split by radix digit or by sample quantiles.  So
// the base case is a counting sort on NB linear bins (1x the capacity for
// <= 4-byte keys, 2x for 8/16-byte keys: measured) of
// (key - lo) >> shift, shift = bitlen(hi - lo) - log2 NB:
//   1. block min/max, then one fire-and-forget shared atomic per key (bin
//      counts);
//   2. exclusive scan of the bin counts (16-bit, two per word) -- thread t
//      owns BPT consecutive bins in 16-byte groups padded so LDS.128/STS.128
//      are conflict-free;
//      the same pass reduces sum(count^2) and the largest bin;
//   3. keys scattered to smem grouped by bin, each taking the next slot of
//      its bin with a returning atomic on the prefix (padding keys fill
//      [size, TOTAL));
//   4. each thread takes ITEMS consecutive positions into registers and the
//      warp runs C rounds of odd-even transposition sort, C = largest bin:
//      pairs from different bins are already ordered and never swap, so C
//      rounds sort every bin of <= C keys (about 1 min/max per key per round;
//      the thread-boundary pair goes through one shuffle each way);
//   5. bins straddling a warp boundary (<= one per boundary) are repaired by
//      insertion sort in smem; coalesced decode + store.
// Clustered items (sum c^2 > 4*size + 256, or a bin above 64 keys) return
// false before touching the output; the caller sorts them with the network.
// Equal keys are bitwise identical in the transformed domain, so the order
// among them is immaterial.
template <typename W, int THREADS, int ITEMS>
struct BinSort {
  static constexpr int kTotal = THREADS * ITEMS;
  // bins per key slot: 1 for <= 4-byte keys (their odd-even rounds are one
  // VIMNMX per key: fewer counters beat smaller bins), 2 for wider keys
  static constexpr int kNB = (sizeof(W) <= 4 || kTotal > 4096) ? kTotal : 2 * kTotal;
  static constexpr int kBPT = kNB / THREADS;  // bins per thread in the scan
  static constexpr int kNBBits = kNB == 128 ? 7 : kNB == 256 ? 8 : kNB == 512 ? 9 : kNB == 1024 ? 10 : kNB == 2048 ? 11 : kNB == 4096 ? 12 : kNB == 8192 ? 13 : 14;
  // 8/16-byte keys: bin counters are 16-bit halves packed two per word (bin
  // b: word b/2, half b&1), half the smem of 32-bit counters for the zero
  // fill, the scan and its write-back (counts and prefixes are < 2^16).
  // <= 4-byte keys keep one 32-bit counter per bin: their kernel is issue-
  // bound, and neighbouring bins sharing a word serialise their atomics.
  static constexpr bool kPacked = sizeof(W) >= 8;
  static constexpr int kBinsPerWord = kPacked ? 2 : 1;
  static constexpr int kWords = kNB / kBinsPerWord;
  static constexpr int kWPT = kBPT / kBinsPerWord;  // words per thread in the scan
  static constexpr int kEnd = kWords + kWords / 8;  // padded word of bin NB (end sentinel, low half)
  static constexpr int kDummy = kEnd + 1;           // word of bin NB + kBinsPerWord (padding keys, low half)
  static constexpr int kCnt = (kDummy + 4) & ~3;
  static constexpr int kMaxBin = 64;
  static constexpr size_t kSmem = (size_t)kTotal * sizeof(W) + (size_t)kCnt * 4;
  static_assert(kTotal < 1024 || ((1 << kNBBits) == kNB && kWPT % 4 == 0 && kBPT <= 32), "bin count");  // (class 0 never bins)
  // 4 pad words after every 32 counter words: the 16-byte groups of 8
  // threads in one LDS.128 phase land on distinct banks
  __host__ __device__ static __forceinline__ int wslot(int w) { return w + ((w >> 3) & ~3); }
  __device__ static __forceinline__ unsigned half(const unsigned* cnt, int b) {
    if constexpr (kPacked) return (cnt[wslot(b >> 1)] >> ((b & 1) << 4)) & 0xFFFFu;
    else return cnt[wslot(b)];
  }
  // smem position of key p: the 16-byte chunks of row r = p / ITEMS are
  // XOR-swizzled by r & 7 so the per-thread row loads/stores (LDS.128 /
  // STS.128, rows 64-256 B apart) are conflict-free.  Each chunk bit is
  // XORed with a strictly higher bit, so this is a bijection.
  static constexpr int kLogItems = ITEMS == 4 ? 2 : ITEMS == 8 ? 3 : ITEMS == 16 ? 4 : 5;
  static constexpr int kLogKpc = sizeof(W) == 2 ? 3 : sizeof(W) == 4 ? 2 : sizeof(W) == 8 ? 1 : 0;
  // (rows of a single chunk are consecutive chunks already: no swizzle)
  static constexpr int kNV = ITEMS * (int)sizeof(W) / 16;
  static constexpr int kSwz = kNV >= 2 ? 7 : 0;
  __device__ static __forceinline__ int swz(int p) { return p ^ (((p >> kLogItems) & kSwz) << kLogKpc); }
};

// Block min / max of k[] over all THREADS*ITEMS slots (the caller pads with
// a copy of a real key, so no per-slot validity test is needed).
template <typename W>
__device__ __forceinline__ W key_min2(const W& a, const W& b) { return key_lt(b, a) ? b : a; }
template <typename W>
__device__ __forceinline__ W key_max2(const W& a, const W& b) { return key_lt(a, b) ? b : a; }
template <>
__device__ __forceinline__ uint32_t key_min2<uint32_t>(const uint32_t& a, const uint32_t& b) { return umin(a, b); }
template <>
__device__ __forceinline__ uint32_t key_max2<uint32_t>(const uint32_t& a, const uint32_t& b) { return umax(a, b); }

template <typename W, int THREADS, int ITEMS>
__device__ __forceinline__ void block_minmax(const W (&k)[ITEMS], W& lo, W& hi, W* red_lo, W* red_hi) {
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (sizeof(W) == 8) {
    // 64-bit keys: bounds from the 32-bit high words (two VIMNMX per key);
    // only when every key shares one high word are the low words reduced.
    // [lo, hi] then brackets the keys, which is all the binning needs.
    unsigned* rl = reinterpret_cast<unsigned*>(red_lo);
    unsigned* rh = reinterpret_cast<unsigned*>(red_hi);
    auto reduce = [&](unsigned a, unsigned b, int slot, unsigned& oa, unsigned& ob) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a = umin(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = umax(b, __shfl_xor_sync(0xffffffffu, b, o));
      }
      if (lane == 0) {
        rl[2 * warp + slot] = a;
        rh[2 * warp + slot] = b;
      }
      __syncthreads();
      oa = rl[slot];
      ob = rh[slot];
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        oa = umin(oa, rl[2 * w + slot]);
        ob = umax(ob, rh[2 * w + slot]);
      }
    };
    unsigned a = (unsigned)(k[0] >> 32), b = a;
#pragma unroll
    for (int i = 1; i < ITEMS; ++i) {
      a = umin(a, (unsigned)(k[i] >> 32));
      b = umax(b, (unsigned)(k[i] >> 32));
    }
    unsigned mh, xh;
    reduce(a, b, 0, mh, xh);
    if (mh != xh) {  // block-uniform
      lo = W((unsigned long long)mh << 32);
      hi = W(((unsigned long long)xh << 32) | 0xFFFFFFFFull);
      return;
    }
    a = (unsigned)k[0];
    b = a;
#pragma unroll
    for (int i = 1; i < ITEMS; ++i) {
      a = umin(a, (unsigned)k[i]);
      b = umax(b, (unsigned)k[i]);
    }
    unsigned ml, xl;
    reduce(a, b, 1, ml, xl);
    lo = W(((unsigned long long)mh << 32) | ml);
    hi = W(((unsigned long long)mh << 32) | xl);
    return;
  }
  lo = k[0];
  hi = k[0];
#pragma unroll
  for (int i = 1; i < ITEMS; ++i) {
    lo = key_min2(lo, k[i]);
    hi = key_max2(hi, k[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = key_min2(lo, shfl_xor(lo, o));
    hi = key_max2(hi, shfl_xor(hi, o));
  }
  if (lane == 0) {
    red_lo[warp] = lo;
    red_hi[warp] = hi;
  }
  __syncthreads();
  lo = red_lo[0];
  hi = red_hi[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) {
    lo = key_min2(lo, red_lo[w]);
    hi = key_max2(hi, red_hi[w]);
  }
}

// k[]: keys striped (key i*THREADS + tid), transformed domain, padded
// beyond `size` with a copy of one of the item's keys (neutral for min/max).
// Writes the sorted, decoded item to dst and returns true, or returns false
// (nothing written, k[] untouched) when the bins are too unbalanced.
// smem: BinSort<W,THREADS,ITEMS>::kSmem bytes.
// RANK (8-byte keys, measured faster for them): the counting pass uses a
// returning atomic, so each key knows its rank inside its bin and the
// scatter pass is prefix + rank (cnt then keeps bin STARTS).  Otherwise the
// counting atomics are fire-and-forget and the scatter pass takes slots with
// a returning atomic on the prefix (cnt then ends as bin ENDS).
template <typename W, int THREADS, int ITEMS, bool FLT, bool RANK>
__device__ __forceinline__ bool bin_sort_item(const W (&k)[ITEMS], int size, W* dst, const Xf<W>& X) {
  using BS = BinSort<W, THREADS, ITEMS>;
  constexpr int TOTAL = BS::kTotal;
  constexpr int NW = THREADS / 32;
  constexpr int NV = ITEMS * (int)sizeof(W) / 16;  // uint4 per thread row
  static_assert(NV * 16 == ITEMS * (int)sizeof(W), "vector rows");
  // (the dynamic smem is named here, not through a generic pointer, so every
  // access is a plain LDS/STS off a shared-window symbol)
  extern __shared__ __align__(128) unsigned char bs_dyn[];
  W* sk = reinterpret_cast<W*>(bs_dyn);  // keys grouped by bin, then sorted
  unsigned* cnt = reinterpret_cast<unsigned*>(sk + TOTAL);
  __shared__ W red_lo[NW];
  __shared__ W red_hi[NW];
  __shared__ unsigned s_tot[NW];
  __shared__ unsigned s_sq[NW];
  __shared__ unsigned s_mx[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < BS::kCnt / 4; j += THREADS) reinterpret_cast<uint4*>(cnt)[j] = make_uint4(0, 0, 0, 0);
  W lo, hi;
  block_minmax<W, THREADS, ITEMS>(k, lo, hi, red_lo, red_hi);  // (its barrier covers cnt)
  const int bl = key_bitlen(key_sub(hi, lo));
  const int shift = bl > BS::kNBBits ? bl - BS::kNBBits : 0;
  // 64-bit keys whose high words differ: lo has a zero low word (block_minmax),
  // so (k - lo) >> shift with shift >= 32 is (hi(k) - hi(lo)) >> (shift - 32)
  // exactly -- two 32-bit ops instead of a 64-bit subtract and shift
  const bool hiword = sizeof(W) == 8 && shift >= 32;  // (block-uniform)
  auto bin_of = [&](const W& x) -> unsigned {
    if constexpr (sizeof(W) == 8) {
      if (hiword)
        return ((unsigned)((unsigned long long)x >> 32) - (unsigned)((unsigned long long)lo >> 32)) >> (shift - 32);
    }
    return key_shr32(key_sub(x, lo), shift);
  };
  // pass 1: count.  br[i] = counter word << 17 | half << 16 (| rank, RANK)
  unsigned br[ITEMS];
  unsigned sq = 0;  // sum over bins of count^2 (the cost of the rounds)
  unsigned mx = 0;  // largest bin (RANK: largest rank)
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    // (padding slots take no part in the counting: they keep their own
    // positions [size, TOTAL) in pass 2 -- no same-address atomics on a
    // dummy bin, up to a third of the slots of a half-full item)
    const bool valid = i * THREADS + tid < size;
    const unsigned b = bin_of(k[i]);
    const int w = BS::kPacked ? BS::wslot((int)(b >> 1)) : BS::wslot((int)b);
    const unsigned h = BS::kPacked ? (b & 1u) << 4 : 0u;
    br[i] = ((unsigned)w << 17) | ((h >> 4) << 16);
    if (valid) {
      if constexpr (RANK) {
        const unsigned r = (atomicAdd(&cnt[w], 1u << h) >> h) & 0xFFFFu;
        br[i] |= r;
        sq += 2u * r + 1u;  // sum over keys of 2*rank + 1 = sum over bins of count^2
        mx = umax(mx, r);
      } else {
        atomicAdd(&cnt[w], 1u << h);
      }
    }
  }
  __syncthreads();
  // exclusive scan over the bins; thread t owns bins [t*BPT, (t+1)*BPT)
  uint4* cg = reinterpret_cast<uint4*>(cnt + BS::wslot(tid * BS::kWPT));
  unsigned sum = 0;
  auto acc = [&](unsigned x) {
    if constexpr (BS::kPacked) {
      const unsigned l = x & 0xFFFFu, hh = x >> 16;
      sum += l + hh;
      if constexpr (!RANK) {
        sq += l * l + hh * hh;
        mx = umax(mx, umax(l, hh));
      }
    } else {
      sum += x;
      if constexpr (!RANK) {
        sq += x * x;
        mx = umax(mx, x);
      }
    }
  };
#pragma unroll
  for (int j = 0; j < BS::kWPT / 4; ++j) {
    const uint4 c = cg[j];
    acc(c.x);
    acc(c.y);
    acc(c.z);
    acc(c.w);
  }
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    mx = umax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 31) s_tot[warp] = incl;
  if (lane == 0) {
    s_sq[warp] = sq;
    s_mx[warp] = mx;
  }
  __syncthreads();
  unsigned base = incl - sum, tsq = 0, rounds = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    base += w < warp ? s_tot[w] : 0u;
    tsq += s_sq[w];
    rounds = umax(rounds, s_mx[w]);
  }
  if constexpr (RANK) {
    rounds += 1;  // largest rank + 1 = largest bin
  }
  // block-uniform rejection; cnt is no longer read
  if (tsq > 4u * (unsigned)size + 256u || rounds > (unsigned)BS::kMaxBin) return false;
  auto pre = [&](unsigned x) {  // count(s) -> exclusive prefix(es), same packing
    if constexpr (BS::kPacked) {
      const unsigned l = base, hh = base + (x & 0xFFFFu);
      base = hh + (x >> 16);
      return l | (hh << 16);
    } else {
      const unsigned l = base;
      base += x;
      return l;
    }
  };
#pragma unroll
  for (int j = 0; j < BS::kWPT / 4; ++j) {  // (only this thread touches these counters)
    const uint4 c = cg[j];
    uint4 o;
    o.x = pre(c.x);
    o.y = pre(c.y);
    o.z = pre(c.z);
    o.w = pre(c.w);
    cg[j] = o;
  }
  if (tid == THREADS - 1) {
    cnt[BS::kEnd] = (unsigned)size;
    cnt[BS::kDummy] = (unsigned)size;  // padding keys go to [size, TOTAL)
  }
  __syncthreads();
  // pass 2: scatter grouped by bin
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const unsigned h = ((br[i] >> 16) & 1u) << 4;
    const bool valid = i * THREADS + tid < size;
    unsigned pos = (unsigned)(i * THREADS + tid);  // (padding: its own slot, >= size)
    if (valid) {
      if constexpr (RANK) pos = ((cnt[br[i] >> 17] >> h) & 0xFFFFu) + (br[i] & 0xFFFFu);
      else pos = (atomicAdd(&cnt[br[i] >> 17], 1u << h) >> h) & 0xFFFFu;
    }
    VXS_DCHECK(pos < (unsigned)TOTAL && (valid ? pos < (unsigned)size : true), "base case: bin slot outside the item");
    sk[BS::swz((int)pos)] = valid ? k[i] : key_max<W>();
  }
  __syncthreads();
  // odd-even transposition rounds over this thread's row of ITEMS positions
  // (a warp whose 32 rows hold only padding -- the tail of a part-full item --
  // skips the rounds: the shuffles below stay inside the warp)
  const bool live = warp * 32 * ITEMS < size;  // (warp-uniform)
  W v[ITEMS];
  {
    const uint4* row = reinterpret_cast<const uint4*>(sk);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const uint4 t = row[(tid * NV + q) ^ (tid & BS::kSwz)];
      memcpy(reinterpret_cast<char*>(v) + 16 * q, &t, 16);
    }
  }
  if (rounds > 1 && live) {
#pragma unroll 1
    for (unsigned r = 0; r < rounds; r += 2) {
#pragma unroll
      for (int i = 0; i + 1 < ITEMS; i += 2) cas(v[i], v[i + 1]);
      if (r + 1 >= rounds) break;  // odd largest bin: its last round is an even one (block-uniform)
#pragma unroll
      for (int i = 1; i + 1 < ITEMS; i += 2) cas(v[i], v[i + 1]);
      const W nx = shfl_next(v[0]);
      const W pv = shfl_prev(v[ITEMS - 1]);
      if (lane < 31 && key_lt(nx, v[ITEMS - 1])) v[ITEMS - 1] = nx;
      if (lane > 0 && key_lt(v[0], pv)) v[0] = pv;
    }
  }
  if (rounds > 1 && live) {
    uint4* row = reinterpret_cast<uint4*>(sk);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      uint4 t;
      memcpy(&t, reinterpret_cast<const char*>(v) + 16 * q, 16);
      row[(tid * NV + q) ^ (tid & BS::kSwz)] = t;
    }
  }
  __syncthreads();
  if (NW > 1 && rounds > 1 && lane == 0 && warp > 0) {  // bin straddling the boundary before this warp
    const int p = warp * 32 * ITEMS;
    if (p < size) {
      const int b = (int)key_shr32(key_sub(sk[BS::swz(p)], lo), shift);
      // bin b is [start(b), start(b+1)) (RANK: cnt holds starts) or
      // [end(b-1), end(b)) (cnt holds ends)
      const int s = RANK ? (int)BS::half(cnt, b) : (b > 0 ? (int)BS::half(cnt, b - 1) : 0);
      const int e = RANK ? (int)BS::half(cnt, b + 1) : (int)BS::half(cnt, b);
      if (s < p) {
        for (int a = s + 1; a < e; ++a) {
          const W x = sk[BS::swz(a)];
          int q = a;
          while (q > s && key_lt(x, sk[BS::swz(q - 1)])) {
            sk[BS::swz(q)] = sk[BS::swz(q - 1)];
            --q;
          }
          sk[BS::swz(q)] = x;
        }
      }
    }
    __syncwarp(1u);
  }
  __syncthreads();
  // write-out: key i*THREADS + tid; its swizzle term ((i*THREADS + tid) /
  // ITEMS) & 7 is per-thread constant when THREADS/ITEMS is a multiple of 8,
  // so the loads take immediate offsets; full rounds carry no bounds test
  {
    constexpr int RPI = THREADS / ITEMS;
    const int nfull = size / THREADS;  // block-uniform
    const int trow = tid >> BS::kLogItems;
    // the swizzle only touches bits below 32*KPC <= THREADS, so
    // (i*THREADS + tid) ^ sw == i*THREADS + (tid ^ sw)
    const int e0 = tid ^ ((trow & BS::kSwz) << BS::kLogKpc);
    const int e1 = tid ^ (((RPI + trow) & BS::kSwz) << BS::kLogKpc);
    W* d = dst + tid;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i >= nfull) break;
      const int e = (RPI % 8 == 0 || (i * RPI) % 8 == 0) ? e0
                    : ((i * RPI) % 8 == RPI % 8 ? e1 : tid ^ (((i * RPI + trow) & BS::kSwz) << BS::kLogKpc));
      d[i * THREADS] = dec_x<FLT>(sk[i * THREADS + e], X);
    }
    const int idx = nfull * THREADS + tid;
    if (nfull < ITEMS && idx < size) d[nfull * THREADS] = dec_x<FLT>(sk[BS::swz(idx)], X);
  }
  __syncthreads();
  return true;
}

}  // namespace vxs
