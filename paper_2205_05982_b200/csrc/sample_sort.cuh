// sample_sort.cuh -- device kernels of the multiway (ips4o-style) sample sort.
//
// Reference path being replaced (/root/reference/proj/core/include/vexsort/detail):
//   driver.hpp:123-191   Driver::recurse/sort   -> a device worklist of buckets:
//                        each LEVEL splits every large bucket up to 256 ways
//                        (k_sample, k_hist, k_plan, k_scatter); small buckets
//                        go to the per-CTA base case (k_final); buckets of
//                        equal keys are terminal (k_copy*).
//   pivot.hpp:146-172    PivotSampler::choose_pivot -> k_sample: stratified
//                        random 4-key chunks per bucket, sorted in smem, m
//                        equidistant splitters (m = 2^L - 1, L <= 8).
//   partition.hpp:197-236 Partitioner::partition (2-way, <=pivot left)
//                        -> k_hist + k_scatter: multiway classify (radix
//                        digit, table-guided splitter search or tree in
//                        smem), shared-atomic counts, block scan, smem-staged
//                        buckets, coalesced bucket writes; each key is read
//                        twice and written once per level.
//   driver.hpp:142-151   degenerate recovery via scan_min_max -> equality
//                        buckets: keys equal to a splitter land in a terminal
//                        bucket, so all-equal / low-entropy inputs finish in
//                        one level (no scan, no heapsort fallback).
//   network.hpp:372-404  base case -> k_final (block_sort.cuh bin_sort_item:
//                        counting sort + odd-even transposition rounds).
//
// Every bucket owns a fixed index range [start, start+size) for its whole
// life; keys ping-pong between the caller's array A and the temp array B in
// that range, so the final base-case/copy pass can always write into A.
#pragma once
#include <cstdint>
#include <type_traits>

#include "block_sort.cuh"
#include "keys.cuh"
#include "tile_pipe.cuh"

namespace vxs {

constexpr int kMaxL = 8;            // up to 256-way splitter-based split per level
constexpr int kMaxRadixL = 8;       // radix-certified split fan-out cap (9 measured slower: cursor contention)
constexpr int kChildStride = 512;   // child slots per split bucket (2*(2^L-1)+2 used)
constexpr int kNumSortClasses = 5;  // base-case size classes
constexpr int kListCopySmall = kNumSortClasses;
constexpr int kListCopyBig = kNumSortClasses + 1;
constexpr int kListFallback = kNumSortClasses + 2;  // items the counting sort rejected
constexpr int kNumLists = kNumSortClasses + 3;
constexpr int kMaxSamples = 4096;
constexpr unsigned long long kTileMask = (1ull << 40) - 1;

enum : unsigned { F_IN_B = 1u, F_RAW = 2u };

struct SplitDesc {
  unsigned long long start, size, tile_base;
  unsigned long long aux;  // radix mode: digit multiplier M (digit = f * M >> 32)
  unsigned flags, L;       // L: bits 0-7 fan-out exponent, bit 8 radix mode, bit 9 piecewise
                           //    radix over the splitters, bits 10 / 13 tile cost weight (tile_weight), bit 11 radix over the
                           //    bucket's known bounds (unclamped digit), bit 12 log units (with bit 9),
                           //    bits 16-23 shift, bits 24-31 distinct splitter count when < 2^L - 1
  // Cost-weighted tile order of the level (k_sample's last CTA, level_ranges):
  // the bucket's tiles start at virtual position vbase and are `weight` units
  // long each; CTA b of k_hist / k_scatter owns the tiles that start inside
  // [b * vpc, (b + 1) * vpc).  bfirst / blast: first / last CTA with a tile of
  // this bucket (rows p + bfirst .. p + blast of the offset table).
  unsigned long long vbase;
  unsigned bfirst, blast;
  // Bounds every key of the bucket lies within (transformed domain, <= 8-byte
  // words; the whole word range at the root, a radix parent's digit cell
  // below it -- k_plan).  A radix split over [klo, khi] needs no per-key
  // clamps (L bit 11, classify_mode<5/6>).
  unsigned long long klo, khi;
};
constexpr unsigned kMaxTileWeight = 3;  // (k_sample: plain radix 1, piecewise radix 2, splitter table / tree 3)
// Largest word value as u64 (bucket bounds; 16-byte words carry none).
template <typename W>
__host__ __device__ __forceinline__ unsigned long long word_max_u64() {
  if constexpr (sizeof(W) >= 8) return ~0ull;
  else return (1ull << (8 * sizeof(W))) - 1ull;
}
__host__ __device__ __forceinline__ unsigned tile_weight(unsigned L) {
  return 1u + ((L >> 10) & 1u) + 2u * ((L >> 13) & 1u);
}

struct Item {
  unsigned long long start, size;
  unsigned flags, pad;
  unsigned long long pad2;
};

struct Ctrl {
  unsigned long long split_packed[2];  // (count << 40) | tiles, per split list
  unsigned long long item_count[kNumLists];
  unsigned long long partition_calls, keys_partitioned, base_cases;
  unsigned error;
  unsigned sample_done;  // k_sample CTAs finished (the last one lays out the level's CTA tile ranges)
  unsigned modes[8][4];  // (diagnostics) buckets per level: splitter table/tree, radix, piecewise radix, ... over log units
};

// Compile-time configuration per key word: the classify/scatter tile (keys
// per tile), the CTA sizes of the two streaming kernels, and the base-case
// capacity (largest class).
template <typename W>
struct Cfg {
  static constexpr int kTile = 8192;
  static constexpr int kHistThreads = 512;
  static constexpr int kScatThreads = 512;
  static constexpr int kHistCopies = 1;
  static constexpr int kScatMinBlocks = 2;
  static constexpr int kHistMinBlocks = 2;
  static constexpr int kHistStages = 3;  // two tiles in flight while one is counted
  static constexpr int kCap = 8192;
};
template <>
struct Cfg<unsigned long long> {
  static constexpr int kTile = 4096;
  static constexpr int kHistThreads = 512;
  static constexpr int kScatThreads = 512;
  static constexpr int kHistCopies = 1;
  static constexpr int kScatMinBlocks = 2;
  static constexpr int kHistMinBlocks = 2;
#ifdef VXS_U64_HIST3
  static constexpr int kHistStages = 3;
#else
  static constexpr int kHistStages = 2;  // (3 would cost an SM's second CTA)
#endif
  static constexpr int kCap = 8192;
};
template <>
struct Cfg<uint16_t> {
  static constexpr int kTile = 8192;
  static constexpr int kHistThreads = 512;
  static constexpr int kScatThreads = 512;
  static constexpr int kHistCopies = 1;
  static constexpr int kScatMinBlocks = 1;
  static constexpr int kHistMinBlocks = 2;
  static constexpr int kHistStages = 3;
  static constexpr int kCap = 8192;
};
template <>
struct Cfg<U128> {
  static constexpr int kTile = 2048;
  static constexpr int kHistThreads = 256;
  static constexpr int kScatThreads = 256;
  static constexpr int kHistCopies = 1;
  static constexpr int kScatMinBlocks = 2;
  static constexpr int kHistMinBlocks = 4;
  static constexpr int kHistStages = 2;
  static constexpr int kCap = 4096;
};
constexpr int kStages = 2;  // TMA tile pipeline depth (k_scatter; k_hist uses Cfg::kHistStages)

// Base-case classes (THREADS, ITEMS); capacity THREADS*ITEMS.  The smallest
// class merges inside the warp with the __shfl_xor_sync network (WARP_NET).
template <int C>
struct SortClass;
template <>
struct SortClass<0> {
  static constexpr int T = 64, I = 4;
  static constexpr bool kWarpNet = true;
};
template <>
struct SortClass<1> {
  static constexpr int T = 64, I = 16;
  static constexpr bool kWarpNet = false;
};
template <>
struct SortClass<2> {
  static constexpr int T = 128, I = 16;
  static constexpr bool kWarpNet = false;
};
template <>
struct SortClass<3> {
  static constexpr int T = 256, I = 16;
  static constexpr bool kWarpNet = false;
};
template <>
struct SortClass<4> {
  static constexpr int T = 512, I = 16;
  static constexpr bool kWarpNet = false;
};

// Radix-mode buckets aim for final items of about this many keys (just
// under the 2048-key base-case class).
constexpr double kFinalTarget = 1900.0;

// Adjacent small children are grouped into one base-case item until the
// group holds at least this many keys (never more than Cap).
constexpr unsigned long long kGroupTarget = 1024;

__host__ __device__ inline int class_for(unsigned long long size) {
  if (size <= 256) return 0;
  if (size <= 1024) return 1;
  if (size <= 2048) return 2;
  if (size <= 4096) return 3;
  return 4;
}

template <typename W>
struct Params {
  W* a;  // caller's keys; final destination
  W* b;  // temp (same length)
  unsigned long long n;
  int xf;          // key transform (keys.cuh)
  int cur;         // split list read this level; children go to cur^1
  int level;
  int part_mode;   // 1: vxs_partition (caller splitters, output decoded into `out`)
  unsigned long long seed;
  Ctrl* ctrl;
  SplitDesc* split[2];
  W* splitters;                 // [cap_split][256]
  unsigned long long* counts;   // [cap_split][kChildStride] per-child totals (k_plan)
  unsigned long long* seg;      // [cap_split + grid][kChildStride] per-(bucket p, CTA b) child
                                //   counts (k_hist) -> absolute offsets (k_plan), slot p + b
  unsigned long long* childbase;  // [cap_split][kChildStride] absolute start of each child
  unsigned short* tilecnt;      // [tiles][kChildStride] per-tile child counts (k_hist -> k_scatter)
  int grid;                     // CTAs of k_hist and k_scatter (identical tile ranges)
  unsigned long long* cta_t0;   // [grid + 1] first tile of every CTA this level (level_ranges)
  int root_init;                // k_sample sets up the root bucket (level-0 launch; see k_sample)
  Item* items[kNumLists];
  unsigned long long cap_split, cap_items;
  W* out;                       // part_mode output
  // Output positions that must end up sorted (vxs_sort_range; [0, n) for a
  // full sort).  Children whose final range misses [rlo, rhi) are not split
  // or sorted further -- only moved back into A (nth_element / partial_sort).
  unsigned long long rlo, rhi;
  // vxs_partition_exchange: segment i is written to ((W*)xdst[i]) + xoff[i]
  // (a peer's receive buffer over NVLink, or a local one); 0 = off
  int xchg;
  const unsigned long long* xdst;
  const unsigned long long* xoff;
};

// Programmatic dependent launch: the host may launch the next kernel of the
// chain early (PDL attribute); every kernel first waits for its predecessor
// to complete (griddepcontrol.wait -- a no-op without PDL) and then lets its
// own successor be scheduled.  All grids here are a single resident wave,
// so early-scheduled successors only take SM slots the tail frees.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename W>
__device__ __forceinline__ int ntiles_dev(unsigned long long size) {
  constexpr int TILE = Cfg<W>::kTile;
  return (int)((size + TILE - 1) / TILE);
}

// Fan-out exponent for a bucket: children target ~Cap/4 keys, <= 256 ways.
template <typename W>
__device__ __forceinline__ int fanout_L(unsigned long long size) {
  const unsigned long long target = Cfg<W>::kCap / 4;
  int L = 1;
  while (L < kMaxL && (size >> L) > target) ++L;
  return L;
}

// ---- block helpers ---------------------------------------------------------
// Exclusive scan of v over the block (THREADS threads, one value each);
// returns the exclusive prefix, writes the total to *total.
template <int THREADS, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* total, T* scratch /*[32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = THREADS / 32;
    T s = lane < NW ? scratch[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NW) scratch[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const T warp_excl = warp == 0 ? T(0) : scratch[warp - 1];
  *total = scratch[THREADS / 32 - 1];
  const T r = warp_excl + x - v;
  __syncthreads();
  return r;
}

// Splitters of one bucket in shared memory, with a two-level lookup table
// that guides classification.  The splitter range [lo, hi] is cut into 2^21
// fine units of 2^shift codes; the top 9 bits of a key's fine unit pick a
// first-level bucket, and each bucket owns 2^k consecutive table cells (k
// from the number of splitters in it: 0 for <= 1, else ~4-8 cells per
// splitter), so clustered splitter sets (normal floats, skewed keys) get
// their resolution where the splitters are.  lut[c] = (#splitters < first key
// of cell c, same for cell c+1): a key's child index (its lower bound among
// the splitters) lies in that range, so typical keys need two table loads and
// 0-1 splitter comparisons instead of an 8-level tree walk (binary search
// inside the rare wider cell keeps any splitter set exact).
constexpr int kLutBits = 12;
constexpr int kLut = 1 << kLutBits;  // table cells
constexpr int kL1Bits = 9;           // first-level buckets
constexpr int kL1 = 1 << kL1Bits;
constexpr int kSubBits = 12;         // fine-unit bits below a first-level bucket

// Radix-mode digit of x: f = (max(x, lo) - lo) >> shift (top ~24 varying
// bits of the bucket's sample range, saturated to 32 bits for keys far above
// it), digit = min(umulhi(f, mul), m).  Monotone in x, so child ids ascend
// with the keys; a single IMAD.HI per key instead of a 64-bit product.
__device__ __forceinline__ unsigned radix_digit(uint16_t x, uint16_t lo, int shift, unsigned mul, unsigned m) {
  const unsigned xl = x > lo ? x : lo;
  return umin(__umulhi((xl - lo) >> shift, mul), m);
}
__device__ __forceinline__ unsigned radix_digit(uint32_t x, uint32_t lo, int shift, unsigned mul, unsigned m) {
  const unsigned xl = umax(x, lo);
  return umin(__umulhi((xl - lo) >> shift, mul), m);
}
__device__ __forceinline__ unsigned radix_digit(unsigned long long x, unsigned long long lo, int shift, unsigned mul,
                                                unsigned m) {
  const unsigned long long f = ((x > lo ? x : lo) - lo) >> shift;
  return umin(__umulhi((f >> 32) ? 0xFFFFFFFFu : (unsigned)f, mul), m);
}
// 64-bit keys whose bucket range spans >= 56 bits (shift >= 32): the digit
// is taken from the high words alone, hi(x) - hi(lo) (32-bit ops; never
// saturates).  It can differ from the exact (x - lo) >> shift by one unit
// before the shift where lo(x) < lo(lo) -- still monotone in x, and every
// kernel uses this same function, so the split stays consistent.
__device__ __forceinline__ unsigned radix_digit_hi(unsigned long long x, unsigned long long lo, int shift,
                                                   unsigned mul, unsigned m) {
  const unsigned xh = (unsigned)(x >> 32), lh = (unsigned)(lo >> 32);
  const unsigned f = (xh - lh) >> (shift - 32);
  return umin(__umulhi(xh < lh ? 0u : f, mul), m);
}
__device__ __forceinline__ unsigned radix_digit(const U128& x, const U128& lo, int shift, unsigned mul, unsigned m) {
  if (key_lt(x, lo)) return 0u;
  return umin(__umulhi(key_shr32(key_sub(x, lo), shift), mul), m);
}

// Digit of x in a bucket whose keys are KNOWN to lie in [lo, hi] (SplitDesc
// klo / khi) with the multiplier fitted to hi: no clamp below, none above.
template <typename W>
__device__ __forceinline__ unsigned radix_digit_unc(const W& x, const W& lo, int shift, unsigned mul) {
  return __umulhi(key_shr32(key_sub(x, lo), shift), mul);
}
// (<= 32-bit words: the shift is < 32 -- at most 8 -- so no guarded shift)
__device__ __forceinline__ unsigned radix_digit_unc(const uint32_t& x, const uint32_t& lo, int shift, unsigned mul) {
  return __umulhi((x - lo) >> shift, mul);
}
__device__ __forceinline__ unsigned radix_digit_unc(const uint16_t& x, const uint16_t& lo, int shift, unsigned mul) {
  return __umulhi((unsigned)(uint16_t)(x - lo) >> shift, mul);
}
// (64-bit words below the high-word mode: shift < 32 and (x - lo) >> shift < 2^25, no saturation)
__device__ __forceinline__ unsigned radix_digit_unc(const unsigned long long& x, const unsigned long long& lo, int shift,
                                                    unsigned mul) {
  return __umulhi((unsigned)((x - lo) >> shift), mul);
}
// Same on the high words (64-bit keys, shift >= 32; lo has a zero low word,
// so hi(x) - hi(lo) is exact).
__device__ __forceinline__ unsigned radix_digit_unc_hi(unsigned long long x, unsigned long long lo, int shift,
                                                       unsigned mul) {
  return __umulhi(((unsigned)(x >> 32) - (unsigned)(lo >> 32)) >> (shift - 32), mul);
}

template <typename W>
struct SplSmem {
  W srt[257];  // m splitters, padded with the maximum up to 255, + sentinel
  union {
    W tree[256];      // implicit BST over srt[0..254] in BFS order (tree[1..255]), tree mode
    unsigned t1[kL1];  // first-level table: cell base | k << 16, table mode
  };
  W lo;
  unsigned cmax;  // table modes: raw unit of the last splitter (keys above clamp to it)
  int lshift;     // table modes: fine unit = min(raw unit, cmax) << lshift (small ranges)
  int tdepth;     // tree mode: levels (2^tdepth - 1 >= m; shallow for few splitters)
  int shift, m, use_tree;  // use_tree: 0 table, 1 tree, 2 radix (equal-width digits),
                           //   3 radix on the high word (64-bit keys, shift >= 32), 4 piecewise
                           //   radix, 5 / 6 = 2 / 3 over the bucket's known bounds (unclamped), 7 piecewise
                           //   radix over log units (skewed integers)
  unsigned mul;  // radix mode multiplier (radix_digit)
  unsigned short lut[kLut];  // (first, end) splitter index of cell c, packed lo | hi << 8
};

// Table cell of key x (table mode).
// Fine unit (< 2^21) of key x over the splitter range [lo, hi]: raw unit
// (x - lo) >> rsh, clamped to the last splitter's, then << lsh so small ranges
// also spread over all 2^21 units.  Monotone in x.
template <typename W>
__device__ __forceinline__ unsigned fine_unit(const W& x, const W& lo, int rsh, int lsh, unsigned cmax) {
  unsigned cf = key_shr32(key_sub(x, lo), rsh);
  cf = cf < cmax ? cf : cmax;
  cf = key_lt(x, lo) ? 0u : cf;
  return cf << lsh;
}
// First key of fine unit u (false if beyond hi).
template <typename W>
__device__ __forceinline__ bool unit_start(const W& lo, const W& hi, unsigned u, int rsh, int lsh, W& out) {
  if (lsh) return cell_start<W>(lo, hi, (u + (1u << lsh) - 1) >> lsh, 0, out);
  return cell_start<W>(lo, hi, u, rsh, out);
}
// Geometry of a splitter range: rsh / lsh / cmax for fine_unit.
template <typename W>
__device__ __forceinline__ void fine_geometry(const W& range, int& rsh, int& lsh, unsigned& cmax) {
  const int bl = key_bitlen(range);
  rsh = bl > kL1Bits + kSubBits ? bl - (kL1Bits + kSubBits) : 0;
  lsh = bl < kL1Bits + kSubBits ? kL1Bits + kSubBits - bl : 0;
  cmax = key_shr32(range, rsh);
}

// Log-scale fine units (piecewise radix over skewed integers, use_tree 7):
// the unit of y = x - lo is y itself below 2^(kLogM+1), else (bit length,
// top kLogM bits below the leading one) -- a minifloat code of y, monotone
// and < 2^21 for every word type.  Power-law / log-uniform keys (e.g.
// floor(2^64 u^4)) have a smooth density per "exponent band" of this code, as
// floats have in theirs, so equal-width digits inside each first-level bucket
// balance where linear units put most splitters into one bucket.
constexpr int kLogM = 14;
template <typename W>
__device__ __forceinline__ unsigned log_unit_of(const W& y) {
  const int e = key_bitlen(y);
  if (e <= kLogM + 1) return key_shr32(y, 0);
  return ((unsigned)(e - kLogM) << kLogM) | (key_shr32(y, e - 1 - kLogM) & ((1u << kLogM) - 1u));
}
template <typename W>
__device__ __forceinline__ unsigned fine_unit_log(const W& x, const W& lo, unsigned cmax) {
  const unsigned cf = log_unit_of(key_sub(x, lo));
  return key_lt(x, lo) ? 0u : (cf < cmax ? cf : cmax);
}
// First key of log unit u (false if beyond hi).
template <typename W>
__device__ __forceinline__ bool unit_start_log(const W& lo, const W& hi, unsigned u, W& out) {
  if (u < (2u << kLogM)) return cell_start<W>(lo, hi, u, 0, out);
  return cell_start<W>(lo, hi, (1u << kLogM) | (u & ((1u << kLogM) - 1u)), (int)(u >> kLogM) - 1, out);
}

// (first, end) splitter pair of key x's table cell.  A first-level bucket
// with a single cell (<= 1 splitter: the common case for smooth splitter
// sets) keeps its pair in t1 itself (bit 20 set): one table load per key.
constexpr unsigned kT1Direct = 1u << 20;
template <typename W>
__device__ __forceinline__ unsigned lut_pair(const W& x, const SplSmem<W>& S) {
  const unsigned cf = fine_unit(x, S.lo, S.shift, S.lshift, S.cmax);
  const unsigned t = S.t1[cf >> kSubBits];
  if (t & kT1Direct) return t & 0xFFFFu;
  return S.lut[(t & 0xFFFFu) + ((cf & ((1u << kSubBits) - 1)) >> (kSubBits - (t >> 16)))];
}

template <typename W>
__device__ __forceinline__ int lower_bound_smem(const W* srt, int lo, int hi, const W& x) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key_lt(srt[mid], x)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Piecewise-radix digit (use_tree 4): first-level bucket c1 of x holds n
// splitters, t1[c1] = (#splitters before the bucket) | n << 16, and the
// bucket is cut into n equal-width digits.  Digits ascend with the keys (an
// empty bucket's keys join the next bucket's first digit); every digit spans
// about one quantile of the sample when the density is smooth inside a
// bucket (normal floats: a bucket is at most one exponent band), so children
// stay balanced with one near-broadcast table load per key and no splitter
// compare.  Digits lie in [0, m).
template <bool LOG = false, typename W>
__device__ __forceinline__ unsigned pw_digit(const W& x, const W& lo, int rsh, int lsh, unsigned cmax,
                                             const unsigned* t1) {
  const unsigned cf = LOG ? fine_unit_log(x, lo, cmax) : fine_unit(x, lo, rsh, lsh, cmax);
  const unsigned t = t1[cf >> kSubBits];
  return (t & 0xFFFFu) + (((cf & ((1u << kSubBits) - 1)) * (t >> 16)) >> kSubBits);
}

// First-level table over m sorted splitters srt[]: t1[j] = #splitters below
// bucket j | #splitters inside it << 16.  Thread 0 has set lo / shift / cmax
// (and a barrier followed).  Returns the bucket count.
template <typename W>
__device__ __forceinline__ int build_t1(const W* srt, int m, const W& lo, const W& hi, int rsh, int lsh,
                                        unsigned cmax, unsigned* t1, bool logu = false) {
  const int n1 = (int)((cmax << lsh) >> kSubBits) + 1;
  auto ustart = [&](unsigned u, W& out) {
    return logu ? unit_start_log<W>(lo, hi, u, out) : unit_start<W>(lo, hi, u, rsh, lsh, out);
  };
  for (int j = threadIdx.x; j < n1; j += blockDim.x) {
    W s0, s1;
    const unsigned f0 = ustart((unsigned)j << kSubBits, s0) ? lower_bound_smem(srt, 0, m, s0) : m;
    const unsigned f1 = (j + 1 < n1 && ustart((unsigned)(j + 1) << kSubBits, s1)) ? lower_bound_smem(srt, 0, m, s1)
                                                                                  : (unsigned)m;
    t1[j] = f0 | ((f1 - f0) << 16);
  }
  __syncthreads();
  return n1;
}

// Exclusive scan in place over v[0..count), count <= kL1, by the whole CTA
// (two values per thread at most); returns the total to every thread.
__device__ __forceinline__ unsigned block_scan_small(unsigned* v, int count, unsigned* warp_tot /*[32]*/) {
  const int per = (count + (int)blockDim.x - 1) / (int)blockDim.x;  // 1 or 2
  const int j0 = threadIdx.x * per;
  unsigned a = j0 < count ? v[j0] : 0u;
  unsigned b = (per > 1 && j0 + 1 < count) ? v[j0 + 1] : 0u;
  const unsigned mine = a + b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  unsigned before = 0, total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    before += w < warp ? warp_tot[w] : 0u;
    total += warp_tot[w];
  }
  const unsigned ex = before + incl - mine;
  if (j0 < count) v[j0] = ex;
  if (per > 1 && j0 + 1 < count) v[j0 + 1] = ex + a;
  __syncthreads();
  return total;
}

// Shared-histogram slot of child c: even children (key ranges; the only
// ids radix mode produces) fill [0, 256), odd ones (equality buckets)
// [256, 512), so the hot counters are consecutive words over all 32 banks
// instead of every other bank.
__host__ __device__ __forceinline__ int hslot(int c) { return (c >> 1) | ((c & 1) << 8); }
__host__ __device__ __forceinline__ int unslot(int s) { return ((s & 255) << 1) | (s >> 8); }

// Children of a bucket with m splitters: ids 0..2m+1 (the last one is the
// equality bucket of the maximum key, used when the tree pads with it).
__host__ __device__ __forceinline__ int num_children(int L) { return 2 * ((1 << L) - 1) + 2; }

// Implicit BST of depth D over srt[0 .. 2^D - 1) (BFS order, tree[1 ..
// 2^D)); the padding with the maximum key keeps lower-bound semantics.
template <typename W>
__device__ __forceinline__ void build_tree(SplSmem<W>& S, int D) {
  for (int j = threadIdx.x + 1; j < (1 << D); j += blockDim.x) {
    const int d = 31 - __clz(j);
    const int q = j - (1 << d);
    S.tree[j] = S.srt[((2 * q + 1) << (D - 1 - d)) - 1];
  }
  if (threadIdx.x == 0) S.tdepth = D;
}

// Load a bucket's splitters, build the two-level lookup table, and pick the
// classifier: the table when no cell holds more than 2 splitters for more
// than a few splitters, else the 8-level tree (extremely clustered codes).
template <typename W>
__device__ __forceinline__ void load_splitters(const W* g_srt, unsigned lraw, SplSmem<W>& S,
                                               unsigned long long aux = 0) {
  __shared__ int s_wide;
  __shared__ unsigned s_tot[32];
  const int L = (int)(lraw & 0xFFu);
  const int m = (lraw >> 24) ? (int)(lraw >> 24) : (1 << L) - 1;  // deduplicated count, if set
  if (lraw & 0x100u) {  // radix mode: digit = (x - lo) >> shift, no table
    __syncthreads();
    if (threadIdx.x == 0) {
      S.lo = g_srt[0];
      S.shift = (int)((lraw >> 16) & 0xFFu);
      S.lshift = 0;
      S.m = m;
      S.mul = (unsigned)aux;
      S.use_tree = (sizeof(W) == 8 && S.shift >= 32) ? 3 : 2;
      if (lraw & 0x800u) S.use_tree += 3;  // known bounds: unclamped digit
    }
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < 255; i += blockDim.x) S.srt[i] = i < m ? g_srt[i] : key_max<W>();
  if (threadIdx.x == 0) {
    S.srt[255] = key_max<W>();
    S.srt[256] = key_max<W>();
    s_wide = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S.lo = S.srt[0];
    fine_geometry(key_sub(S.srt[m - 1], S.lo), S.shift, S.lshift, S.cmax);
    S.m = m;
  }
  __syncthreads();
  if (m <= 15) {  // few splitters (low-entropy keys): a shallow tree, <= 4 near-broadcast loads
    build_tree(S, 32 - __clz((unsigned)m));
    if (threadIdx.x == 0) S.use_tree = 1;
    __syncthreads();
    return;
  }
  const W lo = S.lo, hi = S.srt[m - 1];
  if ((lraw & 0x1200u) == 0x1200u) {  // piecewise radix over log units (certified by k_sample)
    __syncthreads();
    if (threadIdx.x == 0) {
      S.shift = 0;
      S.lshift = 0;
      S.cmax = log_unit_of(key_sub(hi, lo));
      S.use_tree = 7;
    }
    __syncthreads();
    build_t1(S.srt, m, lo, hi, 0, 0, S.cmax, S.t1, true);
    return;
  }
  const int sh = S.shift, lsh = S.lshift;
  const int n1 = build_t1(S.srt, m, lo, hi, sh, lsh, S.cmax, S.t1);
  if (lraw & 0x200u) {  // piecewise radix (certified by k_sample): t1 is the whole classifier
    if (threadIdx.x == 0) S.use_tree = 4;
    __syncthreads();
    return;
  }
  // two-level table: splitters per bucket -> k (cells 2^k) -> cell bases
  for (int j = threadIdx.x; j < n1; j += blockDim.x) {
    const unsigned c = S.t1[j] >> 16;  // splitters inside bucket j
    const unsigned k = c <= 1 ? 0u : umin(32u - __clz(c - 1) + 2u, (unsigned)kSubBits);
    S.t1[j] = 1u << k;  // (cells; at most 8 per splitter + 1 per bucket: <= 2552 in all)
    S.lut[j] = (unsigned short)k;  // (k parked in the table until the cells are built)
  }
  __syncthreads();
  const unsigned ncell = block_scan_small(S.t1, n1, s_tot);
  for (int j = threadIdx.x; j < n1; j += blockDim.x) S.t1[j] |= (unsigned)S.lut[j] << 16;
  __syncthreads();
  // cells: first splitter index of each cell (low byte), then pack (first, end)
  for (int c = threadIdx.x; c < (int)ncell; c += blockDim.x) {
    int a = 0, b = n1 - 1;  // bucket owning cell c: the last j with base(j) <= c
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if ((S.t1[mid] & 0xFFFFu) <= (unsigned)c) a = mid;
      else b = mid - 1;
    }
    const unsigned t = S.t1[a];
    const unsigned u = ((unsigned)a << kSubBits) + (((unsigned)c - (t & 0xFFFFu)) << (kSubBits - (t >> 16)));
    W cs;
    S.lut[c] = (unsigned short)(unit_start<W>(lo, hi, u, sh, lsh, cs) ? lower_bound_smem(S.srt, 0, m, cs) : m);
  }
  if (threadIdx.x == 0) S.lut[ncell] = (unsigned short)m;  // (ncell <= 2552 < kLut: sentinel slot)
  __syncthreads();
  int wide = 0;
  for (int c0 = 0; c0 < (int)ncell; c0 += blockDim.x) {  // (block-uniform trip count)
    const int c = c0 + threadIdx.x;
    const unsigned e = c < (int)ncell ? S.lut[c + 1] & 0xFFu : 0u;
    __syncthreads();
    if (c < (int)ncell) {
      const unsigned f = S.lut[c] & 0xFFu;
      S.lut[c] = (unsigned short)(f | (e << 8));
      const int occ = (int)e - (int)f;
      if (occ > 2) wide += occ;
    }
    __syncthreads();
  }
  // single-cell buckets: their (first, end) pair goes straight into t1
  for (int j = threadIdx.x; j < n1; j += blockDim.x)
    if ((S.t1[j] >> 16) == 0) S.t1[j] = (unsigned)S.lut[S.t1[j] & 0xFFFFu] | kT1Direct;
  if (wide) atomicAdd(&s_wide, wide);
  __syncthreads();
  const bool tree = s_wide > 8;  // (block-uniform)
  if (tree) build_tree(S, 8);    // the table is too coarse: full tree instead (overwrites t1)
  if (threadIdx.x == 0) S.use_tree = tree ? 1 : 0;
  __syncthreads();
}

// Child id of key x: i = #splitters < x (lower bound); an equal splitter sends
// x to the equality bucket 2i+1, else the normal bucket 2i.  Ids ascend in key
// order: normal_0 < eq_0 < normal_1 < ... < normal_m.
//
// Table path: keys below the first splitter use cell 0, keys above the last
// use the last cell; the answer always lies in [first(c), end(c)], so one or
// two splitter compares finish any cell holding <= 2 splitters; wider cells
// return -1 for classify_slow.
// Tree path: branch-free 8-level walk over the padded implicit BST (padding
// with the maximum key keeps lower-bound semantics; the maximum key itself
// lands in equality bucket 2m+1).
template <int MODE, typename W>
__device__ __forceinline__ int classify_mode(const W& x, const SplSmem<W>& S) {
  if constexpr (MODE == 7) {
    return 2 * (int)pw_digit<true>(x, S.lo, 0, 0, S.cmax, S.t1);
  } else if constexpr (MODE == 6 && sizeof(W) == 8) {
    return 2 * (int)radix_digit_unc_hi(x, S.lo, S.shift, S.mul);
  } else if constexpr (MODE >= 5) {
    return 2 * (int)radix_digit_unc(x, S.lo, S.shift, S.mul);
  } else if constexpr (MODE == 4) {
    return 2 * (int)pw_digit(x, S.lo, S.shift, S.lshift, S.cmax, S.t1);
  } else if constexpr (MODE == 3 && sizeof(W) == 8) {
    return 2 * (int)radix_digit_hi(x, S.lo, S.shift, S.mul, (unsigned)S.m);
  } else if constexpr (MODE >= 2) {
    // equal-width digits over the sample range (the sample certified them
    // balanced); keys below/above the range clamp to the first/last digit
    return 2 * (int)radix_digit(x, S.lo, S.shift, S.mul, (unsigned)S.m);
  } else if constexpr (MODE == 1) {
    const int D = S.tdepth;  // (block-uniform)
    int j = 1;
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < D) j = 2 * j + (key_lt(S.tree[j], x) ? 1 : 0);
    const int i = j - (1 << D);
    const int eq = (i < (1 << D) - 1 && key_eq(S.srt[i], x)) ? 1 : 0;
    return 2 * i + eq;
  } else {
    // Cell c holds splitters [i, e).  e == i: answer i, no equality possible
    // (srt[i] >= end of cell > x).  e == i+1: one compare with srt[i] gives
    // the answer and the equality bit.  Wider cells take the slow path.
    const unsigned pr = lut_pair(x, S);
    const int i = (int)(pr & 0xFFu);
    const int e = (int)(pr >> 8);
    const W sp = S.srt[i];
    const bool has = e > i;
    const bool lt = has && key_lt(sp, x);
    bool eq = has && !lt && key_eq(sp, x);
    int r = i + (lt ? 1 : 0);
    if (e - i == 2 && lt) {  // two splitters in the cell (e.g. -0.0 / +0.0, adjacent codes): one more compare
      const W sp1 = S.srt[i + 1];
      const bool lt1 = key_lt(sp1, x);
      r += lt1 ? 1 : 0;
      eq = !lt1 && key_eq(sp1, x);
    }
    return e - i > 2 ? -1 : 2 * r + (eq ? 1 : 0);
  }
}

// Radix-mode classifier parameters hoisted into registers (the write-out
// loop of k_scatter recomputes child ids instead of staging them in smem).
template <typename W>
struct RadixReg {
  W lo;
  int shift;
  unsigned m;
  unsigned mul;
  __device__ __forceinline__ explicit RadixReg(const SplSmem<W>& S)
      : lo(S.lo), shift(S.shift), m((unsigned)S.m), mul(S.mul) {}
  // shared-histogram slot of x's child (= its digit: radix children are even, hslot(2d) = d);
  // UNC: the bucket's known-bounds digit (modes 5 / 6)
  template <bool UNC>
  __device__ __forceinline__ int slot(const W& x) const {
    if constexpr (sizeof(W) == 8) {  // (high-word modes 3 / 6 only)
      if constexpr (UNC) return (int)radix_digit_unc_hi(x, lo, shift, mul);
      else return (int)radix_digit_hi(x, lo, shift, mul, m);
    } else {
      if constexpr (UNC) return (int)radix_digit_unc(x, lo, shift, mul);
      else return (int)radix_digit(x, lo, shift, mul, m);
    }
  }
};

template <typename W>
__device__ __forceinline__ int classify_fast(const W& x, const SplSmem<W>& S) {
  return S.use_tree == 7 ? classify_mode<7>(x, S)
         : S.use_tree == 6 ? classify_mode<6>(x, S)
         : S.use_tree == 5 ? classify_mode<5>(x, S)
         : S.use_tree == 4 ? classify_mode<4>(x, S)
         : S.use_tree == 3 ? classify_mode<3>(x, S)
                        : S.use_tree == 2 ? classify_mode<2>(x, S)
                                          : (S.use_tree ? classify_mode<1>(x, S) : classify_mode<0>(x, S));
}

template <typename W>
__device__ __noinline__ int classify_slow(const W& x, const SplSmem<W>& S) {
  const unsigned pr = lut_pair(x, S);
  const int i = lower_bound_smem(S.srt, (int)(pr & 0xFFu), (int)(pr >> 8), x);
  const int eq = (i < S.m && key_eq(S.srt[i], x)) ? 1 : 0;
  return 2 * i + eq;
}

template <typename W>
__device__ __forceinline__ int classify(const W& x, const SplSmem<W>& S) {
  const int b = classify_fast(x, S);
  return b >= 0 ? b : classify_slow(x, S);
}

// Find the split bucket owning global tile t (binary search on tile_base).
__device__ __forceinline__ int find_bucket(const SplitDesc* list, int nb, unsigned long long t) {
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (list[mid].tile_base <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Cost-weighted CTA tile ranges of one level (run by ONE CTA after every
// bucket's classifier is known).  A tile of a radix bucket costs 1 unit, a
// tile of a splitter-table / tree / piecewise bucket 2 (measured ~2x per key
// in k_hist): with equal tile counts per CTA the CTAs inside such buckets set
// the pace of the whole level (normal floats: 4% of the level-1 buckets made
// k_hist 2x and k_scatter 1.4x slower).  Ranges stay contiguous and ordered,
// so the (bucket p, CTA b) offset rows p + b are still unique along the tile
// order.  Writes SplitDesc::vbase / bfirst / blast and P.cta_t0[0 .. grid].
template <typename W>
__device__ __forceinline__ void level_ranges(const Params<W>& P, SplitDesc* list, int nb, unsigned long long T) {
  __shared__ unsigned long long lr_scan[32];
  __shared__ unsigned long long lr_carry;
  constexpr int kVbCache = 1024;  // vbase of the first buckets cached for the searches below
  __shared__ unsigned long long lr_vb[kVbCache];
  const int THREADS = (int)blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = THREADS >> 5;
  const unsigned long long G = (unsigned long long)P.grid;
  if (nb == 1) {  // (root level, vxs_partition: closed form, no scan, no search)
    const unsigned long long w = tile_weight(__ldcg(&list[0].L));
    unsigned long long vpc = (T * w + G - 1) / G;
    if (vpc < w) vpc = w;  // (see below)
    if (threadIdx.x == 0) {
      list[0].vbase = 0;
      list[0].bfirst = 0;
      list[0].blast = (unsigned)(T ? (T - 1) * w / vpc : 0);
    }
    for (unsigned long long b = threadIdx.x; b <= G; b += THREADS) {
      const unsigned long long i = (b * vpc + w - 1) / w;
      P.cta_t0[b] = i < T ? i : T;
    }
    return;
  }
  if (threadIdx.x == 0) lr_carry = 0;
  __syncthreads();
  for (int p0 = 0; p0 < nb; p0 += THREADS) {  // exclusive scan of ntiles * weight over the buckets
    const int q = p0 + (int)threadIdx.x;
    unsigned long long v = 0;
    if (q < nb) v = (unsigned long long)ntiles_dev<W>(__ldcg(&list[q].size)) * tile_weight(__ldcg(&list[q].L));
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) lr_scan[warp] = x;
    __syncthreads();
    unsigned long long before = lr_carry, all = 0;
    for (int w2 = 0; w2 < nw; ++w2) {
      before += w2 < warp ? lr_scan[w2] : 0ull;
      all += lr_scan[w2];
    }
    if (q < nb) {
      list[q].vbase = before + x - v;
      if (q < kVbCache) lr_vb[q] = before + x - v;
    }
    __syncthreads();
    if (threadIdx.x == 0) lr_carry += all;
    __syncthreads();
  }
  const unsigned long long V = lr_carry;
  // vpc >= the largest weight: every CTA between a bucket's first and last
  // then owns at least one of its tiles (k_plan / k_segscan_root read the
  // offset rows of ALL those CTAs)
  unsigned long long vpc = (V + G - 1) / G;
  if (vpc < kMaxTileWeight) vpc = kMaxTileWeight;
  for (int q = threadIdx.x; q < nb; q += THREADS) {
    const unsigned long long vb = list[q].vbase;
    const unsigned long long nt = (unsigned long long)ntiles_dev<W>(__ldcg(&list[q].size));
    list[q].bfirst = (unsigned)(vb / vpc);
    list[q].blast = (unsigned)((vb + (nt - 1) * tile_weight(__ldcg(&list[q].L))) / vpc);
  }
  // first tile of CTA b = the first tile whose virtual start is >= b * vpc
  for (unsigned long long b = threadIdx.x; b <= G; b += THREADS) {
    const unsigned long long x = b * vpc;
    unsigned long long t = T;
    if (nb > 0 && x < V) {
      int lo = 0, hi = nb - 1;  // last bucket with vbase <= x
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((mid < kVbCache ? lr_vb[mid] : list[mid].vbase) <= x) lo = mid;
        else hi = mid - 1;
      }
      const unsigned long long w = tile_weight(__ldcg(&list[lo].L));
      const unsigned long long nt = (unsigned long long)ntiles_dev<W>(__ldcg(&list[lo].size));
      const unsigned long long i = (x - (lo < kVbCache ? lr_vb[lo] : list[lo].vbase) + w - 1) / w;
      const unsigned long long tb = __ldcg(&list[lo].tile_base);
      t = i < nt ? tb + i : tb + nt;  // (tb + nt: the next bucket's first tile, or T)
    }
    P.cta_t0[b] = t;
  }
}

// Key bounds of child c of bucket d (SplitDesc::klo / khi of the child).
// Every child inherits its parent's bounds; an even child 2*dd of a radix
// split is further confined to its digit's cell: with f = (x - lo) >> sh
// (or the same on the high words) and digit = f * mul >> 32, digit dd holds
// exactly the f in [ceil(dd * 2^32 / mul), ceil((dd + 1) * 2^32 / mul)).  A
// clamped split (digits over the sample range) leaves digit 0 open below and
// its last digit -- and any digit reached by a saturated f -- open above.
// Must mirror radix_digit / radix_digit_hi / radix_digit_unc* exactly: the
// unclamped digit of the NEXT level trusts these bounds.
template <typename W>
__device__ __forceinline__ void child_bounds(const SplitDesc& d, unsigned long long lo, int c,
                                             unsigned long long& klo, unsigned long long& khi) {
  klo = d.klo;
  khi = d.khi;
  if (sizeof(W) > 8 || !(d.L & 0x100u) || (c & 1)) return;
  const unsigned long long mul = d.aux;
  if (mul == 0) return;
  const int sh = (int)((d.L >> 16) & 0xFFu);
  const unsigned long long dd = (unsigned long long)(c >> 1);
  const unsigned long long m = (1ull << (d.L & 0xFFu)) - 1ull;  // last digit of a clamped split
  const bool clamped = !(d.L & 0x800u);
  const unsigned long long fmin = dd == 0 ? 0ull : ((dd << 32) + mul - 1) / mul;
  const unsigned long long fnext = (((dd + 1) << 32) + mul - 1) / mul;  // first f of the next digit
  const unsigned long long maxw = word_max_u64<W>();
  unsigned long long a, b = 0;
  bool has_b = true;
  if (sizeof(W) == 8 && sh >= 32) {
    const unsigned long long lh = lo >> 32;
    const int s2 = sh - 32;
    const unsigned long long ah = lh + (fmin << s2), bh = lh + (fnext << s2);
    a = ah > 0xFFFFFFFFull ? maxw : ah << 32;
    if (bh > 0xFFFFFFFFull) has_b = false;
    else b = (bh << 32) - 1ull;
  } else {
    const unsigned long long room = (maxw - lo) >> sh;  // largest f a word can have
    a = fmin > room ? maxw : lo + (fmin << sh);
    if (fnext > room || fnext >= 0xFFFFFFFFull) has_b = false;  // (>= 2^32 - 1: f may be saturated)
    else b = lo + (fnext << sh) - 1ull;
  }
  if (!(clamped && dd == 0) && a > klo) klo = a;
  if (has_b && !(clamped && dd >= m) && b < khi) khi = b;
}

// ---- kernels ---------------------------------------------------------------

// Root setup: reset counters; the whole array becomes one split bucket or one
// base-case item (driver.hpp:172-191's n<=1 / n<=256 / recurse dispatch).
template <typename W>
__device__ __forceinline__ void init_root(const Params<W>& P) {
  Ctrl* c = P.ctrl;
  c->split_packed[0] = 0;
  c->split_packed[1] = 0;
  for (int i = 0; i < kNumLists; ++i) c->item_count[i] = 0;
  c->partition_calls = c->keys_partitioned = c->base_cases = 0;
  c->error = 0;
  c->sample_done = 0;
  for (int i = 0; i < 32; ++i) c->modes[i / 4][i % 4] = 0;
  if (P.n > (unsigned long long)Cfg<W>::kCap || P.part_mode) {
    SplitDesc d;
    d.start = 0;
    d.size = P.n;
    d.tile_base = 0;
    d.flags = F_RAW;
    d.L = 0;
    d.aux = 0;
    d.vbase = 0;
    d.bfirst = d.blast = 0;
    d.klo = 0;
    d.khi = word_max_u64<W>();
    P.split[0][0] = d;
    c->split_packed[0] = (1ull << 40) | (unsigned long long)ntiles_dev<W>(P.n);
  } else if (P.n > 1) {
    Item it;
    it.start = 0;
    it.size = P.n;
    it.flags = F_RAW;
    const int cls = class_for(P.n);
    P.items[cls][0] = it;
    c->item_count[cls] = 1;
    c->base_cases = 1;
  }
}

template <typename W>
__global__ void k_init(Params<W> P) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  init_root(P);
}

// Splitter selection (replaces choose_pivot, pivot.hpp:146-172): stratified
// random 4-key chunks (cache-line friendly like the reference's 64-B chunks,
// PAPER.md:393-398), smem bitonic sort, equidistant splitters.
template <typename W, int THREADS>
__global__ void __launch_bounds__(THREADS) k_sample(Params<W> P) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* s = reinterpret_cast<W*>(smem_raw);
  __shared__ unsigned dcnt[1 << kMaxRadixL];
  __shared__ unsigned s_maxc;
  __shared__ W s_spl[256];     // deduplicated splitters (piecewise certification)
  __shared__ unsigned s_t1[kL1];
  __shared__ W s_pwlo;
  __shared__ int s_pwsh, s_pwlsh;
  __shared__ unsigned s_pwcmax;
  __shared__ W s_red_lo[THREADS / 32];
  __shared__ W s_red_hi[THREADS / 32];
  // P.root_init (the level-0 launch of a sort with n > Cap): the root
  // bucket is set up here by CTA 0 (k_init's work, one launch fewer); the
  // level has exactly that one bucket
  if (P.root_init) {
    if (blockIdx.x != 0) return;
    if (threadIdx.x == 0) init_root(P);
    __syncthreads();
  }
  const unsigned long long packed = P.root_init ? (1ull << 40) : P.ctrl->split_packed[P.cur];
  const int nb = (int)(packed >> 40);
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctrl->split_packed[P.cur ^ 1] = 0;
  SplitDesc* list = P.split[P.cur];
  for (int p = blockIdx.x; p < nb; p += gridDim.x) {
    SplitDesc d = list[p];
    const int L = fanout_L<W>(d.size);
    const int m = (1 << L) - 1;
    int S = 16 << L;
    if (S > kMaxSamples) S = kMaxSamples;
    const W* src = (d.flags & F_IN_B) ? P.b : P.a;
    const int xf = (d.flags & F_RAW) ? P.xf : XF_NONE;
    const int nch = S / 4;
    const unsigned long long stratum = d.size / nch;
    for (int c = threadIdx.x; c < nch; c += THREADS) {
      const unsigned long long lo = (unsigned long long)c * d.size / nch;
      const unsigned long long r = mix64(P.seed ^ mix64(d.start * 0x9E3779B97F4A7C15ull + c) ^
                                         ((unsigned long long)P.level << 56));
      const unsigned long long span = stratum >= 4 ? stratum - 3 : 1;
      const unsigned long long off = __umul64hi(r, span);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        unsigned long long idx = lo + off + e;
        if (idx >= d.size) idx = d.size - 1;
        s[4 * c + e] = enc<W>(ldg(src + d.start + idx), xf);
      }
    }
    __syncthreads();
    // sample min / max (the radix certification needs no sorted sample)
    W slo, shi;
    {
      constexpr int SI = kMaxSamples / THREADS;
      W k[SI];
#pragma unroll
      for (int i = 0; i < SI; ++i) {
        const int idx = i * THREADS + threadIdx.x;
        k[i] = s[idx < S ? idx : 0];
      }
      block_minmax<W, THREADS, SI>(k, slo, shi, s_red_lo, s_red_hi);
    }
    W* g = P.splitters + (unsigned long long)p * 256;
    const int step = S / (m + 1);
    // Radix certification: if equal-width digits over [sample min, max]
    // give no digit more than ~2x its share of the sample, classify by digit
    // (pure ALU) instead of by splitter search.  Radix buckets may split up
    // to 2^kMaxRadixL ways (no splitter table is needed).
    // The digits are tried first over the bucket's KNOWN bounds [klo, khi]
    // (the word range at the root, a radix parent's digit cell below it):
    // such a split needs no per-key clamps (classify_mode<5/6>); then over
    // the sample's [min, max] (keys outside it clamp to the end digits).
    W rlo = slo;       // digit origin
    int dshift = 0;    // f = top 24 bits of (x - rlo)
    unsigned long long rf = 0;
    auto set_range = [&](const W& lo, const W& hi) {
      const W range = key_sub(hi, lo);
      const int bl = key_bitlen(range);
      rlo = lo;
      dshift = bl > 24 ? bl - 24 : 0;
      rf = key_shr32(range, dshift);
    };
    auto certify = [&](int D, unsigned long long& mul) -> bool {
      const int mr = D - 1;
      mul = ((unsigned long long)D << 32) / (rf + 1);
      if (mul > 0xFFFFFFFFull) mul = 0xFFFFFFFFull;  // fewer code values than digits
      for (int k = threadIdx.x; k <= mr; k += THREADS) dcnt[k] = 0;
      if (threadIdx.x == 0) s_maxc = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < S; i += THREADS)
        atomicAdd(&dcnt[radix_digit(s[i], rlo, dshift, (unsigned)mul, (unsigned)mr)], 1u);
      __syncthreads();
      unsigned used = 0;
      for (int k = threadIdx.x; k <= mr; k += THREADS) {
        atomicMax(&s_maxc, dcnt[k]);
        if (dcnt[k]) used = 1;
      }
      const unsigned nused = __syncthreads_count(used ? 1 : 0);
      // every digit within ~2x of the mean over ALL D digits: children stay
      // <= ~2x the target size, so certification never adds a level
      return P.part_mode == 0 && D >= 4 && 2 * nused >= (unsigned)D &&
             (unsigned)s_maxc * (unsigned)D <= 2u * (unsigned)S + 4u * (unsigned)D;
    };
    // Radix fan-out balanced over the levels still needed so the final
    // items land just under the base case's 2048-key class.
    int Dr;
    {
      const double ratio = (double)d.size / (double)kFinalTarget;
      int lv = 1;
      double Dd = ratio;
      // one level while 256-way children still fit the base case (small
      // inputs: an extra level costs more than a fuller base case saves)
      if (Dd * kFinalTarget > 256.0 * Cfg<W>::kCap) {
        while (Dd > 256.0) {
          ++lv;
          Dd = pow(ratio, 1.0 / lv);
        }
      }
      Dr = (int)ceil(Dd);
      Dr = Dr < 4 ? 4 : (Dr > 256 ? 256 : Dr);
    }
    unsigned long long dmul = 0;
    int Lf = L;
    bool radix = false, unc = false;
    if constexpr (sizeof(W) <= 8) {
      W blo, bhi;
      {
        const unsigned long long a = d.klo, b = d.khi;
        memcpy(&blo, &a, sizeof(W));  // (little-endian low bytes)
        memcpy(&bhi, &b, sizeof(W));
      }
      set_range(blo, bhi);
      // (the high-word digit is exact only from an origin with a zero low word)
      const bool ok = !(sizeof(W) == 8 && dshift >= 32 && (unsigned)d.klo != 0u);
      if (ok) radix = unc = certify(Dr, dmul);
    }
    if (!radix) {
      set_range(slo, shi);
      radix = certify(Dr, dmul);
    }
    if (radix) {
      Lf = 2;
      while ((1 << Lf) < Dr) ++Lf;
    }
    unsigned meff = 0;  // distinct splitters when fewer than m (bits 24-31 of L)
    bool pw = false;    // piecewise radix over the splitters (bit 9 of L)
    bool pwlog = false; // ... over log units (bit 12 of L)
    if (radix) {
      if (threadIdx.x == 0) g[0] = rlo;
    } else {
      // sort the S samples (padded to 4096 with the maximum) with the block
      // base-case sort, 512 threads x 8 keys, then stage them back to smem
      {
        constexpr int SI = kMaxSamples / THREADS;
        W k[SI];
#pragma unroll
        for (int i = 0; i < SI; ++i) {
          const int idx = i * THREADS + threadIdx.x;
          k[i] = idx < S ? s[idx] : key_max<W>();
        }
        __syncthreads();
        block_sort<W, THREADS, SI, sizeof(W) <= 4>(k, s);
#pragma unroll
        for (int i = 0; i < SI; ++i) s[threadIdx.x * SI + i] = k[i];
        __syncthreads();
      }
      // Equidistant splitters, deduplicated: low-entropy samples (few
      // distinct values) get a short splitter list, so the lookup table has
      // one splitter per cell and every key takes the fast path.
      static_assert(THREADS >= 255, "one candidate per thread");
      const int k = threadIdx.x;
      W v = key_max<W>();
      unsigned uq = 0;
      if (k < m) {
        v = s[(k + 1) * step - 1];
        uq = (k == 0 || key_lt(s[k * step - 1], v)) ? 1u : 0u;
      }
      unsigned u = 0;
      const unsigned pos = block_exclusive_scan<THREADS>(uq, &u, reinterpret_cast<unsigned*>(dcnt));
      if (uq) {
        g[pos] = v;
        s_spl[pos] = v;
      }
      if (u < (unsigned)m) {
        Lf = 1;
        while ((1u << Lf) - 1u < u) ++Lf;
        meff = u;
      }
      // Piecewise-radix certification (pw_digit): equal-width digits inside
      // each first-level bucket, as many as the bucket holds splitters; taken
      // when no digit gets more than ~2x its share of the sample (smooth
      // densities, e.g. normal floats), so keys skip the table + splitter
      // search.  Low-entropy samples (duplicates) fail it and keep the
      // splitters' equality buckets.
      const int mq = (int)u;
      __syncthreads();
      if (P.part_mode == 0 && mq >= 15) {
        if (threadIdx.x == 0) {
          s_pwlo = s_spl[0];
          fine_geometry(key_sub(s_spl[mq - 1], s_spl[0]), s_pwsh, s_pwlsh, s_pwcmax);
          s_maxc = 0;
        }
        for (int k2 = threadIdx.x; k2 < mq; k2 += THREADS) dcnt[k2] = 0;
        __syncthreads();
        build_t1(s_spl, mq, s_pwlo, s_spl[mq - 1], s_pwsh, s_pwlsh, s_pwcmax, s_t1);
        for (int i = threadIdx.x; i < S; i += THREADS)
          atomicAdd(&dcnt[pw_digit(s[i], s_pwlo, s_pwsh, s_pwlsh, s_pwcmax, s_t1)], 1u);
        __syncthreads();
        for (int k2 = threadIdx.x; k2 < mq; k2 += THREADS) atomicMax(&s_maxc, dcnt[k2]);
        __syncthreads();
        pw = (unsigned)s_maxc * (unsigned)mq <= 2u * (unsigned)S + 4u * (unsigned)mq;
        // Skewed integers (power-law / log-uniform keys put most splitters
        // into one linear first-level bucket): the same test over LOG units
        // (fine_unit_log).  Encoded keys only -- raw floats certify above.
        if (!pw && xf < XF_FLT_ASC) {
          __syncthreads();
          if (threadIdx.x == 0) {
            s_pwcmax = log_unit_of(key_sub(s_spl[mq - 1], s_spl[0]));
            s_maxc = 0;
          }
          for (int k2 = threadIdx.x; k2 < mq; k2 += THREADS) dcnt[k2] = 0;
          __syncthreads();
          build_t1(s_spl, mq, s_pwlo, s_spl[mq - 1], 0, 0, s_pwcmax, s_t1, true);
          for (int i = threadIdx.x; i < S; i += THREADS)
            atomicAdd(&dcnt[pw_digit<true>(s[i], s_pwlo, 0, 0, s_pwcmax, s_t1)], 1u);
          __syncthreads();
          for (int k2 = threadIdx.x; k2 < mq; k2 += THREADS) atomicMax(&s_maxc, dcnt[k2]);
          __syncthreads();
          pwlog = pw = (unsigned)s_maxc * (unsigned)mq <= 2u * (unsigned)S + 4u * (unsigned)mq;
        }
      }
    }
    if (threadIdx.x == 0) {
      // (tile cost weight: plain radix digit 1, piecewise radix 2 (bit 10), splitter
      // table / tree 3 (bit 13) -- level_ranges)
      list[p].L = (unsigned)Lf | (radix ? (0x100u | ((unsigned)dshift << 16)) : (pw ? 0x400u : 0x2000u)) |
                  (pw ? 0x200u : 0u) |
                  (unc ? 0x800u : 0u) | (pwlog ? 0x1000u : 0u) | (meff << 24);
      list[p].aux = dmul;
      atomicAdd(&P.ctrl->modes[P.level < 8 ? P.level : 7][radix ? 1 : (pwlog ? 3 : (pw ? 2 : 0))], 1u);
    }
    __syncthreads();
  }
  // the last CTA to finish lays out the level's cost-weighted CTA tile ranges
  __shared__ unsigned s_ticket;
  bool last = P.root_init != 0;  // (root level: CTA 0 is the only one here)
  if (!last) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // (after the barrier: orders the whole CTA's descriptor writes)
      s_ticket = atomicAdd(&P.ctrl->sample_done, 1u);
    }
    __syncthreads();
    last = s_ticket == gridDim.x - 1;
  }
  if (!last) return;
  if (threadIdx.x == 0) P.ctrl->sample_done = 0;
  __threadfence();
  level_ranges(P, list, nb, P.root_init ? (unsigned long long)ntiles_dev<W>(P.n) : (packed & kTileMask));
}

// Tile t of the current level: owning bucket, first key and key count.
struct TileRef {
  int p;
  unsigned long long lo;
  int cnt;
};

// The issuing thread's walk over tiles: the owning bucket's descriptor and
// the next bucket's first tile stay in registers, so issuing tile t+1 costs
// no dependent global loads except at bucket boundaries.
template <typename W>
struct TileCursor {
  int p;
  unsigned flags;
  unsigned long long start, size, tb, next_tb;
  __device__ __forceinline__ void load(const SplitDesc* list, int nb) {
    const SplitDesc d = list[p];
    start = d.start;
    size = d.size;
    tb = d.tile_base;
    flags = d.flags;
    next_tb = p + 1 < nb ? list[p + 1].tile_base : ~0ull;
  }
  __device__ __forceinline__ TileRef at(const SplitDesc* list, int nb, unsigned long long t) {
    if (t >= next_tb) {
      ++p;
      while (p + 1 < nb && list[p + 1].tile_base <= t) ++p;
      load(list, nb);
    }
    TileRef r;
    r.p = p;
    r.lo = start + (t - tb) * (unsigned long long)Cfg<W>::kTile;
    const unsigned long long end = start + size;
    r.cnt = (int)((end - r.lo) < (unsigned long long)Cfg<W>::kTile ? (end - r.lo) : Cfg<W>::kTile);
    return r;
  }
};

template <typename W>
__device__ __forceinline__ const W* src_of(const Params<W>& P, unsigned flags) {
  return (flags & F_IN_B) ? P.b : P.a;
}

template <typename W>
__host__ __device__ constexpr int stage_bytes() {
  return Cfg<W>::kTile * (int)sizeof(W) + 32;
}

// Per-tile classification histogram (read-only pass over the level's keys).
// Tiles stream through a 2-stage TMA bulk-copy pipeline; counting uses plain
// shared-memory atomics (no __match_any_sync: measured 13x slower than ATOMS
// on B200 with ~500 distinct ids per warp); a warp whose 32 keys share one
// child (low-entropy input) adds 32 with a single atomic.
template <typename W>
__global__ void __launch_bounds__(Cfg<W>::kHistThreads, Cfg<W>::kHistMinBlocks) k_hist(Params<W> P) {
  pdl_enter();
  constexpr int THREADS = Cfg<W>::kHistThreads;
  constexpr int TILE = Cfg<W>::kTile;
  constexpr int ITEMS = TILE / THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ SplSmem<W> S;
  // two histograms, alternating by tile: tile t's counts are flushed (read and
  // zeroed) while tile t+1 is already being counted into the other one, so a
  // full tile costs one barrier
  // (<= 4-byte keys; measured slower for 8-byte keys, which keep one
  // histogram and the barrier after the tile wait)
  constexpr bool kDbl = sizeof(W) <= 4;
  __shared__ unsigned hist2[kDbl ? 2 : 1][kChildStride + 1];  // + dump slot
  __shared__ __align__(8) unsigned long long bars[Cfg<W>::kHistStages];
  __shared__ int s_p;
  const unsigned long long packed = P.ctrl->split_packed[P.cur];
  const int nb = (int)(packed >> 40);
  if (nb == 0) return;
  const unsigned long long t0 = P.cta_t0[blockIdx.x];  // (cost-weighted ranges: level_ranges)
  const unsigned long long t1 = P.cta_t0[blockIdx.x + 1];
  if (t0 >= t1) return;
  const SplitDesc* list = P.split[P.cur];
  TileCursor<W> ic;  // (thread 0: the tile issuer)
  if (threadIdx.x == 0) {
    s_p = find_bucket(list, nb, t0);
    for (int s = 0; s < Cfg<W>::kHistStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ic.p = s_p;
    ic.load(list, nb);
    for (int s = 0; s + 1 < Cfg<W>::kHistStages && t0 + s < t1; ++s) {  // prefetch depth Cfg<W>::kHistStages - 1
      const TileRef r = ic.at(list, nb, t0 + s);
      tile_issue(src_of(P, ic.flags) + r.lo, (unsigned long long)r.cnt * sizeof(W),
                 smem_raw + s * stage_bytes<W>(), &bars[s]);
    }
  }
  for (int i = threadIdx.x; i < (kDbl ? 2 : 1) * (kChildStride + 1); i += THREADS) (&hist2[0][0])[i] = 0;
  __syncthreads();
  int p = s_p;
  SplitDesc d = list[p];
  unsigned long long p_next = p + 1 < nb ? list[p + 1].tile_base : ~0ull;  // next bucket's first tile
  int L = (int)(d.L & 0xFFu);
  load_splitters(P.splitters + (unsigned long long)p * 256, d.L, S, d.aux);
  // this CTA's per-child totals of the current bucket (thread c owns children
  // c*PER ..): the shared histogram is per tile, flushed to P.tilecnt
  constexpr int PER = kChildStride / THREADS > 0 ? kChildStride / THREADS : 1;
  unsigned ctot[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) ctot[j] = 0;
  unsigned phase = 0;
  int st = 0;  // stage of tile t
  for (unsigned long long t = t0; t < t1; ++t, st = st + 1 == Cfg<W>::kHistStages ? 0 : st + 1) {
    if (threadIdx.x == 0 && t + Cfg<W>::kHistStages - 1 < t1) {
      // the stage consumed in the previous iteration (freed by its final barrier)
      const int sn = st == 0 ? Cfg<W>::kHistStages - 1 : st - 1;
      const TileRef r = ic.at(list, nb, t + Cfg<W>::kHistStages - 1);
      tile_issue(src_of(P, ic.flags) + r.lo, (unsigned long long)r.cnt * sizeof(W),
                 smem_raw + sn * stage_bytes<W>(), &bars[sn]);
    }
    if (t >= p_next) {
      // flush and move to the next bucket
      const int nc = num_children(L);
      unsigned long long* sg = P.seg + (unsigned long long)(p + blockIdx.x) * kChildStride;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int c = threadIdx.x * PER + j;
        if (c < nc) sg[c] = ctot[j];
        ctot[j] = 0;
      }
      while (p + 1 < nb && list[p + 1].tile_base <= t) ++p;
      d = list[p];
      p_next = p + 1 < nb ? list[p + 1].tile_base : ~0ull;
      L = (int)(d.L & 0xFFu);
      __syncthreads();
      load_splitters(P.splitters + (unsigned long long)p * 256, d.L, S, d.aux);
    }
    const W* src = src_of(P, d.flags);
    const int xf = (d.flags & F_RAW) ? P.xf : XF_NONE;
    const unsigned long long lo = d.start + (t - d.tile_base) * TILE;
    const unsigned long long end = d.start + d.size;
    const int cnt = (int)((end - lo) < (unsigned long long)TILE ? (end - lo) : TILE);
    const TileSpan span = tile_span(src + lo, (unsigned long long)cnt * sizeof(W));
    unsigned char* stage = smem_raw + st * stage_bytes<W>();
    mbar_wait(&bars[st], (phase >> st) & 1);
    phase ^= 1u << st;
    unsigned* hist = hist2[kDbl ? (t - t0) & 1 : 0];
    // full tiles of <= 8-byte keys are read in 16-byte chunks (TileVec layout:
    // no head / tail fix-up in smem, so no barrier here)
    constexpr bool kVec = sizeof(W) <= 8;
    const unsigned char* kp = stage + (reinterpret_cast<unsigned long long>(src + lo) - span.base);
    if (!(kVec && cnt == TILE)) tile_fixup<W, THREADS>(src + lo, cnt, span, stage);
    if (!(kDbl && cnt == TILE)) __syncthreads();  // (block-uniform)
    unsigned wide = 0;  // items whose cell holds > 2 splitters (rare)
    const Xf<W> X = make_xf<W>(xf);
    const TileVec<W, THREADS> tv(src + lo, span, stage);
    auto count_tile = [&](auto tree_tag, auto flt_tag) {
      constexpr int TREE = decltype(tree_tag)::value;
      constexpr bool FLT = decltype(flt_tag)::value;
      if (cnt == TILE && TREE >= 2) {  // radix: stream classify -> count
        if constexpr (kVec) {  // 16-byte key loads, KPC independent classify chains per load
          constexpr int KPC = TileVec<W, THREADS>::KPC;
#pragma unroll
          for (int q = 0; q < ITEMS / KPC; ++q) {
            W kk[KPC];
            tv.load(q, kk, q == ITEMS / KPC - 1);
#pragma unroll
            for (int e = 0; e < KPC; ++e)
              atomicAdd(&hist[hslot(classify_mode<TREE>(enc_x<FLT>(kk[e], X), S))], 1u);
          }
        } else {
#pragma unroll
          for (int i = 0; i < ITEMS; ++i)
            atomicAdd(&hist[hslot(classify_mode<TREE>(enc_x<FLT>(lds_key<W>(kp, i * THREADS + threadIdx.x), X), S))], 1u);
        }
      } else if (cnt == TILE) {
        int bk[ITEMS];
        if constexpr (kVec) {
          constexpr int KPC = TileVec<W, THREADS>::KPC;
#pragma unroll
          for (int q = 0; q < ITEMS / KPC; ++q) {
            W kk[KPC];
            if constexpr (TREE == 1) {
              // (tree mode, measured: a global-load path inside this loop
              // costs low-entropy inputs 15%.  The last thread of a tile off
              // the 16-byte grid leaves its last chunk slot empty and counts
              // the tile's KPC head / tail keys from global memory instead.)
              const bool ok = tv.load_mid(q, kk, q == ITEMS / KPC - 1);
#pragma unroll
              for (int e = 0; e < KPC; ++e) bk[q * KPC + e] = ok ? classify_mode<TREE>(enc_x<FLT>(kk[e], X), S) : -2;
              if (!ok) {
                for (int e = 0; e < KPC; ++e)
                  atomicAdd(&hist[hslot(classify(enc_x<FLT>(ldg(src + lo + tv.extra_index(e)), X), S))], 1u);
              }
            } else {
              tv.load(q, kk, q == ITEMS / KPC - 1);
#pragma unroll
              for (int e = 0; e < KPC; ++e) bk[q * KPC + e] = classify_mode<TREE>(enc_x<FLT>(kk[e], X), S);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < ITEMS; ++i)
            bk[i] = classify_mode<TREE>(enc_x<FLT>(lds_key<W>(kp, i * THREADS + threadIdx.x), X), S);
        }
        // a warp whose whole sub-tile is one child (low-entropy input) adds
        // once instead of 32*ITEMS same-address atomics
        bool same = bk[0] >= 0;
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) same = same && bk[i] == bk[0];
        const int b0 = __shfl_sync(0xffffffffu, bk[0], 0);
        if (__all_sync(0xffffffffu, same && bk[0] == b0)) {
          if ((threadIdx.x & 31) == 0) atomicAdd(&hist[hslot(b0)], 32u * ITEMS);
        } else {
#pragma unroll
          for (int i = 0; i < ITEMS; ++i) {  // (wide cells and empty slots count into a dump slot)
            atomicAdd(&hist[bk[i] >= 0 ? hslot(bk[i]) : kChildStride], 1u);
            wide |= (bk[i] == -1 ? 1u : 0u) << i;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int idx = i * THREADS + threadIdx.x;
          if (idx < cnt) {
            const int b = classify_mode<TREE>(enc_x<FLT>(lds_key<W>(kp, idx), X), S);
            if (b >= 0) atomicAdd(&hist[hslot(b)], 1u);
            else wide |= 1u << i;
          }
        }
      }
    };
    if (S.use_tree == 4) {
      if (X.flt) count_tile(std::integral_constant<int, 4>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 4>{}, std::false_type{});
    } else if (S.use_tree == 7) {  // (log units: integer keys only -- floats certify the linear units)
      count_tile(std::integral_constant<int, 7>{}, std::false_type{});
    } else if (S.use_tree == 5) {
      if (X.flt) count_tile(std::integral_constant<int, 5>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 5>{}, std::false_type{});
    } else if (sizeof(W) == 8 && S.use_tree == 6) {
      if (X.flt) count_tile(std::integral_constant<int, 6>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 6>{}, std::false_type{});
    } else if (sizeof(W) == 8 && S.use_tree == 3) {
      if (X.flt) count_tile(std::integral_constant<int, 3>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 3>{}, std::false_type{});
    } else if (S.use_tree >= 2) {
      if (X.flt) count_tile(std::integral_constant<int, 2>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 2>{}, std::false_type{});
    } else if (S.use_tree) {
      if (X.flt) count_tile(std::integral_constant<int, 1>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 1>{}, std::false_type{});
    } else {
      if (X.flt) count_tile(std::integral_constant<int, 0>{}, std::true_type{});
      else count_tile(std::integral_constant<int, 0>{}, std::false_type{});
    }
    while (wide) {
      const int i = __ffs(wide) - 1;
      wide &= wide - 1;
      const W kx = (kVec && cnt == TILE) ? ldg(src + lo + tv.index(i)) : lds_key<W>(kp, i * THREADS + threadIdx.x);
      const int b = classify_slow(enc<W>(kx, xf), S);
      VXS_DCHECK(b >= 0 && b < num_children(L), "k_hist: child id out of range");
      atomicAdd(&hist[hslot(b)], 1u);  // rare
    }
    __syncthreads();  // stage st fully consumed before it is refilled; tile counts complete
    {
      // the tile's child counts -> P.tilecnt (k_scatter places keys from
      // them), into this CTA's totals, and the histogram is reset for the
      // next tile (its first read follows that tile's barrier)
      const int nc = num_children(L);
      unsigned short* tc = P.tilecnt + t * kChildStride;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int c = threadIdx.x * PER + j;
        const unsigned v = hist[hslot(c)];
        hist[hslot(c)] = 0;
        if (c < nc) tc[c] = (unsigned short)v;
        ctot[j] += v;
      }
    }
  }
  const int nc = num_children(L);
  unsigned long long* sg = P.seg + (unsigned long long)(p + blockIdx.x) * kChildStride;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int c = threadIdx.x * PER + j;
    if (c < nc) sg[c] = ctot[j];
  }
}

// Column scan of the root level's per-CTA child counts written by k_hist
// (one bucket, every CTA of the grid holds a row): row b becomes the offset
// of CTA b's keys inside each child, the per-child totals go to counts[].
// One CTA per 32-child chunk, its 32 warps split the rows (one round trip of
// loads instead of a serial walk down ~300 rows per lane).  Deeper levels
// scan their handful of rows per bucket in k_plan.
template <typename W>
__global__ void __launch_bounds__(1024) k_segscan_root(Params<W> P) {
  pdl_enter();
  __shared__ unsigned long long part[32][33];
  const unsigned long long packed = P.ctrl->split_packed[P.cur];
  if ((int)(packed >> 40) == 0) return;
  const SplitDesc d = P.split[P.cur][0];
  const int nc = num_children((int)(d.L & 0xFFu));
  const int rows = (int)d.blast + 1;  // CTAs b = 0 .. rows-1 hold tiles
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (rows + 31) / 32;
  constexpr int R = 16;
  for (int c0 = blockIdx.x * 32; c0 < nc; c0 += gridDim.x * 32) {
    const int c = c0 + lane;
    const int r0 = warp * per, r1 = r0 + per < rows ? r0 + per : rows;
    unsigned long long sum = 0;
    for (int r = r0; r < r1; r += R) {
      unsigned long long v[R];
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (r + j < r1 && c < nc) ? P.seg[(unsigned long long)(r + j) * kChildStride + c] : 0ull;
#pragma unroll
      for (int j = 0; j < R; ++j) sum += v[j];
    }
    part[warp][lane] = sum;
    __syncthreads();
    unsigned long long run = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      run += w < warp ? part[w][lane] : 0ull;
      tot += part[w][lane];
    }
    for (int r = r0; r < r1; r += R) {
      unsigned long long v[R];
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (r + j < r1 && c < nc) ? P.seg[(unsigned long long)(r + j) * kChildStride + c] : 0ull;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (r + j < r1 && c < nc) P.seg[(unsigned long long)(r + j) * kChildStride + c] = run;
        run += v[j];
      }
    }
    if (warp == 0 && c < nc) P.counts[c] = tot;
    __syncthreads();
  }
}

// Per split bucket: child offsets -> cursors; children become next-level
// split buckets, base-case items (grouping adjacent small children into one
// item of <= Cap keys) or copy items (equality buckets).
template <typename W>
__global__ void __launch_bounds__(kChildStride) k_plan(Params<W> P) {
  pdl_enter();
  constexpr int THREADS = kChildStride;
  constexpr unsigned long long CAP = Cfg<W>::kCap;
  __shared__ unsigned long long s_cnt[kChildStride];
  __shared__ unsigned long long s_off[kChildStride];
  __shared__ unsigned long long scan_scratch[32];
  __shared__ unsigned char s_kind[kChildStride];
  __shared__ unsigned s_res[kNumLists];  // (32-bit: a 64-bit shared atomicAdd is a CAS loop -- with every
                                         // child of a bucket on one list it was a quarter of this kernel)
  __shared__ unsigned long long s_base[kNumLists];
  __shared__ unsigned long long s_nsort;
  __shared__ unsigned long long s_split_base;
  if (threadIdx.x == 0) s_nsort = 0;
  const unsigned long long packed = P.ctrl->split_packed[P.cur];
  const int nb = (int)(packed >> 40);
  const SplitDesc* list = P.split[P.cur];
  const int nxt = P.cur ^ 1;
  // CTAs beyond the bucket count (most of the grid at the top levels) only
  // scan tile counts into prefixes (below), concurrently with the bucket work
  const bool spare = (int)gridDim.x > nb;
  for (int p = blockIdx.x; p < nb; p += gridDim.x) {
    const SplitDesc d = list[p];
    const int L = (int)(d.L & 0xFFu);
    const int nc = num_children(L);
    const int c = threadIdx.x;
    unsigned long long cnt = 0;
    if (P.level == 0) {
      // the root's per-child totals were reduced over every CTA row by k_segscan_root
      cnt = c < nc ? P.counts[(unsigned long long)p * kChildStride + c] : 0ull;
    } else if (c < nc) {
      // column scan of child c over the CTA rows touching this bucket (a
      // handful below the root): row slots become offsets, the sum the total
      const int b_first = (int)d.bfirst, b_last = (int)d.blast;
      for (int b = b_first; b <= b_last; ++b) {
        unsigned long long* sl = P.seg + (unsigned long long)(p + b) * kChildStride + c;
        const unsigned long long v = *sl;
        *sl = cnt;
        cnt += v;
      }
      P.counts[(unsigned long long)p * kChildStride + c] = cnt;
    }
    unsigned long long total;
    const unsigned long long off = block_exclusive_scan<THREADS>(cnt, &total, scan_scratch);
    VXS_DCHECK(total == d.size, "k_plan: child counts do not add up to the bucket");
    if (c < nc) P.childbase[(unsigned long long)p * kChildStride + c] = d.start + off;
    s_cnt[c] = cnt;
    s_off[c] = off;
    const unsigned child_flags = (d.flags & F_IN_B) ? 0u : F_IN_B;  // raw cleared
    if (P.part_mode) {
      __syncthreads();
      continue;
    }
    // does child c's final range [start + off, + cnt) meet the requested output range?
    const bool rel = d.start + off + cnt > P.rlo && d.start + off < P.rhi;
    // next-level split children
    const bool is_split = c < nc && (c & 1) == 0 && cnt > CAP && rel;
    const unsigned long long my_tiles = is_split ? (unsigned long long)ntiles_dev<W>(cnt) : 0ull;
    const unsigned long long pk = is_split ? ((1ull << 40) | my_tiles) : 0ull;
    unsigned long long pk_total;
    const unsigned long long pk_excl = block_exclusive_scan<THREADS>(pk, &pk_total, scan_scratch);
    if (c == 0 && pk_total) s_split_base = atomicAdd(&P.ctrl->split_packed[nxt], pk_total);
    __syncthreads();
    if (is_split) {
      const unsigned long long base = s_split_base + pk_excl;
      const unsigned long long q = base >> 40;
      if (q < P.cap_split) {
        SplitDesc nd;
        nd.start = d.start + off;
        nd.size = cnt;
        nd.tile_base = base & kTileMask;
        nd.flags = child_flags;
        nd.L = 0;
        nd.aux = 0;
        nd.vbase = 0;
        nd.bfirst = nd.blast = 0;
        {
          unsigned long long org = 0;  // the parent's digit origin (radix splits keep it in splitters[0])
          if ((d.L & 0x100u) && sizeof(W) <= 8) {
            const W g0 = P.splitters[(unsigned long long)p * 256];
            memcpy(&org, &g0, sizeof(W) <= 8 ? sizeof(W) : 8);
          }
          child_bounds<W>(d, org, c, nd.klo, nd.khi);
        }
        P.split[nxt][q] = nd;
      } else {
        P.ctrl->error = 1;
      }
    }
    // Group the remaining children in parallel.  Kinds: SPLIT (handled
    // above), BIGEQ (equality bucket > Cap: one cooperative copy item), SOLO
    // (>= kGroupTarget keys: its own item), SMALL (< kGroupTarget, incl.
    // empty).  Consecutive SMALL children whose parent-relative start offsets
    // fall in the same kGroupTarget window form one item (< 2*kGroupTarget
    // <= Cap keys), so a group never needs a sequential greedy pass.
    const bool eqc = (c & 1) != 0;
    const bool small = c < nc && cnt < kGroupTarget;
    s_kind[c] = c >= nc ? 0 : (small ? 1 : 2);  // 0 none, 1 small, 2 other
    __syncthreads();
    const bool need_copy = (child_flags & F_IN_B) || P.xf != XF_NONE;
    int my_list = -1;
    unsigned long long my_start = 0, my_size = 0;
    if (c < nc && !small) {
      if (!eqc && cnt > CAP && rel) {
        // split child: already queued
      } else if (cnt > CAP) {  // equality bucket, or a child outside the requested range
        if (need_copy) my_list = kListCopyBig;
      } else {
        my_list = (!eqc && cnt > 1 && rel) ? class_for(cnt) : (need_copy ? kListCopySmall : -1);
      }
      my_start = d.start + off;
      my_size = cnt;
    } else if (small) {
      const unsigned long long win = off / kGroupTarget;
      const bool leader = c == 0 || s_kind[c - 1] != 1 || (s_off[c - 1] / kGroupTarget) != win;
      if (leader) {
        unsigned long long gz = 0;
        bool gsort = false;
        for (int e = c; e < nc && s_kind[e] == 1 && (s_off[e] / kGroupTarget) == win; ++e) {
          gz += s_cnt[e];
          gsort = gsort || ((e & 1) == 0 && s_cnt[e] > 1);
        }
        const bool grel = d.start + off + gz > P.rlo && d.start + off < P.rhi;
        if (gz) {
          my_list = (gsort && grel) ? class_for(gz) : (need_copy ? kListCopySmall : -1);
          my_start = d.start + off;
          my_size = gz;
        }
      }
    }
    if (c < kNumLists) s_res[c] = 0;
    __syncthreads();
    unsigned long long my_slot = 0;
    if (my_list >= 0) my_slot = atomicAdd(&s_res[my_list], 1u);
    __syncthreads();
    if (c < kNumLists) {
      const unsigned long long k = s_res[c];
      s_base[c] = k ? atomicAdd(&P.ctrl->item_count[c], k) : 0;
      if (c < kNumSortClasses && k) atomicAdd(&s_nsort, k);
    }
    if (c == 32) {
      atomicAdd(&P.ctrl->partition_calls, 1ull);
      atomicAdd(&P.ctrl->keys_partitioned, d.size);
    }
    __syncthreads();
    if (c == 0 && s_nsort) {
      atomicAdd(&P.ctrl->base_cases, s_nsort);
      s_nsort = 0;
    }
    if (my_list >= 0) {
      const unsigned long long slot = s_base[my_list] + my_slot;
      if (slot < P.cap_items) {
        Item it;
        it.start = my_start;
        it.size = my_size;
        it.flags = child_flags;
        it.pad = 0;
        it.pad2 = 0;
        P.items[my_list][slot] = it;
      } else {
        P.ctrl->error = 2;
      }
    }
    __syncthreads();
  }
  // Per-tile child counts (k_hist) -> exclusive prefixes in place, one warp
  // per tile (lane l owns children 16l .. 16l+15: two 16-byte loads, a warp
  // scan, two stores).  k_scatter then starts every tile from its prefixes
  // instead of a block-wide scan (three barriers per tile fewer).  Entries
  // past the bucket's child count hold stale values; prefixes are causal, so
  // the entries k_scatter reads (<= child count) are exact.
  {
    const unsigned long long T = packed & kTileMask;
    const int lane = threadIdx.x & 31;
    // (with spare CTAs the bucket CTAs skip this pass: it then overlaps their work)
    if (spare && (int)blockIdx.x < nb) return;
    const unsigned long long first = spare ? (unsigned long long)((int)blockIdx.x - nb) : blockIdx.x;
    const unsigned long long nw = (unsigned long long)(spare ? (int)gridDim.x - nb : (int)gridDim.x) * (THREADS / 32);
    // (kU tiles per warp in flight: the loads of all of them are issued
    // before the first scan -- a warp otherwise walks its tiles one global
    // round trip at a time)
    constexpr int kU = 4;
    for (unsigned long long t0 = first * (THREADS / 32) + (threadIdx.x >> 5); t0 < T; t0 += kU * nw) {
      uint4 q[kU][2];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const unsigned long long t = t0 + u * nw;
        if (t < T) {
          const uint4* row = reinterpret_cast<const uint4*>(P.tilecnt + t * kChildStride) + 2 * lane;
          q[u][0] = row[0];
          q[u][1] = row[1];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const unsigned long long t = t0 + u * nw;
        if (t >= T) break;  // (warp-uniform)
        unsigned* w = reinterpret_cast<unsigned*>(q[u]);  // 8 words = 16 u16 counts
        unsigned sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) sum += (w[j] & 0xFFFFu) + (w[j] >> 16);
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned run = incl - sum;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const unsigned a = w[j] & 0xFFFFu, b = w[j] >> 16;
          w[j] = (run & 0xFFFFu) | ((run + a) << 16);
          run += a + b;
        }
        uint4* row = reinterpret_cast<uint4*>(P.tilecnt + t * kChildStride) + 2 * lane;
        row[0] = q[u][0];
        row[1] = q[u][1];
      }
    }
  }
}

// Scatter: classify again (radix digit / table / tree), count per child
// with fire-and-forget shared atomics (one per warp when the warp's whole
// sub-tile falls into one child), exclusive scan over the children, stage
// the tile in smem grouped by child (each key takes the next slot of its
// child with a returning atomic on the prefix; the tile's own TMA stage is
// reused), advance this CTA's private per-child cursors (placement from the
// k_hist / k_segscan offset table: no global atomics), then write each child
// run with consecutive threads (coalesced), recomputing radix child ids
// instead of staging them.  Exchange mode stores a segment's runs straight
// into its owner's receive buffer (vxs_partition_exchange).
template <typename W>
__global__ void __launch_bounds__(Cfg<W>::kScatThreads, Cfg<W>::kScatMinBlocks) k_scatter(Params<W> P) {
  pdl_enter();
  constexpr int THREADS = Cfg<W>::kScatThreads;
  constexpr int TILE = Cfg<W>::kTile;
  constexpr int ITEMS = TILE / THREADS;
  constexpr int PER = kChildStride / THREADS > 0 ? kChildStride / THREADS : 1;  // children per thread
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned short* stage_b = reinterpret_cast<unsigned short*>(smem_raw + kStages * stage_bytes<W>());
  unsigned* whist = reinterpret_cast<unsigned*>(stage_b + TILE);  // [kChildStride] per-child slot counters
  __shared__ SplSmem<W> S;
  __shared__ W* gptr[kChildStride];  // where staged slot 0 of the child in histogram slot s goes (slot j -> gptr[s][j])
  __shared__ unsigned long long gcur[kChildStride];  // this CTA's next global slot per child
  __shared__ __align__(8) unsigned long long bars[kStages];
  __shared__ int s_p;
  const unsigned long long packed = P.ctrl->split_packed[P.cur];
  const int nb = (int)(packed >> 40);
  if (nb == 0) return;
  const unsigned long long t0 = P.cta_t0[blockIdx.x];  // (cost-weighted ranges: level_ranges)
  const unsigned long long t1 = P.cta_t0[blockIdx.x + 1];
  if (t0 >= t1) return;
  const SplitDesc* list = P.split[P.cur];
  TileCursor<W> ic;  // (thread 0: the tile issuer)
  if (threadIdx.x == 0) {
    s_p = find_bucket(list, nb, t0);
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ic.p = s_p;
    ic.load(list, nb);
    const TileRef r = ic.at(list, nb, t0);
    tile_issue(src_of(P, ic.flags) + r.lo, (unsigned long long)r.cnt * sizeof(W), smem_raw, &bars[0]);
  }
  __syncthreads();
  int p = s_p;
  SplitDesc d = list[p];
  unsigned long long p_next = p + 1 < nb ? list[p + 1].tile_base : ~0ull;  // next bucket's first tile
  int L = (int)(d.L & 0xFFu);
  load_splitters(P.splitters + (unsigned long long)p * 256, d.L, S, d.aux);
  auto load_cursors = [&]() {
    const unsigned long long* sg = P.seg + (unsigned long long)(p + blockIdx.x) * kChildStride;
    const unsigned long long* cb = P.childbase + (unsigned long long)p * kChildStride;
    const int ncl = num_children(L);
#pragma unroll
    for (int j = 0; j < PER; ++j) {  // (thread tid owns children tid*PER + j, here and in the tile loop)
      const int c = threadIdx.x * PER + j;
      if (c < ncl) gcur[c] = cb[c] + sg[c];
    }
  };
  load_cursors();
  const int lane = threadIdx.x & 31;
  const int out_xf = P.part_mode ? P.xf : XF_NONE;
  const bool xchg = P.xchg != 0;
  unsigned phase = 0;
  for (unsigned long long t = t0; t < t1; ++t) {
    const int st = (int)((t - t0) & (kStages - 1));
    if (threadIdx.x == 0 && t + 1 < t1) {
      const TileRef r = ic.at(list, nb, t + 1);
      tile_issue(src_of(P, ic.flags) + r.lo, (unsigned long long)r.cnt * sizeof(W),
                 smem_raw + (st ^ 1) * stage_bytes<W>(), &bars[st ^ 1]);
    }
    if (t >= p_next) {
      while (p + 1 < nb && list[p + 1].tile_base <= t) ++p;
      d = list[p];
      p_next = p + 1 < nb ? list[p + 1].tile_base : ~0ull;
      L = (int)(d.L & 0xFFu);
      load_splitters(P.splitters + (unsigned long long)p * 256, d.L, S, d.aux);
      load_cursors();
    }
    W* dst_buf = P.part_mode ? P.out : ((d.flags & F_IN_B) ? P.a : P.b);
    const int nc = num_children(L);
    const W* src = src_of(P, d.flags);
    const int xf = (d.flags & F_RAW) ? P.xf : XF_NONE;
    const unsigned long long lo = d.start + (t - d.tile_base) * TILE;
    const unsigned long long end = d.start + d.size;
    const int cnt = (int)((end - lo) < (unsigned long long)TILE ? (end - lo) : TILE);
    // this tile's child prefixes (k_hist counted, k_plan scanned): issued
    // before the tile wait so their latency hides under it.  tpre[j] = first
    // staging slot of child tid*PER + j; tpre[PER] = end of the last one.
    unsigned tpre[PER + 1];
    {
      const unsigned short* tc = P.tilecnt + t * kChildStride;
#pragma unroll
      for (int j = 0; j <= PER; ++j) {
        const int c = threadIdx.x * PER + j;
        tpre[j] = c < nc ? (unsigned)tc[c] : (unsigned)cnt;
      }
    }
    const TileSpan span = tile_span(src + lo, (unsigned long long)cnt * sizeof(W));
    unsigned char* stage = smem_raw + st * stage_bytes<W>();
    mbar_wait(&bars[st], (phase >> st) & 1);
    phase ^= 1u << st;
    // (full tiles of <= 8-byte keys: TileVec reads the aligned chunks from
    // smem and the head / tail keys from global -- no fix-up, no barrier)
    const unsigned char* kp = stage + (reinterpret_cast<unsigned long long>(src + lo) - span.base);
    if (!(sizeof(W) <= 8 && cnt == TILE)) {  // (block-uniform)
      tile_fixup<W, THREADS>(src + lo, cnt, span, stage);
      __syncthreads();  // tile complete in smem
    }
    W k[ITEMS];
    int bk[ITEMS];
    unsigned wide = 0;
    const Xf<W> X = make_xf<W>(xf);
    // recompute child ids at write-out instead of staging them (cheap for
    // <= 32-bit words and the 64-bit high-word classifier; piecewise radix
    // stages them: f32 1e8 scatter@L0 0.39 -> 0.34 ms)
    const bool unc = S.use_tree >= 5;  // known-bounds digit
    const bool radix = (sizeof(W) <= 4 && (S.use_tree == 2 || S.use_tree == 5)) ||
                       (sizeof(W) == 8 && (S.use_tree == 3 || S.use_tree == 6));
    // bk[] holds each key's shared-histogram SLOT (hslot of its child id; the
    // digit itself in the radix modes), or -1 (wide cell) / -2 (past the tile)
    auto classify_tile = [&](auto tree_tag, auto flt_tag) {
      constexpr int TREE = decltype(tree_tag)::value;
      constexpr bool FLT = decltype(flt_tag)::value;
      auto to_slot = [](int id) {
        if constexpr (TREE >= 2) return id >> 1;  // (even ids: folds to the digit)
        else return id >= 0 ? hslot(id) : id;
      };
      if (cnt == TILE) {  // full tile: no per-key bounds (branch-free classify)
        if constexpr (sizeof(W) <= 8) {  // 16-byte key loads (TileVec layout; any key -> item map works)
          constexpr int KPC = TileVec<W, THREADS>::KPC;
          const TileVec<W, THREADS> tv(src + lo, span, stage);
#pragma unroll
          for (int q = 0; q < ITEMS / KPC; ++q) {
            W kk[KPC];
            tv.load(q, kk, q == ITEMS / KPC - 1);
#pragma unroll
            for (int e = 0; e < KPC; ++e) {
              const int i = q * KPC + e;
              k[i] = enc_x<FLT>(kk[e], X);
              bk[i] = to_slot(classify_mode<TREE>(k[i], S));
              if (bk[i] == -1) wide |= 1u << i;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < ITEMS; ++i) {
            k[i] = enc_x<FLT>(lds_key<W>(kp, i * THREADS + threadIdx.x), X);
            bk[i] = to_slot(classify_mode<TREE>(k[i], S));
            if (bk[i] == -1) wide |= 1u << i;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int idx = i * THREADS + threadIdx.x;
          k[i] = idx < cnt ? enc_x<FLT>(lds_key<W>(kp, idx), X) : key_max<W>();
          bk[i] = idx < cnt ? to_slot(classify_mode<TREE>(k[i], S)) : -2;
          if (bk[i] == -1) wide |= 1u << i;
        }
      }
    };
    if (S.use_tree == 4) {
      if (X.flt) classify_tile(std::integral_constant<int, 4>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 4>{}, std::false_type{});
    } else if (S.use_tree == 7) {  // (log units: integer keys only -- floats certify the linear units)
      classify_tile(std::integral_constant<int, 7>{}, std::false_type{});
    } else if (S.use_tree == 5) {
      if (X.flt) classify_tile(std::integral_constant<int, 5>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 5>{}, std::false_type{});
    } else if (sizeof(W) == 8 && S.use_tree == 6) {
      if (X.flt) classify_tile(std::integral_constant<int, 6>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 6>{}, std::false_type{});
    } else if (sizeof(W) == 8 && S.use_tree == 3) {
      if (X.flt) classify_tile(std::integral_constant<int, 3>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 3>{}, std::false_type{});
    } else if (S.use_tree >= 2) {
      if (X.flt) classify_tile(std::integral_constant<int, 2>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 2>{}, std::false_type{});
    } else if (S.use_tree) {
      if (X.flt) classify_tile(std::integral_constant<int, 1>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 1>{}, std::false_type{});
    } else {
      if (X.flt) classify_tile(std::integral_constant<int, 0>{}, std::true_type{});
      else classify_tile(std::integral_constant<int, 0>{}, std::false_type{});
    }
    if (wide) {  // rare; static indices keep k[] / bk[] in registers
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (bk[i] == -1) bk[i] = hslot(classify_slow(k[i], S));
    }
    // child offsets inside the tile (the prefixes k_plan scanned) become the
    // children's slot counters; this CTA's private cursors give each child
    // run its global place (no global atomics).
    {
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int c = threadIdx.x * PER + j;
        const unsigned ex = tpre[j], tcnt = tpre[j + 1] - tpre[j];
        VXS_DCHECK(tpre[j] <= tpre[j + 1] && tpre[j + 1] <= (unsigned)cnt,
                   "k_scatter: tile prefixes do not fit the tile");
        whist[hslot(c)] = ex;
        if (tcnt) {
          const unsigned long long gres = gcur[c];
          gcur[c] = gres + tcnt;
          // (vxs_partition_exchange: segment c/2 goes straight to its owner's
          // receive buffer at this rank's offset there -- the fused exchange)
          W* base = dst_buf;
          if (xchg) {
            const int sg = c >> 1;
            base = reinterpret_cast<W*>(P.xdst[sg]) + P.xoff[sg] - P.childbase[2 * sg];
          }
          gptr[hslot(c)] = base + ((long long)gres - (long long)ex);
        }
      }
    }
    // (this barrier also orders every key read from the stage -- the keys
    // are in registers by now -- before the staging writes)
    __syncthreads();  // slot counters and gptr ready

    // stage the tile grouped by child: each key takes the next slot of its
    // child (returning shared atomic); the tile's own TMA stage is reused
    {
      W* staged = reinterpret_cast<W*>(stage);
      auto put = [&](unsigned pos, int i) {
        VXS_DCHECK(pos < (unsigned)cnt, "k_scatter: staging slot outside the tile (k_hist/k_scatter counts differ)");
        staged[pos] = k[i];
        if (!radix) stage_b[pos] = (unsigned short)bk[i];
      };
      // (random keys leave here at once: the first and last lane's first
      // keys already differ, and neither fast path below can apply)
      const int b0 = __shfl_sync(0xffffffffu, bk[0], 0);
      const bool ends = __shfl_sync(0xffffffffu, bk[0], 31) == b0;  // (warp-uniform)
      bool same = false;
      if (ends) {
        same = bk[0] >= 0;
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) same = same && bk[i] == bk[0];
      }
      if (ends && __all_sync(0xffffffffu, same && bk[0] == b0)) {
        // the warp's whole sub-tile is one child: one atomic for 32*ITEMS keys
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&whist[b0], 32u * ITEMS);
        base = __shfl_sync(0xffffffffu, base, 0) + lane * ITEMS;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) put(base + i, i);
      } else if (cnt == TILE && ends) {
        // presorted-looking warp (its first 32-key slice is one child): slice
        // by slice, one atomic per uniform slice -- 32 lanes would otherwise
        // serialise on the same counter
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int ci = __shfl_sync(0xffffffffu, bk[i], 0);
          if (__all_sync(0xffffffffu, bk[i] == ci)) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&whist[ci], 32u);
            put(__shfl_sync(0xffffffffu, base, 0) + lane, i);
          } else {
            put(atomicAdd(&whist[bk[i]], 1u), i);
          }
        }
      } else if (cnt == TILE) {  // full tile: every id is valid (straight-line code)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) put(atomicAdd(&whist[bk[i]], 1u), i);
      } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
          if (bk[i] >= 0) put(atomicAdd(&whist[bk[i]], 1u), i);
      }
    }
    W* staged = reinterpret_cast<W*>(stage);
    __syncthreads();
#ifdef VXS_CHECKS
    // every staged slot j of child c lands inside child c's range
    auto chk = [&](int slot, int j) {
      const int c = unslot(slot);
      VXS_DCHECK(slot >= 0 && c < nc, "k_scatter: child id out of range");
      const W* base = dst_buf;  // (exchange: the segment's place in its owner's window)
      if (P.xchg) base = reinterpret_cast<const W*>(P.xdst[c >> 1]) + P.xoff[c >> 1] - P.childbase[2 * (c >> 1)];
      const long long idx = (long long)((gptr[slot] + j) - base);
      const unsigned long long b0 = P.childbase[(unsigned long long)p * kChildStride + c];
      const unsigned long long n0 = P.counts[(unsigned long long)p * kChildStride + c];
      VXS_DCHECK(idx >= (long long)b0 && (unsigned long long)idx < b0 + n0, "k_scatter: key stored outside its child");
    };
#else
    auto chk = [](int, int) {};
#endif
    if (radix && out_xf == XF_NONE && cnt == TILE) {  // full tile: unrolled, no bounds
      const RadixReg<W> R(S);
      if (unc) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int j = i * THREADS + threadIdx.x;
          const W v = staged[j];
          chk(R.template slot<true>(v), j);
          gptr[R.template slot<true>(v)][j] = v;
        }
      } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int j = i * THREADS + threadIdx.x;
          const W v = staged[j];
          chk(R.template slot<false>(v), j);
          gptr[R.template slot<false>(v)][j] = v;
        }
      }
    } else if (out_xf == XF_NONE && cnt == TILE) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int j = i * THREADS + threadIdx.x;
        chk(stage_b[j], j);
        gptr[stage_b[j]][j] = staged[j];
      }
    } else if (radix) {
      const RadixReg<W> R(S);
      if (out_xf == XF_NONE) {
        for (int j = threadIdx.x; j < cnt; j += THREADS) {
          const W v = staged[j];
          const int sl = unc ? R.template slot<true>(v) : R.template slot<false>(v);
          chk(sl, j);
          gptr[sl][j] = v;
        }
      } else {
        for (int j = threadIdx.x; j < cnt; j += THREADS) {
          const W v = staged[j];
          gptr[unc ? R.template slot<true>(v) : R.template slot<false>(v)][j] = dec<W>(v, out_xf);
        }
      }
    } else if (out_xf == XF_NONE) {
      for (int j = threadIdx.x; j < cnt; j += THREADS) {
        chk(stage_b[j], j);
        gptr[stage_b[j]][j] = staged[j];
      }
    } else {  // vxs_partition: decode into the caller's encoding
      for (int j = threadIdx.x; j < cnt; j += THREADS) {
        chk(stage_b[j], j);
        gptr[stage_b[j]][j] = dec<W>(staged[j], out_xf);
      }
    }
    __syncthreads();  // (measured: deferring the next tile's TMA issue to drop this barrier does not pay)
  }
  if (P.xchg) __threadfence_system();  // peer stores visible before the exchange's barrier
}

// Register budget of the counting-sort classes (8 or 16 keys per thread):
// 40/64 (<= 4-byte keys), 64/80 (8-byte) or 128 (16-byte) registers per
// thread, so several CTAs share an SM and hide each other's item loads.
template <typename W, int CLS>
constexpr int final_min_blocks() {
  constexpr int I = SortClass<CLS>::I;
  constexpr int R = sizeof(W) <= 4 ? (I <= 8 ? 40 : 64) : sizeof(W) == 8 ? (I <= 8 ? 64 : 80) : 128;
  constexpr int B = 65536 / (SortClass<CLS>::T * R);
  return CLS == 0 ? 1 : (B < 1 ? 1 : B);
}

// Base case over one size class: load <= T*I keys (pad: transformed maximum),
// sort them -- class 0 (<= 256 keys) with the warp bitonic network, larger
// classes with the counting sort (block_sort.cuh bin_sort_item) -- decode,
// write back into A.
template <typename W, int CLS>
__global__ void __launch_bounds__(SortClass<CLS>::T, final_min_blocks<W, CLS>()) k_final(Params<W> P) {
  pdl_enter();
  constexpr int THREADS = SortClass<CLS>::T;
  constexpr int ITEMS = SortClass<CLS>::I;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  const unsigned long long nitems = P.ctrl->item_count[CLS];
  const Item* items = P.items[CLS];
  const Xf<W> X = make_xf<W>(P.xf);
  // the next item's descriptor is loaded while this one is sorted (one
  // dependent global round trip fewer per item)
  Item nxt{};
  if (blockIdx.x < nitems) nxt = items[blockIdx.x];
  for (unsigned long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    const Item item = nxt;
    if (it + gridDim.x < nitems) nxt = items[it + gridDim.x];
    const W* src = (item.flags & F_IN_B) ? P.b : P.a;
    const int size = (int)item.size;
    VXS_DCHECK(item.size >= 1 && item.size <= (unsigned long long)(THREADS * ITEMS) && item.start + item.size <= P.n,
               "k_final: item outside the array or its class");
    W k[ITEMS];
    // padding: the maximum for the network (class 0); a copy of the item's
    // first key for the counting sort (neutral for its min / max)
    if (item.flags & F_RAW) {  // only the root item of a small input is raw
      const W pad = CLS >= 1 ? enc<W>(ldg(src + item.start), P.xf) : key_max<W>();
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int idx = i * THREADS + threadIdx.x;
        k[i] = idx < size ? enc<W>(ldcs(src + item.start + idx), P.xf) : pad;
      }
    } else {
      const W pad = CLS >= 1 ? ldg(src + item.start) : key_max<W>();
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int idx = i * THREADS + threadIdx.x;
        k[i] = idx < size ? ldcs(src + item.start + idx) : pad;
      }
    }
    W* dst = P.a + item.start;
    if constexpr (CLS >= 1) {
      // counting-sort base case; items it rejects (clustered keys, decided
      // block-uniformly) go to the full-width network fallback kernel
      // (rank-in-count for 8-byte keys was faster until the padding slots left the
      // counting pass; re-measured after: fire-and-forget counts win there too,
      // k_final<u64> 0.630 -> 0.603 ms)
      constexpr bool RANK = false;
      const bool done = X.flt ? bin_sort_item<W, THREADS, ITEMS, true, RANK>(k, size, dst, X)
                              : bin_sort_item<W, THREADS, ITEMS, false, RANK>(k, size, dst, X);
      if (!done && threadIdx.x == 0) {
        const unsigned long long slot = atomicAdd(&P.ctrl->item_count[kListFallback], 1ull);
        if (slot < P.cap_items) P.items[kListFallback][slot] = item;
        else P.ctrl->error = 3;
      }
    } else {
      // smallest class: bitonic network merged inside the warp (__shfl_xor_sync)
      block_sort<W, THREADS, ITEMS, true>(k, sm);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) sm[pad_idx<W>(threadIdx.x * ITEMS + i)] = k[i];
      __syncthreads();
      if (X.flt) {
        for (int idx = threadIdx.x; idx < size; idx += THREADS) dst[idx] = dec_x<true>(sm[pad_idx<W>(idx)], X);
      } else {
        for (int idx = threadIdx.x; idx < size; idx += THREADS) dst[idx] = dec_x<false>(sm[pad_idx<W>(idx)], X);
      }
      __syncthreads();
    }
  }
}

// Full-width bitonic/merge-path sort of the items the counting sort rejected
// (persistent; reads the fallback count on the device, usually zero).
template <typename W>
__global__ void __launch_bounds__(SortClass<4>::T) k_final_fallback(Params<W> P) {
  pdl_enter();
  constexpr int THREADS = SortClass<4>::T;
  constexpr int ITEMS = (sizeof(W) >= 16) ? 8 : 16;  // capacity >= Cap
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  const unsigned long long nitems = P.ctrl->item_count[kListFallback];
  const Item* items = P.items[kListFallback];
  const Xf<W> X = make_xf<W>(P.xf);
  // the next item's descriptor is loaded while this one is sorted (one
  // dependent global round trip fewer per item)
  Item nxt{};
  if (blockIdx.x < nitems) nxt = items[blockIdx.x];
  for (unsigned long long it = blockIdx.x; it < nitems; it += gridDim.x) {
    const Item item = nxt;
    if (it + gridDim.x < nitems) nxt = items[it + gridDim.x];
    const W* src = (item.flags & F_IN_B) ? P.b : P.a;
    const int size = (int)item.size;
    W k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * THREADS + threadIdx.x;
      k[i] = idx < size ? ((item.flags & F_RAW) ? enc<W>(ldcs(src + item.start + idx), P.xf)
                                                : ldcs(src + item.start + idx))
                        : key_max<W>();
    }
    block_sort<W, THREADS, ITEMS, false>(k, sm);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) sm[pad_idx<W>(threadIdx.x * ITEMS + i)] = k[i];
    __syncthreads();
    W* dst = P.a + item.start;
    for (int idx = threadIdx.x; idx < size; idx += THREADS) dst[idx] = dec<W>(sm[pad_idx<W>(idx)], P.xf);
    __syncthreads();
  }
}

// Copy (decode) sorted runs that need no sorting: equality buckets and groups
// of single keys, B -> A or decode-in-place in A.
template <typename W>
__global__ void __launch_bounds__(256) k_copy(Params<W> P) {
  pdl_enter();
  // small items: one CTA per item
  {
    const unsigned long long nitems = P.ctrl->item_count[kListCopySmall];
    const Item* items = P.items[kListCopySmall];
    for (unsigned long long it = blockIdx.x; it < nitems; it += gridDim.x) {
      const Item item = items[it];
      const W* src = ((item.flags & F_IN_B) ? P.b : P.a) + item.start;
      W* dst = P.a + item.start;
      for (unsigned long long i = threadIdx.x; i < item.size; i += 256) dst[i] = dec<W>(ldcs(src + i), P.xf);
    }
  }
  // big items: one flat space of 4096-key chunks over all items, grid-strided
  // (each CTA walks the item list forward as its chunk index grows)
  {
    const unsigned long long nitems = P.ctrl->item_count[kListCopyBig];
    const Item* items = P.items[kListCopyBig];
    constexpr unsigned long long CH = 4096;
    unsigned long long it = 0, base = 0;
    Item item{};
    unsigned long long nch = 0;
    if (nitems) {
      item = items[0];
      nch = (item.size + CH - 1) / CH;
    }
    for (unsigned long long ch = blockIdx.x; it < nitems; ch += gridDim.x) {
      while (it < nitems && ch >= base + nch) {
        base += nch;
        if (++it < nitems) {
          item = items[it];
          nch = (item.size + CH - 1) / CH;
        }
      }
      if (it >= nitems) break;
      const unsigned long long c0 = (ch - base) * CH;
      const unsigned long long e = c0 + CH < item.size ? c0 + CH : item.size;
      const W* src = ((item.flags & F_IN_B) ? P.b : P.a) + item.start;
      W* dst = P.a + item.start;
      unsigned long long i = c0 + threadIdx.x;
      for (; i + 3 * 256 < e; i += 4 * 256) {  // 4 independent loads in flight per thread
        const W v0 = ldcs(src + i), v1 = ldcs(src + i + 256), v2 = ldcs(src + i + 512), v3 = ldcs(src + i + 768);
        dst[i] = dec<W>(v0, P.xf);
        dst[i + 256] = dec<W>(v1, P.xf);
        dst[i + 512] = dec<W>(v2, P.xf);
        dst[i + 768] = dec<W>(v3, P.xf);
      }
      for (; i < e; i += 256) dst[i] = dec<W>(ldcs(src + i), P.xf);
    }
  }
}

// Sampling for the distributed sort: s keys (transformed domain), stratified.
template <typename W>
__global__ void k_sample_out(const W* keys, unsigned long long n, int xf, unsigned long long seed, W* out,
                             int s) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < s; c += gridDim.x * blockDim.x) {
    const unsigned long long lo = (unsigned long long)c * n / s;
    const unsigned long long hi = (unsigned long long)(c + 1) * n / s;
    const unsigned long long span = hi > lo ? hi - lo : 1;
    const unsigned long long r = mix64(seed ^ mix64(0xA5A5ull + c));
    unsigned long long idx = lo + __umul64hi(r, span);
    if (idx >= n) idx = n - 1;
    out[c] = enc<W>(ldg(keys + idx), xf);
  }
}

// Distributed partition: install the caller's splitters (transformed domain,
// sorted, nspl of them) as the root bucket's tree, padded with the maximum.
template <typename W>
__global__ void k_part_setup(Params<W> P, const W* spl, int nspl, int L) {
  const int m = (1 << L) - 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) P.splitters[i] = i < nspl ? spl[i] : key_max<W>();
  for (int i = threadIdx.x; i < kChildStride; i += blockDim.x) P.counts[i] = 0;
  if (threadIdx.x == 0) P.split[0][0].L = (unsigned)L;
  __syncthreads();
  level_ranges(P, P.split[0], 1, (unsigned long long)ntiles_dev<W>(P.n));
}

// Per-segment counts: segment i holds children 2i (keys between splitters)
// and 2i+1 (keys equal to splitter i).
template <typename W>
__global__ void k_part_counts(Params<W> P, int nseg, unsigned long long* seg_counts) {
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) seg_counts[i] = P.counts[2 * i] + P.counts[2 * i + 1];
}

}  // namespace vxs
