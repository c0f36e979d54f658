/*
 * vexsort_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU sort path (vexsort, a clean-room
 * vqsort restatement under /root/reference/proj) used as the CHECKER for the
 * B200 product.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library.  The product path never calls it.
 *
 * What is restated (file:line under /root/reference/proj):
 *   - Sfc64 generator                      core/include/vexsort/detail/pivot.hpp:25-45
 *   - bounded_offset                       pivot.hpp:49-53
 *   - five_draws_for_nine_offsets          pivot.hpp:66-82
 *   - median3_keys / reduce_medians        pivot.hpp:107-142
 *   - choose_pivot (9/6/3 64-byte chunks)  pivot.hpp:146-172
 *   - 2-way partition, <=pivot goes left   partition.hpp:1-10, 197-236 (scalar form)
 *   - base case for n <= 256               network.hpp:372-404 (restated as an
 *                                          insertion sort: same output, the
 *                                          output of a sort under a total order
 *                                          is unique)
 *   - depth_budget / default_seed          driver.hpp:38-46
 *   - scan_min_max degenerate recovery     driver.hpp:67-93, 142-151
 *   - heap_sort fallback                   driver.hpp:96-121
 *   - recurse / sort + SortStats           driver.hpp:26-32, 123-191
 *   - key order (precedes)                 traits.hpp:51-64 (lane keys),
 *                                          traits.hpp:151-170 (K128 hi,lo)
 *   - harness generators (Dist)            tools/bench/harness.cpp:56-70, 179-219
 *
 * Deliberate, documented divergence: the reference rejects NaN
 * (driver.hpp:176-180) and leaves +-0 unordered.  This oracle instead uses the
 * canonical total order the B200 build commits to:
 *   ascending : -inf < ... < -0.0 < +0.0 < ... < +inf < NaN (NaNs by raw bits)
 *   descending: +inf > ... > +0.0 > -0.0 > ... > -inf, then NaN (raw bits asc)
 * which refines the reference's IEEE '<' order (identical on NaN-free inputs
 * up to the relative order of -0.0/+0.0, the harness's own exemption,
 * harness.cpp:286-298).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "vexsort_oracle.h"

/* ---- Sfc64 (pivot.hpp:25-45) ------------------------------------------- */
typedef struct {
  uint64_t a, b, c, counter;
} sfc64_t;

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static inline uint64_t sfc64_next(sfc64_t* s) {
  const uint64_t result = s->a + s->b + s->counter++;
  s->a = s->b ^ (s->b >> 11);
  s->b = s->c + (s->c << 3);
  s->c = rotl64(s->c, 24) + result;
  return result;
}

static inline void sfc64_init(sfc64_t* s, uint64_t seed) {
  s->a = s->b = s->c = seed;
  s->counter = 1;
  for (int i = 0; i < 12; ++i) sfc64_next(s);
}

void vxo_sfc64_stream(uint64_t seed, uint64_t* out, size_t n) {
  sfc64_t s;
  sfc64_init(&s, seed);
  for (size_t i = 0; i < n; ++i) out[i] = sfc64_next(&s);
}

/* pivot.hpp:49-53 */
static inline uint32_t bounded_offset(uint64_t random, uint32_t bound) {
  const uint64_t r32 = (uint32_t)random;
  return (uint32_t)((r32 * bound) >> 32);
}

uint32_t vxo_bounded_offset(uint64_t random, uint32_t bound) { return bounded_offset(random, bound); }

/* pivot.hpp:66-82: always five draws, nine 32-bit pieces. */
static void five_draws_for_nine(sfc64_t* rng, uint32_t bound, size_t num, uint32_t* idx) {
  uint32_t pieces[10];
  for (int i = 0; i < 5; ++i) {
    const uint64_t d = sfc64_next(rng);
    pieces[2 * i] = (uint32_t)d;
    pieces[2 * i + 1] = (uint32_t)(d >> 32);
  }
  for (size_t i = 0; i < num; ++i) idx[i] = bounded_offset(pieces[i], bound);
}

void vxo_five_draws(uint64_t seed, uint32_t bound, size_t num, uint32_t* idx) {
  sfc64_t s;
  sfc64_init(&s, seed);
  five_draws_for_nine(&s, bound, num, idx);
}

/* driver.hpp:38-46 */
size_t vxo_depth_budget(size_t n) {
  if (n <= 1) return 4;
  size_t w = 0;
  for (size_t v = n - 1; v; v >>= 1) ++w; /* std::bit_width */
  return 2 * w + 4;
}

uint64_t vxo_default_seed(const void* keys, size_t n) {
  return 0x9E3779B97F4A7C15ULL ^ (uint64_t)(uintptr_t)keys ^ ((uint64_t)n * 0xD1B54A32D192ED03ULL);
}

/* ---- canonical key orders ---------------------------------------------- */
/* precedes(a, b): a comes strictly before b in the requested order.
 * Integers: traits.hpp:58-64. K128: traits.hpp:163-170 (hi, then lo). */
typedef struct {
  uint64_t lo, hi;
} k128_t;

#define INT_PRECEDES(a, b, asc) ((asc) ? ((a) < (b)) : ((b) < (a)))

static inline int f32_precedes(float a, float b, int asc) {
  const int na = isnan(a), nb = isnan(b);
  if (na || nb) {
    if (!na) return 1; /* non-NaN before NaN, both orders */
    if (!nb) return 0;
    uint32_t ua, ub;
    memcpy(&ua, &a, 4);
    memcpy(&ub, &b, 4);
    return ua < ub; /* NaNs by raw bits */
  }
  if (a == b) {
    if (a != 0.0f) return 0;
    const int sa = signbit(a) != 0, sb = signbit(b) != 0;
    return asc ? (sa && !sb) : (!sa && sb);
  }
  return asc ? (a < b) : (b < a);
}

static inline int f64_precedes(double a, double b, int asc) {
  const int na = isnan(a), nb = isnan(b);
  if (na || nb) {
    if (!na) return 1;
    if (!nb) return 0;
    uint64_t ua, ub;
    memcpy(&ua, &a, 8);
    memcpy(&ub, &b, 8);
    return ua < ub;
  }
  if (a == b) {
    if (a != 0.0) return 0;
    const int sa = signbit(a) != 0, sb = signbit(b) != 0;
    return asc ? (sa && !sb) : (!sa && sb);
  }
  return asc ? (a < b) : (b < a);
}

static inline int k128_precedes(k128_t a, k128_t b, int asc) {
  const int lt = a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
  const int gt = b.hi < a.hi || (b.hi == a.hi && b.lo < a.lo);
  return asc ? lt : gt;
}

/* ---- generic quicksort body, instantiated per key type ----------------- */
/* PREC(a,b) must be defined; K is the key type; KEYS_PER_CHUNK = 64/sizeof(K)
 * for lane keys and 4 for K128 (a 64-byte chunk holds 4 pairs). */
#define DEFINE_SORT(NAME, K, PREC, KEY_EQ)                                               \
  static inline K NAME##_median3(K a, K b, K c, int asc) {                              \
    /* pivot.hpp:107-112 */                                                             \
    const K lo = PREC(c, a, asc) ? c : a;                                               \
    const K hi = PREC(c, a, asc) ? a : c;                                               \
    const K mid = PREC(b, lo, asc) ? lo : b;                                            \
    return PREC(hi, mid, asc) ? hi : mid;                                               \
  }                                                                                     \
  static K NAME##_choose_pivot(const K* keys, size_t n, sfc64_t* rng, int asc) {        \
    /* pivot.hpp:146-172 */                                                             \
    const size_t ck = 64 / sizeof(K) ? 64 / sizeof(K) : 1;                              \
    const size_t total_chunks = n / ck;                                                 \
    const size_t use = total_chunks >= 9 ? 9 : (total_chunks >= 6 ? 6 : 3);             \
    const size_t rounds = use / 3;                                                      \
    uint32_t idx[9];                                                                    \
    five_draws_for_nine(rng, (uint32_t)total_chunks, use, idx);                         \
    K med[3 * 64], other[3 * 64];                                                       \
    for (size_t r = 0; r < rounds; ++r) {                                               \
      const size_t o0 = idx[3 * r] * ck, o1 = idx[3 * r + 1] * ck, o2 = idx[3 * r + 2] * ck; \
      for (size_t j = 0; j < ck; ++j)                                                   \
        med[r * ck + j] = NAME##_median3(keys[o0 + j], keys[o1 + j], keys[o2 + j], asc); \
    }                                                                                   \
    /* reduce_medians, pivot.hpp:118-142: triples (i, i+K, i+2K) */                     \
    K* cur = med;                                                                       \
    K* oth = other;                                                                     \
    size_t count = rounds * ck;                                                         \
    while (count >= 3) {                                                                \
      const size_t stride = count / 3;                                                  \
      for (size_t i = 0; i < stride; ++i)                                               \
        oth[i] = NAME##_median3(cur[i], cur[i + stride], cur[i + 2 * stride], asc);     \
      count = stride;                                                                   \
      K* t = cur;                                                                       \
      cur = oth;                                                                        \
      oth = t;                                                                          \
    }                                                                                   \
    return cur[0];                                                                      \
  }                                                                                     \
  static size_t NAME##_partition(K* keys, size_t n, K pivot, int asc) {                 \
    /* keys that do not follow the pivot go left (partition.hpp:1-10) */                \
    size_t w = 0;                                                                       \
    for (size_t i = 0; i < n; ++i) {                                                    \
      if (!PREC(pivot, keys[i], asc)) {                                                 \
        K t = keys[w];                                                                  \
        keys[w] = keys[i];                                                              \
        keys[i] = t;                                                                    \
        ++w;                                                                            \
      }                                                                                 \
    }                                                                                   \
    return w;                                                                           \
  }                                                                                     \
  static void NAME##_base_case(K* keys, size_t n, int asc) {                            \
    for (size_t i = 1; i < n; ++i) {                                                    \
      K v = keys[i];                                                                    \
      size_t j = i;                                                                     \
      while (j > 0 && PREC(v, keys[j - 1], asc)) {                                      \
        keys[j] = keys[j - 1];                                                          \
        --j;                                                                            \
      }                                                                                 \
      keys[j] = v;                                                                      \
    }                                                                                   \
  }                                                                                     \
  static void NAME##_sift(K* keys, size_t root, size_t limit, int asc) {              \
    for (;;) {                                                                          \
      const size_t left = 2 * root + 1;                                                 \
      if (left >= limit) break;                                                         \
      size_t next = left;                                                               \
      if (left + 1 < limit && PREC(keys[left], keys[left + 1], asc)) next = left + 1;   \
      if (!PREC(keys[root], keys[next], asc)) break;                                    \
      K t = keys[root];                                                                 \
      keys[root] = keys[next];                                                          \
      keys[next] = t;                                                                   \
      root = next;                                                                      \
    }                                                                                   \
  }                                                                                     \
  static void NAME##_heap_sort(K* keys, size_t n, int asc) {                            \
    /* driver.hpp:96-121 */                                                             \
    if (n <= 1) return;                                                                 \
    for (size_t i = n / 2; i-- > 0;) NAME##_sift(keys, i, n, asc);                      \
    for (size_t end = n - 1; end > 0; --end) {                                          \
      K t = keys[0];                                                                    \
      keys[0] = keys[end];                                                              \
      keys[end] = t;                                                                    \
      NAME##_sift(keys, 0, end, asc);                                                   \
    }                                                                                   \
  }                                                                                     \
  static void NAME##_scan(const K* keys, size_t n, K* first, K* last, int asc) {        \
    /* driver.hpp:67-93 */                                                              \
    *first = keys[0];                                                                   \
    *last = keys[0];                                                                    \
    for (size_t i = 1; i < n; ++i) {                                                    \
      if (PREC(keys[i], *first, asc)) *first = keys[i];                                 \
      if (PREC(*last, keys[i], asc)) *last = keys[i];                                   \
    }                                                                                   \
  }                                                                                     \
  static void NAME##_recurse(K* keys, size_t n, K pivot, size_t budget, size_t depth,   \
                             sfc64_t* rng, int asc, vxo_stats* st) {                    \
    /* driver.hpp:123-170 (loop form for the tail call) */                              \
    for (;;) {                                                                          \
      if (budget == 0) {                                                                \
        NAME##_heap_sort(keys, n, asc);                                                 \
        st->fallback_triggered = 1;                                                     \
        return;                                                                         \
      }                                                                                 \
      if (depth > st->max_depth) st->max_depth = depth;                                 \
      const size_t bound = NAME##_partition(keys, n, pivot, asc);                       \
      st->partition_calls += 1;                                                         \
      st->keys_partitioned += n;                                                        \
      if (bound == n) {                                                                 \
        K first, last;                                                                  \
        NAME##_scan(keys, n, &first, &last, asc);                                       \
        if (KEY_EQ(first, last)) return;                                                \
        pivot = first;                                                                  \
        budget -= 1;                                                                    \
        depth += 1;                                                                     \
        continue;                                                                       \
      }                                                                                 \
      K* left = keys;                                                                   \
      const size_t nl = bound;                                                          \
      K* right = keys + bound;                                                          \
      const size_t nr = n - bound;                                                      \
      if (nl <= 256) {                                                                  \
        NAME##_base_case(left, nl, asc);                                                \
        st->base_case_calls += 1;                                                       \
      } else {                                                                          \
        const K p = NAME##_choose_pivot(left, nl, rng, asc);                            \
        NAME##_recurse(left, nl, p, budget - 1, depth + 1, rng, asc, st);               \
      }                                                                                 \
      if (nr <= 256) {                                                                  \
        NAME##_base_case(right, nr, asc);                                               \
        st->base_case_calls += 1;                                                       \
        return;                                                                         \
      }                                                                                 \
      pivot = NAME##_choose_pivot(right, nr, rng, asc);                                 \
      keys = right;                                                                     \
      n = nr;                                                                           \
      budget -= 1;                                                                      \
      depth += 1;                                                                       \
    }                                                                                   \
  }                                                                                     \
  static void NAME##_sort(K* keys, size_t n, uint64_t seed, int asc, vxo_stats* st) {   \
    /* driver.hpp:172-191 */                                                            \
    memset(st, 0, sizeof(*st));                                                         \
    if (n <= 1) return;                                                                 \
    if (n <= 256) {                                                                     \
      NAME##_base_case(keys, n, asc);                                                   \
      st->base_case_calls = 1;                                                          \
      return;                                                                           \
    }                                                                                   \
    sfc64_t rng;                                                                        \
    sfc64_init(&rng, seed);                                                             \
    const K pivot = NAME##_choose_pivot(keys, n, &rng, asc);                            \
    NAME##_recurse(keys, n, pivot, vxo_depth_budget(n), 1, &rng, asc, st);              \
  }

#define EQ_PLAIN(a, b) ((a) == (b))
#define EQ_F32(a, b) (memcmp(&(a), &(b), 4) == 0)
#define EQ_F64(a, b) (memcmp(&(a), &(b), 8) == 0)
#define EQ_K128(a, b) ((a).lo == (b).lo && (a).hi == (b).hi)
#define PREC_INT(a, b, asc) INT_PRECEDES(a, b, asc)

DEFINE_SORT(i16, int16_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(u16, uint16_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(i32, int32_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(u32, uint32_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(i64, int64_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(u64, uint64_t, PREC_INT, EQ_PLAIN)
DEFINE_SORT(f32, float, f32_precedes, EQ_F32)
DEFINE_SORT(f64, double, f64_precedes, EQ_F64)
DEFINE_SORT(k128, k128_t, k128_precedes, EQ_K128)

int vxo_sort(void* keys, size_t n, int key_type, int descending, uint64_t seed, vxo_stats* stats) {
  vxo_stats local;
  vxo_stats* st = stats ? stats : &local;
  const int asc = !descending;
  switch (key_type) {
    case VXO_I16: i16_sort((int16_t*)keys, n, seed, asc, st); return 0;
    case VXO_U16: u16_sort((uint16_t*)keys, n, seed, asc, st); return 0;
    case VXO_I32: i32_sort((int32_t*)keys, n, seed, asc, st); return 0;
    case VXO_U32: u32_sort((uint32_t*)keys, n, seed, asc, st); return 0;
    case VXO_F32: f32_sort((float*)keys, n, seed, asc, st); return 0;
    case VXO_I64: i64_sort((int64_t*)keys, n, seed, asc, st); return 0;
    case VXO_U64: u64_sort((uint64_t*)keys, n, seed, asc, st); return 0;
    case VXO_F64: f64_sort((double*)keys, n, seed, asc, st); return 0;
    case VXO_K128: k128_sort((k128_t*)keys, n, seed, asc, st); return 0;
    default: return -1;
  }
}

/* Pairwise predicate exposed for tests (canonical order). */
int vxo_precedes(const void* a, const void* b, int key_type, int descending) {
  const int asc = !descending;
  switch (key_type) {
    case VXO_I16: return PREC_INT(*(const int16_t*)a, *(const int16_t*)b, asc);
    case VXO_U16: return PREC_INT(*(const uint16_t*)a, *(const uint16_t*)b, asc);
    case VXO_I32: return PREC_INT(*(const int32_t*)a, *(const int32_t*)b, asc);
    case VXO_U32: return PREC_INT(*(const uint32_t*)a, *(const uint32_t*)b, asc);
    case VXO_F32: return f32_precedes(*(const float*)a, *(const float*)b, asc);
    case VXO_I64: return PREC_INT(*(const int64_t*)a, *(const int64_t*)b, asc);
    case VXO_U64: return PREC_INT(*(const uint64_t*)a, *(const uint64_t*)b, asc);
    case VXO_F64: return f64_precedes(*(const double*)a, *(const double*)b, asc);
    case VXO_K128: return k128_precedes(*(const k128_t*)a, *(const k128_t*)b, asc);
    default: return -1;
  }
}

/* Heap sort alone (driver.hpp:96-121), for the reference's heap_sort tests. */
int vxo_heap_sort(void* keys, size_t n, int key_type, int descending) {
  const int asc = !descending;
  switch (key_type) {
    case VXO_U16: u16_heap_sort((uint16_t*)keys, n, asc); return 0;
    case VXO_U32: u32_heap_sort((uint32_t*)keys, n, asc); return 0;
    case VXO_U64: u64_heap_sort((uint64_t*)keys, n, asc); return 0;
    case VXO_K128: k128_heap_sort((k128_t*)keys, n, asc); return 0;
    default: return -1;
  }
}

/* ---- harness generators (tools/bench/harness.cpp:179-219) --------------- */
/* dist: 0 uniform, 1 equal, 2 lowentropy, 3 asc, 4 desc, 5 twovalue.
 * Restated for the integer/K128 types and f32/f64 (uniform [0,1e6),
 * harness.cpp:56-63). */
static int key_bytes(int t) {
  switch (t) {
    case VXO_I16: case VXO_U16: return 2;
    case VXO_I32: case VXO_U32: case VXO_F32: return 4;
    case VXO_I64: case VXO_U64: case VXO_F64: return 8;
    case VXO_K128: return 16;
  }
  return 0;
}

static void put_u(void* out, size_t i, int t, uint64_t v) {
  switch (key_bytes(t)) {
    case 2: ((uint16_t*)out)[i] = (uint16_t)v; break;
    case 4: ((uint32_t*)out)[i] = (uint32_t)v; break;
    case 8: ((uint64_t*)out)[i] = v; break;
  }
}

static void put_widened(void* out, size_t i, int t, uint16_t v) {
  /* widen16<T>, harness.cpp:30-37 */
  if (t == VXO_K128) {
    ((k128_t*)out)[i].lo = v;
    ((k128_t*)out)[i].hi = 0;
  } else if (t == VXO_F32) {
    ((float*)out)[i] = (float)v;
  } else if (t == VXO_F64) {
    ((double*)out)[i] = (double)v;
  } else if (t == VXO_I16) {
    ((int16_t*)out)[i] = (int16_t)v;
  } else {
    put_u(out, i, t, v);
  }
}

static void put_index(void* out, size_t i, int t, size_t idx) {
  /* from_index<T>, harness.cpp:39-55 */
  if (t == VXO_K128) {
    ((k128_t*)out)[i].lo = idx;
    ((k128_t*)out)[i].hi = 0;
  } else if (t == VXO_F32) {
    ((float*)out)[i] = (float)idx;
  } else if (t == VXO_F64) {
    ((double*)out)[i] = (double)idx;
  } else if (key_bytes(t) == 2) {
    put_u(out, i, t, (uint64_t)(idx % 65536));
  } else {
    put_u(out, i, t, (uint64_t)idx);
  }
}

static int cmp_generic_asc(const void* a, const void* b, int t) {
  if (vxo_precedes(a, b, t, 0)) return -1;
  if (vxo_precedes(b, a, t, 0)) return 1;
  return 0;
}

static int g_sort_type;
static int qsort_cmp(const void* a, const void* b) { return cmp_generic_asc(a, b, g_sort_type); }

int vxo_generate(void* out, size_t n, int key_type, int dist, uint64_t seed) {
  sfc64_t rng;
  sfc64_init(&rng, seed ^ (0x6A09E667F3BCC909ULL + (uint64_t)n));
  const int kb = key_bytes(key_type);
  if (kb == 0) return -1;
  switch (dist) {
    case 0: /* uniform_key<T>, harness.cpp:56-69 */
      for (size_t i = 0; i < n; ++i) {
        if (key_type == VXO_K128) {
          ((k128_t*)out)[i].lo = sfc64_next(&rng);
          ((k128_t*)out)[i].hi = sfc64_next(&rng);
        } else if (key_type == VXO_F32) {
          ((float*)out)[i] = (float)(sfc64_next(&rng) >> 40) * (1.0f / (1 << 24)) * 1e6f;
        } else if (key_type == VXO_F64) {
          ((double*)out)[i] = (double)(sfc64_next(&rng) >> 11) * (1.0 / (double)(1ULL << 53)) * 1e6;
        } else {
          put_u(out, i, key_type, sfc64_next(&rng));
        }
      }
      return 0;
    case 1:
      for (size_t i = 0; i < n; ++i) put_widened(out, i, key_type, 0x2A);
      return 0;
    case 2:
      for (size_t i = 0; i < n; ++i) put_widened(out, i, key_type, (uint16_t)sfc64_next(&rng));
      return 0;
    case 3:
    case 4:
      for (size_t i = 0; i < n; ++i) put_index(out, i, key_type, i);
      if (key_type != VXO_K128) {
        g_sort_type = key_type;
        qsort(out, n, (size_t)kb, qsort_cmp);
      }
      if (dist == 4) {
        char* p = (char*)out;
        char tmp[16];
        for (size_t i = 0, j = n ? n - 1 : 0; i < j; ++i, --j) {
          memcpy(tmp, p + i * kb, kb);
          memcpy(p + i * kb, p + j * kb, kb);
          memcpy(p + j * kb, tmp, kb);
        }
      }
      return 0;
    case 5:
      for (size_t i = 0; i < n; ++i) put_widened(out, i, key_type, (sfc64_next(&rng) & 1) ? 2 : 1);
      return 0;
  }
  return -1;
}

/* choose_pivot alone for u64 keys (pivot.hpp:146-172), to pin against the
 * reference's PivotSampler<ScalarTag>. */
uint64_t vxo_choose_pivot_u64(const uint64_t* keys, size_t n, uint64_t seed, int descending) {
  sfc64_t rng;
  sfc64_init(&rng, seed);
  return u64_choose_pivot(keys, n, &rng, !descending);
}
