/* vexsort_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 * C restatement of /root/reference/proj's sort path; see vexsort_oracle.c. */
#ifndef VEXSORT_ORACLE_H_
#define VEXSORT_ORACLE_H_
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Key-type codes: same numbering as include/vxsort_b200.h's vxs_key_type. */
enum { VXO_I16 = 0, VXO_U16, VXO_I32, VXO_U32, VXO_F32, VXO_I64, VXO_U64, VXO_F64, VXO_K128 };

/* Mirrors vexsort::SortStats (driver.hpp:26-32). */
typedef struct {
  size_t max_depth;
  size_t partition_calls;
  size_t base_case_calls;
  size_t keys_partitioned;
  int fallback_triggered;
} vxo_stats;

int vxo_sort(void* keys, size_t n, int key_type, int descending, uint64_t seed, vxo_stats* stats);
int vxo_precedes(const void* a, const void* b, int key_type, int descending);
int vxo_heap_sort(void* keys, size_t n, int key_type, int descending);
int vxo_generate(void* out, size_t n, int key_type, int dist, uint64_t seed);
void vxo_sfc64_stream(uint64_t seed, uint64_t* out, size_t n);
uint32_t vxo_bounded_offset(uint64_t random, uint32_t bound);
void vxo_five_draws(uint64_t seed, uint32_t bound, size_t num, uint32_t* idx);
size_t vxo_depth_budget(size_t n);
uint64_t vxo_default_seed(const void* keys, size_t n);
uint64_t vxo_choose_pivot_u64(const uint64_t* keys, size_t n, uint64_t seed, int descending);

#ifdef __cplusplus
}
#endif
#endif
