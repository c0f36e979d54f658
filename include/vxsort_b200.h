/*
 * vxsort_b200.h -- C ABI of the B200 sort (libvxsort_b200.so).
 *
 * Drop-in boundary for the reference's sort surface
 *   vexsort::sort(std::span<T> keys, const SortConfig&) -> SortStats
 *   /root/reference/proj/core/include/vexsort/vexsort.hpp:121-129
 *   (dispatch: proj/core/src/vexsort.cpp:11-49; SortConfig vexsort.hpp:112-119;
 *    SortStats driver.hpp:26-32; scratch_bytes vexsort.hpp:58-66).
 * Plain pointers and sizes only.  include/vexsort_b200.hpp wraps this ABI in
 * the reference's C++ overload set (recompile-only drop-in); INTEGRATION.md
 * shows the binding.
 *
 * Errors: the reference throws std::invalid_argument (scratch too small,
 * vexsort.cpp:23-25) and std::logic_error (config.hpp:55-59).  A C ABI cannot
 * throw: every entry point returns a vxs_status and vxs_last_error() holds a
 * thread-local message; the C++ wrapper rethrows.
 *
 * Threading: every call is reentrant per (device, stream); no global mutable
 * state beyond per-device caches behind a mutex (reference: SPEC.md:504).
 */
#ifndef VXSORT_B200_H_
#define VXSORT_B200_H_
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The nine reference key types (vexsort.hpp:121-129) plus KV64, an alias of
 * the K128 layout {lo = payload, hi = key} that sorts by key, then payload. */
typedef enum {
  VXS_I16 = 0,
  VXS_U16 = 1,
  VXS_I32 = 2,
  VXS_U32 = 3,
  VXS_F32 = 4,
  VXS_I64 = 5,
  VXS_U64 = 6,
  VXS_F64 = 7,
  VXS_K128 = 8,
  VXS_KV64 = 9
} vxs_key_type;

/* vexsort::Order (vexsort.hpp:31) */
typedef enum { VXS_ASCENDING = 0, VXS_DESCENDING = 1 } vxs_order;

typedef enum {
  VXS_OK = 0,
  VXS_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  VXS_CUDA_ERROR = 2,       /* reference: none (std::runtime_error in C++) */
  VXS_OUT_OF_MEMORY = 3,
  VXS_INTERNAL = 4,         /* reference: std::logic_error (DASSERT) */
  VXS_NO_DEVICE = 5
} vxs_status;

/* vexsort::SortStats (driver.hpp:26-32) first, then device extras.
 *   max_depth         -> multiway levels executed
 *   partition_calls   -> buckets split (multiway partitions)
 *   base_case_calls   -> base-case items sorted (CTA-level sorts)
 *   keys_partitioned  -> keys moved by partition passes
 *   fallback_triggered-> more levels than the size-based estimate were needed */
typedef struct {
  size_t max_depth;
  size_t partition_calls;
  size_t base_case_calls;
  size_t keys_partitioned;
  int fallback_triggered;
  int kernel_launches; /* kernels this call launched */
  size_t workspace_bytes;
} vxs_stats;

/* Device workspace a vxs_sort call of n keys needs (CUB-style two-phase). */
vxs_status vxs_sort_workspace_bytes(size_t n, vxs_key_type type, size_t* bytes);

/* In-place sort of n keys at DEVICE pointer d_keys, stream-ordered on
 * `stream` (a cudaStream_t; NULL = legacy default stream).  d_workspace may
 * be NULL (then it is allocated stream-ordered).  The call synchronises the
 * stream once (to read the device bucket scheduler's level count) unless the
 * stream is being captured into a CUDA graph (see vxs_workspace_status); if
 * stats is non-NULL it is filled.  seed/has_seed mirror SortConfig.seed
 * (vexsort.hpp:112-119): the output never depends on it. */
vxs_status vxs_sort(void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed,
                    int has_seed, void* d_workspace, size_t workspace_bytes, void* stream,
                    vxs_stats* stats);

/* The reference's host-span semantics (vexsort.cpp:11-49): h_keys is a HOST
 * pointer; copies to the device, sorts, copies back, synchronises. */
vxs_status vxs_sort_host(void* h_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed,
                         int has_seed, vxs_stats* stats);

/* Partial sort / selection (std::nth_element and
 * std::partial_sort semantics, generalised to an output range): after the
 * call d_keys[lo, hi) holds, sorted, exactly the keys of sorted ranks
 * lo..hi-1; every key before lo precedes (or equals) them and every key from
 * hi on follows (or equals) them in the requested order; d_keys stays a
 * permutation of the input.  Buckets whose final range misses [lo, hi) are
 * never split or sorted -- they are only moved back into place -- so
 * selecting one rank costs one multiway pass plus the narrowing levels.
 * nth_element(k) = [k, k+1); top-k / partial_sort(k) = [0, k).  Requires
 * lo <= hi <= n (lo == hi: no-op).  Workspace as vxs_sort_workspace_bytes. */
vxs_status vxs_sort_range(void* d_keys, size_t n, vxs_key_type type, vxs_order order, size_t lo, size_t hi,
                          uint64_t seed, int has_seed, void* d_workspace, size_t workspace_bytes, void* stream,
                          vxs_stats* stats);

/* Stable argsort and key+value sort (the row-id trick of
 * "appending a unique row identifier to the least
 * significant bits" -- applied on the device).  Each key is packed with its
 * index into one wider word (64-bit for 16/32-bit keys while n <= 2^32,
 * 128-bit {lo = index, hi = key} otherwise and for 64-bit keys) and the
 * packed words are sorted; ties therefore keep ascending index order in
 * both directions (a stable sort).  128-bit keys (K128/KV64) are not
 * supported (VXS_INVALID_ARGUMENT).
 * vxs_argsort: d_indices[i] = original position of the i-th key in sorted
 *   order; if d_sorted_keys is non-NULL it receives the sorted keys.  d_keys
 *   is not modified.
 * vxs_sort_pairs: sorts d_keys in place and permutes d_values (n elements of
 *   value_bytes = 1, 2, 4, 8 or 16) alongside. */
vxs_status vxs_argsort_workspace_bytes(size_t n, vxs_key_type type, size_t value_bytes, size_t* bytes);
vxs_status vxs_argsort(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t* d_indices,
                       void* d_sorted_keys, uint64_t seed, int has_seed, void* d_workspace,
                       size_t workspace_bytes, void* stream, vxs_stats* stats);
vxs_status vxs_sort_pairs(void* d_keys, void* d_values, size_t value_bytes, size_t n, vxs_key_type type,
                          vxs_order order, uint64_t seed, int has_seed, void* d_workspace,
                          size_t workspace_bytes, void* stream, vxs_stats* stats);

/* Distributed sample sort building blocks.
 * vxs_sample: s stratified random samples of d_keys written to d_out as
 *   ORDER-TRANSFORMED unsigned words of the key width (sortable as unsigned).
 * vxs_partition: multiway partition of d_keys into nspl+1 segments by sorted
 *   transformed-domain splitters (segment i = keys k with spl[i-1] < k <=
 *   spl[i]); output keys (original encoding) grouped by segment in d_out,
 *   per-segment counts (uint64) in d_seg_counts. */
vxs_status vxs_sample(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed,
                      void* d_out, int s, void* stream);
vxs_status vxs_partition(const void* d_keys, size_t n, vxs_key_type type, vxs_order order,
                         const void* d_splitters, int nspl, void* d_out, uint64_t* d_seg_counts,
                         void* d_workspace, size_t workspace_bytes, void* stream);

/* Fused exchange for the distributed sort: a partition split
 * in two so the all-to-all rides on the scatter's own stores.
 * vxs_partition_counts: phase 1 (read-only): per-segment counts of d_keys by
 *   the splitters into d_seg_counts; the (required) workspace keeps the
 *   per-CTA offsets for phase 2.
 * vxs_partition_exchange: phase 2: segment i's keys (original encoding) are
 *   stored at ((key*)d_dst[i]) + d_dst_offsets[i] -- device arrays of nspl+1
 *   addresses / element offsets, typically peers' receive buffers mapped with
 *   vxs_ipc_open.  Same keys, n, type, order, nspl and workspace as phase 1.
 * vxs_device_alloc / vxs_device_free: IPC-exportable device blocks.
 * vxs_ipc_handle: 64-byte cudaIpcMemHandle_t of a vxs_device_alloc block.
 * vxs_ipc_open / vxs_ipc_close: map / unmap a peer's block (P2P). */
vxs_status vxs_partition_counts(const void* d_keys, size_t n, vxs_key_type type, vxs_order order,
                                const void* d_splitters, int nspl, uint64_t* d_seg_counts, void* d_workspace,
                                size_t workspace_bytes, void* stream);
vxs_status vxs_partition_exchange(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, int nspl,
                                  const uint64_t* d_dst, const uint64_t* d_dst_offsets, void* d_workspace,
                                  size_t workspace_bytes, void* stream);
vxs_status vxs_device_alloc(size_t bytes, void** d_ptr);
vxs_status vxs_device_free(void* d_ptr);
vxs_status vxs_ipc_handle(void* d_ptr, void* handle64);
vxs_status vxs_ipc_open(const void* handle64, void** d_ptr);
vxs_status vxs_ipc_close(void* d_ptr);

/* ---- distributed sample sort (SURVEY §8b vxs_dist_sort, §8e) ----------------
 * Extends the reference's single-array surface (vexsort.hpp:121-129; the
 * reference itself has no parallel sort) to one rank per GPU:
 * rank r ends up holding the r-th key range of the union of every rank's
 * keys, sorted; concatenation in rank order equals the single-array sort.
 *
 * vxs_dist_group describes the process group.  With nccl_comm (an
 * ncclComm_t, e.g. from vxs_nccl_comm_create) the small collectives run on
 * the device over NCCL; without one, `allgather` (a host callback: every rank
 * contributes `bytes` from send, recv receives world*bytes in rank order;
 * returns 0 on success) carries them -- e.g. an MPI/gloo bootstrap, or ranks
 * sharing one GPU, which NCCL refuses.
 *
 * vxs_dist_create keeps per-group state across calls: the symmetric receive
 * window (one IPC-exported block per rank, mapped by every peer: P2P over
 * NVLink / NVSwitch), the partition workspace and staging.  Collective: every
 * rank of the group calls it (and every vxs_dist_sort / vxs_dist_destroy).
 *
 * vxs_dist_sort: local sampling (vxs_sample), all-gather of samples, the same
 * world-1 splitters on every rank, then
 *   exchange = VXS_EXCHANGE_FUSED: vxs_partition_counts, all-gather of the
 *     world x world count matrix, vxs_partition_exchange storing each segment
 *     straight into its owner's window (the all-to-all rides on the scatter's
 *     stores), a barrier;
 *   exchange = VXS_EXCHANGE_NCCL: vxs_partition into a local buffer, NCCL
 *     grouped send/recv (needs nccl_comm);
 * then a local vxs_sort of the received keys.  *d_out points at this rank's
 * sorted slice (*n_out keys) inside the context's window: valid until the
 * next vxs_dist_sort / vxs_dist_destroy on the context.  Synchronises
 * `stream` (the count matrix sizes the window).  Stats: the local sort's, with
 * kernel_launches counting every kernel of the call. */
typedef struct {
  int rank;
  int world;
  void* nccl_comm;
  int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes);
  void* allgather_ctx;
} vxs_dist_group;

typedef enum { VXS_EXCHANGE_FUSED = 0, VXS_EXCHANGE_NCCL = 1 } vxs_exchange;

typedef struct vxs_dist_ctx_s* vxs_dist_ctx;

vxs_status vxs_dist_create(const vxs_dist_group* group, vxs_dist_ctx* out);
vxs_status vxs_dist_destroy(vxs_dist_ctx ctx);
vxs_status vxs_dist_sort(vxs_dist_ctx ctx, const void* d_keys, size_t n, vxs_key_type type, vxs_order order,
                         uint64_t seed, vxs_exchange exchange, void** d_out, size_t* n_out, void* stream,
                         vxs_stats* stats);
/* Per-rank key counts of the last vxs_dist_sort (world entries: keys each
 * rank received) and this rank's per-destination send counts. */
vxs_status vxs_dist_last_counts(vxs_dist_ctx ctx, uint64_t* recv_per_rank, uint64_t* sent_per_rank);

/* NCCL bootstrap helpers for hosts without their own (NCCL is loaded at run
 * time; these fail with VXS_CUDA_ERROR when libnccl.so.2 is absent).
 * vxs_nccl_unique_id writes the 128-byte ncclUniqueId rank 0 must share. */
vxs_status vxs_nccl_unique_id(void* id128);
vxs_status vxs_nccl_comm_create(const void* id128, int world, int rank, void** comm);
vxs_status vxs_nccl_comm_destroy(void* comm);

/* CUDA graphs: vxs_sort / vxs_sort_range / vxs_argsort / vxs_sort_pairs on a
 * stream under capture launch without any host round trip (the expected
 * number of levels plus two guard levels -- an idle level exits at once --
 * and every base-case class, item counts read on the device), so the call
 * can be captured once and replayed.  Stats then hold only the launch count.
 * vxs_workspace_status reads the device control block of the last sort that
 * ran in d_workspace (n, type as for that sort): its stats, and
 * VXS_INTERNAL if it overflowed a device list or (captured) needed more
 * levels than were launched.  Synchronises `stream`. */
vxs_status vxs_workspace_status(const void* d_workspace, size_t n, vxs_key_type type, void* stream,
                                vxs_stats* stats);

/* Key transform as used inside the kernels (exposed for tests): encodes
 * (inverse=0) or decodes (inverse=1) n keys in place on the device. */
vxs_status vxs_transform(void* d_keys, size_t n, vxs_key_type type, vxs_order order, int inverse,
                         void* stream);

/* Measurement hooks (bench.py): when enabled, every kernel the library
 * launches is bracketed by CUDA events on its launching stream; read()
 * resolves them (synchronising) into per-kernel launch counts and device
 * milliseconds.  Off by default; costs two event records per launch. */
typedef struct {
  char name[32];
  long long launches;
  double total_ms;
} vxs_kernel_profile;
vxs_status vxs_profile_enable(int on);
void vxs_profile_reset(void);
int vxs_profile_read(vxs_kernel_profile* out, int cap);

/* Thread-local message for the last non-OK status. */
const char* vxs_last_error(void);

/* Size in bytes of one key of this type (2, 4, 8 or 16; 0 if invalid). */
size_t vxs_key_bytes(vxs_key_type type);

/* Base-case capacity (keys per CTA sort) for this type. */
size_t vxs_base_case_capacity(vxs_key_type type);

/* Library version string. */
const char* vxs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VXSORT_B200_H_ */
