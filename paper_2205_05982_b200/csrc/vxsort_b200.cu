// vxsort_b200.cu -- host orchestration (device bucket scheduler) + C ABI.
//
// Host side of the reference's Driver (driver.hpp:172-191) and the public
// dispatch (vexsort.cpp:11-49), re-designed for the device: the host only
// launches a fixed sequence of persistent kernels per level; the bucket
// worklists, splitter trees, per-child cursors and base-case item lists all
// live in device memory.  One stream synchronisation per call reads the
// scheduler's control block (remaining split work, item counts, stats).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/vxsort_b200.h"
#include "sample_sort.cuh"

namespace vxs {
namespace {

thread_local char g_err[512];

vxs_status fail(vxs_status s, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return s;
}

vxs_status cuda_fail(cudaError_t e, const char* where) {
  std::snprintf(g_err, sizeof(g_err), "vxsort_b200: CUDA error in %s: %s", where, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? VXS_OUT_OF_MEMORY : VXS_CUDA_ERROR;
}

#define VXS_CK(expr, where)                     \
  do {                                          \
    cudaError_t e_ = (expr);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- optional per-kernel event timing (measurement tools only) -----------
enum KernelId : int {
  K_INIT = 0, K_SAMPLE, K_HIST, K_SEGSCAN, K_PLAN, K_SCATTER, K_FINAL0, K_FINAL1, K_FINAL2, K_FINAL3, K_FINAL4,
  K_FALLBACK, K_COPY, K_PART, K_MISC, K_COUNT
};
const char* kKernelNames[K_COUNT] = {"k_init", "k_sample", "k_hist", "k_segscan", "k_plan", "k_scatter", "k_final_c0",
                                     "k_final_c1", "k_final_c2", "k_final_c3", "k_final_c4",
                                     "k_final_fallback", "k_copy", "k_part", "k_misc"};
struct Prof {
  bool on = false;
  std::mutex mu;
  struct Rec { int id; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  // slot = kernel id + K_COUNT * (level + 1) for per-level kernels
  static constexpr int kSlots = K_COUNT * 9;
  double ms[kSlots] = {};
  long long launches[kSlots] = {};
} g_prof;

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII bracket around one launch on stream st.
struct ProfScope {
  int id;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int id_, cudaStream_t st_) : id(id_), st(st_) {
    if (!g_prof.on) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    a = prof_event();
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    cudaEvent_t b = prof_event();
    cudaEventRecord(b, st);
    g_prof.pending.push_back({id, a, b});
  }
};

// ---- per-device caches (behind a mutex) -----------------------------------
struct DevInfo {
  int sms = 0;
  std::unordered_map<const void*, int> occ;
};
std::mutex g_mu;
std::unordered_map<int, DevInfo> g_dev;

// Keep stream-ordered allocations (workspace, host-path key buffers) cached
// in the device's default pool instead of returning them at every sync.
void ensure_pool(int dev, DevInfo& di) {
  if (di.sms != 0) return;
  cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

int grid_for(const void* fn, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& di = g_dev[dev];
  ensure_pool(dev, di);
  auto it = di.occ.find(fn);
  int occ;
  if (it == di.occ.end()) {
    if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
    if (occ < 1) occ = 1;
    di.occ[fn] = occ;
  } else {
    occ = it->second;
  }
  return di.sms * occ;
}

// ---- workspace layout ------------------------------------------------------
constexpr int kMaxGrid = 4096;  // upper bound on the streaming kernels' grid

template <typename W>
constexpr size_t hist_smem();
template <typename W>
constexpr size_t scatter_smem();

// k_hist and k_scatter run with the SAME grid so CTA b owns the same tile
// range in both (the per-(bucket, CTA) offset table relies on it).
template <typename W>
int stream_grid() {
  const int gh = grid_for((const void*)k_hist<W>, Cfg<W>::kHistThreads, hist_smem<W>());
  const int gs = grid_for((const void*)k_scatter<W>, Cfg<W>::kScatThreads, scatter_smem<W>());
  int g = gh < gs ? gh : gs;
  return g < kMaxGrid ? g : kMaxGrid;
}
struct Layout {
  size_t tmp, split0, split1, splitters, counts, childbase, seg, items[kNumLists], ctrl, total;
  unsigned long long cap_split, cap_items;
};

template <typename W>
Layout layout_for(size_t n) {
  Layout L{};
  const unsigned long long cap = Cfg<W>::kCap;
  L.cap_split = n / cap + 2;
  L.cap_items = 32 * (n / cap) + 1024;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.tmp = take(n * sizeof(W));
  L.split0 = take(L.cap_split * sizeof(SplitDesc));
  L.split1 = take(L.cap_split * sizeof(SplitDesc));
  L.splitters = take(L.cap_split * 256 * sizeof(W));
  L.counts = take(L.cap_split * kChildStride * sizeof(unsigned long long));
  L.childbase = take(L.cap_split * kChildStride * sizeof(unsigned long long));
  L.seg = take((L.cap_split + kMaxGrid) * kChildStride * sizeof(unsigned long long));
  for (int i = 0; i < kNumLists; ++i) L.items[i] = take(L.cap_items * sizeof(Item));
  L.ctrl = take(sizeof(Ctrl));
  L.total = off;
  return L;
}

template <typename W>
Params<W> make_params(W* keys, size_t n, int xf, uint64_t seed, unsigned char* ws, const Layout& L) {
  Params<W> P{};
  P.a = keys;
  P.b = reinterpret_cast<W*>(ws + L.tmp);
  P.n = n;
  P.xf = xf;
  P.cur = 0;
  P.level = 0;
  P.part_mode = 0;
  P.seed = seed;
  P.ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  P.split[0] = reinterpret_cast<SplitDesc*>(ws + L.split0);
  P.split[1] = reinterpret_cast<SplitDesc*>(ws + L.split1);
  P.splitters = reinterpret_cast<W*>(ws + L.splitters);
  P.counts = reinterpret_cast<unsigned long long*>(ws + L.counts);
  P.seg = reinterpret_cast<unsigned long long*>(ws + L.seg);
  P.childbase = reinterpret_cast<unsigned long long*>(ws + L.childbase);
  P.grid = stream_grid<W>();
  for (int i = 0; i < kNumLists; ++i) P.items[i] = reinterpret_cast<Item*>(ws + L.items[i]);
  P.cap_split = L.cap_split;
  P.cap_items = L.cap_items;
  P.out = nullptr;
  return P;
}

template <typename W>
constexpr size_t sample_smem() {
  return (size_t)padded_size<W>(kMaxSamples) * sizeof(W);
}
template <typename W>
constexpr size_t hist_smem() {
  return (size_t)kStages * stage_bytes<W>();
}
template <typename W>
constexpr size_t scatter_smem() {
  return (size_t)kStages * stage_bytes<W>() + (size_t)Cfg<W>::kTile * sizeof(unsigned short) +
         (size_t)Cfg<W>::kHistCopies * kChildStride * sizeof(unsigned);
}

// Levels a uniform input of n keys needs (>=128-way shrink per level).
int expected_levels(size_t n, size_t cap) {
  int lv = 0;
  size_t s = n;
  while (s > cap) {
    s = (s + 127) / 128;
    ++lv;
  }
  return lv;
}

template <typename W>
vxs_status launch_level(Params<W>& P, cudaStream_t st, int& launches) {
  constexpr int kSampleThreads = 512;
  {
    ProfScope ps(K_SAMPLE + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_sample<W, kSampleThreads>;
    const int g = grid_for((const void*)fn, kSampleThreads, sample_smem<W>());
    fn<<<g, kSampleThreads, sample_smem<W>(), st>>>(P);
  }
  {
    ProfScope ps(K_HIST + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_hist<W>;
    fn<<<P.grid, Cfg<W>::kHistThreads, hist_smem<W>(), st>>>(P);
  }
  {
    ProfScope ps(K_SEGSCAN + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_segscan<W>;
    const int g = grid_for((const void*)fn, 128, 0);
    fn<<<g, 128, 0, st>>>(P);
  }
  {
    ProfScope ps(K_PLAN + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_plan<W>;
    const int g = grid_for((const void*)fn, kChildStride, 0);
    fn<<<g, kChildStride, 0, st>>>(P);
  }
  {
    ProfScope ps(K_SCATTER + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_scatter<W>;
    fn<<<P.grid, Cfg<W>::kScatThreads, scatter_smem<W>(), st>>>(P);
  }
  launches += 5;
  VXS_CK(cudaGetLastError(), "level launch");
  return VXS_OK;
}

template <typename W, int CLS>
void launch_final(Params<W>& P, unsigned long long count, cudaStream_t st) {
  constexpr int T = SortClass<CLS>::T;
  constexpr int TOT = T * SortClass<CLS>::I;
  constexpr size_t smem_a = (size_t)padded_size<W>(TOT) * sizeof(W);
  constexpr size_t smem_b = (size_t)TOT * sizeof(W) + (size_t)padded_size<unsigned>(TOT) * sizeof(unsigned);
  constexpr size_t smem = smem_a > smem_b ? smem_a : smem_b;
  ProfScope ps(K_FINAL0 + CLS, st);
  auto fn = k_final<W, CLS>;
  int g = grid_for((const void*)fn, T, smem);
  if ((unsigned long long)g > count) g = (int)count;
  fn<<<g, T, smem, st>>>(P);
}

template <typename W>
vxs_status run_sort(W* keys, size_t n, int xf, uint64_t seed, void* ws, size_t ws_bytes, cudaStream_t st,
                    vxs_stats* stats) {
  const Layout L = layout_for<W>(n);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->workspace_bytes = L.total;
  }
  if (n <= 1) return VXS_OK;
  void* owned = nullptr;
  if (ws == nullptr) {
    VXS_CK(cudaMallocAsync(&owned, L.total, st), "workspace alloc");
    ws = owned;
  } else if (ws_bytes < L.total) {
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
  }
  Params<W> P = make_params<W>(keys, n, xf, seed, static_cast<unsigned char*>(ws), L);
  int launches = 0;
  {
    ProfScope ps(K_INIT, st);
    k_init<W><<<1, 32, 0, st>>>(P);
  }
  ++launches;
  Ctrl h{};
  int levels = 0;
  bool fallback = false;
  const int expect = expected_levels(n, Cfg<W>::kCap);
  if (n > (size_t)Cfg<W>::kCap) {
    int batch = expect;
    for (;;) {
      for (int i = 0; i < batch; ++i) {
        P.level = levels;
        vxs_status s = launch_level<W>(P, st, launches);
        if (s != VXS_OK) return s;
        P.cur ^= 1;
        ++levels;
      }
      VXS_CK(cudaMemcpyAsync(&h, P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "ctrl readback");
      VXS_CK(cudaStreamSynchronize(st), "level sync");
      if (h.error) {  // (final-phase overflow is checked by the error flag below)
        if (owned) cudaFreeAsync(owned, st);
        return fail(VXS_INTERNAL, "vxsort_b200: device scheduler list overflow");
      }
      if ((h.split_packed[P.cur] >> 40) == 0) break;
      fallback = true;
      batch = 1;
      if (levels > 64) {
        if (owned) cudaFreeAsync(owned, st);
        return fail(VXS_INTERNAL, "vxsort_b200: bucket recursion did not converge");
      }
    }
  } else {
    VXS_CK(cudaMemcpyAsync(&h, P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "ctrl readback");
    VXS_CK(cudaStreamSynchronize(st), "ctrl sync");
  }
  if (h.item_count[0]) { launch_final<W, 0>(P, h.item_count[0], st); ++launches; }
  if (h.item_count[1]) { launch_final<W, 1>(P, h.item_count[1], st); ++launches; }
  if (h.item_count[2]) { launch_final<W, 2>(P, h.item_count[2], st); ++launches; }
  if (h.item_count[3]) { launch_final<W, 3>(P, h.item_count[3], st); ++launches; }
  if constexpr (Cfg<W>::kCap >= 8192) {
    if (h.item_count[4]) { launch_final<W, 4>(P, h.item_count[4], st); ++launches; }
  }
  if constexpr (sizeof(W) >= 8) {
    // items rejected by the prefix-compressed base case (count lives on the device)
    if (h.item_count[0] + h.item_count[1] + h.item_count[2] + h.item_count[3] + h.item_count[4]) {
      ProfScope ps(K_FALLBACK, st);
      constexpr int ITEMS = sizeof(W) >= 16 ? 8 : 16;
      constexpr size_t smem = (size_t)padded_size<W>(SortClass<4>::T * ITEMS) * sizeof(W);
      auto fn = k_final_fallback<W>;
      const int g = grid_for((const void*)fn, SortClass<4>::T, smem);
      fn<<<g, SortClass<4>::T, smem, st>>>(P);
      ++launches;
    }
  }
  if (h.item_count[kListCopySmall] || h.item_count[kListCopyBig]) {
    ProfScope ps(K_COPY, st);
    auto fn = k_copy<W>;
    const int g = grid_for((const void*)fn, 256, 0);
    fn<<<g, 256, 0, st>>>(P);
    ++launches;
  }
  VXS_CK(cudaGetLastError(), "final launch");
  if (owned) VXS_CK(cudaFreeAsync(owned, st), "workspace free");
  if (stats) {
    stats->max_depth = (size_t)levels;
    stats->partition_calls = (size_t)h.partition_calls;
    stats->base_case_calls = (size_t)h.base_cases;
    stats->keys_partitioned = (size_t)h.keys_partitioned;
    stats->fallback_triggered = fallback ? 1 : 0;
    stats->kernel_launches = launches;
  }
  return VXS_OK;
}

// key type -> (word, transform)
int xform_for(vxs_key_type t, vxs_order o) {
  const bool d = o == VXS_DESCENDING;
  switch (t) {
    case VXS_U16: case VXS_U32: case VXS_U64: case VXS_K128: case VXS_KV64:
      return d ? XF_NOT : XF_NONE;
    case VXS_I16: case VXS_I32: case VXS_I64:
      return d ? XF_SIGN_NOT : XF_SIGN;
    case VXS_F32: case VXS_F64:
      return d ? XF_FLT_DESC : XF_FLT_ASC;
  }
  return XF_NONE;
}

int word_bytes(vxs_key_type t) {
  switch (t) {
    case VXS_I16: case VXS_U16: return 2;
    case VXS_I32: case VXS_U32: case VXS_F32: return 4;
    case VXS_I64: case VXS_U64: case VXS_F64: return 8;
    case VXS_K128: case VXS_KV64: return 16;
  }
  return 0;
}

template <class F>
vxs_status with_word(vxs_key_type t, F&& f) {
  switch (word_bytes(t)) {
    case 2: return f((uint16_t*)nullptr);
    case 4: return f((uint32_t*)nullptr);
    case 8: return f((unsigned long long*)nullptr);
    case 16: return f((U128*)nullptr);
  }
  return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: unknown key type");
}

bool valid_order(vxs_order o) { return o == VXS_ASCENDING || o == VXS_DESCENDING; }

uint64_t seed_for(uint64_t seed, int has_seed, const void* keys, size_t n) {
  // default_seed, driver.hpp:43-46 (address-dependent unless cfg.seed given)
  if (has_seed) return seed;
  return 0x9E3779B97F4A7C15ull ^ (uint64_t)(uintptr_t)keys ^ ((uint64_t)n * 0xD1B54A32D192ED03ull);
}

template <typename W>
__global__ void k_xform(W* keys, unsigned long long n, int xf, int inverse) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    keys[i] = inverse ? dec<W>(keys[i], xf) : enc<W>(keys[i], xf);
}

}  // namespace
}  // namespace vxs

using namespace vxs;

extern "C" {

vxs_status vxs_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on != 0;
  return VXS_OK;
}

void vxs_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (auto& r : g_prof.pending) {
    cudaEventSynchronize(r.b);
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
  for (int i = 0; i < Prof::kSlots; ++i) {
    g_prof.ms[i] = 0;
    g_prof.launches[i] = 0;
  }
}

int vxs_profile_read(vxs_kernel_profile* out, int cap) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (auto& r : g_prof.pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    g_prof.ms[r.id] += ms;
    g_prof.launches[r.id] += 1;
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.pending.clear();
  int k = 0;
  for (int i = 0; i < Prof::kSlots && k < cap; ++i) {
    if (!g_prof.launches[i]) continue;
    const int kid = i % K_COUNT, lv = i / K_COUNT;
    if (lv == 0) std::snprintf(out[k].name, sizeof(out[k].name), "%s", kKernelNames[kid]);
    else std::snprintf(out[k].name, sizeof(out[k].name), "%s@L%d", kKernelNames[kid], lv - 1);
    out[k].launches = g_prof.launches[i];
    out[k].total_ms = g_prof.ms[i];
    ++k;
  }
  return k;
}

const char* vxs_version(void) { return "vxsort_b200 0.1 (sm_100a)"; }

const char* vxs_last_error(void) { return g_err; }

size_t vxs_key_bytes(vxs_key_type type) { return (size_t)word_bytes(type); }

size_t vxs_base_case_capacity(vxs_key_type type) {
  switch (word_bytes(type)) {
    case 2: return Cfg<uint16_t>::kCap;
    case 4: return Cfg<uint32_t>::kCap;
    case 8: return Cfg<unsigned long long>::kCap;
    case 16: return Cfg<U128>::kCap;
  }
  return 0;
}

vxs_status vxs_sort_workspace_bytes(size_t n, vxs_key_type type, size_t* bytes) {
  if (!bytes) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: bytes is NULL");
  return with_word(type, [&](auto* tag) {
    using W = std::remove_pointer_t<decltype(tag)>;
    *bytes = layout_for<W>(n).total;
    return VXS_OK;
  });
}

vxs_status vxs_sort(void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed, int has_seed,
                    void* d_workspace, size_t workspace_bytes, void* stream, vxs_stats* stats) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (n > 0 && d_keys == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: keys is NULL");
  const int xf = xform_for(type, order);
  const uint64_t s = seed_for(seed, has_seed, d_keys, n);
  return with_word(type, [&](auto* tag) {
    using W = std::remove_pointer_t<decltype(tag)>;
    return run_sort<W>(static_cast<W*>(d_keys), n, xf, s, d_workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream), stats);
  });
}

vxs_status vxs_sort_host(void* h_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed, int has_seed,
                         vxs_stats* stats) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  const size_t kb = (size_t)word_bytes(type);
  if (kb == 0) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: unknown key type");
  if (n > 0 && h_keys == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: keys is NULL");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (n <= 1) return VXS_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(VXS_NO_DEVICE, "vxsort_b200: no CUDA device");
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    ensure_pool(dev, g_dev[dev]);
  }
  cudaStream_t st;
  VXS_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream create");
  void* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, n * kb, st);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    return cuda_fail(e, "key buffer alloc");
  }
  vxs_status s = VXS_OK;
  e = cudaMemcpyAsync(d, h_keys, n * kb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) s = cuda_fail(e, "H2D");
  if (s == VXS_OK) s = vxs_sort(d, n, type, order, seed_for(seed, has_seed, h_keys, n), 1, nullptr, 0, st, stats);
  if (s == VXS_OK) {
    e = cudaMemcpyAsync(h_keys, d, n * kb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) s = cuda_fail(e, "D2H");
  }
  cudaFreeAsync(d, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess && s == VXS_OK) s = cuda_fail(e, "sync");
  cudaStreamDestroy(st);
  if (stats) stats->kernel_launches += 0;
  return s;
}

vxs_status vxs_transform(void* d_keys, size_t n, vxs_key_type type, vxs_order order, int inverse, void* stream) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  const int xf = xform_for(type, order);
  return with_word(type, [&](auto* tag) {
    using W = std::remove_pointer_t<decltype(tag)>;
    if (n == 0) return VXS_OK;
    const int g = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_xform<W><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<W*>(d_keys), n, xf, inverse);
    VXS_CK(cudaGetLastError(), "transform");
    return VXS_OK;
  });
}

vxs_status vxs_sample(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t seed, void* d_out,
                      int s, void* stream) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (n == 0 || s <= 0) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: sample needs n > 0 and s > 0");
  const int xf = xform_for(type, order);
  return with_word(type, [&](auto* tag) {
    using W = std::remove_pointer_t<decltype(tag)>;
    const int g = std::min((s + 255) / 256, 1024);
    k_sample_out<W><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const W*>(d_keys), n, xf, seed,
                                                                       static_cast<W*>(d_out), s);
    VXS_CK(cudaGetLastError(), "sample");
    return VXS_OK;
  });
}

vxs_status vxs_partition(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, const void* d_splitters,
                         int nspl, void* d_out, uint64_t* d_seg_counts, void* d_workspace, size_t workspace_bytes,
                         void* stream) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (nspl < 0 || nspl > 255) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: nspl must be in [0, 255]");
  const int xf = xform_for(type, order);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return with_word(type, [&](auto* tag) -> vxs_status {
    using W = std::remove_pointer_t<decltype(tag)>;
    const int nseg = nspl + 1;
    if (n == 0) {
      VXS_CK(cudaMemsetAsync(d_seg_counts, 0, nseg * sizeof(uint64_t), st), "memset");
      return VXS_OK;
    }
    const Layout Lay = layout_for<W>(n);
    void* owned = nullptr;
    void* ws = d_workspace;
    if (ws == nullptr) {
      VXS_CK(cudaMallocAsync(&owned, Lay.total, st), "workspace alloc");
      ws = owned;
    } else if (workspace_bytes < Lay.total) {
      return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
    }
    Params<W> P = make_params<W>(const_cast<W*>(static_cast<const W*>(d_keys)), n, xf, 0,
                                 static_cast<unsigned char*>(ws), Lay);
    P.part_mode = 1;
    P.out = static_cast<W*>(d_out);
    int L = 1;
    while ((1 << L) - 1 < nspl) ++L;
    k_init<W><<<1, 32, 0, st>>>(P);
    k_part_setup<W><<<1, 256, 0, st>>>(P, static_cast<const W*>(d_splitters), nspl, L);
    {
      auto fn = k_hist<W>;
      fn<<<P.grid, Cfg<W>::kHistThreads, hist_smem<W>(), st>>>(P);
    }
    k_segscan<W><<<16, 128, 0, st>>>(P);
    k_plan<W><<<1, kChildStride, 0, st>>>(P);
    {
      auto fn = k_scatter<W>;
      fn<<<P.grid, Cfg<W>::kScatThreads, scatter_smem<W>(), st>>>(P);
    }
    k_part_counts<W><<<1, 256, 0, st>>>(P, nseg, reinterpret_cast<unsigned long long*>(d_seg_counts));
    VXS_CK(cudaGetLastError(), "partition");
    if (owned) VXS_CK(cudaFreeAsync(owned, st), "workspace free");
    return VXS_OK;
  });
}

}  // extern "C"
