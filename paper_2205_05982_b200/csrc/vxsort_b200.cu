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
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/vxsort_b200.h"
#include "host_pipe.cuh"
#include "sample_sort.cuh"

namespace vxs {

thread_local char g_err[512];
void set_error(const char* msg) { std::snprintf(g_err, sizeof(g_err), "%s", msg); }

namespace {

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
  K_FALLBACK, K_COPY, K_PART, K_MISC, K_FINAL_PHASE, K_COUNT
};
const char* kKernelNames[K_COUNT] = {"k_init", "k_sample", "k_hist", "k_segscan", "k_plan", "k_scatter", "k_final_c0",
                                     "k_final_c1", "k_final_c2", "k_final_c3", "k_final_c4",
                                     "k_final_fallback", "k_copy", "k_part", "k_misc",
                                     "k_final_phase" /* wall time of all base-case launches of one sort */};
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

// Stream-ordered allocations (own workspace, host-path key buffers) come
// from a PRIVATE per-device pool that keeps its memory cached between calls.
// The device's default pool is left untouched: its attributes belong to the
// host application (and to torch's allocator next to us).
std::unordered_map<int, cudaMemPool_t> g_pool;

void ensure_pool(int dev, DevInfo& di) {
  if (di.sms != 0) return;
  cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
}

// (caller holds g_mu)
cudaMemPool_t pool_for(int dev) {
  auto it = g_pool.find(dev);
  if (it != g_pool.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    return g_pool[dev] = nullptr;
  }
  unsigned long long thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  return g_pool[dev] = pool;
}

cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    pool = pool_for(dev);
  }
  if (pool == nullptr) return cudaMallocAsync(p, bytes, st);
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

// Library-owned stream-ordered buffer: freed on `st` on every exit path.
struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  AsyncBuf() = default;
  AsyncBuf(const AsyncBuf&) = delete;
  AsyncBuf& operator=(const AsyncBuf&) = delete;
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    st = s;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (cap == cudaStreamCaptureStatusActive) return cudaMallocAsync(&p, bytes, s);  // graph memory node
    return lib_malloc_async(&p, bytes, s);
  }
  cudaError_t free() {
    if (!p) return cudaSuccess;
    const cudaError_t e = cudaFreeAsync(p, st);
    p = nullptr;
    return e;
  }
  ~AsyncBuf() { free(); }
};

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
  size_t tmp, split0, split1, splitters, counts, childbase, seg, tilecnt, cta_t0, items[kNumLists], ctrl, total;
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
  // per-tile child counts of one level: at most n / Tile full tiles plus one
  // partial tile per split bucket
  L.tilecnt = take((n / Cfg<W>::kTile + L.cap_split + 1) * kChildStride * sizeof(unsigned short));
  L.cta_t0 = take((kMaxGrid + 1) * sizeof(unsigned long long));
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
  P.tilecnt = reinterpret_cast<unsigned short*>(ws + L.tilecnt);
  P.grid = stream_grid<W>();
  P.cta_t0 = reinterpret_cast<unsigned long long*>(ws + L.cta_t0);
  for (int i = 0; i < kNumLists; ++i) P.items[i] = reinterpret_cast<Item*>(ws + L.items[i]);
  P.cap_split = L.cap_split;
  P.cap_items = L.cap_items;
  P.out = nullptr;
  P.rlo = 0;
  P.rhi = n;
  return P;
}

template <typename W>
constexpr size_t sample_smem() {
  return (size_t)padded_size<W>(kMaxSamples) * sizeof(W);
}
template <typename W>
constexpr size_t hist_smem() {
  return (size_t)Cfg<W>::kHistStages * stage_bytes<W>();
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

// Launch with programmatic stream serialization (the kernels open with
// pdl_enter); plain launch while per-kernel profiling events sit between
// launches.
template <typename PT>
void pdl_launch(void (*fn)(PT), int grid, int block, size_t smem, cudaStream_t st, const PT& P) {
  if (g_prof.on) {
    fn<<<grid, block, smem, st>>>(P);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, fn, P);
}

template <typename W>
vxs_status launch_level(Params<W>& P, cudaStream_t st, int& launches) {
  constexpr int kSampleThreads = 512;
  {
    ProfScope ps(K_SAMPLE + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_sample<W, kSampleThreads>;
    const int g = grid_for((const void*)fn, kSampleThreads, sample_smem<W>());
    pdl_launch(fn, g, kSampleThreads, sample_smem<W>(), st, P);
  }
  {
    ProfScope ps(K_HIST + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_hist<W>;
    pdl_launch(fn, P.grid, Cfg<W>::kHistThreads, hist_smem<W>(), st, P);
  }
  if (P.level == 0) {  // the root bucket: every CTA holds a row (deeper levels: k_plan scans)
    ProfScope ps(K_SEGSCAN + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    pdl_launch(k_segscan_root<W>, (kChildStride + 31) / 32, 1024, 0, st, P);
  }
  {
    ProfScope ps(K_PLAN + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_plan<W>;
    const int g = grid_for((const void*)fn, kChildStride, 0);
    pdl_launch(fn, g, kChildStride, 0, st, P);
  }
  {
    ProfScope ps(K_SCATTER + K_COUNT * (1 + (P.level < 7 ? P.level : 7)), st);
    auto fn = k_scatter<W>;
    pdl_launch(fn, P.grid, Cfg<W>::kScatThreads, scatter_smem<W>(), st, P);
  }
  launches += P.level == 0 ? 5 : 4;
  P.root_init = 0;  // (only the first level's k_sample sets up the root)
  VXS_CK(cudaGetLastError(), "level launch");
  return VXS_OK;
}

template <typename W, int CLS>
void launch_final(Params<W>& P, unsigned long long count, cudaStream_t st) {
  constexpr int T = SortClass<CLS>::T;
  constexpr int TOT = T * SortClass<CLS>::I;
  constexpr size_t smem = CLS >= 1 ? BinSort<W, T, SortClass<CLS>::I>::kSmem : (size_t)padded_size<W>(TOT) * sizeof(W);
  ProfScope ps(K_FINAL0 + CLS, st);
  auto fn = k_final<W, CLS>;
  int g = grid_for((const void*)fn, T, smem);
  if ((unsigned long long)g > count) g = (int)count;
  fn<<<g, T, smem, st>>>(P);
}

// Graph-capture mode (run_sort): levels launched beyond the expected count,
// and the base-case classes launched without host-side counts.
constexpr int kCaptureGuardLevels = 2;

#define VXS_CK_STATUS(expr)        \
  do {                             \
    const vxs_status s_ = (expr);  \
    if (s_ != VXS_OK) return s_;   \
  } while (0)

// Unconverged split work after the last captured level -> error flag.
template <typename W>
__global__ void k_check_done(Params<W> P) {
  if ((P.ctrl->split_packed[P.cur] >> 40) != 0) P.ctrl->error = 4;
}

template <typename W>
int launch_final_all(Params<W>& P, cudaStream_t st) {
  constexpr unsigned long long kAll = ~0ull;  // grid = occupancy; counts are read on the device
  launch_final<W, 0>(P, kAll, st);
  launch_final<W, 1>(P, kAll, st);
  launch_final<W, 2>(P, kAll, st);
  launch_final<W, 3>(P, kAll, st);
  int launches = 4;
  if constexpr (Cfg<W>::kCap >= 8192) {
    launch_final<W, 4>(P, kAll, st);
    ++launches;
  }
  {
    auto fn = k_copy<W>;
    const int g = grid_for((const void*)fn, 256, 0);
    fn<<<g, 256, 0, st>>>(P);
  }
  {
    constexpr int ITEMS = sizeof(W) >= 16 ? 8 : 16;
    constexpr size_t smem = (size_t)padded_size<W>(SortClass<4>::T * ITEMS) * sizeof(W);
    auto fn = k_final_fallback<W>;
    const int g = grid_for((const void*)fn, SortClass<4>::T, smem);
    fn<<<g, SortClass<4>::T, smem, st>>>(P);
  }
  return launches + 2;
}

// Control-block readback through mapped pinned memory written by a 1-warp
// kernel: no copy engine involved, so the per-call sync never queues behind
// a large D2H transfer on another stream (host pipeline, user copies).
__global__ void k_ctrl_out(const Ctrl* c, Ctrl* out) {
  const unsigned* s = reinterpret_cast<const unsigned*>(c);
  volatile unsigned* d = reinterpret_cast<volatile unsigned*>(out);
  for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += 32) d[i] = s[i];
  __threadfence_system();
}

// Per (thread, device) side stream + fork/join events for the base-case
// classes (run_sort).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
struct SideStreams {
  std::unordered_map<int, SideStream> m;
  ~SideStreams() {
    for (auto& kv : m) {
      cudaEventDestroy(kv.second.fork);
      cudaEventDestroy(kv.second.join);
      cudaStreamDestroy(kv.second.s);
    }
  }
};
// Per (thread, device) cached streams: kSideBaseCase carries the base-case
// classes under the main one (run_sort); kSideHost the small host-pointer path.
enum SideKind : int { kSideBaseCase = 0, kSideHost = 1 };
SideStream* side_stream(int kind = kSideBaseCase) {
  thread_local SideStreams ts[2];
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = ts[kind].m.find(dev);
  if (it != ts[kind].m.end()) return &it->second;
  SideStream x;
  if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  return &(ts[kind].m[dev] = x);
}

struct CtrlMirror {
  std::unordered_map<int, Ctrl*> buf;
  ~CtrlMirror() {
    for (auto& kv : buf) cudaFreeHost(kv.second);
  }
};

// Per (thread, device) mapped mirror; run_sort has at most one outstanding
// readback per thread (it synchronises before returning).
Ctrl* ctrl_mirror() {
  thread_local CtrlMirror m;
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = m.buf.find(dev);
  if (it != m.buf.end()) return it->second;
  Ctrl* p = nullptr;
  if (cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(Ctrl), cudaHostAllocMapped) != cudaSuccess) return nullptr;
  m.buf[dev] = p;
  return p;
}

vxs_status read_ctrl(const Ctrl* d_ctrl, Ctrl& h, cudaStream_t st) {
  Ctrl* m = ctrl_mirror();
  if (m == nullptr) {
    VXS_CK(cudaMemcpyAsync(&h, d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "ctrl readback");
    VXS_CK(cudaStreamSynchronize(st), "ctrl sync");
    return VXS_OK;
  }
  k_ctrl_out<<<1, 32, 0, st>>>(d_ctrl, m);
  VXS_CK(cudaGetLastError(), "ctrl readback");
  VXS_CK(cudaStreamSynchronize(st), "ctrl sync");
  std::memcpy(&h, const_cast<const Ctrl*>(m), sizeof(Ctrl));
  return VXS_OK;
}

template <typename W>
vxs_status run_sort(W* keys, size_t n, int xf, uint64_t seed, void* ws, size_t ws_bytes, cudaStream_t st,
                    vxs_stats* stats, size_t rlo = 0, size_t rhi = ~size_t(0)) {
  const Layout L = layout_for<W>(n);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->workspace_bytes = L.total;
  }
  if (n <= 1) return VXS_OK;
  AsyncBuf owned;  // released on every exit path (stream-ordered)
  if (ws == nullptr) {
    VXS_CK(owned.alloc(L.total, st), "workspace alloc");
    ws = owned.p;
  } else if (ws_bytes < L.total) {
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
  }
  Params<W> P = make_params<W>(keys, n, xf, seed, static_cast<unsigned char*>(ws), L);
  P.rlo = rlo;
  P.rhi = std::min(rhi, n);
  int launches = 0;
  if (n > (size_t)Cfg<W>::kCap) {
    P.root_init = 1;  // the first k_sample sets up the root bucket
  } else {
    ProfScope ps(K_INIT, st);
    k_init<W><<<1, 32, 0, st>>>(P);
    ++launches;
  }
  Ctrl h{};
  int levels = 0;
  bool fallback = false;
  const int expect = expected_levels(n, Cfg<W>::kCap);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  VXS_CK(cudaStreamIsCapturing(st, &cap), "capture query");
  if (cap == cudaStreamCaptureStatusActive) {
    // Graph capture: no host round trip.  The expected levels plus
    // kCaptureGuardLevels more are launched (a level with no split work
    // exits at once), then every base-case class with an occupancy grid
    // reading its item count on the device.  A sort that would need still
    // more levels raises the control block's error flag instead
    // (vxs_workspace_status reports it).
    const int nlev = n > (size_t)Cfg<W>::kCap ? expect + kCaptureGuardLevels : 0;
    for (int i = 0; i < nlev; ++i) {
      P.level = i;
      VXS_CK_STATUS(launch_level<W>(P, st, launches));
      P.cur ^= 1;
    }
    k_check_done<W><<<1, 1, 0, st>>>(P);
    ++launches;
    launches += launch_final_all<W>(P, st);
    VXS_CK(cudaGetLastError(), "capture launches");
    VXS_CK(owned.free(), "workspace free");
    if (stats) {
      stats->max_depth = (size_t)nlev;
      stats->kernel_launches = launches;
    }
    return VXS_OK;
  }
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
      {
        const vxs_status rs = read_ctrl(P.ctrl, h, st);
        if (rs != VXS_OK) return rs;
        ++launches;
      }
      if (h.error)  // (final-phase overflow is checked by the error flag below)
        return fail(VXS_INTERNAL, "vxsort_b200: device scheduler list overflow");
      if ((h.split_packed[P.cur] >> 40) == 0) break;
      fallback = true;
      batch = 1;
      if (levels > 64) return fail(VXS_INTERNAL, "vxsort_b200: bucket recursion did not converge");
    }
  } else {
    const vxs_status rs = read_ctrl(P.ctrl, h, st);
    if (rs != VXS_OK) return rs;
    ++launches;
  }
  if (std::getenv("VXSORT_TRACE"))
    std::fprintf(stderr, "[vxsort n=%zu levels=%d] items c0..c4 %llu %llu %llu %llu %llu copy %llu/%llu\n", n, levels,
                 h.item_count[0], h.item_count[1], h.item_count[2], h.item_count[3], h.item_count[4],
                 h.item_count[kListCopySmall], h.item_count[kListCopyBig]);
  if (std::getenv("VXSORT_TRACE"))
    for (int l = 0; l < levels && l < 8; ++l)
      std::fprintf(stderr, "  level %d buckets: splitters %u radix %u piecewise %u piecewise-log %u\n", l, h.modes[l][0],
                   h.modes[l][1], h.modes[l][2], h.modes[l][3]);
  ProfScope phase(K_FINAL_PHASE, st);  // (closes at the end of run_sort's final block)
  // The size classes and the equality-bucket copy touch disjoint items: the
  // class holding the most keys runs on the caller's stream, the rest on a
  // side stream underneath it (forked and joined with events, no host sync);
  // the fallback for rejected items follows the join.
  {
    constexpr unsigned long long kClassCap[5] = {256, 1024, 2048, 4096, 8192};
    int main_cls = 0;
    for (int c = 1; c < kNumSortClasses; ++c)
      if (h.item_count[c] * kClassCap[c] > h.item_count[main_cls] * kClassCap[main_cls]) main_cls = c;
    const bool copy = h.item_count[kListCopySmall] || h.item_count[kListCopyBig];
    int others = copy ? 1 : 0;
    for (int c = 0; c < kNumSortClasses; ++c) others += (c != main_cls && h.item_count[c]) ? 1 : 0;
    static const bool serial = std::getenv("VXSORT_SERIAL_CLASSES") != nullptr;  // (diagnostics)
    SideStream* ss = (others && !serial) ? side_stream() : nullptr;
    cudaStream_t sd = ss ? ss->s : st;
    if (ss) {
      VXS_CK(cudaEventRecord(ss->fork, st), "fork");
      VXS_CK(cudaStreamWaitEvent(sd, ss->fork, 0), "fork wait");
    }
    auto launch_cls = [&](int c, cudaStream_t s2) {
      switch (c) {
        case 0: launch_final<W, 0>(P, h.item_count[0], s2); break;
        case 1: launch_final<W, 1>(P, h.item_count[1], s2); break;
        case 2: launch_final<W, 2>(P, h.item_count[2], s2); break;
        case 3: launch_final<W, 3>(P, h.item_count[3], s2); break;
        default:
          if constexpr (Cfg<W>::kCap >= 8192) launch_final<W, 4>(P, h.item_count[4], s2);
          break;
      }
      ++launches;
    };
    for (int c = 0; c < kNumSortClasses; ++c)
      if (c != main_cls && h.item_count[c]) launch_cls(c, sd);
    if (copy) {
      ProfScope ps(K_COPY, sd);
      auto fn = k_copy<W>;
      const int g = grid_for((const void*)fn, 256, 0);
      fn<<<g, 256, 0, sd>>>(P);
      ++launches;
    }
    if (h.item_count[main_cls]) launch_cls(main_cls, st);
    if (ss) {
      // always join (even after a failed record/launch): the workspace is
      // released on st and must outlive the side-stream kernels
      const cudaError_t ej = cudaEventRecord(ss->join, sd);
      const cudaError_t ew = ej == cudaSuccess ? cudaStreamWaitEvent(st, ss->join, 0) : cudaErrorUnknown;
      if (ej != cudaSuccess || ew != cudaSuccess) {
        cudaStreamSynchronize(sd);  // last resort: order by the host
        return cuda_fail(ej != cudaSuccess ? ej : ew, "join");
      }
    }
  }
  {
    // items rejected by the counting-sort base case (count lives on the device)
    if (h.item_count[1] + h.item_count[2] + h.item_count[3] + h.item_count[4]) {
      ProfScope ps(K_FALLBACK, st);
      constexpr int ITEMS = sizeof(W) >= 16 ? 8 : 16;
      constexpr size_t smem = (size_t)padded_size<W>(SortClass<4>::T * ITEMS) * sizeof(W);
      auto fn = k_final_fallback<W>;
      const int g = grid_for((const void*)fn, SortClass<4>::T, smem);
      fn<<<g, SortClass<4>::T, smem, st>>>(P);
      ++launches;
    }
  }
  VXS_CK(cudaGetLastError(), "final launch");
  VXS_CK(owned.free(), "workspace free");
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

// ---- host-pointer pipeline (kernels in host_pipe.cuh) --------

// Host-side "first k stages are ready" counter shared with a copy thread.
struct Ready {
  std::mutex mu;
  std::condition_variable cv;
  int k = 0;
  void post(int v) {
    {
      std::lock_guard<std::mutex> lk(mu);
      k = v;
    }
    cv.notify_all();
  }
  void wait(int v) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return k >= v; });
  }
};

// Fixed pool of host threads for pageable <-> pinned staging copies (one
// memcpy thread measured ~14 GB/s on the GPU box's host, 8 threads ~60 GB/s,
// i.e. faster than PCIe).
class CopyPool {
 public:
  explicit CopyPool(int nthreads) : n_(nthreads) {
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // Parallel memcpy; returns when every part is copied.
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(1) << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = static_cast<unsigned char*>(dst);
    src_ = static_cast<const unsigned char*>(src);
    bytes_ = bytes;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void loop(int i) {
    unsigned long long seen = 0;
    for (;;) {
      unsigned char* d;
      const unsigned char* s;
      size_t b;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        d = dst_;
        s = src_;
        b = bytes_;
      }
      const size_t per = ((b + n_ - 1) / n_ + 63) & ~size_t(63);  // n_ * per >= b
      const size_t lo = std::min(b, per * i), hi = std::min(b, lo + per);
      if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  unsigned char* dst_ = nullptr;
  const unsigned char* src_ = nullptr;
  size_t bytes_ = 0;
  int pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

constexpr int kMergeStreams = 4;
constexpr int kStageSlots = 4;                        // per direction
constexpr size_t kStageBytes = size_t(8) << 20;       // per slot

// Per-device pipeline context: streams, events and the pinned staging ring,
// created once and reused (one host-pointer sort at a time per device).
struct PipeCtx {
  int dev = 0;
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr, s_mrg[kMergeStreams] = {};
  cudaEvent_t ev_in[kPipeMaxChunks], ev_sl[kPipeMaxSlices], ev_alloc, ev_done, ev_mrg[kMergeStreams];
  unsigned char* stage = nullptr;  // 2 * kStageSlots * kStageBytes pinned
  cudaEvent_t ev_stage[2 * kStageSlots];
  std::unique_ptr<CopyPool> pool;
  std::mutex busy;
  bool ok = false;
  explicit PipeCtx(int d) : dev(d) {
    bool good = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&s_cmp, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& s : s_mrg) good = good && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& e : ev_in) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    for (auto& e : ev_sl) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    for (auto& e : ev_mrg) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    for (auto& e : ev_stage) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    good = good && cudaEventCreateWithFlags(&ev_alloc, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) == cudaSuccess;
    ok = good;
  }
  // Pinned staging ring + copy threads, only when a pageable source shows up.
  bool ensure_staging() {
    if (stage) return true;
    if (cudaHostAlloc(reinterpret_cast<void**>(&stage), 2 * kStageSlots * kStageBytes, cudaHostAllocDefault) !=
        cudaSuccess) {
      stage = nullptr;
      cudaGetLastError();
      return false;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    pool = std::make_unique<CopyPool>((int)std::max(1u, std::min(8u, hc ? hc / 2 : 4u)));
    return true;
  }
  unsigned char* slot(int i) { return stage + (size_t)i * kStageBytes; }
};

std::mutex g_pipe_mu;
std::unordered_map<int, std::unique_ptr<PipeCtx>> g_pipe;

PipeCtx* pipe_ctx(int dev) {
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  auto& p = g_pipe[dev];
  if (!p) p = std::make_unique<PipeCtx>(dev);
  return p->ok ? p.get() : nullptr;
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct GatherSet {
  unsigned long long src[kPipeMaxChunks];
  unsigned long long len[kPipeMaxChunks];
  unsigned long long dst[kPipeMaxChunks];
};

// blockIdx.y = chunk piece; copies the piece's keys of one slice into place.
template <typename W>
__global__ void k_gather(const W* a, W* b, GatherSet g) {
  const int c = blockIdx.y;
  const W* src = a + g.src[c];
  W* dst = b + g.dst[c];
  const unsigned long long len = g.len[c];
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < len;
       i += (unsigned long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Chunks / slices of the pipeline: VXSORT_HOST_CHUNKS=1 disables it (one
// H2D, one device sort, one D2H).
void pipe_dims(size_t n, size_t kb, int& C, int& S) {
  const size_t bytes = n * kb;
  // (16 chunks: swept 4-32 on 400 MB.  Pinned sources are within noise from
  // 6 to 16 -- fewer chunks shorten the run of small tail sorts, more merge
  // rounds cost nothing visible -- and the staged pageable path needs the
  // finer pipelining: 20.3 ms with 16 chunks against 25.6 with 8)
  C = bytes >= (size_t(64) << 20) ? 16 : 1;
  S = bytes >= (size_t(256) << 20) ? 64 : 32;
  if (const char* e = std::getenv("VXSORT_HOST_CHUNKS")) C = std::atoi(e);
  if (const char* e = std::getenv("VXSORT_HOST_SLICES")) S = std::atoi(e);
  C = std::max(1, std::min(C, kPipeMaxChunks));
  int s2 = 2;
  while (s2 * 2 <= std::min(std::max(S, 2), kPipeMaxSlices)) s2 *= 2;
  S = s2;
  if ((size_t)C * 4096 > n) C = 1;
}

// Chunk boundaries: equal chunks, then a geometric tail (1/2, 1/4, 1/8 of a
// chunk) so the sort of the last chunk to land -- the only one not hidden
// under the transfer -- is short.
void chunk_bounds(size_t n, int C, ChunkSet& cs) {
  cs.C = C;
  double w[kPipeMaxChunks];
  double tot = 0;
  int taper = 3;  // the last chunks shrink (1/2, 1/4, 1/8): the sort exposed after the last H2D is short
  if (const char* e = std::getenv("VXSORT_HOST_TAPER")) taper = std::atoi(e);
  for (int c = 0; c < C; ++c) {
    const int from_end = C - 1 - c;
    w[c] = (C >= 6 && from_end < taper) ? 1.0 / (double)(1 << (taper - from_end)) : 1.0;
    tot += w[c];
  }
  double acc = 0;
  cs.off[0] = 0;
  for (int c = 0; c < C; ++c) {
    acc += w[c];
    cs.off[c + 1] = c + 1 == C ? n : (unsigned long long)((double)n * acc / tot);
  }
}

void add_stats(vxs_stats& acc, const vxs_stats& s) {
  acc.max_depth = std::max(acc.max_depth, s.max_depth);
  acc.partition_calls += s.partition_calls;
  acc.base_case_calls += s.base_case_calls;
  acc.keys_partitioned += s.keys_partitioned;
  acc.fallback_triggered |= s.fallback_triggered;
  acc.kernel_launches += s.kernel_launches;
  acc.workspace_bytes = std::max(acc.workspace_bytes, s.workspace_bytes);
}

template <typename W>
vxs_status host_pipeline(PipeCtx& X, W* h, size_t n, int xf, uint64_t seed, int C, int S, vxs_stats* stats) {
  const int dev = X.dev;
  const bool staged = !host_is_pinned(h);
  if (staged && !X.ensure_staging()) return fail(VXS_OUT_OF_MEMORY, "vxsort_b200: pinned staging alloc failed");
  const bool trace = std::getenv("VXSORT_PIPE_TRACE") != nullptr;
  cudaEvent_t tev[6];  // start, H2D done, chunk sorts done, bounds done, first slice merged, D2H done
  if (trace)
    for (auto& t : tev) cudaEventCreate(&t);
  vxs_stats acc{};
  W *A = nullptr, *B = nullptr;
  unsigned char* small = nullptr;
  const size_t bounds_bytes = sizeof(unsigned long long) * C * (S + 1);
  vxs_status st = VXS_OK;
  cudaError_t e = lib_malloc_async(reinterpret_cast<void**>(&A), n * sizeof(W), X.s_cmp);
  if (e == cudaSuccess) e = lib_malloc_async(reinterpret_cast<void**>(&B), n * sizeof(W), X.s_cmp);
  if (e == cudaSuccess) e = lib_malloc_async(reinterpret_cast<void**>(&small), 256 + sizeof(W) * kPipeMaxSlices + bounds_bytes, X.s_cmp);
  if (e != cudaSuccess) st = cuda_fail(e, "pipeline alloc");
  W* spl = reinterpret_cast<W*>(small);
  unsigned long long* d_bounds = reinterpret_cast<unsigned long long*>(small + 256 + sizeof(W) * kPipeMaxSlices);
  cudaEventRecord(X.ev_alloc, X.s_cmp);
  cudaStreamWaitEvent(X.s_in, X.ev_alloc, 0);
  cudaStreamWaitEvent(X.s_out, X.ev_alloc, 0);
  ChunkSet cs{};
  chunk_bounds(n, C, cs);

  // 1. chunked H2D on its own thread (a pageable source goes through the
  //    pinned staging ring: parallel memcpy of piece i+1 overlaps the DMA of
  //    piece i)
  Ready in_ready, out_ready;
  std::vector<unsigned long long> sl_off(S + 1, 0);
  cudaError_t thread_err[2] = {cudaSuccess, cudaSuccess};
  const bool ok_alloc = st == VXS_OK;
  if (trace) cudaEventRecord(tev[0], X.s_in);
  std::thread tin([&] {
    cudaSetDevice(dev);
    int piece = 0;
    for (int c = 0; c < C; ++c) {
      if (ok_alloc && thread_err[0] == cudaSuccess) {
        const size_t b0 = cs.off[c] * sizeof(W), b1 = cs.off[c + 1] * sizeof(W);
        const unsigned char* src = reinterpret_cast<const unsigned char*>(h);
        unsigned char* dst = reinterpret_cast<unsigned char*>(A);
        if (!staged) {
          const cudaError_t ce = cudaMemcpyAsync(dst + b0, src + b0, b1 - b0, cudaMemcpyHostToDevice, X.s_in);
          if (ce != cudaSuccess) thread_err[0] = ce;
        } else {
          for (size_t p = b0; p < b1 && thread_err[0] == cudaSuccess; p += kStageBytes, ++piece) {
            const int sl = piece % kStageSlots;
            const size_t len = std::min(kStageBytes, b1 - p);
            cudaEventSynchronize(X.ev_stage[sl]);  // slot's previous DMA done
            X.pool->copy(X.slot(sl), src + p, len);
            cudaError_t ce = cudaMemcpyAsync(dst + p, X.slot(sl), len, cudaMemcpyHostToDevice, X.s_in);
            if (ce == cudaSuccess) ce = cudaEventRecord(X.ev_stage[sl], X.s_in);
            if (ce != cudaSuccess) thread_err[0] = ce;
          }
        }
      }
      cudaEventRecord(X.ev_in[c], X.s_in);
      if (trace && c == C - 1) cudaEventRecord(tev[1], X.s_in);
      in_ready.post(c + 1);
    }
  });
  // 3b. D2H of finished slices, in order (own thread for the same reason)
  std::thread tout([&] {
    cudaSetDevice(dev);
    struct Pend {
      int slot;
      unsigned char* dst;
      size_t len;
    };
    Pend q[kStageSlots];
    int qh = 0, qn = 0, next = 0;
    auto drain_one = [&] {
      Pend& p = q[qh];
      cudaEventSynchronize(X.ev_stage[kStageSlots + p.slot]);
      X.pool->copy(p.dst, X.slot(kStageSlots + p.slot), p.len);
      qh = (qh + 1) % kStageSlots;
      --qn;
    };
    if (!staged) {
      // Pinned destination: slices leave in groups of 1, 1, 2, 4, 8, ... --
      // one cudaMemcpyAsync per group.  The merges run several times faster
      // than PCIe drains them, so only the first slices are latency-critical;
      // 64 separate copies cost ~0.5 ms of per-copy overhead on a 7.2 ms D2H.
      int s = 0, gsz = 1, ngroups = 0;
      while (s < S) {
        const int s1 = std::min(S, s + gsz);
        out_ready.wait(s1);
        const unsigned long long b0 = sl_off[s], b1 = sl_off[s1];
        if (b1 > b0 && thread_err[1] == cudaSuccess) {
          for (int j = s; j < s1; ++j)
            if (sl_off[j + 1] > sl_off[j]) cudaStreamWaitEvent(X.s_out, X.ev_sl[j], 0);
          const cudaError_t ce = cudaMemcpyAsync(h + b0, B + b0, (b1 - b0) * sizeof(W), cudaMemcpyDeviceToHost, X.s_out);
          if (ce != cudaSuccess) thread_err[1] = ce;
        }
        s = s1;
        if (++ngroups >= 2) gsz *= 2;
      }
      return;
    }
    for (int s = 0; s < S; ++s) {
      out_ready.wait(s + 1);
      const unsigned long long len = sl_off[s + 1] - sl_off[s];
      if (len == 0 || thread_err[1] != cudaSuccess) continue;
      cudaStreamWaitEvent(X.s_out, X.ev_sl[s], 0);
      if (!staged) {
        const cudaError_t ce =
            cudaMemcpyAsync(h + sl_off[s], B + sl_off[s], len * sizeof(W), cudaMemcpyDeviceToHost, X.s_out);
        if (ce != cudaSuccess) thread_err[1] = ce;
        continue;
      }
      const unsigned char* src = reinterpret_cast<const unsigned char*>(B + sl_off[s]);
      unsigned char* dst = reinterpret_cast<unsigned char*>(h + sl_off[s]);
      for (size_t p = 0; p < (size_t)(len * sizeof(W)) && thread_err[1] == cudaSuccess; p += kStageBytes) {
        if (qn == kStageSlots) drain_one();
        const int sl = next;
        next = (next + 1) % kStageSlots;
        const size_t l = std::min(kStageBytes, (size_t)(len * sizeof(W)) - p);
        cudaError_t ce = cudaMemcpyAsync(X.slot(kStageSlots + sl), src + p, l, cudaMemcpyDeviceToHost, X.s_out);
        if (ce == cudaSuccess) ce = cudaEventRecord(X.ev_stage[kStageSlots + sl], X.s_out);
        if (ce != cudaSuccess) {
          thread_err[1] = ce;
          break;
        }
        q[(qh + qn) % kStageSlots] = Pend{sl, dst + p, l};
        ++qn;
      }
    }
    while (qn) drain_one();
  });
  // 1b. sort each chunk as it lands (one workspace for all the chunk sorts:
  //     no stream-ordered alloc / free pair per chunk)
  std::vector<cudaEvent_t> tcs;  // (trace: per-chunk sort completion)
  unsigned char* cws = nullptr;
  size_t cws_bytes = 0;
  for (int c = 0; c < C; ++c) cws_bytes = std::max(cws_bytes, layout_for<W>(cs.off[c + 1] - cs.off[c]).total);
  if (st == VXS_OK) {
    e = lib_malloc_async(reinterpret_cast<void**>(&cws), cws_bytes, X.s_cmp);
    if (e != cudaSuccess) st = cuda_fail(e, "pipeline workspace alloc");
  }
  for (int c = 0; c < C; ++c) {
    in_ready.wait(c + 1);
    if (st != VXS_OK) continue;
    cudaStreamWaitEvent(X.s_cmp, X.ev_in[c], 0);
    vxs_stats sc{};
    st = run_sort<W>(A + cs.off[c], cs.off[c + 1] - cs.off[c], xf, seed + (uint64_t)c * 0x9E3779B97F4A7C15ull,
                     cws, cws_bytes, X.s_cmp, &sc);
    add_stats(acc, sc);
    if (trace) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, X.s_cmp);
      tcs.push_back(ev);
    }
  }
  // 2. global splitters from a regular sample of the sorted chunks; bounds
  std::vector<unsigned long long> hb((size_t)C * (S + 1), 0);
  if (trace) cudaEventRecord(tev[2], X.s_cmp);
  if (st == VXS_OK) {
    const size_t smem = (size_t)padded_size<W>(kPipeCand) * sizeof(W);
    cudaFuncSetAttribute(k_pick_splitters<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pick_splitters<W><<<1, 512, smem, X.s_cmp>>>(A, cs, xf, S, spl);
    k_slice_bounds<W><<<(C * (S + 1) + 255) / 256, 256, 0, X.s_cmp>>>(A, cs, xf, S, spl, d_bounds);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(hb.data(), d_bounds, bounds_bytes, cudaMemcpyDeviceToHost, X.s_cmp);
    if (trace) cudaEventRecord(tev[3], X.s_cmp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(X.s_cmp);
    if (e != cudaSuccess) st = cuda_fail(e, "pipeline splitters");
    acc.kernel_launches += 2;
  }
  // 3. per slice: merge the C sorted sub-runs (pairwise merge-path rounds,
  //    no host sync; slices round-robin over kMergeStreams streams, each with
  //    its own ping-pong buffer), hand the slice to the D2H thread
  W* Tb = nullptr;
  unsigned long long max_len = 0;
  if (st == VXS_OK) {
    for (int s = 0; s < S; ++s) {
      unsigned long long len = 0;
      for (int c = 0; c < C; ++c) len += hb[(size_t)c * (S + 1) + s + 1] - hb[(size_t)c * (S + 1) + s];
      max_len = std::max(max_len, len);
    }
    max_len = std::max<unsigned long long>(max_len, 1);
    e = lib_malloc_async(reinterpret_cast<void**>(&Tb), kMergeStreams * max_len * sizeof(W), X.s_cmp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(X.s_cmp);
    if (e != cudaSuccess) st = cuda_fail(e, "pipeline merge buffer");
  }
  constexpr int kMT = 256, kMI = 8, kMTile = kMT * kMI;
  const size_t merge_smem = (size_t)padded_size<W>(kMTile) * sizeof(W);
  int used_streams = 0;
  for (int s = 0; s < S; ++s) {
    unsigned long long len = 0;
    Runs R{};
    if (st == VXS_OK) {
      for (int c = 0; c < C; ++c) {
        const unsigned long long b0 = hb[(size_t)c * (S + 1) + s], b1 = hb[(size_t)c * (S + 1) + s + 1];
        if (b1 == b0) continue;
        R.src[R.m] = cs.off[c] + b0;
        R.len[R.m] = b1 - b0;
        ++R.m;
        len += b1 - b0;
      }
    }
    sl_off[s + 1] = sl_off[s] + len;
    if (len) {
      const int k = used_streams % kMergeStreams;
      ++used_streams;
      cudaStream_t ms = X.s_mrg[k];
      W* tmp = Tb + (size_t)k * max_len;
      if (R.m == 1) {
        GatherSet g{};
        g.src[0] = R.src[0];
        g.len[0] = len;
        g.dst[0] = sl_off[s];
        const int gx = (int)std::min<unsigned long long>((len + 2047) / 2048, 1184);
        k_gather<W><<<dim3(gx, 1), 256, 0, ms>>>(A, B, g);
        acc.kernel_launches += 1;
      } else {
        int rounds = 0;
        while ((1 << rounds) < R.m) ++rounds;
        bool to_b = (rounds & 1) != 0;
        const W* in = A;
        const unsigned grid = (unsigned)((len + kMTile - 1) / kMTile);
        for (int r = 0; r < rounds; ++r) {
          W* out = to_b ? B + sl_off[s] : tmp;
          k_merge_pairs<W, kMT, kMI><<<grid, kMT, merge_smem, ms>>>(in, R, out, xf);
          acc.kernel_launches += 1;
          Runs R2{};
          R2.m = (R.m + 1) / 2;
          unsigned long long pos = 0;
          for (int j = 0; j < R2.m; ++j) {
            R2.src[j] = pos;
            R2.len[j] = R.len[2 * j] + (2 * j + 1 < R.m ? R.len[2 * j + 1] : 0ull);
            pos += R2.len[j];
          }
          R = R2;
          in = out;
          to_b = !to_b;
        }
      }
      e = cudaGetLastError();
      if (e != cudaSuccess && st == VXS_OK) st = cuda_fail(e, "pipeline merge");
      cudaEventRecord(X.ev_sl[s], ms);
      if (trace && sl_off[s] == 0) cudaEventRecord(tev[4], ms);
    }
    out_ready.post(s + 1);
  }
  tin.join();
  tout.join();
  // frees are ordered after the merges and the D2H copies
  for (int k = 0; k < kMergeStreams; ++k) {
    cudaEventRecord(X.ev_mrg[k], X.s_mrg[k]);
    cudaStreamWaitEvent(X.s_cmp, X.ev_mrg[k], 0);
  }
  cudaEventRecord(X.ev_done, X.s_out);
  if (trace) {
    cudaEventRecord(tev[5], X.s_out);
    cudaEventSynchronize(tev[5]);
    float t[6] = {};
    for (int i = 1; i < 6; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[i]);
    std::fprintf(stderr,
                 "[vxsort pipe C=%d S=%d %s] h2d %.3f  chunk-sorts %.3f  bounds %.3f  slice0 %.3f  d2h-done %.3f ms\n",
                 C, S, staged ? "staged" : "pinned", t[1], t[2], t[3], t[4], t[5]);
    std::fprintf(stderr, "  chunk sorts done at (ms):");
    for (auto& ev : tcs) {
      float ms = 0;
      cudaEventElapsedTime(&ms, tev[0], ev);
      std::fprintf(stderr, " %.2f", ms);
      cudaEventDestroy(ev);
    }
    std::fprintf(stderr, "\n");
    for (auto& x : tev) cudaEventDestroy(x);
  }
  cudaStreamWaitEvent(X.s_cmp, X.ev_done, 0);
  if (A) cudaFreeAsync(A, X.s_cmp);
  if (B) cudaFreeAsync(B, X.s_cmp);
  if (small) cudaFreeAsync(small, X.s_cmp);
  if (Tb) cudaFreeAsync(Tb, X.s_cmp);
  if (cws) cudaFreeAsync(cws, X.s_cmp);
  e = cudaStreamSynchronize(X.s_cmp);
  if (st == VXS_OK && e != cudaSuccess) st = cuda_fail(e, "pipeline sync");
  if (st == VXS_OK && thread_err[0] != cudaSuccess) st = cuda_fail(thread_err[0], "H2D");
  if (st == VXS_OK && thread_err[1] != cudaSuccess) st = cuda_fail(thread_err[1], "D2H");
  if (st == VXS_OK && sl_off[S] != n) st = fail(VXS_INTERNAL, "vxsort_b200: pipeline slices do not cover the input");
  if (stats) {
    acc.max_depth += 1;  // the slice merge stage
    acc.workspace_bytes += (2 * n + kMergeStreams * max_len) * sizeof(W);
    *stats = acc;
  }
  return st;
}

// ---- stable argsort / key+value sort ------------------------
// Key and index packed into one word (PAPER.md:907-910 row-id trick): the
// packed words are distinct, so the sort is stable by construction.

__device__ __forceinline__ void pack_kv(unsigned long long& p, unsigned long long k, unsigned long long i) {
  p = (k << 32) | i;
}
__device__ __forceinline__ void pack_kv(U128& p, unsigned long long k, unsigned long long i) { p = U128{i, k}; }
__device__ __forceinline__ unsigned long long packed_idx(const unsigned long long& p) { return p & 0xFFFFFFFFull; }
__device__ __forceinline__ unsigned long long packed_idx(const U128& p) { return p.lo; }
__device__ __forceinline__ unsigned long long packed_key(const unsigned long long& p) { return p >> 32; }
__device__ __forceinline__ unsigned long long packed_key(const U128& p) { return p.hi; }

template <typename WK, typename WP>
__global__ void k_pack_index(const WK* keys, WP* out, unsigned long long n, int xf) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    WP p;
    pack_kv(p, (unsigned long long)enc<WK>(ldcs(keys + i), xf), i);
    out[i] = p;
  }
}

template <typename WK, typename WP, typename V>
__global__ void k_unpack_index(const WP* packed, unsigned long long n, int xf, unsigned long long* idx_out,
                               WK* keys_out, const V* vals_in, V* vals_out) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const WP p = packed[i];
    const unsigned long long j = packed_idx(p);
    if (idx_out) idx_out[i] = j;
    if (keys_out) keys_out[i] = dec<WK>((WK)packed_key(p), xf);
    if (vals_out) vals_out[i] = vals_in[j];
  }
}

bool pack_wide(size_t n, size_t kb) { return kb >= 8 || n > (size_t(1) << 32); }

struct PackLayout {
  size_t packed, sort_ws, sort_ws_bytes, vals, total;
};

PackLayout pack_layout(size_t n, size_t kb, size_t vb) {
  PackLayout L{};
  const bool wide = pack_wide(n, kb);
  size_t off = 0;
  L.packed = off;
  off = align_up(off + n * (wide ? 16 : 8), 256);
  L.sort_ws = off;
  L.sort_ws_bytes = wide ? layout_for<U128>(n).total : layout_for<unsigned long long>(n).total;
  off = align_up(off + L.sort_ws_bytes, 256);
  L.vals = off;
  off = align_up(off + n * vb, 256);
  L.total = off;
  return L;
}

bool valid_value_bytes(size_t vb) { return vb == 1 || vb == 2 || vb == 4 || vb == 8 || vb == 16; }

template <class F>
vxs_status with_value(size_t vb, F&& f) {
  switch (vb) {
    case 1: return f((uint8_t*)nullptr);
    case 2: return f((uint16_t*)nullptr);
    case 4: return f((uint32_t*)nullptr);
    case 8: return f((unsigned long long*)nullptr);
    case 16: return f((U128*)nullptr);
  }
  return f((uint8_t*)nullptr);
}

// keys_in -> (idx_out?, keys_out?, values permuted in place?)
template <typename WK, typename WP, typename V>
vxs_status run_packed(const WK* keys_in, size_t n, int xf, uint64_t seed, unsigned long long* idx_out, WK* keys_out,
                      V* vals, size_t vb, void* ws, size_t ws_bytes, cudaStream_t st, vxs_stats* stats) {
  const PackLayout L = pack_layout(n, sizeof(WK), vals ? vb : 0);
  AsyncBuf owned;
  if (ws == nullptr) {
    VXS_CK(owned.alloc(std::max<size_t>(L.total, 256), st), "workspace alloc");
    ws = owned.p;
  } else if (ws_bytes < L.total) {
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
  }
  unsigned char* base = static_cast<unsigned char*>(ws);
  WP* packed = reinterpret_cast<WP*>(base + L.packed);
  V* vtmp = reinterpret_cast<V*>(base + L.vals);
  const int g = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  {
    ProfScope ps(K_MISC, st);
    k_pack_index<WK, WP><<<g, 256, 0, st>>>(keys_in, packed, n, xf);
  }
  VXS_CK(cudaGetLastError(), "pack");
  vxs_status s = run_sort<WP>(packed, n, XF_NONE, seed, base + L.sort_ws, L.sort_ws_bytes, st, stats);
  if (s != VXS_OK) return s;
  {
    ProfScope ps(K_MISC, st);
    k_unpack_index<WK, WP, V><<<g, 256, 0, st>>>(packed, n, xf, idx_out, keys_out, vals, vals ? vtmp : nullptr);
  }
  VXS_CK(cudaGetLastError(), "unpack");
  if (vals) VXS_CK(cudaMemcpyAsync(vals, vtmp, n * vb, cudaMemcpyDeviceToDevice, st), "values copy");
  VXS_CK(owned.free(), "workspace free");
  if (stats) {
    stats->kernel_launches += 2;
    stats->workspace_bytes = L.total;
  }
  return VXS_OK;
}

template <typename WK, typename V>
vxs_status dispatch_packed(const WK* keys_in, size_t n, int xf, uint64_t seed, unsigned long long* idx_out,
                           WK* keys_out, V* vals, size_t vb, void* ws, size_t ws_bytes, cudaStream_t st,
                           vxs_stats* stats) {
  if (pack_wide(n, sizeof(WK)))
    return run_packed<WK, U128, V>(keys_in, n, xf, seed, idx_out, keys_out, vals, vb, ws, ws_bytes, st, stats);
  return run_packed<WK, unsigned long long, V>(keys_in, n, xf, seed, idx_out, keys_out, vals, vb, ws, ws_bytes, st,
                                               stats);
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

vxs_status vxs_workspace_status(const void* d_workspace, size_t n, vxs_key_type type, void* stream,
                                vxs_stats* stats) {
  if (!d_workspace) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: workspace is NULL");
  return with_word(type, [&](auto* tag) -> vxs_status {
    using W = std::remove_pointer_t<decltype(tag)>;
    const Layout L = layout_for<W>(n);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (n <= 1) {  // a sort of <= 1 key never touches the workspace (run_sort)
      if (stats) stats->workspace_bytes = L.total;
      return VXS_OK;
    }
    Ctrl h{};
    VXS_CK_STATUS(read_ctrl(reinterpret_cast<const Ctrl*>(static_cast<const unsigned char*>(d_workspace) + L.ctrl), h,
                            static_cast<cudaStream_t>(stream)));
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      int lv = 0;
      for (int l = 0; l < 8; ++l)
        if (h.modes[l][0] + h.modes[l][1] + h.modes[l][2]) lv = l + 1;
      stats->max_depth = (size_t)lv;
      stats->partition_calls = (size_t)h.partition_calls;
      stats->base_case_calls = (size_t)h.base_cases;
      stats->keys_partitioned = (size_t)h.keys_partitioned;
      stats->workspace_bytes = L.total;
    }
    if (h.error) return fail(VXS_INTERNAL, h.error == 4 ? "vxsort_b200: captured sort needed more levels than launched"
                                                        : "vxsort_b200: device scheduler list overflow");
    return VXS_OK;
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
  {
    int C = 1, S = 2;
    pipe_dims(n, kb, C, S);
    int dev = 0;
    cudaGetDevice(&dev);
    PipeCtx* X = C > 1 ? pipe_ctx(dev) : nullptr;
    if (X) {
      const int xf = xform_for(type, order);
      const uint64_t sd = seed_for(seed, has_seed, h_keys, n);
      std::lock_guard<std::mutex> lk(X->busy);
      return with_word(type, [&](auto* tag) {
        using W = std::remove_pointer_t<decltype(tag)>;
        return host_pipeline<W>(*X, static_cast<W*>(h_keys), n, xf, sd, C, S, stats);
      });
    }
  }
  // small inputs: copy in, sort, copy out on this thread's cached stream
  SideStream* hs = side_stream(kSideHost);
  if (hs == nullptr) return fail(VXS_CUDA_ERROR, "vxsort_b200: stream create failed");
  cudaStream_t st = hs->s;
  vxs_status s = VXS_OK;
  {
    AsyncBuf d;
    cudaError_t e = d.alloc(n * kb, st);
    if (e != cudaSuccess) return cuda_fail(e, "key buffer alloc");
    e = cudaMemcpyAsync(d.p, h_keys, n * kb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) s = cuda_fail(e, "H2D");
    if (s == VXS_OK) s = vxs_sort(d.p, n, type, order, seed_for(seed, has_seed, h_keys, n), 1, nullptr, 0, st, stats);
    if (s == VXS_OK) {
      e = cudaMemcpyAsync(h_keys, d.p, n * kb, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) s = cuda_fail(e, "D2H");
    }
  }
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess && s == VXS_OK) s = cuda_fail(e, "sync");
  return s;
}

vxs_status vxs_sort_range(void* d_keys, size_t n, vxs_key_type type, vxs_order order, size_t lo, size_t hi,
                          uint64_t seed, int has_seed, void* d_workspace, size_t workspace_bytes, void* stream,
                          vxs_stats* stats) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (n > 0 && d_keys == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: keys is NULL");
  if (lo > hi || hi > n) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: sort_range needs lo <= hi <= n");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (lo == hi) return VXS_OK;
  const int xf = xform_for(type, order);
  const uint64_t s = seed_for(seed, has_seed, d_keys, n);
  return with_word(type, [&](auto* tag) {
    using W = std::remove_pointer_t<decltype(tag)>;
    return run_sort<W>(static_cast<W*>(d_keys), n, xf, s, d_workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream), stats, lo, hi);
  });
}

vxs_status vxs_argsort_workspace_bytes(size_t n, vxs_key_type type, size_t value_bytes, size_t* bytes) {
  if (!bytes) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: bytes is NULL");
  const size_t kb = (size_t)word_bytes(type);
  if (kb == 0 || kb == 16) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: argsort supports 16/32/64-bit keys");
  if (value_bytes && !valid_value_bytes(value_bytes))
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: value_bytes must be 1, 2, 4, 8 or 16");
  *bytes = pack_layout(n, kb, value_bytes).total;
  return VXS_OK;
}

vxs_status vxs_argsort(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, uint64_t* d_indices,
                       void* d_sorted_keys, uint64_t seed, int has_seed, void* d_workspace, size_t workspace_bytes,
                       void* stream, vxs_stats* stats) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  const size_t kb = (size_t)word_bytes(type);
  if (kb == 0 || kb == 16) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: argsort supports 16/32/64-bit keys");
  if (n > 0 && (d_keys == nullptr || d_indices == nullptr))
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: keys/indices is NULL");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (n == 0) return VXS_OK;
  const int xf = xform_for(type, order);
  const uint64_t sd = seed_for(seed, has_seed, d_keys, n);
  return with_word(type, [&](auto* tag) -> vxs_status {
    using WK = std::remove_pointer_t<decltype(tag)>;
    if constexpr (sizeof(WK) == 16) {
      return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: argsort supports 16/32/64-bit keys");
    } else {
      return dispatch_packed<WK, uint8_t>(static_cast<const WK*>(d_keys), n, xf, sd,
                                          reinterpret_cast<unsigned long long*>(d_indices),
                                          static_cast<WK*>(d_sorted_keys), nullptr, 0, d_workspace, workspace_bytes,
                                          static_cast<cudaStream_t>(stream), stats);
    }
  });
}

vxs_status vxs_sort_pairs(void* d_keys, void* d_values, size_t value_bytes, size_t n, vxs_key_type type,
                          vxs_order order, uint64_t seed, int has_seed, void* d_workspace, size_t workspace_bytes,
                          void* stream, vxs_stats* stats) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  const size_t kb = (size_t)word_bytes(type);
  if (kb == 0 || kb == 16) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: sort_pairs supports 16/32/64-bit keys");
  if (!valid_value_bytes(value_bytes))
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: value_bytes must be 1, 2, 4, 8 or 16");
  if (n > 0 && (d_keys == nullptr || d_values == nullptr))
    return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: keys/values is NULL");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (n <= 1) return VXS_OK;
  const int xf = xform_for(type, order);
  const uint64_t sd = seed_for(seed, has_seed, d_keys, n);
  return with_word(type, [&](auto* tag) -> vxs_status {
    using WK = std::remove_pointer_t<decltype(tag)>;
    if constexpr (sizeof(WK) == 16) {
      return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: sort_pairs supports 16/32/64-bit keys");
    } else {
      return with_value(value_bytes, [&](auto* vtag) -> vxs_status {
        using V = std::remove_pointer_t<decltype(vtag)>;
        return dispatch_packed<WK, V>(static_cast<const WK*>(d_keys), n, xf, sd, nullptr, static_cast<WK*>(d_keys),
                                      static_cast<V*>(d_values), value_bytes, d_workspace, workspace_bytes,
                                      static_cast<cudaStream_t>(stream), stats);
      });
    }
  });
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
    AsyncBuf owned;
    void* ws = d_workspace;
    if (ws == nullptr) {
      VXS_CK(owned.alloc(Lay.total, st), "workspace alloc");
      ws = owned.p;
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
    k_segscan_root<W><<<(kChildStride + 31) / 32, 1024, 0, st>>>(P);
    k_plan<W><<<grid_for((const void*)k_plan<W>, kChildStride, 0), kChildStride, 0, st>>>(P);  // (+ the tile prefixes)
    {
      auto fn = k_scatter<W>;
      fn<<<P.grid, Cfg<W>::kScatThreads, scatter_smem<W>(), st>>>(P);
    }
    k_part_counts<W><<<1, 256, 0, st>>>(P, nseg, reinterpret_cast<unsigned long long*>(d_seg_counts));
    VXS_CK(cudaGetLastError(), "partition");
    VXS_CK(owned.free(), "workspace free");
    return VXS_OK;
  });
}

// Fused exchange, phase 1: the read-only half of a partition -- classify
// every key by the splitters, per-(bucket, CTA) counts, offsets, per-segment
// totals in d_seg_counts.  The workspace keeps that state for phase 2.
vxs_status vxs_partition_counts(const void* d_keys, size_t n, vxs_key_type type, vxs_order order,
                                const void* d_splitters, int nspl, uint64_t* d_seg_counts, void* d_workspace,
                                size_t workspace_bytes, void* stream) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (nspl < 0 || nspl > 255) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: nspl must be in [0, 255]");
  if (d_workspace == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: partition_counts needs a workspace");
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
    if (workspace_bytes < Lay.total) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
    Params<W> P = make_params<W>(const_cast<W*>(static_cast<const W*>(d_keys)), n, xf, 0,
                                 static_cast<unsigned char*>(d_workspace), Lay);
    P.part_mode = 1;
    int L = 1;
    while ((1 << L) - 1 < nspl) ++L;
    k_init<W><<<1, 32, 0, st>>>(P);
    k_part_setup<W><<<1, 256, 0, st>>>(P, static_cast<const W*>(d_splitters), nspl, L);
    k_hist<W><<<P.grid, Cfg<W>::kHistThreads, hist_smem<W>(), st>>>(P);
    k_segscan_root<W><<<(kChildStride + 31) / 32, 1024, 0, st>>>(P);
    k_plan<W><<<grid_for((const void*)k_plan<W>, kChildStride, 0), kChildStride, 0, st>>>(P);  // (+ the tile prefixes)
    k_part_counts<W><<<1, 256, 0, st>>>(P, nseg, reinterpret_cast<unsigned long long*>(d_seg_counts));
    VXS_CK(cudaGetLastError(), "partition_counts");
    return VXS_OK;
  });
}

// Fused exchange, phase 2: the classify + scatter pass, with segment i's keys
// stored straight into ((key type*)d_dst[i]) + d_dst_offsets[i] -- another
// rank's receive buffer mapped over NVLink (vxs_ipc_open), so the
// all-to-all rides on the scatter's own stores.  Same keys, n, type, order,
// nspl and workspace as the phase-1 call; d_dst / d_dst_offsets are device
// arrays of nspl+1 entries.  Ends with a system-scope fence per CTA.
vxs_status vxs_partition_exchange(const void* d_keys, size_t n, vxs_key_type type, vxs_order order, int nspl,
                                  const uint64_t* d_dst, const uint64_t* d_dst_offsets, void* d_workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!valid_order(order)) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: invalid order");
  if (nspl < 0 || nspl > 255) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: nspl must be in [0, 255]");
  if (d_workspace == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: partition_exchange needs a workspace");
  const int xf = xform_for(type, order);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return with_word(type, [&](auto* tag) -> vxs_status {
    using W = std::remove_pointer_t<decltype(tag)>;
    if (n == 0) return VXS_OK;
    const Layout Lay = layout_for<W>(n);
    if (workspace_bytes < Lay.total) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: provided workspace is too small");
    Params<W> P = make_params<W>(const_cast<W*>(static_cast<const W*>(d_keys)), n, xf, 0,
                                 static_cast<unsigned char*>(d_workspace), Lay);
    P.part_mode = 1;
    P.xchg = 1;
    P.xdst = reinterpret_cast<const unsigned long long*>(d_dst);
    P.xoff = reinterpret_cast<const unsigned long long*>(d_dst_offsets);
    {
      ProfScope ps(K_PART, st);
      k_scatter<W><<<P.grid, Cfg<W>::kScatThreads, scatter_smem<W>(), st>>>(P);
    }
    VXS_CK(cudaGetLastError(), "partition_exchange");
    return VXS_OK;
  });
}

// Symmetric receive buffers for the fused exchange: plain cudaMalloc blocks
// (IPC-exportable), their 64-byte IPC handles, and peer mappings (P2P over
// NVLink via cudaIpcMemLazyEnablePeerAccess).
vxs_status vxs_device_alloc(size_t bytes, void** d_ptr) {
  if (d_ptr == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: null out pointer");
  VXS_CK(cudaMalloc(d_ptr, bytes ? bytes : 16), "device alloc");
  return VXS_OK;
}
vxs_status vxs_device_free(void* d_ptr) {
  VXS_CK(cudaFree(d_ptr), "device free");
  return VXS_OK;
}
vxs_status vxs_ipc_handle(void* d_ptr, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (handle64 == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: null handle buffer");
  cudaIpcMemHandle_t h;
  VXS_CK(cudaIpcGetMemHandle(&h, d_ptr), "ipc get handle");
  std::memcpy(handle64, &h, sizeof(h));
  return VXS_OK;
}
vxs_status vxs_ipc_open(const void* handle64, void** d_ptr) {
  if (handle64 == nullptr || d_ptr == nullptr) return fail(VXS_INVALID_ARGUMENT, "vxsort_b200: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  VXS_CK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc open handle");
  return VXS_OK;
}
vxs_status vxs_ipc_close(void* d_ptr) {
  VXS_CK(cudaIpcCloseMemHandle(d_ptr), "ipc close handle");
  return VXS_OK;
}

}  // extern "C"
