// dist_sort.cu -- the distributed sample sort behind the C ABI (vxs_dist_*).
//
// SURVEY §8b names vxs_dist_sort as the multi-GPU extension of the
// reference's sort surface (vexsort.hpp:121-129; the reference has no
// parallel sort), and §8e gives the algorithm: local sampling,
// all-gather of samples, identical splitters everywhere, one exchange step,
// local sort.  This file is host orchestration only: every kernel it runs is
// one of the library's own entry points (vxs_sample, vxs_sort,
// vxs_partition_counts / vxs_partition_exchange, vxs_partition) plus one
// splitter-pick kernel.  The fused exchange stores every segment straight
// into its owner's receive window (one cudaMalloc block per rank, exported
// with CUDA IPC and mapped by every peer: P2P stores over NVLink / NVSwitch),
// so the all-to-all is the partition kernel's own coalesced stores.
//
// Collectives go through NCCL when the group carries a communicator (loaded
// with dlopen: the library itself never links NCCL), else through the
// group's host all-gather callback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/vxsort_b200.h"

namespace vxs {
void set_error(const char* msg);  // vxsort_b200.cu: the thread-local slot vxs_last_error() reads
}

namespace {

vxs_status dfail(vxs_status s, const char* msg) {
  vxs::set_error(msg);
  return s;
}

vxs_status dcuda(cudaError_t e, const char* where) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "vxsort_b200 dist: CUDA error in %s: %s", where, cudaGetErrorString(e));
  vxs::set_error(buf);
  return e == cudaErrorMemoryAllocation ? VXS_OUT_OF_MEMORY : VXS_CUDA_ERROR;
}

#define DCK(expr, where)                       \
  do {                                         \
    cudaError_t e_ = (expr);                   \
    if (e_ != cudaSuccess) return dcuda(e_, where); \
  } while (0)

// A library call failed: its own message is already in vxs_last_error().
#define VCK(expr)                 \
  do {                            \
    vxs_status s_ = (expr);       \
    if (s_ != VXS_OK) return s_;  \
  } while (0)

// ---- NCCL, resolved at run time --------------------------------------------
struct Nccl {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // an NCCL already loaded in the process (e.g. torch's) is reused
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define LOADSYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
    LOADSYM(get_unique_id, "ncclGetUniqueId");
    LOADSYM(comm_init_rank, "ncclCommInitRank");
    LOADSYM(comm_destroy, "ncclCommDestroy");
    LOADSYM(all_gather, "ncclAllGather");
    LOADSYM(all_reduce, "ncclAllReduce");
    LOADSYM(send, "ncclSend");
    LOADSYM(recv, "ncclRecv");
    LOADSYM(group_start, "ncclGroupStart");
    LOADSYM(group_end, "ncclGroupEnd");
    LOADSYM(error_string, "ncclGetErrorString");
#undef LOADSYM
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather && n.all_reduce && n.send &&
           n.recv && n.group_start && n.group_end && n.error_string;
  });
  return n;
}

vxs_status nccl_fail(ncclResult_t r, const char* where) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "vxsort_b200 dist: NCCL error in %s: %s", where,
                nccl().error_string ? nccl().error_string(r) : "?");
  vxs::set_error(buf);
  return VXS_CUDA_ERROR;
}

#define NCK(expr, where)                           \
  do {                                             \
    ncclResult_t r_ = (expr);                      \
    if (r_ != ncclSuccess) return nccl_fail(r_, where); \
  } while (0)

// ---- per-group state ---------------------------------------------------------
template <typename T>
struct DevBuf {  // persistent, grow-only device buffer
  T* p = nullptr;
  size_t cap = 0;  // elements
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    const size_t want = std::max(n, cap + cap / 4);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const cudaError_t e = cudaMalloc(&p, std::max<size_t>(want * sizeof(T), 256));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

struct vxs_dist_ctx_s {
  vxs_dist_group g{};
  int device = 0;
  // symmetric receive window: peers[r] = rank r's block (own one at rank)
  size_t win_bytes = 0;
  std::vector<void*> peers;
  DevBuf<uint64_t> d_addrs, d_offs;       // exchange destinations / offsets
  DevBuf<unsigned char> ws, part;         // partition workspace / nccl-exchange staging
  DevBuf<unsigned char> smp, gathered, spl;
  DevBuf<uint64_t> counts, allcounts, one;
  DevBuf<unsigned char> hbuf_dev;         // collective staging on the device (handles)
  std::vector<uint64_t> last_recv, last_sent;
};

namespace {

size_t word_bytes(vxs_key_type t) {
  switch (t) {
    case VXS_I16: case VXS_U16: return 2;
    case VXS_I32: case VXS_U32: case VXS_F32: return 4;
    case VXS_I64: case VXS_U64: case VXS_F64: return 8;
    case VXS_K128: case VXS_KV64: return 16;
  }
  return 0;
}

vxs_key_type word_type(size_t kb) {
  return kb == 2 ? VXS_U16 : kb == 4 ? VXS_U32 : kb == 8 ? VXS_U64 : VXS_K128;
}

// All-gather of `bytes` per rank, device buffers, ordered on `st`.
vxs_status allgather_dev(vxs_dist_ctx c, const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) {
  if (c->g.world == 1) {
    if (d_send != d_recv) DCK(cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, st), "allgather");
    return VXS_OK;
  }
  if (c->g.nccl_comm) {
    NCK(nccl().all_gather(d_send, d_recv, bytes, ncclUint8, static_cast<ncclComm_t>(c->g.nccl_comm), st),
        "ncclAllGather");
    return VXS_OK;
  }
  std::vector<unsigned char> hs(bytes), hr(bytes * (size_t)c->g.world);
  DCK(cudaMemcpyAsync(hs.data(), d_send, bytes, cudaMemcpyDeviceToHost, st), "allgather D2H");
  DCK(cudaStreamSynchronize(st), "allgather sync");
  if (c->g.allgather(c->g.allgather_ctx, hs.data(), hr.data(), bytes) != 0)
    return dfail(VXS_INTERNAL, "vxsort_b200 dist: host allgather callback failed");
  DCK(cudaMemcpyAsync(d_recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st), "allgather H2D");
  DCK(cudaStreamSynchronize(st), "allgather sync");  // (hr goes out of scope)
  return VXS_OK;
}

// All-gather of host bytes (small control data: IPC handles, barriers).
vxs_status allgather_host(vxs_dist_ctx c, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  if (c->g.world == 1) {
    std::memcpy(recv, send, bytes);
    return VXS_OK;
  }
  if (!c->g.nccl_comm) {
    if (c->g.allgather(c->g.allgather_ctx, send, recv, bytes) != 0)
      return dfail(VXS_INTERNAL, "vxsort_b200 dist: host allgather callback failed");
    return VXS_OK;
  }
  DCK(c->hbuf_dev.ensure(bytes * (size_t)(c->g.world + 1)), "staging alloc");
  unsigned char* ds = c->hbuf_dev.p;
  unsigned char* dr = c->hbuf_dev.p + bytes;
  DCK(cudaMemcpyAsync(ds, send, bytes, cudaMemcpyHostToDevice, st), "allgather H2D");
  VCK(allgather_dev(c, ds, dr, bytes, st));
  DCK(cudaMemcpyAsync(recv, dr, bytes * (size_t)c->g.world, cudaMemcpyDeviceToHost, st), "allgather D2H");
  DCK(cudaStreamSynchronize(st), "allgather sync");
  return VXS_OK;
}

vxs_status barrier(vxs_dist_ctx c, cudaStream_t st) {
  int one = 1;
  std::vector<int> all((size_t)c->g.world);
  DCK(cudaStreamSynchronize(st), "barrier sync");
  return allgather_host(c, &one, all.data(), sizeof(int), st);
}

void close_window(vxs_dist_ctx c) {
  for (int r = 0; r < (int)c->peers.size(); ++r)
    if (r != c->g.rank && c->peers[r]) vxs_ipc_close(c->peers[r]);
}

// Grow the symmetric window to >= bytes on every rank (collective; every rank
// computes the same size from the same all-gathered count matrix).
vxs_status ensure_window(vxs_dist_ctx c, size_t bytes, cudaStream_t st) {
  if (bytes <= c->win_bytes) return VXS_OK;
  bytes = std::max(bytes, c->win_bytes + c->win_bytes / 4);
  bytes = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  DCK(cudaStreamSynchronize(st), "window sync");
  // every rank unmaps its peers' blocks before any owner frees its own
  close_window(c);
  if (c->g.world > 1) VCK(barrier(c, st));
  if (!c->peers.empty() && c->peers[c->g.rank]) vxs_device_free(c->peers[c->g.rank]);
  c->peers.assign((size_t)c->g.world, nullptr);
  c->win_bytes = 0;
  void* mine = nullptr;
  VCK(vxs_device_alloc(bytes, &mine));
  c->peers[c->g.rank] = mine;
  if (c->g.world > 1) {
    unsigned char h[64];
    VCK(vxs_ipc_handle(mine, h));
    std::vector<unsigned char> all(64 * (size_t)c->g.world);
    VCK(allgather_host(c, h, all.data(), 64, st));
    for (int r = 0; r < c->g.world; ++r)
      if (r != c->g.rank) VCK(vxs_ipc_open(all.data() + 64 * r, &c->peers[r]));
  }
  std::vector<uint64_t> addrs((size_t)c->g.world);
  for (int r = 0; r < c->g.world; ++r) addrs[r] = (uint64_t)(uintptr_t)c->peers[r];
  DCK(c->d_addrs.ensure(addrs.size()), "addrs alloc");
  DCK(cudaMemcpyAsync(c->d_addrs.p, addrs.data(), addrs.size() * 8, cudaMemcpyHostToDevice, st), "addrs H2D");
  DCK(cudaStreamSynchronize(st), "addrs sync");
  c->win_bytes = bytes;
  return VXS_OK;
}

// The world-1 global splitters: positions (r+1)*s - 1 of the sorted G*s sample.
__global__ void k_pick(const unsigned char* sorted, unsigned char* spl, int nspl, int s, int kb) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nspl * kb; i += gridDim.x * blockDim.x) {
    const int r = i / kb, b = i % kb;
    spl[i] = sorted[((size_t)(r + 1) * s - 1) * kb + b];
  }
}

void add_stats(vxs_stats& acc, const vxs_stats& s) {
  acc.kernel_launches += s.kernel_launches;
}

}  // namespace

extern "C" {

vxs_status vxs_dist_create(const vxs_dist_group* group, vxs_dist_ctx* out) {
  if (!group || !out) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: null argument");
  if (group->world < 1 || group->rank < 0 || group->rank >= group->world)
    return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: need 0 <= rank < world");
  if (group->world > 1 && !group->nccl_comm && !group->allgather)
    return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: world > 1 needs nccl_comm or an allgather callback");
  if (group->nccl_comm && !nccl().ok)
    return dfail(VXS_CUDA_ERROR, "vxsort_b200 dist: nccl_comm given but libnccl.so.2 could not be loaded");
  auto* c = new vxs_dist_ctx_s();
  c->g = *group;
  cudaGetDevice(&c->device);
  *out = c;
  return VXS_OK;
}

vxs_status vxs_dist_destroy(vxs_dist_ctx c) {
  if (!c) return VXS_OK;
  vxs_status s = VXS_OK;
  cudaDeviceSynchronize();
  close_window(c);
  if (c->g.world > 1 && !c->peers.empty()) s = barrier(c, 0);
  if (!c->peers.empty() && c->peers[c->g.rank]) vxs_device_free(c->peers[c->g.rank]);
  delete c;
  return s;
}

vxs_status vxs_dist_last_counts(vxs_dist_ctx c, uint64_t* recv_per_rank, uint64_t* sent_per_rank) {
  if (!c) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: null context");
  if (c->last_recv.empty()) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: no sort ran on this context");
  if (recv_per_rank) std::memcpy(recv_per_rank, c->last_recv.data(), c->last_recv.size() * 8);
  if (sent_per_rank) std::memcpy(sent_per_rank, c->last_sent.data(), c->last_sent.size() * 8);
  return VXS_OK;
}

vxs_status vxs_dist_sort(vxs_dist_ctx c, const void* d_keys, size_t n, vxs_key_type type, vxs_order order,
                         uint64_t seed, vxs_exchange exchange, void** d_out, size_t* n_out, void* stream,
                         vxs_stats* stats) {
  if (!c || !d_out || !n_out) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: null argument");
  const size_t kb = word_bytes(type);
  if (kb == 0) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: unknown key type");
  if (order != VXS_ASCENDING && order != VXS_DESCENDING)
    return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: invalid order");
  if (n > 0 && !d_keys) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: keys is NULL");
  if (exchange == VXS_EXCHANGE_NCCL && c->g.world > 1 && !c->g.nccl_comm)
    return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: the NCCL exchange needs nccl_comm");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = c->g.world, me = c->g.rank;
  vxs_stats acc{};
  if (stats) std::memset(stats, 0, sizeof(*stats));

  // 1. local stratified samples (order-transformed words); an empty rank
  //    contributes maximum words
  const int kOversample = 256;
  const int s = kOversample * G;
  DCK(c->smp.ensure((size_t)s * kb), "sample alloc");
  DCK(c->gathered.ensure((size_t)G * s * kb), "sample alloc");
  DCK(c->spl.ensure((size_t)std::max(1, G - 1) * kb), "splitter alloc");
  if (n > 0) {
    VCK(vxs_sample(d_keys, n, type, order, seed ^ ((uint64_t)me * 0x9E3779B97F4A7C15ull), c->smp.p, s, st));
  } else {
    DCK(cudaMemsetAsync(c->smp.p, 0xFF, (size_t)s * kb, st), "sample fill");
  }
  acc.kernel_launches += 1;
  // 2. all-gather; every rank sorts the same G*s words and picks the same splitters
  VCK(allgather_dev(c, c->smp.p, c->gathered.p, (size_t)s * kb, st));
  vxs_stats ss{};
  VCK(vxs_sort(c->gathered.p, (size_t)G * s, word_type(kb), VXS_ASCENDING, 1, 1, nullptr, 0, st, &ss));
  add_stats(acc, ss);
  if (G > 1) {
    k_pick<<<1, 256, 0, st>>>(c->gathered.p, c->spl.p, G - 1, s, (int)kb);
    DCK(cudaGetLastError(), "splitter pick");
    acc.kernel_launches += 1;
  }
  // 3. per-destination counts and the world x world matrix
  DCK(c->counts.ensure((size_t)G), "counts alloc");
  DCK(c->allcounts.ensure((size_t)G * G), "counts alloc");
  size_t wsb = 0;
  VCK(vxs_sort_workspace_bytes(std::max<size_t>(n, 1), type, &wsb));
  DCK(c->ws.ensure(wsb), "workspace alloc");
  if (G == 1) {  // one rank: the exchange is the identity; sort a copy in the window
    VCK(ensure_window(c, std::max<size_t>(n * kb, 256), st));
    if (n) DCK(cudaMemcpyAsync(c->peers[0], d_keys, n * kb, cudaMemcpyDeviceToDevice, st), "copy");
    if (n > 1) {
      vxs_stats ls{};
      VCK(vxs_sort(c->peers[0], n, type, order, seed, 1, nullptr, 0, st, &ls));
      ls.kernel_launches += acc.kernel_launches;
      acc = ls;
    }
    c->last_recv.assign(1, n);
    c->last_sent.assign(1, n);
    *d_out = c->peers[0];
    *n_out = n;
    if (stats) *stats = acc;
    return VXS_OK;
  }
  const bool fused = exchange == VXS_EXCHANGE_FUSED;
  if (n > 0) {
    if (fused) {
      VCK(vxs_partition_counts(d_keys, n, type, order, c->spl.p, G - 1, c->counts.p, c->ws.p, c->ws.cap, st));
    } else {
      DCK(c->part.ensure(n * kb), "partition buffer alloc");
      VCK(vxs_partition(d_keys, n, type, order, c->spl.p, G - 1, c->part.p, c->counts.p, c->ws.p, c->ws.cap, st));
    }
    acc.kernel_launches += 6;
  } else {
    DCK(cudaMemsetAsync(c->counts.p, 0, (size_t)G * 8, st), "counts fill");
  }
  VCK(allgather_dev(c, c->counts.p, c->allcounts.p, (size_t)G * 8, st));
  std::vector<uint64_t> m((size_t)G * G);
  DCK(cudaMemcpyAsync(m.data(), c->allcounts.p, m.size() * 8, cudaMemcpyDeviceToHost, st), "counts D2H");
  DCK(cudaStreamSynchronize(st), "counts sync");
  // this rank's element offset inside every destination (senders land in rank order)
  std::vector<uint64_t> offs((size_t)G, 0), recv_of((size_t)G, 0);
  for (int r = 0; r < G; ++r)
    for (int q = 0; q < G; ++q) {
      recv_of[r] += m[(size_t)q * G + r];
      if (q < me) offs[r] += m[(size_t)q * G + r];
    }
  const uint64_t recv = recv_of[me];
  const uint64_t need = *std::max_element(recv_of.begin(), recv_of.end());
  VCK(ensure_window(c, std::max<size_t>(need * kb, 256), st));
  // 4. exchange
  if (fused) {
    if (n > 0) {
      DCK(c->d_offs.ensure((size_t)G), "offsets alloc");
      DCK(cudaMemcpyAsync(c->d_offs.p, offs.data(), (size_t)G * 8, cudaMemcpyHostToDevice, st), "offsets H2D");
      VCK(vxs_partition_exchange(d_keys, n, type, order, G - 1, c->d_addrs.p, c->d_offs.p, c->ws.p, c->ws.cap, st));
      acc.kernel_launches += 1;
    }
    // order every peer's stores (each exchange CTA ends with a system fence)
    // before anyone reads its window
    if (G > 1) {
      if (c->g.nccl_comm) {
        DCK(c->one.ensure(1), "flag alloc");
        NCK(nccl().all_reduce(c->one.p, c->one.p, 1, ncclUint64, ncclSum, static_cast<ncclComm_t>(c->g.nccl_comm),
                              st),
            "ncclAllReduce");
      } else {
        VCK(barrier(c, st));
      }
    }
  } else {
    // baseline: NCCL grouped send/recv of the partitioned segments
    unsigned char* win = static_cast<unsigned char*>(c->peers[me]);
    std::vector<uint64_t> soff((size_t)G + 1, 0), roff((size_t)G + 1, 0);
    for (int r = 0; r < G; ++r) {
      soff[r + 1] = soff[r] + m[(size_t)me * G + r];
      roff[r + 1] = roff[r] + m[(size_t)r * G + me];
    }
    NCK(nccl().group_start(), "ncclGroupStart");
    for (int r = 0; r < G; ++r) {
      const size_t sb = (soff[r + 1] - soff[r]) * kb, rb = (roff[r + 1] - roff[r]) * kb;
      if (r == me) {
        if (sb) DCK(cudaMemcpyAsync(win + roff[r] * kb, c->part.p + soff[r] * kb, sb, cudaMemcpyDeviceToDevice, st),
                    "self copy");
        continue;
      }
      if (sb) NCK(nccl().send(c->part.p + soff[r] * kb, sb, ncclUint8, r, static_cast<ncclComm_t>(c->g.nccl_comm), st),
                  "ncclSend");
      if (rb) NCK(nccl().recv(win + roff[r] * kb, rb, ncclUint8, r, static_cast<ncclComm_t>(c->g.nccl_comm), st),
                  "ncclRecv");
    }
    NCK(nccl().group_end(), "ncclGroupEnd");
  }
  // 5. local sort of the received range
  void* out = c->peers[me];
  if (recv > 1) {
    vxs_stats ls{};
    VCK(vxs_sort(out, recv, type, order, seed, 1, nullptr, 0, st, &ls));
    acc.max_depth = ls.max_depth;
    acc.partition_calls = ls.partition_calls;
    acc.base_case_calls = ls.base_case_calls;
    acc.keys_partitioned = ls.keys_partitioned;
    acc.fallback_triggered = ls.fallback_triggered;
    acc.workspace_bytes = ls.workspace_bytes;
    add_stats(acc, ls);
  }
  c->last_recv = recv_of;
  c->last_sent.assign(m.begin() + (size_t)me * G, m.begin() + (size_t)(me + 1) * G);
  *d_out = out;
  *n_out = recv;
  if (stats) *stats = acc;
  return VXS_OK;
}

vxs_status vxs_nccl_unique_id(void* id128) {
  if (!id128) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: null id buffer");
  if (!nccl().ok) return dfail(VXS_CUDA_ERROR, "vxsort_b200 dist: libnccl.so.2 could not be loaded");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NCK(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof(id));
  return VXS_OK;
}

vxs_status vxs_nccl_comm_create(const void* id128, int world, int rank, void** comm) {
  if (!id128 || !comm) return dfail(VXS_INVALID_ARGUMENT, "vxsort_b200 dist: null argument");
  if (!nccl().ok) return dfail(VXS_CUDA_ERROR, "vxsort_b200 dist: libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  NCK(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
  *comm = c;
  return VXS_OK;
}

vxs_status vxs_nccl_comm_destroy(void* comm) {
  if (!comm) return VXS_OK;
  if (!nccl().ok) return dfail(VXS_CUDA_ERROR, "vxsort_b200 dist: libnccl.so.2 could not be loaded");
  NCK(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return VXS_OK;
}

}  // extern "C"
