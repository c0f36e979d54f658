// C++ host calling the distributed sort through the C ABI (vexsort::DistSorter
// over vxs_dist_*), checked against std::sort:
//   world1 : one rank, with a native NCCL communicator and without one;
//   fork2  : two processes sharing GPU 0 (NCCL refuses that), collectives
//            through a host all-gather over shared memory; the parent (no
//            CUDA) checks the concatenated rank outputs.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "vexsort_b200.hpp"

namespace {

std::vector<std::uint64_t> keys_for(int rank, std::size_t n) {
  std::mt19937_64 g(1234 + 77 * rank);
  std::vector<std::uint64_t> v(n);
  for (auto& x : v) x = g();
  return v;
}

constexpr int kWorld = 2;
constexpr std::size_t kMaxMsg = 1 << 20;
constexpr std::size_t kMaxOut = 1 << 20;  // keys per rank

struct Shm {
  std::atomic<unsigned> arrive, gen;
  unsigned char msg[kWorld][kMaxMsg];
  std::size_t n_out[kWorld];
  std::uint64_t out[kWorld][kMaxOut];
};

void shm_barrier(Shm* s) {
  const unsigned g = s->gen.load();
  if (s->arrive.fetch_add(1) + 1 == kWorld) {
    s->arrive.store(0);
    s->gen.fetch_add(1);
  } else {
    while (s->gen.load() == g) usleep(20);
  }
}

struct CbCtx {
  Shm* shm;
  int rank;
};

int shm_allgather(void* ctx, const void* send, void* recv, std::size_t bytes) {
  auto* c = static_cast<CbCtx*>(ctx);
  if (bytes > kMaxMsg) return 1;
  std::memcpy(c->shm->msg[c->rank], send, bytes);
  shm_barrier(c->shm);
  for (int r = 0; r < kWorld; ++r) std::memcpy(static_cast<unsigned char*>(recv) + r * bytes, c->shm->msg[r], bytes);
  shm_barrier(c->shm);
  return 0;
}

int sort_and_check_world1(void* comm, vxs_exchange ex) {
  const std::size_t n = 1'000'003;
  auto h = keys_for(0, n);
  std::uint64_t* d = nullptr;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  vxs_dist_group g{0, 1, comm, nullptr, nullptr};
  vexsort::DistSorter ds(g);
  vexsort::SortConfig cfg;
  cfg.order = vexsort::Order::kDescending;
  std::span<std::uint64_t> out = ds.sort(d, n, cfg, nullptr, ex);
  std::vector<std::uint64_t> got(out.size());
  cudaMemcpy(got.data(), out.data(), out.size() * 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  std::sort(h.begin(), h.end(), std::greater<>());
  return got == h ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "world1";
  if (mode == "world1") {
    unsigned char id[128];
    void* comm = nullptr;
    if (vxs_nccl_unique_id(id) != VXS_OK || vxs_nccl_comm_create(id, 1, 0, &comm) != VXS_OK) {
      std::printf("nccl unavailable: %s\n", vxs_last_error());
      return 3;
    }
    int bad = sort_and_check_world1(comm, VXS_EXCHANGE_FUSED) + sort_and_check_world1(comm, VXS_EXCHANGE_NCCL) +
              sort_and_check_world1(nullptr, VXS_EXCHANGE_FUSED);
    vxs_nccl_comm_destroy(comm);
    if (bad) return 1;
    std::puts("ok");
    return 0;
  }
  // fork2: no CUDA in the parent before the fork
  auto* shm = static_cast<Shm*>(mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0));
  if (shm == MAP_FAILED) return 4;
  new (shm) Shm();
  const std::size_t n_of[kWorld] = {300'000, 170'001};
  pid_t pids[kWorld];
  for (int r = 0; r < kWorld; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) {
      cudaSetDevice(0);
      auto h = keys_for(r, n_of[r]);
      std::uint64_t* d = nullptr;
      cudaMalloc(&d, h.size() * 8);
      cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      CbCtx cb{shm, r};
      int rc = 0;
      try {
        vexsort::DistSorter ds(vxs_dist_group{r, kWorld, nullptr, shm_allgather, &cb});
        for (int rep = 0; rep < 2; ++rep) {  // (second call reuses the window)
          std::span<std::uint64_t> out = ds.sort(d, h.size());
          if (out.size() > kMaxOut) {
            rc = 5;
            break;
          }
          shm->n_out[r] = out.size();
          cudaMemcpy(shm->out[r], out.data(), out.size() * 8, cudaMemcpyDeviceToHost);
        }
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
        rc = 6;
      }
      cudaFree(d);
      _exit(rc);
    }
  }
  int bad = 0;
  for (int r = 0; r < kWorld; ++r) {
    int st = 0;
    waitpid(pids[r], &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) bad = 1;
  }
  if (bad) return 1;
  std::vector<std::uint64_t> all, got;
  for (int r = 0; r < kWorld; ++r) {
    auto h = keys_for(r, n_of[r]);
    all.insert(all.end(), h.begin(), h.end());
    got.insert(got.end(), shm->out[r], shm->out[r] + shm->n_out[r]);
  }
  std::sort(all.begin(), all.end());
  if (all != got) return 2;
  std::puts("ok");
  return 0;
}
