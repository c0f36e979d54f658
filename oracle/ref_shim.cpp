// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim compiled TOGETHER WITH the unmodified reference sources where
// they lie (/root/reference/proj/core/src/vexsort.cpp + headers, and
// /root/reference/proj/tools/bench/harness.cpp) into oracle/_ref/libvexsort_ref.so
// by oracle/Makefile.  Nothing from the reference is copied into this repo.
// It lets the Python tests and bench.py's CPU-baseline leg call the real
// reference:
//   vexsort::sort(std::span<T>, SortConfig)   vexsort.hpp:121-129
//   Driver::heap_sort / depth_budget          driver.hpp:38-41, 96-121
//   PivotSampler::choose_pivot, Sfc64         pivot.hpp:25-172
//   vexbench::generate<T>                     harness.cpp:179-219
//   vexbench::run_partition_bench             harness.cpp:409-489
#include <atomic>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "bench/harness.hpp"
#include "vexsort/detail/driver.hpp"
#include "vexsort/detail/pivot.hpp"
#include "vexsort/vexsort.hpp"

namespace {

thread_local char g_err[256];

struct RefStats {
  std::size_t max_depth, partition_calls, base_case_calls, keys_partitioned;
  int fallback_triggered;
};

template <class F>
auto with_type(int t, F&& f) {
  switch (t) {
    case 0: return f(std::type_identity<std::int16_t>{});
    case 1: return f(std::type_identity<std::uint16_t>{});
    case 2: return f(std::type_identity<std::int32_t>{});
    case 3: return f(std::type_identity<std::uint32_t>{});
    case 4: return f(std::type_identity<float>{});
    case 5: return f(std::type_identity<std::int64_t>{});
    case 6: return f(std::type_identity<std::uint64_t>{});
    case 7: return f(std::type_identity<double>{});
    default: return f(std::type_identity<vexsort::K128>{});
  }
}

int sort_one(void* keys, std::size_t n, int type, int desc, std::uint64_t seed,
             int has_seed, int backend, RefStats* out) {
  try {
    vexsort::SortConfig cfg;
    cfg.order = desc ? vexsort::Order::kDescending : vexsort::Order::kAscending;
    cfg.backend = backend == 1 ? vexsort::Backend::kScalar
                               : (backend == 2 ? vexsort::Backend::kWide
                                               : vexsort::Backend::kAuto);
    if (has_seed) cfg.seed = seed;
    const vexsort::SortStats st = with_type(type, [&](auto tag) {
      using T = typename decltype(tag)::type;
      return vexsort::sort(std::span<T>(static_cast<T*>(keys), n), cfg);
    });
    if (out) {
      out->max_depth = st.max_depth;
      out->partition_calls = st.partition_calls;
      out->base_case_calls = st.base_case_calls;
      out->keys_partitioned = st.keys_partitioned;
      out->fallback_triggered = st.fallback_triggered ? 1 : 0;
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return 1;
  } catch (const std::logic_error& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return 3;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

// Status: 0 ok, 1 std::invalid_argument, 2 std::logic_error, 3 other.
int ref_sort(void* keys, std::size_t n, int type, int desc, std::uint64_t seed,
             int has_seed, int backend, RefStats* stats) {
  return sort_one(keys, n, type, desc, seed, has_seed, backend, stats);
}

// Independent instances, one std::thread per buffer (the harness's
// threads>1 mode, harness.cpp:316-358).  Returns the first non-zero status.
int ref_sort_instances(void** bufs, std::size_t n_bufs, std::size_t n, int type,
                       int desc, std::uint64_t seed) {
  std::vector<std::thread> workers;
  std::atomic<int> status{0};
  for (std::size_t i = 0; i < n_bufs; ++i) {
    workers.emplace_back([&, i]() {
      const int s = sort_one(bufs[i], n, type, desc, seed, 1, 0, nullptr);
      if (s != 0) status.store(s);
    });
  }
  for (auto& w : workers) w.join();
  return status.load();
}

// SortConfig.scratch too small -> std::invalid_argument (vexsort.cpp:19-31).
int ref_sort_with_scratch(void* keys, std::size_t n, int type, std::size_t scratch_bytes) {
  try {
    vexsort::SortScratch scratch(scratch_bytes);
    vexsort::SortConfig cfg;
    cfg.scratch = &scratch;
    cfg.seed = 1;
    with_type(type, [&](auto tag) {
      using T = typename decltype(tag)::type;
      return vexsort::sort(std::span<T>(static_cast<T*>(keys), n), cfg);
    });
    return 0;
  } catch (const std::invalid_argument& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return 1;
  }
}

std::size_t ref_scratch_bytes(int type) {
  return with_type(type, [&](auto tag) {
    using T = typename decltype(tag)::type;
    return vexsort::scratch_bytes<T>();
  });
}

std::size_t ref_depth_budget(std::size_t n) { return vexsort::detail::depth_budget(n); }

void ref_sfc64_stream(std::uint64_t seed, std::uint64_t* out, std::size_t n) {
  vexsort::detail::Sfc64 rng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = rng.next();
}

void ref_five_draws(std::uint64_t seed, std::uint32_t bound, std::size_t num,
                    std::uint32_t* idx) {
  vexsort::detail::Sfc64 rng(seed);
  const auto plan = vexsort::detail::five_draws_for_nine_offsets(rng, bound, num);
  for (std::size_t i = 0; i < num; ++i) idx[i] = plan.chunk_index[i];
}

// choose_pivot on the scalar backend for u64 keys (pivot.hpp:146-172).
std::uint64_t ref_choose_pivot_u64(const std::uint64_t* keys, std::size_t n,
                                   std::uint64_t seed, int desc) {
  using namespace vexsort::detail;
  Sfc64 rng(seed);
  std::vector<std::uint64_t> scratch(1024);
  auto run = [&](auto tr) {
    using TR = decltype(tr);
    return PivotSampler<ScalarTag, TR>::choose_pivot(
        std::span<const std::uint64_t>(keys, n), scratch, rng);
  };
  return desc ? run(LaneKeyTraits<std::uint64_t, false>{})
              : run(LaneKeyTraits<std::uint64_t, true>{});
}

int ref_heap_sort(void* keys, std::size_t n, int type, int desc) {
  using namespace vexsort::detail;
  with_type(type, [&](auto tag) {
    using T = typename decltype(tag)::type;
    using TF = vexsort::detail::TraitsFor<T>;
    using Lane = typename TF::Lane;
    if (desc) {
      Driver<WideTag, typename TF::template Traits<false>>::heap_sort(
          static_cast<Lane*>(keys), n);
    } else {
      Driver<WideTag, typename TF::template Traits<true>>::heap_sort(
          static_cast<Lane*>(keys), n);
    }
    return 0;
  });
  return 0;
}

// dist codes follow vexbench::Dist (harness.hpp:22-29).
int ref_generate(void* out, std::size_t n, int type, int dist, std::uint64_t seed) {
  const auto d = static_cast<vexbench::Dist>(dist);
  return with_type(type, [&](auto tag) {
    using T = typename decltype(tag)::type;
    const std::vector<T> v = vexbench::generate<T>(d, n, seed);
    std::memcpy(out, v.data(), n * sizeof(T));
    return 0;
  });
}

// The reference's own partition-only benchmark (harness.cpp:409-489: 2-way
// Partitioner::partition with a median pivot, verified every rep), at sizes
// 2^10 .. max_n in powers of four.  Fills up to cap (n, median MB/s) pairs;
// returns how many, or -1 on a verification failure.
int ref_partition_bench(int type, std::size_t max_n, std::size_t reps, std::uint64_t seed,
                        std::size_t* n_out, double* mbps_out, int cap) {
  try {
    vexbench::PartitionBenchConfig cfg;
    cfg.type = static_cast<vexbench::KeyType>(type);
    cfg.max_n = max_n;
    cfg.reps = reps;
    cfg.seed = seed;
    const auto res = vexbench::run_partition_bench(cfg);
    int k = 0;
    for (const auto& r : res) {
      if (k >= cap) break;
      n_out[k] = r.n;
      mbps_out[k] = r.mbps_median;
      ++k;
    }
    return k;
  } catch (const std::exception& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return -1;
  }
}

// ISA the shim was compiled for (the reference's wide backend follows it).
const char* ref_isa() {
#if defined(__AVX512VL__) && defined(__AVX512DQ__)
  return "avx2+avx512vl/dq";
#elif defined(__AVX2__)
  return "avx2";
#else
  return "scalar";
#endif
}

}  // extern "C"
