// vexsort_b200.hpp -- recompile-only drop-in for the reference's public API
// (/root/reference/proj/core/include/vexsort/vexsort.hpp:31-132), backed by
// the B200 C ABI (vxsort_b200.h, libvxsort_b200.so).
//
//   std::vector<uint64_t> keys = ...;
//   vexsort::SortStats stats = vexsort::sort(std::span(keys));
//
// Same names, argument meaning and error behaviour as the reference:
//   * nine overloads over host std::span (int16..double, K128), in place;
//   * SortConfig{order, backend, seed, scratch}; a caller scratch smaller than
//     scratch_bytes<T>() throws std::invalid_argument (vexsort.cpp:19-31);
//   * SortStats{max_depth, partition_calls, base_case_calls,
//     keys_partitioned, fallback_triggered} (driver.hpp:26-32), filled with the
//     device analogues (levels, multiway splits, base-case CTAs, keys moved).
// Deliberate differences: NaN keys are sorted last instead of
// rejected; -0.0 precedes +0.0 in ascending order; Backend is accepted but
// every value runs the B200 kernels (no CPU path exists).  Device pointers
// are sorted with vexsort::sort_device().
#ifndef VEXSORT_B200_HPP_
#define VEXSORT_B200_HPP_

#include <cstddef>
#include <cstdint>
#include <new>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>

#include "vxsort_b200.h"

namespace vexsort {

// 128-bit key: low half first, as the reference (traits.hpp:24-31).
struct K128 {
  std::uint64_t lo;
  std::uint64_t hi;
  friend bool operator==(const K128& a, const K128& b) = default;
};

struct SortStats {
  std::size_t max_depth = 0;
  std::size_t partition_calls = 0;
  std::size_t base_case_calls = 0;
  std::size_t keys_partitioned = 0;
  bool fallback_triggered = false;
};

enum class Order { kAscending, kDescending };
enum class Backend { kAuto, kScalar, kWide };

namespace detail {
template <typename T> struct KeyCode;
template <> struct KeyCode<std::int16_t> { static constexpr vxs_key_type v = VXS_I16; static constexpr std::size_t scratch = 512; };
template <> struct KeyCode<std::uint16_t> { static constexpr vxs_key_type v = VXS_U16; static constexpr std::size_t scratch = 512; };
template <> struct KeyCode<std::int32_t> { static constexpr vxs_key_type v = VXS_I32; static constexpr std::size_t scratch = 1024; };
template <> struct KeyCode<std::uint32_t> { static constexpr vxs_key_type v = VXS_U32; static constexpr std::size_t scratch = 1024; };
template <> struct KeyCode<float> { static constexpr vxs_key_type v = VXS_F32; static constexpr std::size_t scratch = 1024; };
template <> struct KeyCode<std::int64_t> { static constexpr vxs_key_type v = VXS_I64; static constexpr std::size_t scratch = 2048; };
template <> struct KeyCode<std::uint64_t> { static constexpr vxs_key_type v = VXS_U64; static constexpr std::size_t scratch = 2048; };
template <> struct KeyCode<double> { static constexpr vxs_key_type v = VXS_F64; static constexpr std::size_t scratch = 2048; };
template <> struct KeyCode<K128> { static constexpr vxs_key_type v = VXS_K128; static constexpr std::size_t scratch = 4096; };
}  // namespace detail

// Same values as the reference's scratch_bytes<T>() (vexsort.hpp:58-66).
template <typename T>
constexpr std::size_t scratch_bytes() {
  return detail::KeyCode<T>::scratch;
}

// 64-byte-aligned reusable scratch buffer. Move-only (vexsort.hpp:69-110).
class SortScratch {
 public:
  SortScratch() = default;
  explicit SortScratch(std::size_t bytes)
      : mem_(static_cast<std::byte*>(::operator new(bytes, std::align_val_t{64}))), size_(bytes) {}
  template <typename T>
  static SortScratch for_key() {
    return SortScratch(scratch_bytes<T>());
  }
  SortScratch(SortScratch&& o) noexcept
      : mem_(std::exchange(o.mem_, nullptr)), size_(std::exchange(o.size_, 0)) {}
  SortScratch& operator=(SortScratch&& o) noexcept {
    if (this != &o) {
      release();
      mem_ = std::exchange(o.mem_, nullptr);
      size_ = std::exchange(o.size_, 0);
    }
    return *this;
  }
  SortScratch(const SortScratch&) = delete;
  SortScratch& operator=(const SortScratch&) = delete;
  ~SortScratch() { release(); }
  std::byte* data() const { return mem_; }
  std::size_t size() const { return size_; }

 private:
  void release() {
    if (mem_ != nullptr) {
      ::operator delete(mem_, std::align_val_t{64});
      mem_ = nullptr;
    }
  }
  std::byte* mem_ = nullptr;
  std::size_t size_ = 0;
};

struct SortConfig {
  Order order = Order::kAscending;
  Backend backend = Backend::kAuto;
  std::optional<std::uint64_t> seed{};
  SortScratch* scratch = nullptr;
};

namespace detail {
inline void throw_status(vxs_status s) {
  if (s == VXS_OK) return;
  const std::string msg = vxs_last_error();
  if (s == VXS_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == VXS_INTERNAL) throw std::logic_error(msg);
  if (s == VXS_OUT_OF_MEMORY) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

inline SortStats to_stats(const vxs_stats& s) {
  SortStats r;
  r.max_depth = s.max_depth;
  r.partition_calls = s.partition_calls;
  r.base_case_calls = s.base_case_calls;
  r.keys_partitioned = s.keys_partitioned;
  r.fallback_triggered = s.fallback_triggered != 0;
  return r;
}

template <typename T>
SortStats sort_typed(std::span<T> keys, const SortConfig& config) {
  if (config.scratch != nullptr && config.scratch->size() < scratch_bytes<T>()) {
    throw std::invalid_argument("vexsort: provided scratch is too small");
  }
  vxs_stats st{};
  throw_status(vxs_sort_host(keys.data(), keys.size(), KeyCode<T>::v,
                             config.order == Order::kAscending ? VXS_ASCENDING : VXS_DESCENDING,
                             config.seed.value_or(0), config.seed.has_value() ? 1 : 0, &st));
  return to_stats(st);
}
}  // namespace detail

inline SortStats sort(std::span<std::int16_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<std::uint16_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<std::int32_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<std::uint32_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<float> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<std::int64_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<std::uint64_t> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<double> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }
inline SortStats sort(std::span<K128> keys, const SortConfig& config = {}) { return detail::sort_typed(keys, config); }

// Device-resident keys (stream-ordered; see vxs_sort).
template <typename T>
SortStats sort_device(T* d_keys, std::size_t n, const SortConfig& config = {}, void* stream = nullptr,
                      void* d_workspace = nullptr, std::size_t workspace_bytes = 0) {
  if (config.scratch != nullptr && config.scratch->size() < scratch_bytes<T>()) {
    throw std::invalid_argument("vexsort: provided scratch is too small");
  }
  vxs_stats st{};
  detail::throw_status(vxs_sort(d_keys, n, detail::KeyCode<T>::v,
                                config.order == Order::kAscending ? VXS_ASCENDING : VXS_DESCENDING,
                                config.seed.value_or(0), config.seed.has_value() ? 1 : 0, d_workspace,
                                workspace_bytes, stream, &st));
  return detail::to_stats(st);
}

// Extensions beyond the reference surface: stable argsort and
// key+value sort of device-resident keys (16/32/64-bit key types).
template <typename T>
SortStats argsort_device(const T* d_keys, std::size_t n, std::uint64_t* d_indices, T* d_sorted_keys = nullptr,
                         const SortConfig& config = {}, void* stream = nullptr, void* d_workspace = nullptr,
                         std::size_t workspace_bytes = 0) {
  vxs_stats st{};
  detail::throw_status(vxs_argsort(d_keys, n, detail::KeyCode<T>::v,
                                   config.order == Order::kAscending ? VXS_ASCENDING : VXS_DESCENDING, d_indices,
                                   d_sorted_keys, config.seed.value_or(0), config.seed.has_value() ? 1 : 0,
                                   d_workspace, workspace_bytes, stream, &st));
  return detail::to_stats(st);
}

template <typename T, typename V>
SortStats sort_pairs_device(T* d_keys, V* d_values, std::size_t n, const SortConfig& config = {},
                            void* stream = nullptr, void* d_workspace = nullptr, std::size_t workspace_bytes = 0) {
  vxs_stats st{};
  detail::throw_status(vxs_sort_pairs(d_keys, d_values, sizeof(V), n, detail::KeyCode<T>::v,
                                      config.order == Order::kAscending ? VXS_ASCENDING : VXS_DESCENDING,
                                      config.seed.value_or(0), config.seed.has_value() ? 1 : 0, d_workspace,
                                      workspace_bytes, stream, &st));
  return detail::to_stats(st);
}

// Distributed sample sort across ranks (one process per GPU),
// RAII over vxs_dist_create / vxs_dist_destroy.  Every rank of the group
// constructs, sorts and destroys together.  sort() returns this rank's sorted
// slice of the union (device memory inside the context's receive window,
// valid until the next sort()).
class DistSorter {
 public:
  explicit DistSorter(const vxs_dist_group& group) { detail::throw_status(vxs_dist_create(&group, &ctx_)); }
  DistSorter(const DistSorter&) = delete;
  DistSorter& operator=(const DistSorter&) = delete;
  ~DistSorter() { vxs_dist_destroy(ctx_); }

  template <typename T>
  std::span<T> sort(const T* d_keys, std::size_t n, const SortConfig& config = {}, void* stream = nullptr,
                    vxs_exchange exchange = VXS_EXCHANGE_FUSED, SortStats* stats = nullptr) {
    void* out = nullptr;
    std::size_t n_out = 0;
    vxs_stats st{};
    detail::throw_status(vxs_dist_sort(ctx_, d_keys, n, detail::KeyCode<T>::v,
                                       config.order == Order::kAscending ? VXS_ASCENDING : VXS_DESCENDING,
                                       config.seed.value_or(1), exchange, &out, &n_out, stream, &st));
    if (stats) *stats = detail::to_stats(st);
    return std::span<T>(static_cast<T*>(out), n_out);
  }

 private:
  vxs_dist_ctx ctx_ = nullptr;
};

// The B200 path is data-parallel device code; kept for source compatibility
// with vexsort.hpp:132.
inline bool wide_backend_is_simd() { return true; }

}  // namespace vexsort

#endif  // VEXSORT_B200_HPP_
