// Microbenchmark: interpolation counting-sort base case vs warp-network sort.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2205_05982_b200/csrc/block_sort.cuh"
#include "../../paper_2205_05982_b200/csrc/tile_pipe.cuh"
using namespace vxs;

template <int THREADS, typename T>
__device__ __forceinline__ T bscan(T v, T* total, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { T y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = THREADS / 32;
    T s = lane < NW ? scratch[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { T y = __shfl_up_sync(0xffffffffu, s, o); if (lane >= o) s += y; }
    if (lane < NW) scratch[lane] = s;
  }
  __syncthreads();
  const T r = (warp == 0 ? T(0) : scratch[warp - 1]) + x - v;
  *total = scratch[THREADS / 32 - 1];
  __syncthreads();
  return r;
}

// items of exactly `item` keys, CAP = THREADS*ITEMS >= item
template <typename W, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_interp(const W* in, W* out, int item, int nitems, int* fallbacks) {
  constexpr int CAP = THREADS * ITEMS;
  constexpr int NW = THREADS / 32;
  __shared__ W sk[CAP];
  __shared__ unsigned cnt[CAP + 1];
  __shared__ W rlo[NW], rhi[NW];
  __shared__ unsigned rmx[NW];
  __shared__ unsigned scr[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const W* src = in + (size_t)it * item;
    W* dst = out + (size_t)it * item;
    const int n = item;
    W k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) { const int idx = i * THREADS + threadIdx.x; k[i] = idx < n ? __ldcs(src + idx) : key_max<W>(); }
    W lo = k[0], hi = k[0];
#pragma unroll
    for (int i = 1; i < ITEMS; ++i) if (i * THREADS + (int)threadIdx.x < n) { lo = key_lt(k[i], lo) ? k[i] : lo; hi = key_lt(hi, k[i]) ? k[i] : hi; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { W a = shfl_xor(lo, o), b = shfl_xor(hi, o); lo = key_lt(a, lo) ? a : lo; hi = key_lt(hi, b) ? b : hi; }
    if (lane == 0) { rlo[warp] = lo; rhi[warp] = hi; }
    const int log2d = n <= 1 ? 0 : 32 - __clz(n - 1);
    const int D = 1 << log2d;
    for (int i = threadIdx.x; i <= D; i += THREADS) cnt[i] = 0;
    __syncthreads();
    lo = rlo[0]; hi = rhi[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) { lo = key_lt(rlo[w], lo) ? rlo[w] : lo; hi = key_lt(hi, rhi[w]) ? rhi[w] : hi; }
    const int bl = key_bitlen(key_sub(hi, lo));
    const int shift = bl > log2d ? bl - log2d : 0;
    unsigned dr[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) if (i * THREADS + (int)threadIdx.x < n) {
      const unsigned d = key_shr32(key_sub(k[i], lo), shift);
      dr[i] = (d << 16) | atomicAdd(&cnt[d], 1u);
    }
    __syncthreads();
    const int per = (D + THREADS - 1) / THREADS;
    const int c0 = threadIdx.x * per;
    unsigned sum = 0, mx = 0;
    for (int j = 0; j < per; ++j) { const unsigned v = c0 + j < D ? cnt[c0 + j] : 0u; sum += v; mx = v > mx ? v : mx; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { unsigned y = __shfl_xor_sync(0xffffffffu, mx, o); mx = y > mx ? y : mx; }
    if (lane == 0) rmx[warp] = mx;
    unsigned tot;
    unsigned ex = bscan<THREADS>(sum, &tot, scr);
    mx = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) mx = rmx[w] > mx ? rmx[w] : mx;
    if (mx > 16) { if (threadIdx.x == 0) atomicAdd(fallbacks, 1); __syncthreads(); continue; }
    for (int j = 0; j < per; ++j) if (c0 + j < D) { const unsigned v = cnt[c0 + j]; cnt[c0 + j] = ex; ex += v; }
    if (threadIdx.x == 0) cnt[D] = n;
    __syncthreads();
    unsigned pos[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) if (i * THREADS + (int)threadIdx.x < n) { pos[i] = cnt[dr[i] >> 16] + (dr[i] & 0xFFFFu); sk[pos[i]] = k[i]; }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) if (i * THREADS + (int)threadIdx.x < n) {
      const unsigned d = dr[i] >> 16;
      const unsigned b0 = cnt[d], b1 = cnt[d + 1];
      unsigned r = b0;
      if (b1 - b0 > 1) {
        for (unsigned q = b0; q < b1; ++q) { const W y = sk[q]; r += (key_lt(y, k[i]) || (q < pos[i] && key_eq(y, k[i]))) ? 1u : 0u; }
      }
      dst[r] = k[i];
    }
    __syncthreads();
  }
}

template <typename W, int T, int I>
void run(const char* name, int item, bool narrow) {
  const int nitems = (1 << 26) / item;
  const size_t n = (size_t)nitems * item;
  std::vector<W> h(n);
  unsigned long long s = 88172645463325252ull;
  for (size_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    W v = (W)s;
    if (narrow) { // item-local range like a level-2 bucket: base + 16..48 varying bits
      const size_t it = i / item;
      W base = (W)(it * 0x9E3779B97F4A7C15ull);
      v = base + (W)(s >> (sizeof(W) == 4 ? 48 : 16));
    }
    h[i] = v;
  }
  W *in, *out; int* fb;
  cudaMalloc(&in, n * sizeof(W)); cudaMalloc(&out, n * sizeof(W)); cudaMalloc(&fb, 4); cudaMemset(fb, 0, 4);
  cudaMemcpy(in, h.data(), n * sizeof(W), cudaMemcpyHostToDevice);
  auto fn = k_interp<W, T, I>;
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * occ;
  fn<<<grid, T>>>(in, out, item, nitems, fb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) fn<<<grid, T>>>(in, out, item, nitems, fb);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
  std::vector<W> o(n); int hfb = 0;
  cudaMemcpy(o.data(), out, n * sizeof(W), cudaMemcpyDeviceToHost);
  cudaMemcpy(&hfb, fb, 4, cudaMemcpyDeviceToHost);
  bool ok = true;
  for (int it = 0; it < nitems && ok; it += 97) {
    std::vector<W> e(h.begin() + (size_t)it * item, h.begin() + (size_t)(it + 1) * item);
    std::sort(e.begin(), e.end());
    ok = std::equal(e.begin(), e.end(), o.begin() + (size_t)it * item);
  }
  printf("%-24s item=%5d occ=%2d narrow=%d %.3f ms %.1f Gkeys/s %s fallbacks=%d err=%s\n", name, item, occ, narrow, ms,
         n / ms / 1e6, ok ? "ok" : "WRONG(or fallback)", hfb, cudaGetErrorString(cudaGetLastError()));
  cudaFree(in); cudaFree(out); cudaFree(fb);
}

int main() {
  run<unsigned, 128, 16>("u32 interp 128x16", 1536, true);
  run<unsigned, 128, 16>("u32 interp 128x16", 1536, false);
  run<unsigned, 256, 8>("u32 interp 256x8", 1536, true);
  run<unsigned, 64, 32>("u32 interp 64x32", 1536, true);
  run<unsigned long long, 128, 16>("u64 interp 128x16", 1536, true);
  run<unsigned long long, 256, 8>("u64 interp 256x8", 1536, true);
  run<unsigned long long, 128, 16>("u64 interp 128x16", 1024, true);
  return 0;
}
