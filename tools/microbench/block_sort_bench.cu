// Microbenchmark: CTA-level base-case sort variants on random items.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2205_05982_b200/csrc/block_sort.cuh"
using namespace vxs;

template <typename W, int THREADS, int ITEMS, bool WN>
__global__ void __launch_bounds__(THREADS) kb(const W* in, W* out, int item, int nitems) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  W* sm = reinterpret_cast<W*>(smem_raw);
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const W* src = in + (size_t)it * item;
    W k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int idx = i * THREADS + threadIdx.x;
      k[i] = idx < item ? src[idx] : key_max<W>();
    }
    block_sort<W, THREADS, ITEMS, WN>(k, sm);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) sm[pad_idx<W>(threadIdx.x * ITEMS + i)] = k[i];
    __syncthreads();
    W* dst = out + (size_t)it * item;
    for (int idx = threadIdx.x; idx < item; idx += THREADS) dst[idx] = sm[pad_idx<W>(idx)];
    __syncthreads();
  }
}

template <typename W, int T, int I, bool WN>
void run(const char* name, int item) {
  const int nitems = (1 << 26) / item;  // 64M keys
  const size_t n = (size_t)nitems * item;
  std::vector<W> h(n);
  unsigned long long s = 88172645463325252ull;
  for (auto& x : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = (W)s; }
  W *in, *out;
  cudaMalloc(&in, n * sizeof(W)); cudaMalloc(&out, n * sizeof(W));
  cudaMemcpy(in, h.data(), n * sizeof(W), cudaMemcpyHostToDevice);
  const size_t smem = padded_size<W>(T * I) * sizeof(W);
  auto fn = kb<W, T, I, WN>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T, smem);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * occ;
  fn<<<grid, T, smem>>>(in, out, item, nitems);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) fn<<<grid, T, smem>>>(in, out, item, nitems);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
  std::vector<W> o(n);
  cudaMemcpy(o.data(), out, n * sizeof(W), cudaMemcpyDeviceToHost);
  bool ok = true;
  for (int it = 0; it < nitems && ok; it += 97) {
    std::vector<W> e(h.begin() + (size_t)it * item, h.begin() + (size_t)(it + 1) * item);
    std::sort(e.begin(), e.end());
    ok = std::equal(e.begin(), e.end(), o.begin() + (size_t)it * item);
  }
  printf("%-28s item=%5d occ=%d  %.3f ms  %.1f Gkeys/s  %s  err=%s\n", name, item, occ, ms, n / ms / 1e6,
         ok ? "ok" : "WRONG", cudaGetErrorString(cudaGetLastError()));
  cudaFree(in); cudaFree(out);
}

int main() {
  run<unsigned, 128, 16, true>("u32 128x16 warpnet", 2048);
  run<unsigned, 32, 64, true>("u32 32x64 warpnet", 2048);
  run<unsigned, 32, 32, true>("u32 32x32 warpnet", 1024);
  run<unsigned, 64, 16, true>("u32 64x16 warpnet", 1024);
  run<unsigned, 128, 16, true>("u32 128x16 warpnet", 1900);
  run<unsigned, 32, 64, true>("u32 32x64 warpnet", 1900);
  return 0;
}
