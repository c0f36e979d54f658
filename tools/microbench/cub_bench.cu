// cub_bench.cu -- library reference point: cub::DeviceRadixSort on the same
// sizes as the BASELINE configs (device-resident keys, CUDA-event timing,
// L2 flushed by the >126 MB inputs themselves).  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o cub_bench cub_bench.cu
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>

template <typename T>
__global__ void fill(T* k, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    k[i] = (T)z;
  }
}

template <typename T>
void run(const char* name, size_t n, int reps, bool pairs) {
  T *a, *b, *src;
  uint32_t *va = nullptr, *vb = nullptr;
  cudaMalloc(&a, n * sizeof(T));
  cudaMalloc(&b, n * sizeof(T));
  cudaMalloc(&src, n * sizeof(T));
  if (pairs) {
    cudaMalloc(&va, n * 4);
    cudaMalloc(&vb, n * 4);
  }
  fill<<<1184, 256>>>(src, n, 12345);
  size_t tmp_bytes = 0;
  void* tmp = nullptr;
  if (pairs)
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, a, b, va, vb, (int64_t)n);
  else
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int64_t)n);
  cudaMalloc(&tmp, tmp_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ms;
  for (int r = 0; r < reps + 3; ++r) {
    cudaMemcpy(a, src, n * sizeof(T), cudaMemcpyDeviceToDevice);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    if (pairs)
      cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, a, b, va, vb, (int64_t)n);
    else
      cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int64_t)n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    if (r >= 3) ms.push_back(t);
  }
  float best = 1e30f, sum = 0;
  for (float t : ms) {
    best = t < best ? t : best;
    sum += t;
  }
  printf("%-28s n=%zu  mean %.3f ms  best %.3f ms  %.1f Gkeys/s  (err=%s)\n", name, n, sum / ms.size(), best,
         n / (sum / ms.size()) / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(a);
  cudaFree(b);
  cudaFree(src);
  cudaFree(tmp);
  if (pairs) {
    cudaFree(va);
    cudaFree(vb);
  }
}

int main() {
  run<uint32_t>("cub SortKeys u32", 100000000, 10, false);
  run<uint64_t>("cub SortKeys u64", 100000000, 10, false);
  run<uint32_t>("cub SortPairs u32/u32", 100000000, 10, true);
  run<uint64_t>("cub SortKeys u64 2^30", 1ull << 30, 3, false);
  run<uint64_t>("cub SortKeys u64 1e6", 1000000, 20, false);
  return 0;
}
