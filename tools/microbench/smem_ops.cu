// Microbenchmark: shared-memory atomics / loads / MATCH.ANY throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void k(unsigned* out, int iters, int mask) {
  __shared__ unsigned sh[16 * 512];
  for (int i = threadIdx.x; i < 16 * 512; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  unsigned acc = 0;
  unsigned s = hsh(threadIdx.x * 7919 + blockIdx.x * 104729);
  const int w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    s = hsh(s + it);
    unsigned b = s & mask;
    if (MODE == 0) atomicAdd(&sh[b], 1u);                       // block-shared hist, no return
    if (MODE == 1) acc += atomicAdd(&sh[w * 512 + b], 1u);      // per-warp hist, with return
    if (MODE == 2) acc += sh[w * 512 + b];                      // plain LDS random
    if (MODE == 3) acc += __match_any_sync(0xffffffffu, b);     // MATCH.ANY
    if (MODE == 4) { sh[w * 512 + b] += 1; }                    // non-atomic RMW (racy, timing only)
    if (MODE == 5) atomicAdd(&sh[w * 512 + b], 1u);             // per-warp hist, no return
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc + sh[threadIdx.x];
}
int main() {
  unsigned* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"atoms_block_noret", "atoms_warp_ret", "lds_random", "match_any", "lds_sts_rmw", "atoms_warp_noret"};
  for (int mask : {511, 0}) for (int mode = 0; mode < 6; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 4096, threads = 512, blocks = sms * 2;
    auto launch = [&]() {
      switch (mode) { case 0: k<0><<<blocks, threads>>>(out, iters, mask); break; case 1: k<1><<<blocks, threads>>>(out, iters, mask); break;
        case 2: k<2><<<blocks, threads>>>(out, iters, mask); break; case 3: k<3><<<blocks, threads>>>(out, iters, mask); break;
        case 4: k<4><<<blocks, threads>>>(out, iters, mask); break; case 5: k<5><<<blocks, threads>>>(out, iters, mask); break; }
    };
    launch(); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-18s mask=%3d: %.3f ms, %.2f lane-ops/cycle/SM, %.3f Gops/s total\n", names[mode], mask, ms, ops / cyc / sms, ops / ms / 1e6);
  }
  return 0;
}
