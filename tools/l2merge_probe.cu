// Probe: do concurrent misses from many SMs to the same lines get merged in L2?
// Each iteration, every CTA reads the same fresh `region` bytes (cold in L2).
// Compare dram__bytes_read (ncu) with iters * region.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void same_region(const int4* __restrict__ buf, size_t region16, int iters, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    const int4* r = buf + (size_t)it * region16;
    for (size_t i = threadIdx.x; i < region16; i += blockDim.x) {
      int4 v = __ldcg(r + i);
      acc.x ^= v.x; acc.y ^= v.y;
    }
    __syncthreads();
  }
  if (acc.x == 0x1234567) sink[0] = acc;
}
int main() {
  const size_t region = 786432;          // H[b] at cfg3
  const int iters = 256;
  int4* buf; cudaMalloc(&buf, region * iters);
  cudaMemset(buf, 1, region * iters);
  int4* sink; cudaMalloc(&sink, 64);
  // flush L2 by touching a big buffer
  char* fl; cudaMalloc(&fl, 512 << 20); cudaMemset(fl, 0, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  same_region<<<148, 512>>>(buf, region / 16, iters, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("iters=%d region=%zu expected_dram=%.1f MB time=%.3f ms L2-side BW=%.1f GB/s\n", iters, region,
         region * iters / 1e6, ms, 148.0 * region * iters / ms / 1e6);
  return 0;
}
