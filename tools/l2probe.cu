// Microbenchmark: L2-resident streaming read bandwidth and 1.5 KB row-gather
// bandwidth (the access pattern of the Sparton backward), plus device facts.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

__global__ void stream_read(const int4* __restrict__ buf, size_t n16, int reps, int4* sink) {
  int4 acc = make_int4(0,0,0,0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(buf + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// warp per (pair): gather row idx[p] of `rows` (row = D bf16 = D*2 bytes), FMA-accumulate.
template <int CPL>
__global__ void gather_rows(const int4* __restrict__ rows, const int* __restrict__ idx, int npairs,
                            int row16, float* out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int p = warp; p < npairs; p += nw) {
    const int4* r = rows + (size_t)idx[p] * row16;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      int4 v = __ldg(r + lane + 32 * c);
      acc += __int_as_float(v.x) + __int_as_float(v.y) + __int_as_float(v.z) + __int_as_float(v.w);
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int optin = 0; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"clock_khz\":%d}\n", p.name,
         p.multiProcessorCount, p.l2CacheSize, optin, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int4* sink; cudaMalloc(&sink, 64);
  for (size_t mb : {16, 48, 96, 1024}) {
    size_t bytes = mb << 20; int4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
    int reps = mb >= 1024 ? 2 : 20;
    stream_read<<<p.multiProcessorCount * 8, 512>>>(buf, bytes / 16, 1, sink);
    cudaEventRecord(e0);
    stream_read<<<p.multiProcessorCount * 8, 512>>>(buf, bytes / 16, reps, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"stream_read\",\"mb\":%zu,\"GBps\":%.1f}\n", mb, bytes * (double)reps / ms / 1e6);
    cudaFree(buf);
  }
  // gather: rows of 1536 B (D=768 bf16), from a pool of R rows
  for (size_t pool_mb : {1, 48, 400}) {
    int row16 = 96; size_t R = (pool_mb << 20) / 1536;
    int4* rows; cudaMalloc(&rows, R * 1536); cudaMemset(rows, 0, R * 1536);
    int np = 1 << 22; std::vector<int> h(np); std::mt19937 g(1);
    for (int i = 0; i < np; ++i) h[i] = g() % R;
    int* d; cudaMalloc(&d, np * 4); cudaMemcpy(d, h.data(), np * 4, cudaMemcpyHostToDevice);
    float* o; cudaMalloc(&o, 4);
    gather_rows<3><<<p.multiProcessorCount * 4, 512>>>(rows, d, np, row16, o);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) gather_rows<3><<<p.multiProcessorCount * 4, 512>>>(rows, d, np, row16, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"gather_1536B\",\"pool_mb\":%zu,\"GBps\":%.1f}\n", pool_mb, 5.0 * np * 1536 / ms / 1e6);
    cudaFree(rows); cudaFree(d); cudaFree(o);
  }
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
