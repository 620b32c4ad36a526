// Microbenchmark for the dH floor: random 1536-B row gathers (D = 768 bf16)
// from an L2-resident 52 MB slice of E, through
//   (a) LDG.128 into registers, U rows in flight per warp, W warps per SM;
//   (b) cp.async.bulk (TMA) into a per-warp smem ring, then LDS.128;
//   (c) a plain L2 streaming read (the L2 ceiling for this box).
// Reports GB/s of row bytes delivered to registers and the SM clock measured
// inside the kernel (clock64 over the event time), so the numbers can be
// compared at equal clocks.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int ROW16 = 96;   // 1536 B = 96 x 16 B; a lane owns 3 x 16 B

__device__ __forceinline__ float fold(int4 v) {
  return __int_as_float(v.x) + __int_as_float(v.y) + __int_as_float(v.z) + __int_as_float(v.w);
}

template <int U>
__global__ void gather_ldg(const int4* __restrict__ rows, const int* __restrict__ idx, long long npairs,
                           float* out, long long* clk) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  long long t0 = clock64();
  float acc = 0.f;
  for (long long p0 = warp * U; p0 + U <= npairs; p0 += nw * U) {   // tail (< U pairs per warp) dropped
    int4 x[U][3];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int r = __ldg(idx + p0 + q);
      const int4* src = rows + (size_t)r * ROW16 + lane;
#pragma unroll
      for (int c = 0; c < 3; ++c) x[q][c] = __ldg(src + 32 * c);
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc += fold(x[q][c]);
  }
  if (acc == 1.2345f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void gather_tma(const int4* __restrict__ rows, const int* __restrict__ idx, long long npairs,
                           float* out, long long* clk) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  uint8_t* ring = sm + (size_t)wib * NS * 1536;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)(blockDim.x >> 5) * NS * 1536) + wib * NS;
  if (lane == 0)
    for (int i = 0; i < NS; ++i)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(smem_u32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  long long t0 = clock64();
  float acc = 0.f;
  auto issue = [&](long long p, int slot) {
    if (lane == 0) {
      const int r = __ldg(idx + p);
      const uint32_t bar = smem_u32(&bars[slot]);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 1536;" :: "r"(bar) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1536, [%2];"
                   :: "r"(smem_u32(ring + slot * 1536)), "l"(rows + (size_t)r * ROW16), "r"(bar) : "memory");
    }
  };
  long long n_mine = 0;
  for (long long p = warp; p < npairs; p += nw) ++n_mine;   // pairs warp, warp+nw, ...
  for (int i = 0; i < NS && i < n_mine; ++i) issue(warp + i * nw, i);
  uint32_t ph = 0;
  for (long long i = 0; i < n_mine; ++i) {
    const int slot = (int)(i % NS);
    const uint32_t bar = smem_u32(&bars[slot]);
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}\n"
                 :: "r"(bar), "r"(ph) : "memory");
    const int4* s = reinterpret_cast<const int4*>(ring + slot * 1536) + lane;
    int4 x0 = s[0], x1 = s[32], x2 = s[64];
    acc += fold(x0) + fold(x1) + fold(x2);
    __syncwarp();
    if (i + NS < n_mine) issue(warp + (i + NS) * nw, slot);
    if (slot == NS - 1) ph ^= 1;
  }
  if (acc == 1.2345f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

// (d) LDGSTS (cp.async 16 B per lane, L2 -> smem without holding registers):
// per-warp ring of NS row slots, one commit group per row, then LDS.128.
template <int NS>
__global__ void gather_ldgsts(const int4* __restrict__ rows, const int* __restrict__ idx, long long npairs,
                              float* out, long long* clk) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  uint8_t* ring = sm + (size_t)wib * NS * 1536;
  long long t0 = clock64();
  float acc = 0.f;
  auto issue = [&](long long p, int slot) {
    if (p < npairs) {
      const int r = __ldg(idx + p);
      const int4* src = rows + (size_t)r * ROW16 + lane;
      const uint32_t dst = smem_u32(ring + slot * 1536 + lane * 16);
#pragma unroll
      for (int c = 0; c < 3; ++c)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst + c * 512), "l"(src + 32 * c) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int i = 0; i < NS - 1; ++i) issue(warp + i * nw, i);
  int slot = 0;
  for (long long p = warp; p < npairs; p += nw) {
    issue(p + (NS - 1) * nw, (slot + NS - 1) % NS);
    asm volatile("cp.async.wait_group %0;" :: "n"(NS - 1) : "memory");
    const int4* s = reinterpret_cast<const int4*>(ring + slot * 1536) + lane;   // own lanes' bytes only
    acc += fold(s[0]) + fold(s[32]) + fold(s[64]);
    slot = slot + 1 == NS ? 0 : slot + 1;
  }
  if (acc == 1.2345f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

__global__ void stream_l2(const int4* __restrict__ buf, long long n16, int reps, float* out, long long* clk) {
  long long t0 = clock64();
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
      acc += fold(__ldcg(buf + i));
  if (acc == 1.2345f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t nrows = (52ull << 20) / 1536;
  int4* rows;
  cudaMalloc(&rows, nrows * 1536);
  cudaMemset(rows, 0, nrows * 1536);
  const long long npairs = 32ll << 20;
  std::vector<int> h(npairs);
  std::mt19937 g(1);
  for (auto& x : h) x = (int)(g() % nrows);
  int* idx;
  cudaMalloc(&idx, npairs * 4);
  cudaMemcpy(idx, h.data(), npairs * 4, cudaMemcpyHostToDevice);
  float* out;
  long long* clk;
  cudaMalloc(&out, 64);
  cudaMalloc(&clk, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char* name, double bytes, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    long long c = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) { best = ms; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost); }
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"probe\": \"%s\", \"ms\": %.4f, \"GBps\": %.1f, \"sm_ghz\": %.3f, \"B_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n",
           name, best, bytes / best / 1e6, c / best / 1e6, bytes / (c * (double)sms), cudaGetErrorString(e));
  };
  const double gbytes = (double)npairs * 1536;
  for (int wps : {16, 20, 24, 32}) {
    char nm[64];
    snprintf(nm, sizeof nm, "ldg_u4_w%d", wps);
    report(nm, gbytes, [&] { gather_ldg<4><<<sms, wps * 32>>>(rows, idx, npairs, out, clk); });
    if (wps <= 20) {
      snprintf(nm, sizeof nm, "ldg_u8_w%d", wps);
      report(nm, gbytes, [&] { gather_ldg<8><<<sms, wps * 32>>>(rows, idx, npairs, out, clk); });
    }
  }
  for (int wps : {40, 48, 64}) {
    char nm[64];
    snprintf(nm, sizeof nm, "ldg_u2_w%d", wps);
    report(nm, gbytes, [&] { gather_ldg<2><<<2 * sms, wps * 16>>>(rows, idx, npairs, out, clk); });
    snprintf(nm, sizeof nm, "ldg_u3_w%d", wps);
    if (wps <= 48) report(nm, gbytes, [&] { gather_ldg<3><<<2 * sms, wps * 16>>>(rows, idx, npairs, out, clk); });
  }
  for (int wps : {8, 16, 24}) {
    const int ns = wps == 8 ? 16 : (wps == 16 ? 8 : 5);
    const int smem = wps * ns * 1536 + wps * ns * 8;
    char nm[64];
    snprintf(nm, sizeof nm, "tma_ns%d_w%d", ns, wps);
    if (ns == 16) {
      cudaFuncSetAttribute(gather_tma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      report(nm, gbytes, [&] { gather_tma<16><<<sms, wps * 32, smem>>>(rows, idx, npairs, out, clk); });
    } else if (ns == 8) {
      cudaFuncSetAttribute(gather_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      report(nm, gbytes, [&] { gather_tma<8><<<sms, wps * 32, smem>>>(rows, idx, npairs, out, clk); });
    } else {
      cudaFuncSetAttribute(gather_tma<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      report(nm, gbytes, [&] { gather_tma<5><<<sms, wps * 32, smem>>>(rows, idx, npairs, out, clk); });
    }
  }
  {
    auto run = [&](auto kern, int ns, int wps) {
      const int smem = wps * ns * 1536;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      char nm[64];
      snprintf(nm, sizeof nm, "ldgsts_ns%d_w%d", ns, wps);
      report(nm, gbytes, [&] { kern<<<sms, wps * 32, smem>>>(rows, idx, npairs, out, clk); });
    };
    run(gather_ldgsts<9>, 9, 16);
    run(gather_ldgsts<7>, 7, 20);
    run(gather_ldgsts<6>, 6, 24);
    run(gather_ldgsts<4>, 4, 32);
    run(gather_ldgsts<8>, 8, 12);
  }
  const long long n16 = (long long)(nrows * 1536 / 16);
  report("stream_l2_52MB", (double)n16 * 16 * 400, [&] { stream_l2<<<sms * 4, 512>>>(rows, n16, 400, out, clk); });
  return 0;
}
