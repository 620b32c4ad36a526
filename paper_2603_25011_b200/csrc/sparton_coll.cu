// sparton_coll.cu — the vocab-sharded head's dH reduction over NVLink peer
// memory, as one kernel per rank instead of an
// NCCL all-reduce.
//
// Each rank's backward leaves its partial dH (fp32, B·S·D elements: the
// contribution of its vocabulary shard, fused.py:267-273) in a buffer every
// rank can address (torch symmetric memory, or CUDA IPC in the one-GPU test).
// After a barrier, rank r owns the slice of float4 units [r·c, (r+1)·c) with
// c = ⌈n/4 / P⌉ and, for every unit of its slice,
//   * peers:    loads the unit from all P partial buffers (P2P loads over
//               NVLink), sums them in rank order 0..P-1 — the same order on
//               every rank, so the result is deterministic and identical
//               everywhere — and stores it (fp32, or bf16 rounded once) into
//               all P output buffers (P2P stores);
//   * multimem: one multimem.ld_reduce.add.v4.f32 on the partial buffers'
//               NVLS multicast address (the switch sums the P copies) and one
//               multimem.st to the output buffers' multicast address (the
//               switch writes every rank's copy).
// A second barrier publishes the outputs.  Traffic per rank: the partials of
// one slice from each peer in, the reduced slice to each peer out — the bytes
// of a reduce-scatter + all-gather, in one launch (multimem: one slice in and
// one out through the switch).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "sparton_internal.h"

namespace sparton {

namespace {

constexpr int kCollThreads = 512;

struct PeerPtrs {
  const float4* part[kMaxPeers];
  void* out[kMaxPeers];
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

template <bool BF16>
__global__ void __launch_bounds__(kCollThreads)
allreduce_peers_kernel(const PeerPtrs p, int nranks, long long u0, long long u1) {
  for (long long u = u0 + (long long)blockIdx.x * kCollThreads + threadIdx.x; u < u1;
       u += (long long)gridDim.x * kCollThreads) {
    // Rank-ordered sum; .cg: the partials were written by other GPUs (and
    // this kernel's launch already invalidated L1), keep them out of L1.
    float4 s = __ldcg(p.part[0] + u);
    for (int q = 1; q < nranks; ++q) {
      const float4 x = __ldcg(p.part[q] + u);
      s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    if constexpr (BF16) {
      const uint2 o = make_uint2(pack_bf16x2(s.x, s.y), pack_bf16x2(s.z, s.w));
      for (int q = 0; q < nranks; ++q) reinterpret_cast<uint2*>(p.out[q])[u] = o;
    } else {
      for (int q = 0; q < nranks; ++q) reinterpret_cast<float4*>(p.out[q])[u] = s;
    }
  }
}

template <bool BF16>
__global__ void __launch_bounds__(kCollThreads)
allreduce_multimem_kernel(const float* mc_part, void* mc_out, long long u0, long long u1) {
  for (long long u = u0 + (long long)blockIdx.x * kCollThreads + threadIdx.x; u < u1;
       u += (long long)gridDim.x * kCollThreads) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc_part + 4 * u) : "memory");
    if constexpr (BF16) {
      asm volatile("multimem.st.relaxed.sys.global.v2.bf16x2 [%0], {%1, %2};"
                   :: "l"(reinterpret_cast<uint16_t*>(mc_out) + 4 * u), "r"(pack_bf16x2(a, b)),
                      "r"(pack_bf16x2(c, d)) : "memory");
    } else {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
                   :: "l"(reinterpret_cast<float*>(mc_out) + 4 * u), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
    }
  }
}

// This rank's slice of float4 units.
void slice_units(long long n, int nranks, int rank, long long& u0, long long& u1) {
  const long long units = n / 4;
  const long long c = (units + nranks - 1) / nranks;
  u0 = (long long)rank * c;
  if (u0 > units) u0 = units;
  u1 = u0 + c;
  if (u1 > units) u1 = units;
}

int coll_grid(long long units) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (units + kCollThreads - 1) / kCollThreads;
  const long long cap = 4ll * sms;   // a few CTAs per SM keep enough loads in flight
  if (want > cap) want = cap;
  return want < 1 ? 1 : (int)want;
}

}  // namespace

int launch_allreduce_peers(const float* const* parts, void* const* outs, int nranks, int rank, bool bf16,
                           long long n, cudaStream_t stream) {
  PeerPtrs p = {};
  for (int q = 0; q < nranks; ++q) {
    p.part[q] = reinterpret_cast<const float4*>(parts[q]);
    p.out[q] = outs[q];
  }
  long long u0, u1;
  slice_units(n, nranks, rank, u0, u1);
  if (u1 <= u0) return SPARTON_OK;
  const int grid = coll_grid(u1 - u0);
  if (bf16) allreduce_peers_kernel<true><<<grid, kCollThreads, 0, stream>>>(p, nranks, u0, u1);
  else allreduce_peers_kernel<false><<<grid, kCollThreads, 0, stream>>>(p, nranks, u0, u1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPARTON_OK : set_cuda_error("launch allreduce_peers_kernel", e);
}

int launch_allreduce_multimem(const float* mc_part, void* mc_out, int nranks, int rank, bool bf16, long long n,
                              cudaStream_t stream) {
  long long u0, u1;
  slice_units(n, nranks, rank, u0, u1);
  if (u1 <= u0) return SPARTON_OK;
  const int grid = coll_grid(u1 - u0);
  if (bf16) allreduce_multimem_kernel<true><<<grid, kCollThreads, 0, stream>>>(mc_part, mc_out, u0, u1);
  else allreduce_multimem_kernel<false><<<grid, kCollThreads, 0, stream>>>(mc_part, mc_out, u0, u1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPARTON_OK : set_cuda_error("launch allreduce_multimem_kernel", e);
}

}  // namespace sparton
