// sparton_bwd.cu — K2/K3: the argmax-routed sparse backward on sm_100a.
//
// Replaces backward_fused (/root/reference/pkg/src/fusedhead/fused.py:215-278)
// which reads only the saved (Y, I) pair:
//   g[b,v]    = dY[b,v] * exp(-Y[b,v])      for Y[b,v] > 0, else the pair is inactive
//   dE[v,:]   = sum_b g[b,v] * H[b, I[b,v], :]        (embed_block, fused.py:255-265)
//   db[v]     = sum_b g[b,v]
//   dH[b,s,:] = sum_{v: I[b,v]=s} g[b,v] * E[v,:]     (hidden_row,  fused.py:267-273)
//
// Determinism without atomics (SPEC.md "Gradient accumulation determinism"):
// every output element has exactly one owner that accumulates in the
// reference's order — b ascending for dE/db, v ascending for dH.
//
//   K2 sparton_bwd_de_kernel  : CTA owns 32 vocab rows x one D slice; warps own
//                               4 rows each, lanes own 8-wide D chunks; (g, I)
//                               tiles for 32 batch rows are staged in smem and
//                               the H rows at the argmax are gathered (16-B
//                               vector loads, 4 rows in flight per warp).
//   K3a sparton_bwd_route_kernel : CTA per batch row: a stable counting sort of
//                               the active (v, g) pairs by argmax position s,
//                               giving per-(b,s) lists in ascending v.
//   K3b sparton_bwd_dh_kernel : warp owns one (b, s) row (x D slice) and sums
//                               g * E[v,:] over its list in ascending v.
// All arithmetic is fp32 (inputs bf16), exactly one owner per output element.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cmath>

#include "ptx.cuh"
#include "sparton_internal.h"

namespace sparton {

namespace {

constexpr int DE_VB = 32;       // vocab rows per CTA
constexpr int DE_BC = 32;       // batch rows staged per smem tile
constexpr int DE_THREADS = 256; // 8 warps x 4 vocab rows
constexpr int ROUTE_THREADS = 1024;
constexpr int ROUTE_SMEM_INTS = 48 * 1024;  // per-warp histograms (192 KB)
constexpr int DH_THREADS = 256;

__device__ __forceinline__ float pair_grad(float y, float dy) {
  // exp(-Y) == 1/(1+rawmax) (fused.py:247-249); accurate expf, no fast-math.
  return dy * expf(-y);
}

__device__ __forceinline__ void fma8(float* acc, float g, const int4& raw) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    acc[2 * i] = fmaf(g, f.x, acc[2 * i]);
    acc[2 * i + 1] = fmaf(g, f.y, acc[2 * i + 1]);
  }
}

template <typename OutT>
__device__ __forceinline__ void store8(OutT* dst, const float* acc);

template <>
__device__ __forceinline__ void store8<float>(float* dst, const float* acc) {
  reinterpret_cast<float4*>(dst)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* dst, const float* acc) {
  int4 o;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
  *reinterpret_cast<int4*>(dst) = o;
}

// ------------------------------------------------------------------ K2: dE, db
template <int CPL, typename OutT>
__global__ void __launch_bounds__(DE_THREADS)
sparton_bwd_de_kernel(const BwdParams p) {
  __shared__ float g_s[DE_BC][DE_VB];
  __shared__ int i_s[DE_BC][DE_VB];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int v0 = blockIdx.x * DE_VB;
  const int d0 = blockIdx.y * (256 * CPL);

  float acc[4][CPL * 8];
  float gsum[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    gsum[r] = 0.f;
#pragma unroll
    for (int i = 0; i < CPL * 8; ++i) acc[r][i] = 0.f;
  }
  bool dvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) dvalid[c] = (d0 + c * 256 + lane * 8) < p.D;

  for (int b0 = 0; b0 < p.B; b0 += DE_BC) {
    // Stage g and I for DE_BC batch rows x DE_VB vocab rows (coalesced rows of 128 B).
    for (int e = threadIdx.x; e < DE_BC * DE_VB; e += DE_THREADS) {
      const int bb = e / DE_VB, vv = e % DE_VB;
      const int b = b0 + bb, v = v0 + vv;
      float g = 0.f;
      int idx = -1;
      if (b < p.B && v < p.V) {
        const float y = p.Y[(size_t)b * p.ldY + v];
        if (y > 0.f) {
          g = pair_grad(y, p.dY[(size_t)b * p.ldDY + v]);
          idx = p.I[(size_t)b * p.ldY + v];
        }
      }
      g_s[bb][vv] = g;
      i_s[bb][vv] = idx;
    }
    __syncthreads();
    const int nb = min(DE_BC, p.B - b0);
    for (int bb = 0; bb < nb; ++bb) {
      const size_t hbase = (size_t)(b0 + bb) * p.S;
      int4 raw[4][CPL];
      float g[4];
      bool act[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int vv = warp + 8 * r;
        const int idx = i_s[bb][vv];
        g[r] = g_s[bb][vv];
        act[r] = idx >= 0;
        const __nv_bfloat16* row = p.H + (hbase + (act[r] ? idx : 0)) * (size_t)p.D + d0 + lane * 8;
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          raw[r][c] = (act[r] && dvalid[c]) ? __ldg(reinterpret_cast<const int4*>(row + c * 256))
                                           : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (act[r]) {
          gsum[r] += g[r];
#pragma unroll
          for (int c = 0; c < CPL; ++c) fma8(&acc[r][c * 8], g[r], raw[r][c]);
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int v = v0 + warp + 8 * r;
    if (v >= p.V) continue;
    OutT* dst = reinterpret_cast<OutT*>(p.dE) + (size_t)v * p.D + d0 + lane * 8;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (dvalid[c]) store8<OutT>(dst + c * 256, &acc[r][c * 8]);
    if (blockIdx.y == 0 && lane == 0 && p.db != nullptr)
      p.db[v] = p.include_bias_grad ? gsum[r] : 0.f;
  }
}

// ------------------------------------------------------------------ K3a: route
// One CTA per batch row b.  Stable counting sort of the active pairs of row b
// by key s = I[b,v]: the vocabulary is cut into `nseg` contiguous segments,
// one per warp; per-(segment, s) counts give every warp its own cursors, and
// within a warp equal keys are ranked by lane order (match.any), so each
// (b, s) list ends up in ascending v.  Output: pairs[b*V + k] = (v, g bits),
// offsets[b*(S+1) + s] = start of list s (offsets[..S] = number of pairs).
__global__ void __launch_bounds__(ROUTE_THREADS)
sparton_bwd_route_kernel(const BwdParams p, int nseg) {
  extern __shared__ int hist[];            // [nseg][S] (+ scan scratch)
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int S = p.S;
  int* scan_tmp = hist + nseg * S;         // [32] warp totals for the block scan

  for (int i = threadIdx.x; i < nseg * S; i += ROUTE_THREADS) hist[i] = 0;
  __syncthreads();

  const float* Yb = p.Y + (size_t)b * p.ldY;
  const int32_t* Ib = p.I + (size_t)b * p.ldY;
  const long long seg_len = ((long long)p.V + nseg - 1) / nseg;

  // Phase 1: per-segment histograms.
  if (warp < nseg) {
    const int vs = (int)min((long long)p.V, warp * seg_len);
    const int ve = (int)min((long long)p.V, (warp + 1) * seg_len);
    int* h = hist + warp * S;
    for (int v = vs + lane; v < ve; v += 32) {
      if (Yb[v] > 0.f) atomicAdd(&h[Ib[v]], 1);
    }
  }
  __syncthreads();

  // Phase 2: exclusive scan over s of the per-s totals (block-wide), then
  // per-s exclusive scan over segments -> cursors, written back into hist.
  int* off = p.offsets + (size_t)b * (S + 1);
  int carry = 0;
  for (int s0 = 0; s0 < S; s0 += ROUTE_THREADS) {
    const int s = s0 + threadIdx.x;
    int tot = 0;
    if (s < S)
      for (int w = 0; w < nseg; ++w) tot += hist[w * S + s];
    // inclusive warp scan
    int x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scan_tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int t = scan_tmp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      scan_tmp[lane] = t;   // inclusive warp-total prefix
    }
    __syncthreads();
    const int excl = carry + (warp > 0 ? scan_tmp[warp - 1] : 0) + x - tot;
    if (s < S) {
      off[s] = excl;
      int cur = excl;
      for (int w = 0; w < nseg; ++w) {
        const int c = hist[w * S + s];
        hist[w * S + s] = cur;
        cur += c;
      }
    }
    carry += scan_tmp[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) off[S] = carry;
  __syncthreads();

  // Phase 3: stable scatter of (v, g) into the per-s lists.
  if (warp < nseg) {
    const int vs = (int)min((long long)p.V, warp * seg_len);
    const int ve = (int)min((long long)p.V, (warp + 1) * seg_len);
    int* cur = hist + warp * S;
    int2* out = p.pairs + (size_t)b * p.V;
    const float* dYb = p.dY + (size_t)b * p.ldDY;
    for (int base = vs; base < ve; base += 32) {
      const int v = base + lane;
      bool active = false;
      int key = 0;
      float g = 0.f;
      if (v < ve) {
        const float y = Yb[v];
        if (y > 0.f) {
          active = true;
          key = Ib[v];
          g = pair_grad(y, dYb[v]);
        }
      }
      const unsigned amask = __ballot_sync(0xffffffffu, active);
      if (active) {
        const unsigned peers = __match_any_sync(amask, key);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int pos = cur[key] + rank;
        out[pos] = make_int2(v, __float_as_int(g));
        __syncwarp(amask);
        if (rank == 0) cur[key] += __popc(peers);
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------ K3b: dH
template <int CPL, typename OutT>
__global__ void __launch_bounds__(DH_THREADS)
sparton_bwd_dh_kernel(const BwdParams p) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long rowid = (long long)blockIdx.x * (DH_THREADS / 32) + warp;   // b*S + s
  if (rowid >= (long long)p.B * p.S) return;
  const int b = (int)(rowid / p.S);
  const int s = (int)(rowid - (long long)b * p.S);
  const int d0 = blockIdx.y * (256 * CPL);
  const int* off = p.offsets + (size_t)b * (p.S + 1);
  const int k0 = off[s], k1 = off[s + 1];
  const int2* lst = p.pairs + (size_t)b * p.V;

  bool dvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) dvalid[c] = (d0 + c * 256 + lane * 8) < p.D;
  float acc[CPL * 8];
#pragma unroll
  for (int i = 0; i < CPL * 8; ++i) acc[i] = 0.f;

  for (int kb = k0; kb < k1; kb += 32) {
    const int n = min(32, k1 - kb);
    int2 mine = make_int2(0, 0);
    if (lane < n) mine = lst[kb + lane];
    int j = 0;
    for (; j + 2 <= n; j += 2) {
      const int va = __shfl_sync(0xffffffffu, mine.x, j);
      const float ga = __int_as_float(__shfl_sync(0xffffffffu, mine.y, j));
      const int vb = __shfl_sync(0xffffffffu, mine.x, j + 1);
      const float gb = __int_as_float(__shfl_sync(0xffffffffu, mine.y, j + 1));
      const __nv_bfloat16* ra = p.E + (size_t)va * p.D + d0 + lane * 8;
      const __nv_bfloat16* rb = p.E + (size_t)vb * p.D + d0 + lane * 8;
      int4 xa[CPL], xb[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        xa[c] = dvalid[c] ? __ldg(reinterpret_cast<const int4*>(ra + c * 256)) : make_int4(0, 0, 0, 0);
        xb[c] = dvalid[c] ? __ldg(reinterpret_cast<const int4*>(rb + c * 256)) : make_int4(0, 0, 0, 0);
      }
      // ascending v: a before b
#pragma unroll
      for (int c = 0; c < CPL; ++c) fma8(&acc[c * 8], ga, xa[c]);
#pragma unroll
      for (int c = 0; c < CPL; ++c) fma8(&acc[c * 8], gb, xb[c]);
    }
    if (j < n) {
      const int va = __shfl_sync(0xffffffffu, mine.x, j);
      const float ga = __int_as_float(__shfl_sync(0xffffffffu, mine.y, j));
      const __nv_bfloat16* ra = p.E + (size_t)va * p.D + d0 + lane * 8;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int4 xa = dvalid[c] ? __ldg(reinterpret_cast<const int4*>(ra + c * 256)) : make_int4(0, 0, 0, 0);
        fma8(&acc[c * 8], ga, xa);
      }
    }
  }
  OutT* dst = reinterpret_cast<OutT*>(p.dH) + (size_t)rowid * p.D + d0 + lane * 8;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (dvalid[c]) store8<OutT>(dst + c * 256, &acc[c * 8]);
}

template <int CPL, typename OutT>
int launch_bwd_t(const BwdParams& p, cudaStream_t stream) {
  const int dslices = (p.D + 256 * CPL - 1) / (256 * CPL);
  {
    dim3 grid((p.V + DE_VB - 1) / DE_VB, dslices);
    sparton_bwd_de_kernel<CPL, OutT><<<grid, DE_THREADS, 0, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_de_kernel", e);
  }
  {
    int nseg = ROUTE_SMEM_INTS / (p.S > 0 ? p.S : 1);
    if (nseg > 32) nseg = 32;
    if (nseg < 1) nseg = 1;
    const size_t smem = ((size_t)nseg * p.S + 32) * sizeof(int);
    cudaError_t e = cudaFuncSetAttribute(sparton_bwd_route_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(route)", e);
    sparton_bwd_route_kernel<<<p.B, ROUTE_THREADS, smem, stream>>>(p, nseg);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_route_kernel", e);
  }
  {
    const long long rows = (long long)p.B * p.S;
    dim3 grid((unsigned)((rows + DH_THREADS / 32 - 1) / (DH_THREADS / 32)), dslices);
    sparton_bwd_dh_kernel<CPL, OutT><<<grid, DH_THREADS, 0, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_dh_kernel", e);
  }
  return SPARTON_OK;
}

template <typename OutT>
int launch_bwd_dtype(const BwdParams& p, cudaStream_t stream) {
  if (p.D <= 256) return launch_bwd_t<1, OutT>(p, stream);
  if (p.D <= 512) return launch_bwd_t<2, OutT>(p, stream);
  if (p.D <= 768) return launch_bwd_t<3, OutT>(p, stream);
  return launch_bwd_t<4, OutT>(p, stream);
}

}  // namespace

int bwd_max_seq() { return ROUTE_SMEM_INTS - 32; }

size_t bwd_workspace_bytes(long long B, long long S, long long V) {
  const size_t pairs = (size_t)B * (size_t)V * sizeof(int2);
  const size_t offs = (size_t)B * (size_t)(S + 1) * sizeof(int);
  return ((pairs + 255) & ~size_t(255)) + ((offs + 255) & ~size_t(255));
}

int launch_bwd(const BwdParams& p, int grad_dtype, cudaStream_t stream) {
  if (grad_dtype == SPARTON_BF16) return launch_bwd_dtype<__nv_bfloat16>(p, stream);
  return launch_bwd_dtype<float>(p, stream);
}

}  // namespace sparton
