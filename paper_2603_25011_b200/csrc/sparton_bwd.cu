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
//   K2s sparton_bwd_de_staged_kernel (S <= 832, the default): CTA owns 720
//                               vocab rows x 64 columns of D with fp32 sums in
//                               registers over the whole batch; per batch row
//                               the H[b] slice is staged in smem (TMA multicast
//                               over a 2-CTA cluster, 4 for S > 512) and every pair reads its
//                               argmax row from smem.  db by a column-sum kernel.
//   K2 sparton_bwd_de_kernel  : (S > 832) CTA owns 2*W vocab rows x one D slice; warps own
//                               2 vocab rows, lanes 8-wide D chunks; for each
//                               batch row (ascending) each warp gathers its
//                               argmax H rows with 1-D TMA bulk copies into a
//                               private mbarrier ring, 4 batch rows deep.
//   K3a sparton_bwd_route_kernel : CTA per (vocab window, b): one pass over Y/I/dY
//                               computes g and the staged dE's (s, g) records,
//                               then a stable counting sort in smem of the
//                               window's active (v, g) pairs by argmax position
//                               s, written out coalesced as per-(b, window, s)
//                               lists in ascending v.
//   K3b sparton_bwd_dh_kernel : warp owns one (b, s) row (x D slice) and sums
//                               g * E[v,:] over its list in ascending v, in
//                               L2-sized vocabulary chunks (one launch each,
//                               the fp32 partial sums carried between them).
// All arithmetic is fp32 (inputs bf16), exactly one owner per output element.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cmath>
#include <cstdlib>

#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "ptx.cuh"
#include "sparton_internal.h"

namespace sparton {

namespace {

constexpr int DE_RPW = 2;       // vocab rows per warp (a CTA of W warps owns 2*W vocab rows)
constexpr int DH_THREADS = 256;
constexpr int DH_PERSIST_THREADS = 640;
constexpr int DH_FP8_THREADS = 512;
constexpr int DH_FP8_UNROLL = 8;

// A (b, v) pair contributes iff Y > 0 (fused.py:247-249).  An argmax index
// outside [0, S) (saved state from another forward) is treated as inactive
// instead of addressing memory out of bounds; the reference would raise
// IndexError there, the ABI validates shapes only (fused.py:232-235).
__device__ __forceinline__ bool pair_active(float y, int k, int S) {
  return y > 0.f && (unsigned)k < (unsigned)S;
}

__device__ __forceinline__ float pair_grad(float y, float dy) {
  // exp(-Y) == 1/(1+rawmax) (fused.py:247-249); accurate expf, no fast-math.
  return dy * expf(-y);
}

// Sparse-regime decisions (BwdParams::stats): every thread of a launch reads
// the same count, written by the route earlier in stream order.
__device__ __forceinline__ bool de_sparse(const BwdParams& p) {
  return p.stats != nullptr && (long long)__ldg(p.stats) <= p.de_sparse_max;
}
__device__ __forceinline__ bool dh_sparse(const BwdParams& p) {
  return p.stats != nullptr && (long long)__ldg(p.stats) <= p.dh_sparse_max;
}

// acc[0..7] += g * bf16x8(raw), as four packed fp32x2 FMAs (FFMA2: two
// independent round-to-nearest fp32 FMAs, bit-identical to scalar fmaf).
// bf16 -> fp32 is exact: the low half of each 32-bit word moves to the top
// (byte permute), the high half is masked in place — both on the ALU pipe, so
// the FMA pipe only carries the FFMA2s.
__device__ __forceinline__ uint64_t pack_gg(float g) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(g));
  return r;
}

__device__ __forceinline__ void fma8(float* acc, uint64_t gg, const int4& raw) {
  const uint32_t w[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    asm("{\n.reg .b32 lo, hi;\n.reg .b64 x, a;\n"
        "prmt.b32 lo, %2, 0, 0x1044;\n"
        "and.b32 hi, %2, 0xffff0000;\n"
        "mov.b64 x, {lo, hi};\n"
        "mov.b64 a, {%0, %1};\n"
        "fma.rn.f32x2 a, x, %3, a;\n"
        "mov.b64 {%0, %1}, a;\n}\n"
        : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1])
        : "r"(w[i]), "l"(gg));
  }
}

// FP8 operands (sparton_bwd_fp8): acc[0..7] += g * e4m3x8(raw), exact e4m3 ->
// f16 -> f32 conversions (F2FP.F16.E4M3.UNPACK_B + HADD2.F32), then FFMA2.
__device__ __forceinline__ void fma4_e4m3(float* acc, uint64_t gg, uint32_t w) {
  asm("{\n.reg .b16 p0, p1, a0, a1, a2, a3;\n.reg .b32 h0, h1;\n.reg .f32 f0, f1, f2, f3;\n"
      ".reg .b64 x0, x1, c0, c1;\n"
      "mov.b32 {p0, p1}, %4;\n"
      "cvt.rn.f16x2.e4m3x2 h0, p0;\n"
      "cvt.rn.f16x2.e4m3x2 h1, p1;\n"
      "mov.b32 {a0, a1}, h0;\n"
      "mov.b32 {a2, a3}, h1;\n"
      "cvt.f32.f16 f0, a0;\n"
      "cvt.f32.f16 f1, a1;\n"
      "cvt.f32.f16 f2, a2;\n"
      "cvt.f32.f16 f3, a3;\n"
      "mov.b64 x0, {f0, f1};\n"
      "mov.b64 x1, {f2, f3};\n"
      "mov.b64 c0, {%0, %1};\n"
      "mov.b64 c1, {%2, %3};\n"
      "fma.rn.f32x2 c0, x0, %5, c0;\n"
      "fma.rn.f32x2 c1, x1, %5, c1;\n"
      "mov.b64 {%0, %1}, c0;\n"
      "mov.b64 {%2, %3}, c1;\n}\n"
      : "+f"(acc[0]), "+f"(acc[1]), "+f"(acc[2]), "+f"(acc[3])
      : "r"(w), "l"(gg));
}

__device__ __forceinline__ void fma8_e4m3(float* acc, uint64_t gg, const uint2& raw) {
  fma4_e4m3(acc, gg, raw.x);
  fma4_e4m3(acc + 4, gg, raw.y);
}

__device__ __forceinline__ void fma16_e4m3(float* acc, uint64_t gg, const int4& raw) {
  fma4_e4m3(acc, gg, (uint32_t)raw.x);
  fma4_e4m3(acc + 4, gg, (uint32_t)raw.y);
  fma4_e4m3(acc + 8, gg, (uint32_t)raw.z);
  fma4_e4m3(acc + 12, gg, (uint32_t)raw.w);
}

// Dequantisation scale of an e4m3 operand (amax / 448), or 1 for bf16.
__device__ __forceinline__ float dq_scale(const float* amax) { return amax ? __ldg(amax) * (1.0f / 448.0f) : 1.0f; }

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
// CTA = 32 vocab rows x one D slice (DS = 256*CPL columns); 16 warps own 2
// vocab rows each, lanes own 8-wide D chunks, fp32 accumulators in registers.
// Batch rows are visited in ascending order (the reference's order).  Each
// warp runs its own NST-deep TMA pipeline: lanes 0..1 gather the warp's 2
// argmax H rows H[b, I[b,v], slice] for batch row b+NST-1 with 1-D bulk copies
// (cp.async.bulk, one instruction per row) into a private smem ring, lane 0
// arms that stage's mbarrier with the byte count; the warp consumes stage b.
// No register staging and no CTA-wide barrier on the gather path, so ~144 KB
// of rows are in flight per SM.  (g, I) for 32 batch rows at a time are
// staged in smem (double buffered, one __syncthreads per 32 batch rows).
constexpr int DE_BC = 32;       // batch rows per (g, I) tile

template <int CPL, int W>
struct DeCfg {
  static constexpr int DE_WARPS = W;
  static constexpr int DE_VB = W * DE_RPW;
  static constexpr int DE_THREADS = W * 32;
  static constexpr int DS = 256 * CPL;                       // slice width (elements)
  static constexpr int ROW_BYTES = DS * 2;
  static constexpr int NST = CPL >= 2 ? 4 : 8;
  static constexpr int WARP_STAGE_BYTES = DE_RPW * ROW_BYTES;  // DE_RPW rows per warp per stage
  static constexpr int RING_BYTES = DE_WARPS * NST * WARP_STAGE_BYTES;
  static constexpr int GI_BYTES = 2 * DE_BC * DE_VB * 8;      // (I, g) pairs, double buffered
  static constexpr int BAR_BYTES = DE_WARPS * NST * 8;
  static constexpr int SMEM_BYTES = RING_BYTES + GI_BYTES + BAR_BYTES;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int CPL, int W, bool FULL, typename OutT>
__global__ void __launch_bounds__(W * 32, 1)
sparton_bwd_de_kernel(const BwdParams p, int bbeg, int bend) {
  using C = DeCfg<CPL, W>;
  constexpr int DE_WARPS = C::DE_WARPS;
  constexpr int DE_VB = C::DE_VB;
  constexpr int DE_THREADS = C::DE_THREADS;
  extern __shared__ __align__(128) uint8_t de_smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* ring = de_smem + (size_t)warp * C::NST * C::WARP_STAGE_BYTES;       // this warp's ring
  int2* gi_s = reinterpret_cast<int2*>(de_smem + C::RING_BYTES);                // [2][BC][VB] (idx, g)
  uint64_t* bars = reinterpret_cast<uint64_t*>(de_smem + C::RING_BYTES + C::GI_BYTES) + warp * C::NST;

  const int v0 = blockIdx.x * DE_VB;
  const int d0 = blockIdx.y * C::DS;
  const uint32_t slice_bytes = FULL ? (uint32_t)C::ROW_BYTES : (uint32_t)min(C::DS, p.D - d0) * 2u;
  const int nb = bend - bbeg;                // batch rows of this pass (local index lb = b - bbeg)
  const bool first = bbeg == 0;
  const bool last = bend == p.B;

  // Rows of inactive pairs are never copied: the ring must hold finite values
  // so that g = 0 times the stale row adds exactly nothing.
  for (int i = lane; i < C::NST * C::WARP_STAGE_BYTES / 16; i += 32)
    reinterpret_cast<int4*>(ring)[i] = make_int4(0, 0, 0, 0);
  if (lane == 0) {
    for (int i = 0; i < C::NST; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), 1);
    ptx::fence_mbar_init();
  }

  // Stage (I, g) of local batch rows [lb0, lb0 + DE_BC) into buffer `buf`.
  // (I, g) staging is register double-buffered: the raw (Y, dY, I) of the tile
  // after next are loaded right after a tile boundary and only consumed at the
  // next boundary, so their latency never stalls the gather pipeline.
  constexpr int GI_PER_THREAD = DE_BC * DE_VB / DE_THREADS;
  float ry[GI_PER_THREAD], rdy[GI_PER_THREAD];
  int ri[GI_PER_THREAD];
  auto load_gi = [&](int lb0) {
#pragma unroll
    for (int q = 0; q < GI_PER_THREAD; ++q) {
      const int e = threadIdx.x + q * DE_THREADS;
      const int bb = e / DE_VB, vv = e % DE_VB;
      const int lb = lb0 + bb, v = v0 + vv;
      ry[q] = 0.f;
      rdy[q] = 0.f;
      ri[q] = -1;
      if (lb < nb && v < p.V) {
        const size_t b = (size_t)(bbeg + lb);
        ry[q] = p.Y[b * p.ldY + v];
        rdy[q] = p.dY[b * p.ldDY + v];
        ri[q] = p.I[b * p.ldY + v];
      }
    }
  };
  auto store_gi = [&](int buf) {
#pragma unroll
    for (int q = 0; q < GI_PER_THREAD; ++q) {
      const int e = threadIdx.x + q * DE_THREADS;
      const int bb = e / DE_VB, vv = e % DE_VB;
      const bool act = pair_active(ry[q], ri[q], p.S);
      gi_s[(buf * DE_BC + bb) * DE_VB + vv] =
          make_int2(act ? ri[q] : -1, __float_as_int(act ? pair_grad(ry[q], rdy[q]) : 0.f));
    }
  };
  // Lanes 0..DE_RPW-1 gather this warp's rows for local batch row lb into ring
  // stage lb % NST (one bulk copy each); lane 0 arms the stage barrier.  The
  // stage was last read (generic proxy) by this same warp before the
  // __syncwarp that ended the previous step, so no proxy fence is needed for
  // this write-after-read (the reads have retired into registers).
  const char* hslice = reinterpret_cast<const char*>(p.H) + (size_t)d0 * 2;
  const size_t hrow_bytes = (size_t)p.D * 2;
  auto issue = [&](int lb) {
    const int t = lb / DE_BC, bb = lb - t * DE_BC, buf = t & 1;
    const int st = lb % C::NST;
    const uint32_t bar = ptx::smem_u32(&bars[st]);
    const int idx = lane < DE_RPW ? gi_s[(buf * DE_BC + bb) * DE_VB + warp + DE_WARPS * lane].x : -1;
    const unsigned act = __ballot_sync(0xffffffffu, idx >= 0);
    if (lane == 0) ptx::mbar_arrive_expect_tx(bar, (uint32_t)__popc(act) * slice_bytes);
    if (idx >= 0) {
      const size_t hrow = (size_t)(bbeg + lb) * p.S + idx;
      bulk_g2s(ptx::smem_u32(ring + st * C::WARP_STAGE_BYTES + lane * C::ROW_BYTES),
               hslice + hrow * hrow_bytes, slice_bytes, bar);
    }
  };

  float acc[DE_RPW][CPL * 8];
  float gsum[DE_RPW];
  bool dvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) dvalid[c] = FULL || (c * 256 + lane * 8) * 2 < (int)slice_bytes;
  // fp32 carry from the previous pass (the fp32 output itself, or the workspace).
  float* carry = p.dE_acc ? p.dE_acc : reinterpret_cast<float*>(p.dE);
#pragma unroll
  for (int r = 0; r < DE_RPW; ++r) {
    const int v = v0 + warp + DE_WARPS * r;
    gsum[r] = (!first && v < p.V) ? p.db_acc[v] : 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      if (!first && v < p.V && dvalid[c]) {
        const float* src = carry + (size_t)v * p.D + d0 + c * 256 + lane * 8;
        const float4 a = *reinterpret_cast<const float4*>(src);
        const float4 bq = *reinterpret_cast<const float4*>(src + 4);
        acc[r][c * 8 + 0] = a.x; acc[r][c * 8 + 1] = a.y; acc[r][c * 8 + 2] = a.z; acc[r][c * 8 + 3] = a.w;
        acc[r][c * 8 + 4] = bq.x; acc[r][c * 8 + 5] = bq.y; acc[r][c * 8 + 6] = bq.z; acc[r][c * 8 + 7] = bq.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[r][c * 8 + i] = 0.f;
      }
    }
  }

  const int ntiles = (nb + DE_BC - 1) / DE_BC;
  load_gi(0);
  store_gi(0);
  if (ntiles > 1) {
    load_gi(DE_BC);
    store_gi(1);
  }
  if (ntiles > 2) load_gi(2 * DE_BC);
  __syncthreads();
  // Prologue: NST-1 batch rows in flight (all within tiles 0/1, NST-1 < DE_BC).
  for (int lb = 0; lb < C::NST - 1 && lb < nb; ++lb) issue(lb);
  const uint8_t* lane_src = ring + lane * 16;

  // Main loop, unrolled by NST so every ring stage index and phase is a
  // compile-time constant (DE_BC is a multiple of NST: tile boundaries fall on
  // iteration boundaries).
  static_assert(DE_BC % C::NST == 0, "tile must hold whole pipeline rounds");
  for (int lb0 = 0; lb0 < nb; lb0 += C::NST) {
    const int t = lb0 / DE_BC, buf = t & 1;
    if (lb0 % DE_BC == 0 && t > 0) {
      // Tile t is resident (staged one tile ahead); refill the other buffer with
      // tile t+1 once every warp is done with tile t-1.
      __syncthreads();
      if (t + 1 < ntiles) store_gi(buf ^ 1);        // loaded one tile ago
      if (t + 2 < ntiles) load_gi((t + 2) * DE_BC);
      __syncthreads();
    }
    const uint32_t parity = (uint32_t)(lb0 / C::NST) & 1u;
    const int2* gi_row = gi_s + (buf * DE_BC + (lb0 - t * DE_BC)) * DE_VB + warp;
#pragma unroll
    for (int j = 0; j < C::NST; ++j) {
      const int lb = lb0 + j;
      if (lb < nb) {
        // Issue batch row lb+NST-1 (tile t or t+1, both resident) into stage (j-1) mod NST.
        if (lb + C::NST - 1 < nb) issue(lb + C::NST - 1);
        float g[DE_RPW];
#pragma unroll
        for (int r = 0; r < DE_RPW; ++r) g[r] = __int_as_float(gi_row[j * DE_VB + DE_WARPS * r].y);
        ptx::mbar_wait(ptx::smem_u32(&bars[j]), parity);
        const uint8_t* src = lane_src + j * C::WARP_STAGE_BYTES;
#pragma unroll
        for (int r = 0; r < DE_RPW; ++r) {
          gsum[r] += g[r];
          const uint64_t gg = pack_gg(g[r]);
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if (dvalid[c]) {
              const int4 x = *reinterpret_cast<const int4*>(src + r * C::ROW_BYTES + c * 512);
              fma8(&acc[r][c * 8], gg, x);
            }
          }
        }
        __syncwarp();
      }
    }
  }

#pragma unroll
  for (int r = 0; r < DE_RPW; ++r) {
    const int v = v0 + warp + DE_WARPS * r;
    if (v >= p.V) continue;
    if (last) {
      OutT* dst = reinterpret_cast<OutT*>(p.dE) + (size_t)v * p.D + d0 + lane * 8;
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (dvalid[c]) store8<OutT>(dst + c * 256, &acc[r][c * 8]);
      if (blockIdx.y == 0 && lane == 0 && p.db != nullptr)
        p.db[v] = p.include_bias_grad ? gsum[r] : 0.f;
    } else {
      float* dst = carry + (size_t)v * p.D + d0 + lane * 8;
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (dvalid[c]) store8<float>(dst + c * 256, &acc[r][c * 8]);
      if (blockIdx.y == 0 && lane == 0) p.db_acc[v] = gsum[r];
    }
  }
}

// ------------------------------------------------------------------ K2s: staged dE
// dE with on-chip reuse of H instead of per-pair L2 gathers.  A CTA owns a
// block of VB vocab rows x one 64-column slice of D and keeps the VB x 64 fp32
// accumulators in registers for the whole batch (no carry passes).  For each
// batch row b (ascending — the reference's order) the slice H[b, 0:S, d0:d0+64]
// is staged in shared memory (S rows of 128 B) together with the block's
// (s, g) records; every (b, v) pair then reads its argmax row from shared
// memory.  Eight lanes own one vocab row (16 B = 8 columns each), so a warp's
// 128-bit shared load touches four whole 128-B rows: conflict-free for any
// argmax pattern.  The cluster's CL CTAs (2 or 4) hold neighbouring vocab blocks
// of the same slice: each loads S/CL rows of the tile and multicasts them
// to all, so a tile costs one L2 read per cluster.  Warp NW is the TMA
// producer; stage reuse is released cluster-wide (every consumer warp arrives
// on the empty barrier of every CTA, since peers' multicasts write into it).
// Cluster size: 2 CTAs share each tile when S/2 rows fit one TMA box (S <= 512),
// else 4.  Pairs measured 11 % faster than quads at S = 512: every stage waits
// for the slowest consumer of the cluster before it is refilled, and the extra
// L2 traffic of halving the multicast fan-out is cheap here.
int de_cluster(int S) {
  if (const char* ev = dev_env("SPARTON_DE_CL")) {   // experiment switch: 1, 2 or 4
    const int c = atoi(ev);
    if (c == 1 || c == 2 || c == 4) return c;
  }
  return ((S + 1) / 2 + 7) / 8 * 8 <= 256 ? 2 : 4;
}
// A staged row holds the item's 64 columns of D: 128 B of bf16, or (FP8)
// 64 B of e4m3 — half the tile-write and row-read bytes of shared memory for
// the same 720 vocab rows of fp32 accumulators.  Each of the 8 lanes of a row
// group owns 8 columns (16 B bf16 / 8 B e4m3) of every row it reads.
template <int NW, int J, bool FP8 = false>
struct DeStCfg {
  static constexpr int THREADS = (NW + 1) * 32;
  static constexpr int GROUPS = NW * 4;       // 8-lane groups, one vocab row each per step
  static constexpr int VB = GROUPS * J;       // vocab rows per CTA
  static constexpr int GI_BYTES = VB * 8;
  static constexpr int DD = 64;               // D columns per work item
  static constexpr int AW = 8;                // accumulators per (lane, vocab row)
  static constexpr int RB = FP8 ? 64 : 128;   // bytes per staged row
};

__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* m, uint32_t dst, uint32_t bar, int32_t c0,
                                               int32_t c1, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5, %6;"
      :: "r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
      : "memory");
}

template <int NW, int J, int CL, typename OutT, bool FP8 = false>
__global__ void __launch_bounds__(DeStCfg<NW, J, FP8>::THREADS, 1)
sparton_bwd_de_staged_kernel(const __grid_constant__ CUtensorMap tmH, const BwdParams p, int R, int nst,
                             int stage_bytes, int nvg, int nitems) {
  using C = DeStCfg<NW, J, FP8>;
  if (de_sparse(p)) return;   // uniform over the grid: before any cluster barrier
  extern __shared__ __align__(128) uint8_t ds_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ds_smem + (size_t)nst * stage_bytes);
  uint64_t* empty = full + nst;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_ctarank();
  // Persistent: cluster c walks work items c, c + G, ... ; item i = (vocab
  // group i % nvg of CL blocks, D slice i / nvg).  Consecutive clusters
  // share a D slice, so their H tiles are L2-shared.
  const int cl = (int)(blockIdx.x / CL), ncl = (int)(gridDim.x / CL);
  // Stage layout: [zero row][S-row tile][GI records].  s = -1 (inactive pair)
  // addresses the zero row, so inactive pairs never touch H.
  const uint32_t tile_bytes = (uint32_t)(CL * R * C::RB);
  const uint32_t gi_off = 128 + tile_bytes;

  // Zero rows and GI regions start zeroed / (-1, 0): entries past the
  // vocabulary (never copied) read the zero row with g = 0.
  for (int i = threadIdx.x; i < nst * 8; i += C::THREADS)
    reinterpret_cast<int4*>(ds_smem + (size_t)(i / 8) * stage_bytes)[i % 8] = make_int4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < nst * C::GI_BYTES / 16; i += C::THREADS) {
    const int st = i / (C::GI_BYTES / 16), o = i % (C::GI_BYTES / 16);
    reinterpret_cast<int4*>(ds_smem + (size_t)st * stage_bytes + gi_off)[o] = make_int4(-1, 0, -1, 0);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), CL * NW);
    }
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async();   // zeroed GI visible to the async proxy before any bulk copy lands
  ptx::cluster_sync();

  if (warp == NW) {
    if (lane == 0) {
      // ------------------------------------------------ producer
      const uint64_t pol = ptx::policy_evict_normal();
      int st = 0;
      uint32_t ph = 0;
      for (int it = cl; it < nitems; it += ncl) {
      const int v0 = ((it % nvg) * CL + (int)crank) * C::VB;
      const int d0 = (it / nvg) * C::DD;
      const long long vrem = (long long)p.ldGI - v0;          // even
      const uint32_t gi_bytes = (uint32_t)(vrem >= C::VB ? C::GI_BYTES : (vrem > 0 ? vrem * 8 : 0));
      for (int b = 0; b < p.B; ++b) {
        ptx::mbar_wait(ptx::smem_u32(&empty[st]), ph ^ 1);
        const uint32_t sbase = ptx::smem_u32(ds_smem + (size_t)st * stage_bytes);
        const uint32_t fb = ptx::smem_u32(&full[st]);
        ptx::mbar_arrive_expect_tx(fb, tile_bytes + gi_bytes);
        // R rows per CTA in boxes of at most 256 rows (the TMA box limit).
        for (int r0 = 0; r0 < R; r0 += 256)
          tma_load_2d_mc(&tmH, sbase + 128 + (crank * (uint32_t)R + (uint32_t)r0) * (uint32_t)C::RB, fb, d0,
                         b * p.S + (int)crank * R + r0, (uint16_t)((1u << CL) - 1u), pol);
        if (gi_bytes) bulk_g2s(sbase + gi_off, p.gi + (size_t)b * p.ldGI + v0, gi_bytes, fb);
        if (++st == nst) { st = 0; ph ^= 1; }
      }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ consumers
    const int grp = warp * 4 + (lane >> 3);
    const int sub = lane & 7;
    int st = 0;
    uint32_t ph = 0;
    for (int it = cl; it < nitems; it += ncl) {
    const int v0 = ((it % nvg) * CL + (int)crank) * C::VB;
    const int d0 = (it / nvg) * C::DD;
    float acc[J][C::AW];
#pragma unroll
    for (int j = 0; j < J; ++j)
#pragma unroll
      for (int i = 0; i < C::AW; ++i) acc[j][i] = 0.f;
    for (int b = 0; b < p.B; ++b) {
      ptx::mbar_wait(ptx::smem_u32(&full[st]), ph);
      const uint8_t* tile = ds_smem + (size_t)st * stage_bytes;
      const uint8_t* rows = tile + 128 + sub * (C::RB / 8);
      // Group grp owns vocab rows grp + GROUPS*j: one broadcast record load each.
      const int2* gi = reinterpret_cast<const int2*>(tile + gi_off) + grp;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int2 e = gi[C::GROUPS * j];
        if constexpr (FP8) {
          const uint2 x = *reinterpret_cast<const uint2*>(rows + e.x * C::RB);
          fma8_e4m3(acc[j], pack_gg(__int_as_float(e.y)), x);
        } else {
          const int4 x = *reinterpret_cast<const int4*>(rows + e.x * C::RB);
          fma8(acc[j], pack_gg(__int_as_float(e.y)), x);
        }
      }
      // Every lane's shared loads have been consumed by its FMAs (retired), so a
      // relaxed arrival (no MEMBAR) suffices to release the stage to the
      // peers' TMA writes.
      __syncwarp();
      if (lane < CL) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&empty[st]), (uint32_t)lane));
      if (++st == nst) { st = 0; ph ^= 1; }
    }
    const int d = d0 + sub * C::AW;
    if (d < p.D) {
      // FP8: dE = (amax_h / 448) * sum_b g * q_h, scaled once per element.
      const float sc = FP8 ? dq_scale(p.amax_h) : 1.0f;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int v = v0 + grp + C::GROUPS * j;
        if (v < p.V) {
          if constexpr (FP8) {
#pragma unroll
            for (int i = 0; i < C::AW; ++i) acc[j][i] *= sc;
          }
#pragma unroll
          for (int h = 0; h < C::AW; h += 8)
            if (d + h < p.D) store8<OutT>(reinterpret_cast<OutT*>(p.dE) + (size_t)v * p.D + d + h, acc[j] + h);
        }
      }
    }
    }  // items
  }
  // Peers may still multicast into / arrive on this CTA until every CTA is done.
  ptx::cluster_sync();
}

// db[v] = sum_b g[b, v] (b ascending) from the (s, g) records.
__global__ void __launch_bounds__(256)
sparton_bwd_db_kernel(const BwdParams p) {
  const int v = blockIdx.x * 256 + threadIdx.x;
  if (v >= p.V || p.db == nullptr || de_sparse(p)) return;
  float s = 0.f;
  if (p.include_bias_grad) {
    const int2* col = p.gi + v;
    for (int b = 0; b < p.B; ++b) s += __int_as_float(__ldg(&col[(size_t)b * p.ldGI].y));
  }
  p.db[v] = s;
}

// ------------------------------------------------------------------ K2x: sparse dE
// The sparse regime (at most de_sparse_max active pairs; SPLADE
// representations are mostly zeros): staging whole H tiles per batch row
// would pay the dense price for a few pairs.  Warp owns one vocab row v and
// a slice of 256*CPL columns of D (grid.y; lane l: columns d0 + c*256 + l*8
// .. +8).  It scans the route's (s, g)
// records of column v, 32 batch rows per load (lane = b), and gathers
// H[b, s, :] for the active pairs only, in ascending b (the reference's
// order, fused.py:255-265), DES_U rows in flight; db[v] is the ascending sum
// of the same g.  Same fp32 FMA chain per output element as the staged dE
// (which adds g = 0 times a zero row for inactive pairs).
constexpr int DES_THREADS = 512;
constexpr int DES_U = 4;

template <int CPL, bool FULL, typename OutT>
__global__ void __launch_bounds__(DES_THREADS, 1)
sparton_bwd_de_sparse_kernel(const BwdParams p) {
  if (!de_sparse(p)) return;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int d0 = blockIdx.y * (256 * CPL);
  bool dvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) dvalid[c] = FULL || (d0 + c * 256 + lane * 8) < p.D;
  const long long nwarps = (long long)gridDim.x * (DES_THREADS / 32);
  for (long long v = (long long)blockIdx.x * (DES_THREADS / 32) + warp; v < p.V; v += nwarps) {
    float acc[CPL * 8];
#pragma unroll
    for (int i = 0; i < CPL * 8; ++i) acc[i] = 0.f;
    float gsum = 0.f;
    const int2* col = p.gi + v;
    // Records of batch rows b0 + lane and b0 + 32 + lane in flight.
    int2 r0 = lane < p.B ? __ldg(&col[(size_t)lane * p.ldGI]) : make_int2(-1, 0);
    int2 r1 = 32 + lane < p.B ? __ldg(&col[(size_t)(32 + lane) * p.ldGI]) : make_int2(-1, 0);
    for (int b0 = 0; b0 < p.B; b0 += 32) {
      const int2 rec = r0;
      r0 = r1;
      r1 = b0 + 64 + lane < p.B ? __ldg(&col[(size_t)(b0 + 64 + lane) * p.ldGI]) : make_int2(-1, 0);
      unsigned act = __ballot_sync(0xffffffffu, rec.x >= 0);
      while (act) {
        int ln[DES_U];
        float gq[DES_U];
        int4 xq[DES_U][CPL];
#pragma unroll
        for (int q = 0; q < DES_U; ++q) {
          ln[q] = act ? __ffs(act) - 1 : -1;
          act &= act - 1u;
          const int src = ln[q] < 0 ? 0 : ln[q];
          const int s = __shfl_sync(0xffffffffu, rec.x, src);
          gq[q] = __int_as_float(__shfl_sync(0xffffffffu, rec.y, src));
          const __nv_bfloat16* r = p.H + ((size_t)(b0 + src) * p.S + (s < 0 ? 0 : s)) * p.D + d0 + lane * 8;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            xq[q][c] = (ln[q] >= 0 && dvalid[c]) ? __ldg(reinterpret_cast<const int4*>(r + c * 256))
                                                 : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < DES_U; ++q) {
          if (ln[q] >= 0) {
            gsum += gq[q];
            const uint64_t gg = pack_gg(gq[q]);
#pragma unroll
            for (int c = 0; c < CPL; ++c) fma8(&acc[c * 8], gg, xq[q][c]);
          }
        }
      }
    }
    OutT* dst = reinterpret_cast<OutT*>(p.dE) + (size_t)v * p.D + d0 + lane * 8;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (dvalid[c]) store8<OutT>(dst + c * 256, &acc[c * 8]);
    if (blockIdx.y == 0 && lane == 0 && p.db != nullptr) p.db[v] = p.include_bias_grad ? gsum : 0.f;
  }
}

// ------------------------------------------------------------------ K3a: route
// Grid (window, b).  The vocabulary is cut into windows of RT_WIN rows; for
// each (b, window) the CTA performs a stable counting sort of the window's
// active pairs by key s = I[b,v] (counters in shared memory) and scatters the
// sorted (v, g) run into the window's output range, with per-(b, window, s)
// offsets.  Stability: the window is split into `nseg` contiguous segments,
// one per warp; per-(segment, s) counts give every warp its own cursors, and
// equal keys inside a warp are ranked by lane order (match.any), so every
// (b, window, s) sub-list is in ascending v.
constexpr int RT_THREADS = 512;
constexpr int RT_WIN = 8192;
// Three CTAs per SM (40 registers, ~100 B of the register stash spills to
// L1-backed local memory): 30 % faster than two CTAs at 58 registers, and
// ahead of four at 32 (tools/ab_kernels.sh, locked clocks).
constexpr int RT_MINB = 3;
constexpr int RT_SMEM_BUDGET = 200 * 1024;

__global__ void __launch_bounds__(RT_THREADS, RT_MINB)
sparton_bwd_route_kernel(const BwdParams p, int nseg, int nwin, int allow_stash) {
  extern __shared__ int4 rt_smem[];
  const int S = p.S;
  int* hist = reinterpret_cast<int*>(rt_smem);        // [nseg][S]
  int* scan_tmp = hist + nseg * S;                    // [32]
  const int w = blockIdx.x;
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int v0 = w * RT_WIN;
  const int n = min(RT_WIN, p.V - v0);
  const int seg_len = (n + nseg - 1) / nseg;

  __shared__ unsigned int n_active;   // active pairs of this (b, window), for the sparse regime
  for (int i = threadIdx.x; i < nseg * S; i += RT_THREADS) hist[i] = 0;
  if (threadIdx.x == 0) n_active = 0;
  __syncthreads();

  const float* Yb = p.Y + (size_t)b * p.ldY + v0;
  const int32_t* Ib = p.I + (size_t)b * p.ldY + v0;
  const float* dYb = p.dY + (size_t)b * p.ldDY + v0;

  // Phase 1: per-segment histograms.  When a warp's segment fits its register
  // stash (every warp owns a segment: S <= 2125), Y/I/dY are read once here:
  // g and the staged dE's (s, g) record are produced now and (s, g) kept in
  // registers for the scatter, so phase 3 touches no global memory.
  constexpr int RQ = RT_WIN / RT_THREADS;   // stashed elements per lane
  const bool stash = allow_stash && seg_len <= 32 * RQ;
  int rk[RQ];
  float rg[RQ];
  int2* gib = p.gi ? p.gi + (size_t)b * p.ldGI + v0 : nullptr;
  unsigned int nact = 0;
  if (gib != nullptr && w == nwin - 1 && threadIdx.x == 0)
    for (long long v = p.V; v < p.ldGI; ++v) p.gi[(size_t)b * p.ldGI + v] = make_int2(-1, 0);   // row padding
  if (warp < nseg) {
    const int vs = min(n, warp * seg_len), ve = min(n, (warp + 1) * seg_len);
    int* h = hist + warp * S;
    if (stash) {
#pragma unroll
      for (int q0 = 0; q0 < RQ; q0 += 4) {
        float y[4], dy[4];
        int k[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = vs + (q0 + q) * 32 + lane;
          const bool in = v < ve;
          y[q] = in ? Yb[v] : 0.f;
          k[q] = in ? Ib[v] : 0;
          dy[q] = in ? dYb[v] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = vs + (q0 + q) * 32 + lane;
          const bool active = pair_active(y[q], k[q], S);
          const float g = active ? pair_grad(y[q], dy[q]) : 0.f;
          // (s, g) record for the staged dE; inactive pairs get s = -1 (a zero row).
          if (gib != nullptr && v < ve) gib[v] = make_int2(active ? k[q] : -1, __float_as_int(g));
          if (active) atomicAdd(&h[k[q]], 1);
          nact += active;
          rk[q0 + q] = active ? k[q] : -1;
          rg[q0 + q] = g;
        }
      }
    } else {
      for (int base = vs; base < ve; base += 128) {
        float y[4];
        int k[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = base + q * 32 + lane;
          y[q] = v < ve ? Yb[v] : 0.f;
          k[q] = v < ve ? Ib[v] : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (pair_active(y[q], k[q], S)) {
            atomicAdd(&h[k[q]], 1);
            ++nact;
          }
      }
    }
  }
  if (p.stats != nullptr) {
    nact = __reduce_add_sync(0xffffffffu, nact);
    if (lane == 0 && nact) atomicAdd(&n_active, nact);
  }
  __syncthreads();
  if (p.stats != nullptr && threadIdx.x == 0 && n_active)
    atomicAdd(p.stats, (unsigned long long)n_active);

  // Phase 2: exclusive scan over s of the per-s totals -> window-local list
  // offsets; then per-s exclusive scan over segments -> cursors (in hist).
  int* off = p.offsets + ((size_t)b * nwin + w) * (S + 1);
  int carry = 0;
  for (int s0 = 0; s0 < S; s0 += RT_THREADS) {
    const int s = s0 + threadIdx.x;
    int tot = 0;
    if (s < S)
      for (int q = 0; q < nseg; ++q) tot += hist[q * S + s];
    int x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scan_tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int t = lane < RT_THREADS / 32 ? scan_tmp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < RT_THREADS / 32) scan_tmp[lane] = t;
    }
    __syncthreads();
    const int excl = carry + (warp > 0 ? scan_tmp[warp - 1] : 0) + x - tot;
    if (s < S) {
      off[s] = excl;
      int cur = excl;
      for (int q = 0; q < nseg; ++q) {
        const int c = hist[q * S + s];
        hist[q * S + s] = cur;
        cur += c;
      }
    }
    carry += scan_tmp[RT_THREADS / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) off[S] = carry;

  // Phase 3: stable scatter of (v, g) straight to the window's output run
  // (the run's 64 KB is written completely by this CTA, so L2 merges the 8-byte
  // stores; 4 % faster than sorting into shared memory and copying out).
  // Equal keys inside a warp are ranked by lane order (match.any); the bucket
  // cursor then advances.
  int2* dst = p.pairs + (size_t)b * p.V + v0;
  if (warp < nseg) {
    const int vs = min(n, warp * seg_len), ve = min(n, (warp + 1) * seg_len);
    int* cur = hist + warp * S;
    auto place = [&](int k, float g, int v) {
      const bool active = k >= 0;
      const unsigned amask = __ballot_sync(0xffffffffu, active);
      if (active) {
        const unsigned peers = __match_any_sync(amask, k);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int pos = cur[k] + rank;
        dst[pos] = make_int2(v0 + v, __float_as_int(g));
        __syncwarp(amask);
        if (rank == 0) cur[k] += __popc(peers);
      }
      __syncwarp();
    };
    if (stash) {
#pragma unroll
      for (int q = 0; q < RQ; ++q) place(rk[q], rg[q], vs + q * 32 + lane);
    } else {
      for (int base = vs; base < ve; base += 128) {
        float y[4], dy[4];
        int k[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = base + q * 32 + lane;
          const bool in = v < ve;
          y[q] = in ? Yb[v] : 0.f;
          k[q] = in ? Ib[v] : 0;
          dy[q] = in ? dYb[v] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = base + q * 32 + lane;
          const bool active = pair_active(y[q], k[q], S);
          const float g = active ? pair_grad(y[q], dy[q]) : 0.f;
          if (gib != nullptr && v < ve) gib[v] = make_int2(active ? k[q] : -1, __float_as_int(g));
          place(active ? k[q] : -1, g, v);
        }
      }
    }
  }
  __syncthreads();

}

// ------------------------------------------------------------------ K3b: dH
// Warp owns one (b, s) row (x D slice).  The vocabulary is processed in
// L2-sized chunks of `wpc` route windows (~52 MB of E) by successive launches,
// so the E rows every resident warp gathers come from the same window of E.
// Within a chunk the warp walks its (b, window, s) sub-lists in window order,
// each in ascending v, so the accumulation order is exactly the reference's
// (v ascending, hidden_row / np.add.at).  Partial sums carry across launches in
// fp32 (the output itself when it is fp32, else the workspace accumulator).
//
// SPW (sparse regime, bf16 only): one launch walks the whole vocabulary in
// groups of 32 windows without the fp32 carry (the few E rows it gathers need
// no L2-sized chunks); the dense launches exit, or SPW exits when dense.
template <int CPL, int DH_UNROLL, int MINB, bool FULL, typename OutT, int THREADS = DH_THREADS, bool FP8 = false,
          bool SPW = false>
__global__ void __launch_bounds__(THREADS, MINB)
sparton_bwd_dh_kernel(const BwdParams p, int chunk) {
  // Lane l owns columns d0 + c*256 + l*8 .. +8 of its row (bf16: one 16-B
  // load per chunk c; FP8: one 8-B load of e4m3 bytes).
  using XT = typename std::conditional<FP8, uint2, int4>::type;
  constexpr int EB = FP8 ? 1 : 2;   // bytes per E element
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long nrows = (long long)p.B * p.S;
  if (!FP8 && p.stats != nullptr && dh_sparse(p) != SPW) return;
  // Persistent grid-stride over rows (b*S + s): one CTA per SM.
  for (long long rowid = (long long)blockIdx.x * (THREADS / 32) + warp; rowid < nrows;
       rowid += (long long)gridDim.x * (THREADS / 32)) {
  const int b = (int)(rowid / p.S);
  const int s = (int)(rowid - (long long)b * p.S);
  const int d0 = blockIdx.y * (256 * CPL);
  const bool first = SPW || chunk == 0;
  const bool last = SPW || chunk == p.nchunks - 1;
  const int w0 = SPW ? 0 : chunk * p.wpc;
  const int w1 = SPW ? p.nwin : min(p.nwin, w0 + p.wpc);

  bool dvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) dvalid[c] = FULL || (d0 + c * 256 + lane * 8) < p.D;
  float acc[CPL * 8];
  float* accg = p.acc32 ? p.acc32 : reinterpret_cast<float*>(p.dH);   // fp32 carry buffer
  if (first) {
#pragma unroll
    for (int i = 0; i < CPL * 8; ++i) acc[i] = 0.f;
  } else {
    const float* src = accg + (size_t)rowid * p.D + d0 + lane * 8;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      if (dvalid[c]) {
        // The fp32 carry streams through once per pass: evict-first so it does
        // not push the pass's E chunk out of L2.
        const float4 a = __ldcs(reinterpret_cast<const float4*>(src + c * 256));
        const float4 bq = __ldcs(reinterpret_cast<const float4*>(src + c * 256 + 4));
        acc[c * 8 + 0] = a.x; acc[c * 8 + 1] = a.y; acc[c * 8 + 2] = a.z; acc[c * 8 + 3] = a.w;
        acc[c * 8 + 4] = bq.x; acc[c * 8 + 5] = bq.y; acc[c * 8 + 6] = bq.z; acc[c * 8 + 7] = bq.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[c * 8 + i] = 0.f;
      }
    }
  }

  // The row's sub-lists of every window of this pass, read as one flattened
  // list: lane t < nw fetches window wg+t's bounds (one round trip for 32
  // windows), a prefix sum over lanes gives each window's start in the
  // flattened order, and each batch of 32 records is fetched in one load
  // (window order, then ascending v: the reference's summation order).
  // Dense passes span <= 32 windows (wpc is capped on the host): one group.
  for (int wg = w0; SPW ? wg < w1 : wg == w0; wg += 32) {
  const int nw = SPW ? min(32, w1 - wg) : w1 - w0;
  int ks = 0, cnt = 0;
  if (lane < nw) {
    const int* off = p.offsets + ((size_t)b * p.nwin + wg + lane) * (p.S + 1);
    ks = off[s];
    cnt = off[s + 1] - ks;
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int excl = incl - cnt;             // flattened start of window lane (lane < nw)
  const int2* lst0 = p.pairs + (size_t)b * p.V + (size_t)wg * RT_WIN;
  for (int base = 0; base < total; base += 32) {
    const int m = min(32, total - base);
    const int idx = base + lane;
    int wsel = 0, e_sel = 0, k_sel = 0;
    for (int t = 0; t < nw; ++t) {
      const int et = __shfl_sync(0xffffffffu, excl, t);
      const int kt = __shfl_sync(0xffffffffu, ks, t);
      if (idx >= et) { wsel = t; e_sel = et; k_sel = kt; }
    }
    int2 mine = make_int2(0, 0);
    if (lane < m) mine = lst0[(size_t)wsel * RT_WIN + k_sel + (idx - e_sel)];
    int j = 0;
    for (; j + DH_UNROLL <= m; j += DH_UNROLL) {
      float gq[DH_UNROLL];
      XT xq[DH_UNROLL][CPL];
#pragma unroll
      for (int q = 0; q < DH_UNROLL; ++q) {
        const int vq = __shfl_sync(0xffffffffu, mine.x, j + q);
        gq[q] = __int_as_float(__shfl_sync(0xffffffffu, mine.y, j + q));
        const uint8_t* r = reinterpret_cast<const uint8_t*>(p.E) + ((size_t)vq * p.D + d0 + lane * 8) * EB;
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          xq[q][c] = dvalid[c] ? __ldg(reinterpret_cast<const XT*>(r + c * 256 * EB)) : XT{};
      }
#pragma unroll
      for (int q = 0; q < DH_UNROLL; ++q) {
        const uint64_t gg = pack_gg(gq[q]);
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          if constexpr (FP8) fma8_e4m3(&acc[c * 8], gg, xq[q][c]);
          else fma8(&acc[c * 8], gg, xq[q][c]);
        }
      }
    }
    for (; j < m; ++j) {
      const int va = __shfl_sync(0xffffffffu, mine.x, j);
      const float ga = __int_as_float(__shfl_sync(0xffffffffu, mine.y, j));
      const uint8_t* r = reinterpret_cast<const uint8_t*>(p.E) + ((size_t)va * p.D + d0 + lane * 8) * EB;
      const uint64_t gg = pack_gg(ga);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const XT x = dvalid[c] ? __ldg(reinterpret_cast<const XT*>(r + c * 256 * EB)) : XT{};
        if constexpr (FP8) fma8_e4m3(&acc[c * 8], gg, x);
        else fma8(&acc[c * 8], gg, x);
      }
    }
  }
  }  // window groups

  if (last) {
    if constexpr (FP8) {
      // dH = (amax_e / 448) * sum_v g * q_e, scaled once per element.
      const float sc = dq_scale(p.amax_e);
#pragma unroll
      for (int i = 0; i < CPL * 8; ++i) acc[i] *= sc;
    }
    OutT* dst = reinterpret_cast<OutT*>(p.dH) + (size_t)rowid * p.D + d0 + lane * 8;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (dvalid[c]) store8<OutT>(dst + c * 256, &acc[c * 8]);
  } else {
    float* dst = accg + (size_t)rowid * p.D + d0 + lane * 8;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (dvalid[c]) {
        __stcs(reinterpret_cast<float4*>(dst + c * 256), make_float4(acc[c * 8], acc[c * 8 + 1], acc[c * 8 + 2], acc[c * 8 + 3]));
        __stcs(reinterpret_cast<float4*>(dst + c * 256 + 4),
               make_float4(acc[c * 8 + 4], acc[c * 8 + 5], acc[c * 8 + 6], acc[c * 8 + 7]));
      }
  }
  }  // rows
}

int route_nseg(int S) {
  int nseg = (RT_SMEM_BUDGET - RT_WIN * 8 - 128) / (S * 4);
  if (nseg > RT_THREADS / 32) nseg = RT_THREADS / 32;
  if (nseg < 1) nseg = 1;
  return nseg;
}
size_t route_smem_bytes(int S, int nseg) { return ((size_t)nseg * S + 32) * 4; }

template <int CPL, int W, bool FULL, typename OutT>
int launch_de(const BwdParams& p, cudaStream_t stream) {
  using C = DeCfg<CPL, W>;
  constexpr int smem = C::SMEM_BYTES;
  cudaError_t e = cudaFuncSetAttribute(sparton_bwd_de_kernel<CPL, W, FULL, OutT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(de)", e);
  dim3 grid((p.V + C::DE_VB - 1) / C::DE_VB, (p.D + 256 * CPL - 1) / (256 * CPL));
  for (int b0 = 0; b0 < p.B; b0 += p.bchunk) {
    sparton_bwd_de_kernel<CPL, W, FULL, OutT><<<grid, C::DE_THREADS, smem, stream>>>(p, b0, min(p.B, b0 + p.bchunk));
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_de_kernel", e);
  }
  return SPARTON_OK;
}

// Side stream + fork/join events: dE (independent of the route's dH lists)
// runs concurrently with route -> dH so the two gather kernels share the SMs.
// They are per (host thread, device): a call enqueues record(fork) -> wait ->
// dE -> record(join) -> wait without another thread being able to re-record
// the same events in between (two threads calling concurrently on distinct
// streams never see each other's fork/join), and one thread's side-stream
// launches cannot land in another thread's CUDA-graph capture.  Calls from
// one thread are enqueued in program order, so reuse across its calls is safe
// (a later call's dE only queues behind the earlier one on the side stream).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

// Handles of exited threads are parked in a process-wide free list and
// handed to the next thread that needs one: no CUDA call runs in a thread-exit
// destructor (at process exit the runtime may already be torn down).
// (Both intentionally leaked: a thread may exit after static destruction.)
std::mutex& side_mu() { static std::mutex* m = new std::mutex; return *m; }
std::vector<std::pair<int, SideStream>>& side_free() {
  static auto* v = new std::vector<std::pair<int, SideStream>>;
  return *v;
}

struct ThreadSideStreams {
  SideStream dev[64];
  ~ThreadSideStreams() {
    std::lock_guard<std::mutex> lk(side_mu());
    for (int d = 0; d < 64; ++d)
      if (dev[d].s) side_free().emplace_back(d, dev[d]);
  }
};

int side_stream(SideStream& out) {
  thread_local ThreadSideStreams tls;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error("cudaGetDevice", e);
  if (dev >= 64) return set_error(SPARTON_ENOTSUP, "device index >= 64");
  SideStream& c = tls.dev[dev];
  if (!c.s) {
    {
      std::lock_guard<std::mutex> lk(side_mu());
      auto& fl = side_free();
      for (size_t i = 0; i < fl.size(); ++i)
        if (fl[i].first == dev) {
          c = fl[i].second;
          fl.erase(fl.begin() + (long)i);
          break;
        }
    }
    if (!c.s) {
      SideStream n;
      if ((e = cudaStreamCreateWithFlags(&n.s, cudaStreamNonBlocking)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&n.fork, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&n.join, cudaEventDisableTiming)) != cudaSuccess)
        return set_cuda_error("side stream setup", e);
      c = n;
    }
  }
  out = c;
  return SPARTON_OK;
}


int launch_route(const BwdParams& p, cudaStream_t stream) {
  const int nseg = route_nseg(p.S);
  const size_t smem = route_smem_bytes(p.S, nseg);
  // The attribute is the per-function limit, shared by every thread: set it
  // to the budget (a constant), never to this call's size — a concurrent call
  // with a smaller S would otherwise lower it between our set and launch.
  cudaError_t e = cudaFuncSetAttribute(sparton_bwd_route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       RT_SMEM_BUDGET);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(route)", e);
  int allow_stash = 1;
  if (const char* ev = dev_env("SPARTON_ROUTE_STASH")) allow_stash = atoi(ev);   // experiment switch
  sparton_bwd_route_kernel<<<dim3(p.nwin, p.B), RT_THREADS, smem, stream>>>(p, nseg, p.nwin, allow_stash);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_route_kernel", e);
  return SPARTON_OK;
}

template <int CPL, typename OutT, bool FP8 = false>
int launch_dh(const BwdParams& p, cudaStream_t stream) {
  // Persistent: one 640-thread CTA per SM (20 warps x 4 E rows in flight,
  // 96 registers); warps stride over rows independently, so no warp slot
  // idles behind a CTA's slowest row.  11.5 % faster than 3 x 256-thread CTAs
  // per SM with 3 rows in flight (tools/ab_env.sh, locked clocks), and ahead
  // of 24 x 3, 28 x 3, 32 x 2, 16 x 5/6, 20 x 5 and 12 x 8.
  const int dslices = (p.D + 256 * CPL - 1) / (256 * CPL);
  const bool full = p.D % (256 * CPL) == 0;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return set_cuda_error("cudaDeviceGetAttribute(dh)", e);
  const dim3 grid(sms, dslices);
  if constexpr (!FP8) {
    if (p.stats != nullptr) {   // sparse-regime single pass (exits at once when dense)
      if (full)
        sparton_bwd_dh_kernel<CPL, 4, 1, true, OutT, DH_PERSIST_THREADS, false, true><<<grid, DH_PERSIST_THREADS, 0, stream>>>(p, 0);
      else
        sparton_bwd_dh_kernel<CPL, 4, 1, false, OutT, DH_PERSIST_THREADS, false, true><<<grid, DH_PERSIST_THREADS, 0, stream>>>(p, 0);
      e = cudaGetLastError();
      if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_dh_kernel (sparse)", e);
    }
  }
  for (int c = 0; c < p.nchunks; ++c) {
    // FP8 rows are half as wide (8-B loads): 16 warps x 8 rows in flight.
    constexpr int T = FP8 ? DH_FP8_THREADS : DH_PERSIST_THREADS;
    constexpr int U = FP8 ? DH_FP8_UNROLL : 4;
    if (full)
      sparton_bwd_dh_kernel<CPL, U, 1, true, OutT, T, FP8><<<grid, T, 0, stream>>>(p, c);
    else
      sparton_bwd_dh_kernel<CPL, U, 1, false, OutT, T, FP8><<<grid, T, 0, stream>>>(p, c);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_dh_kernel", e);
  }
  return SPARTON_OK;
}

template <int CPL, typename OutT>
int launch_de_sparse(const BwdParams& p, cudaStream_t stream) {
  // One 512-thread CTA per SM, warps striding over vocab rows; the kernel
  // exits at once unless the route counted a sparse batch.
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return set_cuda_error("cudaDeviceGetAttribute(de_sparse)", e);
  const dim3 grid(sms, (p.D + 256 * CPL - 1) / (256 * CPL));
  if (p.D % (256 * CPL) == 0)
    sparton_bwd_de_sparse_kernel<CPL, true, OutT><<<grid, DES_THREADS, 0, stream>>>(p);
  else
    sparton_bwd_de_sparse_kernel<CPL, false, OutT><<<grid, DES_THREADS, 0, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_de_sparse_kernel", e);
  return SPARTON_OK;
}

constexpr int DEST_SMEM_BUDGET = 227 * 1024;

template <int NW, int J, bool FP8 = false>
int de_stage_bytes_t(int CL, int R) {
  using C = DeStCfg<NW, J, FP8>;
  return (128 + CL * R * C::RB + C::GI_BYTES + 127) & ~127;
}
constexpr int DEST_NW = 15, DEST_J = 12;   // 720 vocab rows x 64 columns per CTA (128 regs)
int de_stage_bytes(int CL, int R) { return de_stage_bytes_t<DEST_NW, DEST_J>(CL, R); }

template <int NW, int J, int CL, typename OutT, bool FP8 = false>
int launch_de_staged_t(const BwdParams& p, const CUtensorMap* tmH, cudaStream_t stream) {
  using C = DeStCfg<NW, J, FP8>;
  const int R = de_staged_rows(p.S);
  const int stage_bytes = de_stage_bytes_t<NW, J, FP8>(CL, R);
  int nst = (DEST_SMEM_BUDGET - 128) / stage_bytes;
  if (nst > 4) nst = 4;
  const int smem = nst * stage_bytes + nst * 16;
  auto kern = sparton_bwd_de_staged_kernel<NW, J, CL, OutT, FP8>;
  // Constant limit (the budget), not this call's S-dependent size: see launch_route.
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DEST_SMEM_BUDGET);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(de_staged)", e);
  const int nvb = (p.V + C::VB - 1) / C::VB;
  const int nvg = (nvb + CL - 1) / CL;
  const int nitems = nvg * ((p.D + C::DD - 1) / C::DD);
  int ncl = nitems;
  if (const char* ev = dev_env("SPARTON_DE_CLUSTERS")) {   // persistent grid (SM partition experiments)
    const int n = atoi(ev);
    if (n > 0 && n < ncl) ncl = n;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * CL), 1, 1);
  cfg.blockDim = dim3(C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, *tmH, p, R, nst, stage_bytes, nvg, nitems);
  if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_de_staged_kernel", e);
  sparton_bwd_db_kernel<<<(p.V + 255) / 256, 256, 0, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("launch sparton_bwd_db_kernel", e);
  return SPARTON_OK;
}

// Register budget split between accumulators (reuse: VB vocab rows per staged
// H tile) and loads in flight (latency hiding): 15 consumer warps x 12 rows at
// 128 registers measured 7% faster than 11 x 17 at 168.
template <typename OutT, bool FP8 = false>
int launch_de_staged(const BwdParams& p, const CUtensorMap* tmH, cudaStream_t stream) {
  constexpr int J = DEST_J;
  if (de_cluster(p.S) == 1) return launch_de_staged_t<DEST_NW, J, 1, OutT, FP8>(p, tmH, stream);
  if (de_cluster(p.S) == 2) return launch_de_staged_t<DEST_NW, J, 2, OutT, FP8>(p, tmH, stream);
  return launch_de_staged_t<DEST_NW, J, 4, OutT, FP8>(p, tmH, stream);
}

template <int CPL, int W, typename OutT>
int launch_de_any(const BwdParams& p, cudaStream_t stream) {
  return (p.D % (256 * CPL) == 0) ? launch_de<CPL, W, true, OutT>(p, stream)
                                  : launch_de<CPL, W, false, OutT>(p, stream);
}

template <int CPL, typename OutT>
int launch_bwd_t(const BwdParams& p, const CUtensorMap* tmH, cudaStream_t stream) {
  int mode = 1;
  if (const char* ev = dev_env("SPARTON_BWD_CONCURRENT")) mode = atoi(ev);
  SideStream ss;
  int rc = side_stream(ss);
  if (rc != SPARTON_OK) return rc;
  cudaError_t e;
  auto fork = [&]() -> int {
    e = cudaEventRecord(ss.fork, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ss.s, ss.fork, 0);
    return e == cudaSuccess ? SPARTON_OK : set_cuda_error("fork side stream", e);
  };
  // dH is complete on `stream` when launch_dh returns: a caller's event lets
  // it start consuming dH (e.g. the sharded head's all-reduce) while dE runs.
  auto dh_done = [&]() -> int {
    if (p.dh_ready == nullptr) return SPARTON_OK;
    e = cudaEventRecord(p.dh_ready, stream);
    return e == cudaSuccess ? SPARTON_OK : set_cuda_error("record dh_ready", e);
  };
  auto join = [&]() -> int {
    if ((e = cudaEventRecord(ss.join, ss.s)) != cudaSuccess) return set_cuda_error("record join", e);
    if ((e = cudaStreamWaitEvent(stream, ss.join, 0)) != cudaSuccess) return set_cuda_error("join side stream", e);
    return SPARTON_OK;
  };
  if (p.fp8) {
    // FP8 operands (staged dE only; the ABI checks S): route, then dE || dH.
    if (p.gi == nullptr) return set_error(SPARTON_EINVAL, "the FP8 backward needs the staged dE (S <= 832)");
    if ((rc = launch_route(p, stream)) != SPARTON_OK) return rc;
    if ((rc = fork()) != SPARTON_OK) return rc;
    if ((rc = launch_de_staged<OutT, true>(p, tmH, ss.s)) != SPARTON_OK) return rc;
    if ((rc = launch_dh<CPL, OutT, true>(p, stream)) != SPARTON_OK) return rc;
    if ((rc = dh_done()) != SPARTON_OK) return rc;
    return join();
  }
  if (p.gi != nullptr) {
    // Staged dE needs the route's (s, g) records: route, then dE || dH.  The
    // route also counts the active pairs; the staged dE + db and the sparse
    // dE are both launched and exactly one of them runs (device-side choice).
    if (p.stats != nullptr) {
      e = cudaMemsetAsync(p.stats, 0, sizeof(unsigned long long), stream);
      if (e != cudaSuccess) return set_cuda_error("zero the active-pair count", e);
    }
    if ((rc = launch_route(p, stream)) != SPARTON_OK) return rc;
    auto de = [&](cudaStream_t s) -> int {
      int r = launch_de_staged<OutT>(p, tmH, s);
      if (r == SPARTON_OK && p.stats != nullptr) r = launch_de_sparse<CPL, OutT>(p, s);
      return r;
    };
    if (mode == 0) {
      if ((rc = de(stream)) != SPARTON_OK) return rc;
      if ((rc = launch_dh<CPL, OutT>(p, stream)) != SPARTON_OK) return rc;
      return dh_done();
    }
    // Timing experiments only (tools/bwd_parts.py): one gradient family, the
    // others left unwritten (mode is only ever != 1 in a SPARTON_DEV=1 process).
    if (mode == 3 || mode == 4)
      return mode == 3 ? de(stream) : launch_dh<CPL, OutT>(p, stream);
    if ((rc = fork()) != SPARTON_OK) return rc;
    if ((rc = de(ss.s)) != SPARTON_OK) return rc;
    if ((rc = launch_dh<CPL, OutT>(p, stream)) != SPARTON_OK) return rc;
    if ((rc = dh_done()) != SPARTON_OK) return rc;
    return join();
  }
  if (mode == 0) {
    if ((rc = launch_de_any<CPL, 16, OutT>(p, stream)) != SPARTON_OK) return rc;
    if ((rc = launch_route(p, stream)) != SPARTON_OK) return rc;
    if ((rc = launch_dh<CPL, OutT>(p, stream)) != SPARTON_OK) return rc;
    return dh_done();
  }
  if ((rc = fork()) != SPARTON_OK) return rc;
  rc = (mode == 2) ? launch_de_any<CPL, 16, OutT>(p, ss.s) : launch_de_any<CPL, 8, OutT>(p, ss.s);
  if (rc != SPARTON_OK) return rc;
  if ((rc = launch_route(p, stream)) != SPARTON_OK) return rc;
  if ((rc = launch_dh<CPL, OutT>(p, stream)) != SPARTON_OK) return rc;
  if ((rc = dh_done()) != SPARTON_OK) return rc;
  return join();
}

template <typename OutT>
int launch_bwd_dtype(const BwdParams& p, const CUtensorMap* tmH, cudaStream_t stream) {
  if (p.D <= 256) return launch_bwd_t<1, OutT>(p, tmH, stream);
  if (p.D <= 512 || p.D > 768) return launch_bwd_t<2, OutT>(p, tmH, stream);
  return launch_bwd_t<3, OutT>(p, tmH, stream);
}

}  // namespace

// Rows of H each CTA of a staged-dE cluster loads per batch row (a multiple of
// 8, <= 256 for one TMA box), or 0 when two pipeline stages do not fit.
int de_staged_rows(int S) {
  const int CL = de_cluster(S);
  int R = (S + CL - 1) / CL;
  R = (R + 7) & ~7;
  if (R > 256) R = (R + 255) / 256 * 256;   // whole 256-row boxes
  if (R > 1024) return 0;
  if (2 * de_stage_bytes(CL, R) + 128 > DEST_SMEM_BUDGET) return 0;
  return R;
}

// Largest S the in-smem route supports (one segment of S counters + the window).
int bwd_max_seq() { return (RT_SMEM_BUDGET - RT_WIN * 8 - 128) / 4; }

// E chunk per dH pass: ~52 MB of bf16 rows (4 route windows at D = 768) so it
// stays L2-resident (126 MB L2) next to the streaming pair lists and carries.
// Per backward at cfg3: 8 x 52 MB passes 3.4 % faster than 11 x 38 MB, 7 x 63 MB
// 2 % and 6 x 75 MB 3.5 % (tools/ab_env.sh, locked clocks).
constexpr long long DH_CHUNK_BYTES = 52ll << 20;
constexpr long long DE_CHUNK_BYTES = 48ll << 20;

BwdWorkspace bwd_workspace_layout(long long B, long long S, long long D, long long V, int grad_dtype) {
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  BwdWorkspace w{};
  w.nwin = (int)((V + RT_WIN - 1) / RT_WIN);
  long long chunk_bytes = DH_CHUNK_BYTES;
  if (const char* ev = dev_env("SPARTON_DH_CHUNK_MB")) chunk_bytes = atoll(ev) << 20;   // experiment switch
  long long wpc = chunk_bytes / ((long long)RT_WIN * D * 2);
  if (wpc < 1) wpc = 1;
  if (wpc > w.nwin) wpc = w.nwin;
  if (wpc > 32) wpc = 32;                    // dH reads one pass's window bounds with one warp
  w.wpc = (int)wpc;
  w.nchunks = (w.nwin + w.wpc - 1) / w.wpc;
  w.pairs = 0;
  w.offsets = up((size_t)B * (size_t)V * sizeof(int2));
  // dE passes over batch chunks of ~48 MB of H (L2-resident while every
  // vocab block of the pass gathers from it).
  long long bc = DE_CHUNK_BYTES / (S * D * 2 > 0 ? S * D * 2 : 1);
  if (bc < DE_BC) bc = DE_BC;
  if (bc > B) bc = B;
  w.bchunk = (int)bc;
  const int de_passes = (int)((B + bc - 1) / bc);
  w.db_acc = w.offsets + up((size_t)B * (size_t)w.nwin * (size_t)(S + 1) * sizeof(int));
  w.dE_acc = w.db_acc + up((size_t)V * sizeof(float));
  // Staged dE (S small enough for two smem stages): (s, g) records instead of
  // the gathered dE's fp32 carry.
  w.de_staged = de_staged_rows((int)S) > 0;
  if (const char* ev = dev_env("SPARTON_DE_STAGED")) w.de_staged = w.de_staged && ev[0] != '0';
  w.ldGI = V + (V & 1);
  const bool need_de_acc = !w.de_staged && grad_dtype == SPARTON_BF16 && de_passes > 1;
  w.acc32 = w.dE_acc + (need_de_acc ? up((size_t)V * (size_t)D * sizeof(float)) : 0);
  const bool need_acc = grad_dtype == SPARTON_BF16 && w.nchunks > 1;
  w.gi = w.acc32 + (need_acc ? up((size_t)B * (size_t)S * (size_t)D * sizeof(float)) : 0);
  w.stats = w.gi + (w.de_staged ? up((size_t)B * (size_t)w.ldGI * sizeof(int2)) : 0);
  w.total = w.stats + 256;                   // active-pair count (sparse regime)
  if (!need_acc) w.acc32 = (size_t)-1;
  if (!need_de_acc) w.dE_acc = (size_t)-1;
  return w;
}

int launch_bwd(const BwdParams& p, const CUtensorMap* tmH, int grad_dtype, cudaStream_t stream) {
  if (grad_dtype == SPARTON_BF16) return launch_bwd_dtype<__nv_bfloat16>(p, tmH, stream);
  return launch_bwd_dtype<float>(p, tmH, stream);
}

}  // namespace sparton
