// sparton_fwd.cu — K1: the fused Sparton LM-head forward on sm_100a.
//
// Replaces the reference's forward_fully_fused / forward_hybrid
// (/root/reference/pkg/src/fusedhead/fused.py:160-212 and :115-157) and the
// GEMM stage matmul_bt (tensor.py:130-188).  One persistent, warp-specialised
// kernel per call:
//
//   warp 4        TMA producer: E tile (vocab rows, K-major) and H tile
//                 (sequence rows of one batch row, K-major) -> smem ring.
//   warp 5        TMEM allocator; on the leader CTA, the single-thread
//                 tcgen05.mma issuer (bf16 x bf16 -> f32 in TMEM).
//   warps 0..3    epilogue: tcgen05.ld the accumulator, add bias, apply the
//                 mask (masked -> exactly 0, out-of-range s -> skipped), and
//                 keep a running (max, first argmax) per vocab row in
//                 registers across sequence chunks; log1p(relu(.)) is applied
//                 once per (b, v) after the reduction (fused.py:203).
//
// Work unit = (batch row b, vocab tile of 128*CG rows); the unit loops over
// sequence chunks of 256 positions.  UMMA shape M = 128*CG (vocab on TMEM
// lanes, one lane per vocab row), N = 256 (sequence positions), K = 16.
// Each epilogue thread owns one vocab row and scans its columns in s order,
// so the strict '>' update reproduces the reference's smallest-index tie
// rule (fused.py:200) without cross-lane reductions.
// TMEM holds two 256-column accumulators so the epilogue of chunk i overlaps
// the MMAs of chunk i+1.  CG=2 runs a CTA pair (cta_group::2): each CTA loads
// half of the E tile and half of the H tile, the leader issues M=256 MMAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <algorithm>

#include "ptx.cuh"
#include "sparton_internal.h"

namespace sparton {

// OP: operand format — 0 bf16, 1 e4m3 with per-tensor scales (kind::f8f6f4),
// 2 MXFP8: e4m3 with a ue8m0 scale per 32 K elements of every row, applied
// inside the MMA (kind::mxf8f6f4.block_scale, scale factors in TMEM).
template <int CG, int NP = 1, int OP = 0>
struct FwdCfg {
  static constexpr bool FP8 = OP != 0;           // e4m3 operands
  static constexpr bool MX = OP == 2;            // block-scaled (MXFP8)
  static constexpr int EB = FP8 ? 1 : 2;         // operand element bytes (e4m3 / bf16)
  static constexpr int BM = 128;                 // vocab rows per CTA (TMEM lanes)
  static constexpr int TILE_V = BM * CG * NP;    // vocab rows per unit (NP pairs share H tiles)
  // Sequence positions per chunk (UMMA N).  MX: 240, so columns 240..255 of
  // the first accumulator hold the stage's scale factors (TMEM is otherwise
  // fully taken by the two 256-column accumulators).
  static constexpr int SN = MX ? 240 : 256;
  static constexpr int BN_CTA = SN / CG;         // H rows each CTA holds per chunk
  static constexpr int BN_LOAD = BN_CTA / NP;    // H rows each CTA loads (and multicasts to NP CTAs)
  static constexpr int BK = 128 / EB;            // K per stage = one 128-B swizzle row
  static constexpr int KSTEPS = 4;               // UMMA K = 16 (bf16) / 32 (e4m3): 32 B per step
  static constexpr int A_BYTES = BM * BK * EB;
  static constexpr int B_BYTES = BN_CTA * BK * EB;
  // MX scale factors per stage (4 K blocks of 32): this CTA's 128 E rows
  // (512 B) and the chunk's 256 H-row slots (1 KB), in the tcgen05.cp layout.
  static constexpr int SF_BYTES = MX ? 3 * 512 : 0;
  static constexpr int STAGE_TX = A_BYTES + B_BYTES + SF_BYTES;   // bytes landing per stage
  static constexpr int STAGE_BYTES = (STAGE_TX + 1023) / 1024 * 1024;
  static constexpr int SF_COL = 240;             // MX: TMEM column of SFA (4 cols), SFB follows (8 cols)
  static constexpr int NST = CG == 1 ? 4 : 6;   // 7 stages measured 0.8% slower (tools/ab_fwd.sh)
  static constexpr int UMMA_M = BM * CG;
  static constexpr int NUM_THREADS = 192;
  static constexpr int TMEM_COLS = 512;          // 2 accumulators x 256 columns
  static constexpr int SMEM_BYTES = NST * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

// Per-cluster unit sequence (all warp roles walk the same one).
//
// Large B (B >= 2 * clusters): vocab tiles are grouped (~48 MB of E per
// group); inside a group, cluster c owns the batch rows b = c' + j*nclusters
// (c' = a per-group rotation of c) and, for each of them, walks every vocab
// tile of the group.  H[b] is therefore pulled into L2 once and reused for the
// whole group by one cluster, while the group's E tiles are shared by all
// clusters; clusters never need to stay in lock-step (no drift-induced
// thrashing), and H streams from HBM once per group.
// Default / small B: round-robin over units ordered (vocab group, b, tile).
struct UnitIter {
  int g = 0, j = 0, k = 0;
  unsigned u = 0;
  int c, nc;
  __device__ UnitIter(int cluster, int nclusters) : c(cluster), nc(nclusters) { u = (unsigned)cluster; }
  __device__ __forceinline__ bool next(const FwdParams& p, int& b, int& vt) {
    if (!p.sched_bgroups) {
      // Round-robin over units ordered (vocab group, b, tile): consecutive
      // clusters share H[b] and the group's E tiles stay L2-resident.
      // (num_units < 2^31 is checked on the host: 32-bit index math.)
      if (u >= (unsigned)p.num_units) return false;
      const unsigned per_group = (unsigned)p.group_vt * (unsigned)p.urows;
      const unsigned gg = u / per_group;
      const unsigned r = u - gg * per_group;
      const int gv0 = (int)gg * p.group_vt;
      const unsigned gsz = (unsigned)min(p.group_vt, p.num_vt - gv0);
      const unsigned bb = r / gsz;
      b = (int)bb;
      vt = gv0 + (int)(r - bb * gsz);
      u += (unsigned)nc;
      return true;
    }
    while (true) {
      const int g0 = g * p.group_vt;
      if (g0 >= p.num_vt) return false;
      const int gsz = min(p.group_vt, p.num_vt - g0);
      const int bb = j * nc + (int)(((long long)c + (long long)g * p.rot) % nc);
      if (bb < p.urows) {
        b = bb;
        vt = g0 + k;
        if (++k == gsz) { k = 0; ++j; }
        return true;
      }
      ++g;
      j = 0;
      k = 0;
    }
  }
};

// Reduce 32 accumulator columns (tile columns c0..c0+31 of the current chunk)
// into four interleaved running (max, argmax) pairs; column c goes to slot c&3.
// The comparison runs on the raw dot products x = H.E: the bias is constant
// along s, and fl(. + bias) is monotone, so max_s fl(x_s + bias) =
// fl(max_s x_s + bias) exactly — Y is unchanged and the argmax can only
// differ at positions whose logits tie after rounding (a documented near-tie,
// SURVEY.md §8c).  A masked position has logit exactly 0, i.e. raw value
// -bias (fl(-bias + bias) = +0).
// `keep` bit l: position valid and unmasked (raw x);
// `zero` bit l: position valid but masked (raw -bias, logit 0, still competes);
// neither: position beyond S (skipped).
__device__ __forceinline__ void reduce_group(const float (&r)[32], float nbias, uint32_t keep,
                                             uint32_t zero, int c0, float (&best)[4],
                                             int (&bidx)[4]) {
  if (keep == 0xffffffffu) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (r[c] > best[c & 3]) { best[c & 3] = r[c]; bidx[c & 3] = c0 + c; }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const float x = ((keep >> c) & 1u) ? r[c] : (((zero >> c) & 1u) ? nbias : -INFINITY);
      if (x > best[c & 3]) { best[c & 3] = x; bidx[c & 3] = c0 + c; }
    }
  }
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Unmasked 32-column group, fewer instructions per logit than reduce_group:
// the group maximum m comes from a three-input max tree (block maxima of 8
// columns first); only when some lane of the warp improves its running best
// (m > best) does the warp locate the first column equal to m — first the
// block (reverse select over the 4 block maxima), then the column inside the
// block (the block's 8 values gathered by two select levels, reverse select).
// Same result as the strict '>' scan: first occurrence of the maximum.
__device__ __forceinline__ void reduce_group_fast(const float (&r)[32], int c0, float& best, int& bidx) {
  float bm[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float* x = r + 8 * k;
    bm[k] = max3f(max3f(x[0], x[1], x[2]), max3f(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
  }
  const float m = max3f(bm[0], bm[1], fmaxf(bm[2], bm[3]));
  const bool better = m > best;
  if (__any_sync(0xffffffffu, better)) {
    int kb = 3;
    kb = (bm[2] == m) ? 2 : kb;
    kb = (bm[1] == m) ? 1 : kb;
    kb = (bm[0] == m) ? 0 : kb;
    const bool lo = (kb & 1) != 0, hi = (kb & 2) != 0;
    int kk = 7;
#pragma unroll
    for (int k = 6; k >= 0; --k) {
      const float t0 = lo ? r[8 + k] : r[k];
      const float t1 = lo ? r[24 + k] : r[16 + k];
      kk = ((hi ? t1 : t0) == m) ? k : kk;
    }
    if (better) {
      best = m;
      bidx = c0 + 8 * kb + kk;
    }
  }
}

// One (b, v) result: the caller's output plus any extra destinations (the
// peers' [B, V] copies of a vocab-sharded head, written over NVLink — the
// all-gather fused into the epilogue), or one multimem store to a multicast
// address that the NVSwitch replicates to every rank's copy.  Consecutive lanes hold consecutive v,
// so every destination sees the same coalesced 128-B row segments.
__device__ __forceinline__ void store_yi(const FwdParams& p, size_t o, float y, int i) {
  if (p.mc) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(p.Y + o), "f"(y) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.s32 [%0], %1;" :: "l"(p.I + o), "r"(i) : "memory");
    return;
  }
  p.Y[o] = y;
  p.I[o] = i;
  for (int k = 0; k < p.nx; ++k) {
    p.Yx[k][o] = y;
    p.Ix[k][o] = i;
  }
}

template <int CG, int NP, int OP>
__global__ void __launch_bounds__(FwdCfg<CG, NP, OP>::NUM_THREADS, 1)
sparton_fwd_kernel(const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmH,
                   const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                   const FwdParams p) {
  using C = FwdCfg<CG, NP, OP>;
  constexpr bool FP8 = C::FP8;
  static_assert(!C::MX || (CG == 2 && NP == 1), "MXFP8 runs on the CTA-pair kernel");
  static_assert(NP == 1 || CG == 2, "H multicast across pairs needs CTA pairs");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::NST * C::STAGE_BYTES);
  uint64_t* full = bars;                   // [NST]
  uint64_t* empty = bars + C::NST;         // [NST]
  uint64_t* tfull = bars + 2 * C::NST;     // [2]
  uint64_t* tempty = bars + 2 * C::NST + 2;// [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::NST + 4);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t crank = (CG == 2) ? ptx::cluster_ctarank() : 0;   // rank in the cluster
  const uint32_t rank = crank & (CG - 1);                            // rank in the CTA pair
  const uint32_t pair = crank / CG;                                  // pair index in the cluster
  const uint16_t pair_mask = (uint16_t)(((1u << CG) - 1u) << (pair * CG));
  constexpr uint16_t all_mask = (uint16_t)((1u << (CG * NP)) - 1u);
  const long long cluster = (CG == 2) ? (long long)ptx::cluster_id_x() : (long long)blockIdx.x;
  const long long nclusters = (CG == 2) ? (long long)ptx::nclusters_x() : (long long)gridDim.x;

  // Warp roles.  The SM's four schedulers serve warps wid % 4 and favour the
  // highest wid, so the TMA producer (warp 4) and the MMA issuer (warp 5) sit
  // above the epilogue warps 0/1 that share their schedulers: epilogue
  // instruction bursts never delay an MMA issue or a TMA refill.
  constexpr int kProducer = 4, kMma = 5;
  if (warp == kProducer && lane == 0) {
    ptx::prefetch_tmap(&tmE);
    ptx::prefetch_tmap(&tmH);
    if constexpr (C::MX) {
      ptx::prefetch_tmap(&tmSFA);
      ptx::prefetch_tmap(&tmSFB);
    }
    for (int i = 0; i < C::NST; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), NP);   // one MMA commit per pair (multicast H)
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[i]), 4 * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kMma) ptx::tmem_alloc<CG>(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nsc = (p.S + C::SN - 1) / C::SN;
  const int nkb = (p.D + C::BK - 1) / C::BK;

  if (warp == kProducer) {
    // ------------------------------------------------ TMA producer
    // The whole warp walks the schedule (warp-uniform state); one elected
    // lane issues each stage's barrier arm and TMA loads.
    // L2 policies: 0 evict_normal, 1 evict_last, 2 evict_first (experiment switch)
    auto pol = [](int k) {
      return k == 1 ? ptx::policy_evict_last() : (k == 2 ? ptx::policy_evict_first() : ptx::policy_evict_normal());
    };
    const uint64_t pol_e = pol(p.e_evict_last & 3);
    const uint64_t pol_h = pol((p.e_evict_last >> 2) & 3);
    int st = 0;
    uint32_t ph = 0;
    UnitIter it((int)cluster, (int)nclusters);
    int b, vt;
    while (it.next(p, b, vt)) {
      const int vrow = vt * C::TILE_V + (int)pair * (C::BM * CG) + (int)rank * C::BM;
      for (int sc = 0; sc < nsc; ++sc) {
        // Packed short sequences: unit row b is the batch-row group b*pack .. b*pack+pack-1,
        // whose pack*S = 256 positions are contiguous rows of H.
        // The last chunk of a unit may be narrower (p.n_last columns): the CTA
        // pair then splits those columns evenly, so CTA 1's rows start at n_last/2.
        const int half = (NP == 1 && sc == nsc - 1) ? (p.n_last >> 1) : C::BN_CTA;
        const int hrow = b * p.pack * p.S + sc * C::SN + (int)rank * half + (int)pair * C::BN_LOAD;
        for (int kb = 0; kb < nkb; ++kb) {
          ptx::mbar_wait(ptx::smem_u32(&empty[st]), ph ^ 1);
          if (ptx::elect_one()) {
            const uint32_t sa = ptx::smem_u32(stage_base + st * C::STAGE_BYTES);
            const uint32_t sb = sa + C::A_BYTES;
            const uint32_t fb = ptx::smem_u32(&full[st]);
            if constexpr (CG == 1) {
              ptx::mbar_arrive_expect_tx(fb, C::STAGE_TX);
              ptx::tma_load_2d(&tmE, sa, fb, kb * C::BK, vrow, pol_e);
              ptx::tma_load_2d(&tmH, sb, fb, kb * C::BK, hrow, pol_h);
            } else {
              if (rank == 0) ptx::mbar_arrive_expect_tx(fb, C::STAGE_TX * 2);
              ptx::tma_load_2d_cg2(&tmE, sa, fb, kb * C::BK, vrow, pol_e);
              if constexpr (C::MX) {
                // Scale factors (uint32 rows of 128 = one 512-B chunk): this
                // CTA's E rows (vrow / 128, K group kb) and the chunk's H slot
                // pair ((unit row, chunk), K group kb) — see sparton_quant_mx.
                const uint32_t ssf = sb + C::B_BYTES;
                ptx::tma_load_2d_cg2(&tmSFA, ssf, fb, 0, (vrow >> 7) * nkb + kb, pol_e);
                ptx::tma_load_2d_cg2(&tmSFB, ssf + 512, fb, 0, ((b * nsc + sc) * nkb + kb) * 2, pol_h);
              }
              if constexpr (NP == 1) {
                ptx::tma_load_2d_cg2(&tmH, sb, fb, kb * C::BK, hrow, pol_h);
              } else {
                // Same H rows are needed by CTA `rank` of every pair: each loads
                // 1/NP of them and multicasts to its counterparts.
                const uint16_t mc = (uint16_t)(0x5555u << rank) & all_mask;   // cluster ranks rank, rank+2, ...
                ptx::tma_load_2d_cg2_mc(&tmH, sb + pair * (C::BN_LOAD * C::BK * C::EB), fb, kb * C::BK, hrow, mc,
                                        pol_h);
              }
            }
          }
          __syncwarp();
          if (++st == C::NST) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == kMma) {
    if (rank == 0) {
      // ------------------------------------------------ MMA issuer
      // Warp-uniform loop; one elected lane issues the MMAs and commits.
      auto make_idesc = [](int n) {
        return C::MX ? ptx::umma_idesc_mx(C::UMMA_M, n)
                     : (FP8 ? ptx::umma_idesc_e4m3(C::UMMA_M, n) : ptx::umma_idesc_bf16(C::UMMA_M, n));
      };
      const uint32_t idesc_full = make_idesc(C::SN);
      // Narrow last chunk (S not a multiple of SN): only its columns are computed.
      const uint32_t idesc_last = NP == 1 ? make_idesc(p.n_last) : idesc_full;
      const uint32_t tsfa = tmem_base + C::SF_COL, tsfb = tmem_base + C::SF_COL + 4;
      int st = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      UnitIter it((int)cluster, (int)nclusters);
      int b, vt;
      while (it.next(p, b, vt)) {
        for (int sc = 0; sc < nsc; ++sc) {
          ptx::mbar_wait(ptx::smem_u32(&tempty[acc]), aph ^ 1);
          ptx::tc_fence_after();
          const uint32_t dt = tmem_base + (uint32_t)(acc * 256);
          const uint32_t idesc = (sc == nsc - 1) ? idesc_last : idesc_full;
          for (int kb = 0; kb < nkb; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&full[st]), ph);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
              const uint32_t sa = ptx::smem_u32(stage_base + st * C::STAGE_BYTES);
              const uint64_t da = ptx::umma_desc_sw128(sa);
              const uint64_t db = ptx::umma_desc_sw128(sa + C::A_BYTES);
              if constexpr (C::MX) {
                // Stage scale factors -> TMEM (one slot: tcgen05.cp and
                // tcgen05.mma of this thread execute in issue order, so the
                // copy lands after the previous stage's MMAs have read it).
                const uint32_t ssf = sa + C::A_BYTES + C::B_BYTES;
                ptx::utccp_32x128b_x4<CG>(tsfa, ptx::smem_desc_rows16(ssf));
                ptx::utccp_32x128b_x4<CG>(tsfb, ptx::smem_desc_rows16(ssf + 512));
                ptx::utccp_32x128b_x4<CG>(tsfb + 4, ptx::smem_desc_rows16(ssf + 1024));
              }
#pragma unroll
              for (int k = 0; k < C::KSTEPS; ++k) {
                // +32 bytes along K inside the 128-B swizzle row = +2 in the >>4 address field.
                if constexpr (C::MX)
                  ptx::umma_mx<CG>(dt, da + 2 * k, db + 2 * k, ptx::umma_idesc_mx_sf(idesc, k), tsfa, tsfb,
                                   (kb | k) != 0);
                else if constexpr (FP8) ptx::umma_e4m3<CG>(dt, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                else ptx::umma_bf16<CG>(dt, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
              }
              // The stage's H half was written by every pair's producer: release it cluster-wide.
              ptx::umma_commit<CG>(ptx::smem_u32(&empty[st]), all_mask);
            }
            __syncwarp();
            if (++st == C::NST) { st = 0; ph ^= 1; }
          }
          if (ptx::elect_one()) ptx::umma_commit<CG>(ptx::smem_u32(&tfull[acc]), pair_mask);
          __syncwarp();
          acc ^= 1;
          if (acc == 0) aph ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 0..3)
    // Dequantisation scale of the raw accumulator (FP8: amax_H/448 * amax_E/448).
    float dscale = 1.0f;
    if constexpr (OP == 1) {
      const float ah = __ldg(p.amax_h), ae = __ldg(p.amax_e);
      dscale = (ah > 0.f ? ah / 448.0f : 1.0f) * (ae > 0.f ? ae / 448.0f : 1.0f);
    }
    const int q = warp & 3;                       // TMEM lane quarter this warp may access
    const int row = q * 32 + (int)lane;           // vocab row within this CTA's tile
    const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
    uint32_t tempty0 = ptx::smem_u32(&tempty[0]);
    uint32_t tempty1 = ptx::smem_u32(&tempty[1]);
    if constexpr (CG == 2) {
      tempty0 = ptx::mapa(tempty0, pair * CG);
      tempty1 = ptx::mapa(tempty1, pair * CG);
    }
    int acc = 0;
    uint32_t aph = 0;
    UnitIter it((int)cluster, (int)nclusters);
    int b, vt;
    while (it.next(p, b, vt)) {
      const int v = vt * C::TILE_V + (int)pair * (C::BM * CG) + (int)rank * C::BM + row;
      const float bv = (v < p.V) ? __ldg(p.bias + v) : 0.0f;
      // Raw-space comparisons: logit = dscale * raw + bias with dscale = 1 for
      // bf16 and the product of the two per-tensor e4m3 scales for FP8 (> 0, so
      // the argmax is that of the raw accumulator); a masked position (logit
      // exactly 0) competes as raw -bias / dscale.
      const float nbv = -bv / dscale;
      if (p.pack > 1) {
        // ---- packed chunk: pack = floor(256/S) batch rows of S positions
        // (16 <= S <= 128) occupy the first pack*S columns.
        ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), aph);
        ptx::tc_fence_after();
        const uint32_t tacc = tq + (uint32_t)(acc * 256);
        float cbest = -INFINITY;
        int cidx = 0;
        auto finish_row = [&](int seg) {
          const int bb = b * p.pack + seg;
          if (bb < p.B && v < p.V) {
            const size_t o = (size_t)bb * (size_t)p.ldY + (size_t)v;
            store_yi(p, o, log1pf(fmaxf(fmaf(cbest, dscale, bv), 0.0f)), cidx);
          }
          cbest = -INFINITY;
          cidx = 0;
        };
        auto reduce_masked = [&](float (&r)[32], uint32_t keep, uint32_t zero, int cbase) {
          if (keep == 0xffffffffu) {
            reduce_group_fast(r, cbase, cbest, cidx);
          } else if ((keep | zero) != 0u) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              r[c] = ((keep >> c) & 1u) ? r[c] : (((zero >> c) & 1u) ? nbv : -INFINITY);
            reduce_group_fast(r, cbase, cbest, cidx);
          }
        };
        if ((p.S & 31) == 0) {
          // Each 32-column group belongs to one batch row.
          const int gps = p.S >> 5;                 // groups per batch row
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int seg = j / gps, jj = j - seg * gps;
            if (seg < p.pack) {
              const int bb = b * p.pack + seg;
              const bool brow = bb < p.B;
              const uint32_t keep = __ballot_sync(
                  0xffffffffu, brow && __ldg(p.mask + (size_t)(brow ? bb : 0) * p.S + jj * 32 + lane) != 0);
              float r[32];
              ptx::tmem_ld32(tacc + (uint32_t)(j * 32), r);
              ptx::tmem_ld_wait();
              ptx::reg_fence32(r);
              reduce_masked(r, keep, brow ? ~keep : 0u, jj * 32);
              if (jj == gps - 1) finish_row(seg);
            }
          }
        } else {
          // A group may straddle batch rows (two for S >= 32, up to three for
          // S >= 16): reduce each part separately, finishing a row at its last column.
          const int used = p.pack * p.S;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c0 = j * 32;
            if (c0 < used) {
              const int last = min(c0 + 31, used - 1);
              const int seg_a = c0 / p.S, seg_b = last / p.S;
              const int pcol = c0 + (int)lane;
              const int lseg = pcol / p.S;
              const int lb = b * p.pack + lseg;
              const bool lvalid = pcol < used && lb < p.B;
              const bool lm = lvalid && __ldg(p.mask + (size_t)lb * p.S + (pcol - lseg * p.S)) != 0;
              for (int seg = seg_a; seg <= seg_b; ++seg) {
                const uint32_t keep = __ballot_sync(0xffffffffu, lm && lseg == seg);
                const uint32_t zero = __ballot_sync(0xffffffffu, lvalid && !lm && lseg == seg);
                float r[32];
                ptx::tmem_ld32(tacc + (uint32_t)c0, r);
                ptx::tmem_ld_wait();
                ptx::reg_fence32(r);
                reduce_masked(r, keep, zero, c0 - seg * p.S);
                if ((seg + 1) * p.S - 1 <= last) finish_row(seg);
              }
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          const uint32_t te = acc ? tempty1 : tempty0;
          if constexpr (CG == 2) ptx::mbar_arrive_cluster_relaxed(te);
          else ptx::mbar_arrive(te);
        }
        acc ^= 1;
        if (acc == 0) aph ^= 1;
        continue;
      }
      const uint8_t* mrow = p.mask + (size_t)b * p.S;
      float best = -INFINITY;
      int bidx = 0;
      for (int sc = 0; sc < nsc; ++sc) {
        const int s0 = sc * C::SN;
        // Mask words for the 8 column groups of this chunk (warp-uniform).
        uint32_t keep[8], zero[8];
        if (s0 + C::SN <= p.S) {
          // Full chunk: one base address, eight byte loads, eight ballots
          // (MX: group 7 holds 16 positions).
          const uint8_t* mp = mrow + s0 + lane;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool in = j * 32 + (int)lane < C::SN;
            keep[j] = __ballot_sync(0xffffffffu, in && __ldg(mp + (in ? j * 32 : 0)) != 0);
            zero[j] = __ballot_sync(0xffffffffu, in) & ~keep[j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int s = s0 + j * 32 + (int)lane;
            const bool valid = s < p.S && j * 32 + (int)lane < C::SN;
            const bool m = valid && (__ldg(mrow + (valid ? s : 0)) != 0);
            keep[j] = __ballot_sync(0xffffffffu, m);
            zero[j] = __ballot_sync(0xffffffffu, valid && !m);
          }
        }
        ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), aph);
        ptx::tc_fence_after();
        float cb[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int ci[4] = {0, 0, 0, 0};
        const uint32_t tacc = tq + (uint32_t)(acc * 256);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float r[32];
          ptx::tmem_ld32(tacc + (uint32_t)(j * 32), r);
          ptx::tmem_ld_wait();
          ptx::reg_fence32(r);
          if (p.epi_mode == 1) {
#pragma unroll
            for (int c = 0; c < 32; ++c) cb[c & 3] = fmaxf(cb[c & 3], r[c]);
          } else if (p.epi_mode == 2) {
#pragma unroll
            for (int c = 0; c < 32; ++c) cb[c & 3] = fmaxf(cb[c & 3] + 0.0f * (float)c, r[c]);
          } else if (p.epi_mode == 3) {
#pragma unroll
            for (int c = 0; c < 32; ++c) if (r[c] > cb[c & 3]) cb[c & 3] = r[c];
          } else if (p.epi_mode == 4) {   // experiment switch: the per-element strict '>' scan
            if ((keep[j] | zero[j]) != 0u) reduce_group(r, nbv, keep[j], zero[j], j * 32, cb, ci);
          } else if (keep[j] == 0xffffffffu) {
            reduce_group_fast(r, j * 32, cb[0], ci[0]);
          } else if ((keep[j] | zero[j]) != 0u) {
            // Masked / ragged group: substitute the competing raw values first
            // (masked -> -bias, i.e. logit 0; beyond S -> -inf), then reduce.
            const uint32_t kp = keep[j], zr = zero[j];
            const float nb = nbv;
#pragma unroll
            for (int c = 0; c < 32; ++c)
              r[c] = ((kp >> c) & 1u) ? r[c] : (((zr >> c) & 1u) ? nb : -INFINITY);
            reduce_group_fast(r, j * 32, cb[0], ci[0]);
          }
        }
        // Accumulator fully read: hand it back to the MMA warp.
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          const uint32_t te = acc ? tempty1 : tempty0;
          if constexpr (CG == 2) ptx::mbar_arrive_cluster_relaxed(te);
          else ptx::mbar_arrive(te);
        }
        acc ^= 1;
        if (acc == 0) aph ^= 1;
        // Merge the four interleaved slots: larger value wins, equal values keep the
        // smaller column (first occurrence), then fold into the running pair with a
        // strict '>' (earlier chunks hold smaller s).
        float m = cb[0];
        int mi = ci[0];
#pragma unroll
        for (int k = 1; k < 4; ++k) {
          if (cb[k] > m || (cb[k] == m && ci[k] < mi)) { m = cb[k]; mi = ci[k]; }
        }
        if (m > best) { best = m; bidx = s0 + mi; }
      }
      if (v < p.V) {
        const size_t o = (size_t)b * (size_t)p.ldY + (size_t)v;
        store_yi(p, o, log1pf(fmaxf(fmaf(best, dscale, bv), 0.0f)), bidx);
      }
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == kMma) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

template <int CG, int NP, int OP>
int launch_fwd_impl(const CUtensorMap& tmE, const CUtensorMap& tmH, const CUtensorMap& tmSFA,
                    const CUtensorMap& tmSFB, FwdParams prm, int num_sms, cudaStream_t stream) {
  using C = FwdCfg<CG, NP, OP>;
  constexpr int CL = CG * NP;   // cluster size
  auto kern = sparton_fwd_kernel<CG, NP, OP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(fwd)", e);
  long long want = prm.num_units;
  int grid = (num_sms / CL) * CL;        // persistent: one CTA per SM, whole clusters
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(C::NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CG == 2) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (CG == 2) {
    // Clusters must all be co-resident (static persistent schedule): a GPC
    // with an SM count not divisible by CL leaves SMs no cluster can use, and
    // any cluster beyond the resident limit would run as a serial second wave.
    static int max_clusters[3][8] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& mc = max_clusters[OP][dev & 7];
    if (mc == 0) {
      cfg.gridDim = dim3(grid, 1, 1);
      if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc < 1) {
        cudaGetLastError();
        mc = num_sms / CL;
      }
    }
    if (grid > mc * CL) grid = mc * CL;
  }
  if (want < grid / CL) grid = (int)want * CL;
  if (grid < CL) grid = CL;
  cfg.gridDim = dim3(grid, 1, 1);
  {
    // E group = one vocab tile per resident cluster: the round-robin over
    // (group, b, tile) then hands cluster c tile c of every batch row, so a
    // wave of units covers exactly one batch row (its H[b] read by every
    // cluster at once) and each cluster keeps its E tile for the whole group.
    // Measured against the former fixed 48 MB groups (128 tiles at D = 768):
    // -2.5 ms per cfg3 step (paired in-step A/B on two boxes, the forward's
    // lower energy buys clock) and less DRAM traffic
    // (profiles/r02_fwd_experiments.txt).  Capped at 48 MB of E for wide D;
    // a vocabulary whose whole E fits under the cap stays one group (H then
    // streams once: V = 30522 measured 0.9 % faster that way).
    const long long tile_bytes = (long long)C::TILE_V * prm.D * C::EB;
    const long long cap = 48ll << 20;
    int gv = grid / CL;
    if ((long long)prm.num_vt * tile_bytes <= cap) gv = prm.num_vt;
    if ((long long)gv * tile_bytes > cap) gv = (int)(cap / (tile_bytes > 0 ? tile_bytes : 1));
    if (const char* ev = dev_env("SPARTON_FWD_GROUP_KB")) gv = (int)((atoll(ev) << 10) / (tile_bytes > 0 ? tile_bytes : 1));
    if (gv < 1) gv = 1;
    if (gv > prm.num_vt) gv = prm.num_vt;
    prm.group_vt = gv;
  }
  e = cudaLaunchKernelEx(&cfg, kern, tmE, tmH, tmSFA, tmSFB, prm);
  if (e != cudaSuccess) return set_cuda_error("launch sparton_fwd_kernel", e);
  return SPARTON_OK;
}

static int gcd_int(int a, int b) { while (b) { const int t = a % b; a = b; b = t; } return a; }

int fwd_chunk_cols(int fp8_mode) { return fp8_mode == 2 ? FwdCfg<2, 1, 2>::SN : FwdCfg<2>::SN; }

int fwd_pack(int S, int fp8_mode) {
  const int sn = fwd_chunk_cols(fp8_mode);
  return (S >= 16 && S <= 128 && sn / S > 1) ? sn / S : 1;
}

int launch_fwd(const CUtensorMap& tmE, const CUtensorMap& tmH, const CUtensorMap* tmSFA, const CUtensorMap* tmSFB,
               FwdParams prm, int cluster_ctas, int num_sms, cudaStream_t stream) {
  const int tile_v = 128 * cluster_ctas;
  const int sn = fwd_chunk_cols(prm.fp8);
  prm.num_vt = (prm.V + tile_v - 1) / tile_v;
  // Short sequences (16 <= S <= 128): pack floor(SN/S) batch rows into one
  // chunk so the MMA computes (almost) no padding columns (SPLADE queries).
  prm.pack = fwd_pack(prm.S, prm.fp8);
  if (const char* ev = dev_env("SPARTON_FWD_PACK")) if (ev[0] == '0') prm.pack = 1;
  prm.urows = (prm.B + prm.pack - 1) / prm.pack;
  {
    // UMMA N of the last sequence chunk: the remaining positions rounded up to
    // 16 (cta_group::2 N granularity); packed chunks are always full.
    const int rem = prm.pack > 1 ? prm.pack * prm.S : prm.S - ((prm.S - 1) / sn) * sn;
    prm.n_last = cluster_ctas == 1 ? 256 : ((rem + 15) / 16) * 16;
    if (const char* ev = dev_env("SPARTON_FWD_NLAST")) if (ev[0] == '0') prm.n_last = 256;
  }
  prm.num_units = (long long)prm.num_vt * prm.urows;
  if (prm.num_units >= (1ll << 31) - 4096)
    return set_error(SPARTON_EINVAL, "B * ceil(V / vocab_tile) exceeds the forward scheduler's 31-bit unit index");
  const int nclusters = max(1, num_sms / cluster_ctas);
  // E group (vocab tiles walked for every batch row before the next group,
  // see UnitIter): set per launch in launch_fwd_impl, once the number of
  // resident clusters is known.
  prm.group_vt = 0;
  // Epilogue experiment switch (1-3: max-only variants with WRONG I, 4: the
  // per-element strict '>' scan) — honoured only in a SPARTON_DEV=1 process.
  prm.epi_mode = 0;
  if (const char* ev = dev_env("SPARTON_FWD_EPI")) prm.epi_mode = atoi(ev);
  prm.sched_bgroups = 0;   // measured: the grouped round-robin moves less DRAM (profiles/)
  if (const char* ev = dev_env("SPARTON_FWD_SCHED")) prm.sched_bgroups = ev[0] == '1';
  int rot = (int)(0.618 * nclusters + 0.5);
  if (rot < 1) rot = 1;
  while (gcd_int(rot, nclusters) != 1) ++rot;
  prm.rot = rot % nclusters;
  const CUtensorMap& sfa = tmSFA ? *tmSFA : tmE;   // unused unless MX
  const CUtensorMap& sfb = tmSFB ? *tmSFB : tmE;
  if (prm.fp8 == 2) {
    if (cluster_ctas != 2 || !tmSFA || !tmSFB) return set_error(SPARTON_EINVAL, "MXFP8 runs on CTA pairs (cta_group 2)");
    return launch_fwd_impl<2, 1, 2>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
  }
  if (prm.fp8) {
    if (cluster_ctas == 4) return launch_fwd_impl<2, 2, 1>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
    if (cluster_ctas == 2) return launch_fwd_impl<2, 1, 1>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
    return launch_fwd_impl<1, 1, 1>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
  }
  if (cluster_ctas == 4) return launch_fwd_impl<2, 2, 0>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
  if (cluster_ctas == 2) return launch_fwd_impl<2, 1, 0>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
  return launch_fwd_impl<1, 1, 0>(tmE, tmH, sfa, sfb, prm, num_sms, stream);
}

// ------------------------------------------------------------------ e4m3 quantisation
// Per-tensor scaling for the FP8 forward: amax = max |x| (non-negative floats
// order like their bit patterns, so an integer atomicMax is exact and
// deterministic), then q = e4m3(x * 448 / amax) with round-to-nearest and
// saturation.  The forward dequantises with amax_h/448 * amax_e/448.
__global__ void __launch_bounds__(256) sparton_amax_kernel(const int4* x, long long n16, unsigned* amax_bits) {
  float m = 0.f;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n16; i += (long long)gridDim.x * 256) {
    const int4 a = __ldg(&x[2 * i]), b = __ldg(&x[2 * i + 1]);
    const uint32_t w[8] = {(uint32_t)a.x, (uint32_t)a.y, (uint32_t)a.z, (uint32_t)a.w,
                           (uint32_t)b.x, (uint32_t)b.y, (uint32_t)b.z, (uint32_t)b.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m = fmaxf(m, fabsf(__uint_as_float(w[k] << 16)));
      m = fmaxf(m, fabsf(__uint_as_float(w[k] & 0xffff0000u)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = wm[0];
    for (int k = 1; k < 8; ++k) t = fmaxf(t, wm[k]);
    atomicMax(amax_bits, __float_as_uint(t));
  }
}

__device__ __forceinline__ uint16_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void __launch_bounds__(256) sparton_quant_kernel(const int4* x, long long n16, int4* q,
                                                            const float* amax) {
  const float a = *amax;
  const float inv = a > 0.f ? 448.0f / a : 1.0f;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n16; i += (long long)gridDim.x * 256) {
    const int4 u = __ldg(&x[2 * i]), v = __ldg(&x[2 * i + 1]);
    const uint32_t w[8] = {(uint32_t)u.x, (uint32_t)u.y, (uint32_t)u.z, (uint32_t)u.w,
                           (uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint16_t p0 = e4m3x2(__uint_as_float(w[2 * k] << 16) * inv, __uint_as_float(w[2 * k] & 0xffff0000u) * inv);
      const uint16_t p1 = e4m3x2(__uint_as_float(w[2 * k + 1] << 16) * inv,
                                 __uint_as_float(w[2 * k + 1] & 0xffff0000u) * inv);
      o[k] = (uint32_t)p0 | ((uint32_t)p1 << 16);
    }
    q[i] = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
  }
}

int launch_quantize_e4m3(const void* x, long long n, void* q, float* amax, cudaStream_t stream) {
  const long long n16 = n / 16;
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(float), stream);
  if (e != cudaSuccess) return set_cuda_error("cudaMemsetAsync(amax)", e);
  int blocks = (int)std::min<long long>((n16 + 255) / 256, 148ll * 8);
  if (blocks < 1) blocks = 1;
  sparton_amax_kernel<<<blocks, 256, 0, stream>>>(static_cast<const int4*>(x), n16, reinterpret_cast<unsigned*>(amax));
  sparton_quant_kernel<<<blocks, 256, 0, stream>>>(static_cast<const int4*>(x), n16, static_cast<int4*>(q), amax);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("launch e4m3 quantisation", e);
  return SPARTON_OK;
}

// ------------------------------------------------------------------ MXFP8 quantisation
// OCP MX block scaling with e4m3 elements: every 32 consecutive K elements of
// a row share one ue8m0 scale 2^e, the smallest power of two with
// max|x| / 2^e <= 448 (no saturation), and q = e4m3_rn(x / 2^e).  Scales
// are written in the layout tcgen05.cp expects for the forward's stages: a
// 512-B chunk per (128 rows, 4 K blocks) with row r, block k at
// (r % 32) * 16 + ((r % 128) / 32) * 4 + k.  Rows map to "slots" of
// slot_rows (128 for E's vocab tiles; 256 for H, one per (unit row, sequence
// chunk) of the forward's schedule): slot = (r / group_rows) * slots_per_group
// + (r % group_rows) / chunk_rows, row i = (r % group_rows) % chunk_rows.
// The scale buffer is zeroed first (unused rows / blocks -> scale 2^-127 x 0).
struct MxLayout {
  long long rows;
  int D, nkg, group_rows, chunk_rows, slots_per_group, slot_rows;
};

__global__ void __launch_bounds__(256) sparton_quant_mx_kernel(const uint16_t* __restrict__ x, uint8_t* __restrict__ q,
                                                               uint8_t* __restrict__ sf, const MxLayout L) {
  const int nblk = (L.D + 31) / 32;
  const long long total = L.rows * nblk;
  for (long long t = (long long)blockIdx.x * 256 + threadIdx.x; t < total; t += (long long)gridDim.x * 256) {
    const long long r = t / nblk;
    const int blk = (int)(t - r * nblk);
    const int d0 = blk * 32;
    const int n = min(32, L.D - d0);               // 32, or 16 for a D % 32 == 16 tail
    const int4* src = reinterpret_cast<const int4*>(x + r * L.D + d0);
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int4 v = make_int4(0, 0, 0, 0);
      if (k * 8 < n) v = __ldg(src + k);
      w[4 * k] = (uint32_t)v.x; w[4 * k + 1] = (uint32_t)v.y; w[4 * k + 2] = (uint32_t)v.z; w[4 * k + 3] = (uint32_t)v.w;
    }
    float amax = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[k] << 16)), fabsf(__uint_as_float(w[k] & 0xffff0000u))));
    int e = -127;
    if (amax > 0.f) {
      int ex;
      frexpf(amax, &ex);                            // amax in [2^(ex-1), 2^ex)
      e = ex - 9 + (ldexpf(amax, 9 - ex) > 448.0f ? 1 : 0);
      e = max(-127, min(127, e));
    }
    const float inv = ldexpf(1.0f, -e);
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint16_t p0 = e4m3x2(__uint_as_float(w[2 * k] << 16) * inv, __uint_as_float(w[2 * k] & 0xffff0000u) * inv);
      const uint16_t p1 = e4m3x2(__uint_as_float(w[2 * k + 1] << 16) * inv,
                                 __uint_as_float(w[2 * k + 1] & 0xffff0000u) * inv);
      o[k] = (uint32_t)p0 | ((uint32_t)p1 << 16);
    }
    int4* dst = reinterpret_cast<int4*>(q + r * L.D + d0);
    dst[0] = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
    if (n > 16) dst[1] = make_int4((int)o[4], (int)o[5], (int)o[6], (int)o[7]);
    const long long g = r / L.group_rows;
    const int within = (int)(r - g * L.group_rows);
    const long long slot = g * L.slots_per_group + within / L.chunk_rows;
    const int i = within % L.chunk_rows;
    const long long off = ((slot * L.nkg + blk / 4) * (L.slot_rows / 128) + i / 128) * 512 + (i % 32) * 16 +
                          ((i % 128) / 32) * 4 + (blk % 4);
    sf[off] = (uint8_t)(e + 127);
  }
}

static MxLayout mx_layout(bool h_operand, long long rows_or_B, long long S, int D) {
  MxLayout L{};
  L.D = D;
  L.nkg = (D + 127) / 128;
  if (h_operand) {
    const int sn = fwd_chunk_cols(2), pack = fwd_pack((int)S, 2);
    L.rows = rows_or_B * S;
    L.group_rows = (int)(pack * S);
    L.chunk_rows = sn;
    L.slots_per_group = pack > 1 ? 1 : (int)((S + sn - 1) / sn);
    L.slot_rows = 256;
  } else {
    L.rows = rows_or_B;
    L.group_rows = 128;
    L.chunk_rows = 128;
    L.slots_per_group = 1;
    L.slot_rows = 128;
  }
  return L;
}

long long mx_sf_bytes(bool h_operand, long long rows_or_B, long long S, int D) {
  const MxLayout L = mx_layout(h_operand, rows_or_B, S, D);
  const long long groups = (L.rows + L.group_rows - 1) / L.group_rows;
  return groups * L.slots_per_group * L.nkg * (L.slot_rows / 128) * 512;
}

int launch_quantize_mx(bool h_operand, const void* x, long long rows_or_B, long long S, int D, void* q, void* sf,
                       cudaStream_t stream) {
  const MxLayout L = mx_layout(h_operand, rows_or_B, S, D);
  cudaError_t e = cudaMemsetAsync(sf, 0, (size_t)mx_sf_bytes(h_operand, rows_or_B, S, D), stream);
  if (e != cudaSuccess) return set_cuda_error("cudaMemsetAsync(mx scales)", e);
  const long long work = L.rows * ((D + 31) / 32);
  int blocks = (int)std::min<long long>((work + 255) / 256, 148ll * 16);
  if (blocks < 1) blocks = 1;
  sparton_quant_mx_kernel<<<blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(x), static_cast<uint8_t*>(q),
                                                       static_cast<uint8_t*>(sf), L);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("launch mx quantisation", e);
  return SPARTON_OK;
}

// Rows of H each CTA loads per TMA box for a cluster of `cluster_ctas` CTAs.
int fwd_h_box_rows(int cluster_ctas, int fp8_mode) { return fwd_chunk_cols(fp8_mode) / cluster_ctas; }

int fwd_smem_bytes(int cluster_ctas) {
  return cluster_ctas >= 2 ? FwdCfg<2>::SMEM_BYTES : FwdCfg<1>::SMEM_BYTES;
}

}  // namespace sparton
