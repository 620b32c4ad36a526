/*
 * sparton.h — C ABI of the B200-native fused SPLADE LM head ("Sparton").
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/fusedhead/fused.py).  Every entry point takes plain
 * device pointers, explicit sizes / leading dimensions and a cudaStream_t
 * (passed as void*), so any host language can bind it (ctypes, cgo, JNI, ...).
 * No torch types cross this boundary.
 *
 * Semantics (identical to the reference):
 *   L[b,s,v] = (sum_k H[b,s,k] * E[v,k] + bias[v]) * mask[b,s]     (masked -> exactly 0)
 *   I[b,v]   = smallest s attaining max_s L[b,s,v]                  (int32)
 *   Y[b,v]   = log1p(max(L[b,I[b,v],v], 0))                         (float32)
 *   g[b,v]   = dY[b,v] * exp(-Y[b,v])  if Y[b,v] > 0 else 0
 *   dE[v,:]  = sum_b g[b,v] * H[b, I[b,v], :]     (b ascending, single owner)
 *   db[v]    = sum_b g[b,v]                       (b ascending, single owner)
 *   dH[b,s,:]= sum_{v : I[b,v]=s} g[b,v] * E[v,:] (v ascending, single owner)
 *
 * Layout: H is (B*S) x D row-major bf16 (ld = D), E is V x D row-major bf16,
 * bias f32[V], mask u8[B*S] in {0,1}, Y f32 / I i32 are B x ldY (ldY >= V).
 * H and E must be 16-byte aligned and D a multiple of 8 (TMA stride rule);
 * callers with other D zero-pad the K axis (zero columns add exactly 0).
 *
 * All calls are stream-ordered and asynchronous; outputs and workspace are
 * caller-owned (kernels never allocate).  Only shapes, dtypes and alignment
 * are validated — no device-side value scans — mirroring backward_fused's
 * deliberate "validate shapes only" contract (fused.py:232-245).
 */
#ifndef SPARTON_H_
#define SPARTON_H_

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define SPARTON_API __attribute__((visibility("default")))
#else
#define SPARTON_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python layer maps EINVAL -> ValueError (the reference's
 * shape/dtype errors, reference.py:32-46, fused.py:240-245) and ECUDA /
 * ENOTSUP -> RuntimeError. */
enum {
  SPARTON_OK = 0,
  SPARTON_EINVAL = 1,   /* bad shape / leading dim / alignment / null pointer */
  SPARTON_ECUDA = 2,    /* a CUDA runtime / driver call failed               */
  SPARTON_ENOTSUP = 3   /* device is not sm_100 (B200)                      */
};

/* Gradient output element types for sparton_bwd. */
enum { SPARTON_F32 = 0, SPARTON_BF16 = 1 };

/* ABI version (major*100 + minor). */
SPARTON_API int sparton_abi_version(void);

/* Thread-local description of the last non-OK status on this thread. */
SPARTON_API const char* sparton_last_error(void);

/* Number of SMs of the current device (0 when no device) — lets hosts size
 * shards; pure query, no kernel launch. */
SPARTON_API int sparton_device_sm_count(void);

/*
 * Forward.  Replaces forward_fully_fused / forward_hybrid
 * (fused.py:160-212 / fused.py:115-157): one persistent sm_100a kernel
 * (TMA -> tcgen05.mma bf16 -> TMEM fp32 -> fused bias/mask/max/argmax/log1p
 * epilogue).  Writes only Y and I; the B*S*V logits are never materialised.
 *   H     : bf16 [B*S, D]       E    : bf16 [V, D]
 *   bias  : f32 [V]             mask : u8 [B*S] (row-major B x S)
 *   Y     : f32 [B, ldY]        I    : i32 [B, ldY]
 *   cta_group : CTAs per cluster: 0 = auto (2), 1 = single-CTA UMMA (M=128),
 *               2 = CTA pair (cta_group::2, M=256), 4 = two CTA pairs sharing
 *               each H tile through TMA multicast (halves H L2 traffic)
 */
SPARTON_API int sparton_fwd(const void* H, const void* E, const float* bias, const uint8_t* mask,
                float* Y, int32_t* I,
                int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY,
                int cta_group, void* stream);

/*
 * FP8 forward (the paper's future-work item):
 * H8/E8 are e4m3 with per-tensor scales given as device scalars amax_h/amax_e
 * (logit = amax_h/448 * amax_e/448 * H8·E8 + bias), tensor-core
 * tcgen05.mma kind::f8f6f4 at twice the bf16 rate.  Numerics differ from the
 * bf16/fp32 reference by the e4m3 rounding (3 mantissa bits): Y is
 * approximate and the argmax agrees except where logits lie within the e4m3
 * error.  D must be a multiple of 16.  Otherwise identical to sparton_fwd.
 */
SPARTON_API int sparton_fwd_fp8(const void* H8, const void* E8, const float* amax_h, const float* amax_e,
                const float* bias, const uint8_t* mask, float* Y, int32_t* I,
                int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY,
                int cta_group, void* stream);

/*
 * sparton_fwd writing every (b, v) result to ndst (1..8) destinations with
 * one row stride ldY: Y_dst[k] / I_dst[k] are device pointers (host array of
 * pointers) to the first column this call covers.  For a vocab-sharded head
 * they are the peers' symmetric [B, V] buffers offset to this shard's first
 * column (P2P-mapped over NVLink) — the (Y, I) all-gather is fused into the
 * epilogue's stores (multicast addresses: sparton_fwd_multicast).  Destinations must
 * not overlap.  Replaces no reference function (the reference has no
 * multi-device path); see INTEGRATION.md.
 */
SPARTON_API int sparton_fwd_multi(const void* H, const void* E, const float* bias, const uint8_t* mask,
                                  int ndst, float* const* Y_dst, int32_t* const* I_dst,
                                  int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY,
                                  int cta_group, void* stream);

/*
 * sparton_fwd storing every (b, v) result with multimem.st.relaxed.sys to
 * NVLink SHARP multicast addresses Y_mc / I_mc (first column this call covers,
 * row stride ldY): the multicast object binds every rank's symmetric [B, V]
 * buffer, so one store per result lands in all ranks' copies — the (Y, I)
 * all-gather of a vocab-sharded head done by the switch inside the epilogue.
 * Needs an NVLS-capable NVSwitch system (a multicast object of >= 2 GPUs);
 * otherwise identical to sparton_fwd.  No reference counterpart.
 */
SPARTON_API int sparton_fwd_multicast(const void* H, const void* E, const float* bias, const uint8_t* mask,
                                      float* Y_mc, int32_t* I_mc, int64_t B, int64_t S, int64_t D, int64_t V,
                                      int64_t ldY, int cta_group, void* stream);

/* Per-tensor e4m3 quantisation of n bf16 values (n a multiple of 16, 16-B
 * aligned): amax (device f32 scalar) = max |x|, q = e4m3(x * 448 / amax). */
SPARTON_API int sparton_quantize_e4m3(const void* x_bf16, int64_t n, void* q_e4m3, float* amax, void* stream);

/*
 * MXFP8 forward (tcgen05 block-scaled MXFP8): e4m3
 * operands with one ue8m0 scale per 32 consecutive K elements of every row
 * (OCP MX), applied inside the MMA (tcgen05.mma kind::mxf8f6f4.block_scale,
 * scales staged smem -> TMEM by tcgen05.cp).  Hq/Eq and Hsf/Esf come from
 * sparton_quantize_mx; logit = sum_k 2^(sh-127) qh * 2^(se-127) qe + bias.
 * Sequence chunks are 240 positions (TMEM columns 240..255 hold the scale
 * factors).  D a multiple of 16; otherwise identical to sparton_fwd.
 * Replaces no reference function (the paper's future work).
 */
enum { SPARTON_MX_H = 0, SPARTON_MX_E = 1 };
/* Bytes of the scale-factor buffer of operand H (B, S, D) or E (V, D). */
SPARTON_API int64_t sparton_mx_scales_bytes(int64_t B, int64_t S, int64_t D, int64_t V, int operand);
/* Quantise bf16 x (H as B*S x D, or E as V x D) to e4m3 q (same shape) and
 * ue8m0 scales sf (sf_bytes >= sparton_mx_scales_bytes), in the layout the
 * forward's stages load: 2^e per 32-element block, the smallest power of two
 * with max|x|/2^e <= 448, q = e4m3_rn(x / 2^e). */
SPARTON_API int sparton_quantize_mx(const void* x_bf16, int64_t B, int64_t S, int64_t D, int64_t V, int operand,
                                    void* q_e4m3, void* sf, size_t sf_bytes, void* stream);
SPARTON_API int sparton_fwd_mx(const void* Hq, const void* Hsf, const void* Eq, const void* Esf,
                               const float* bias, const uint8_t* mask, float* Y, int32_t* I,
                               int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, void* stream);

/* Workspace bytes sparton_bwd needs for these sizes: the argmax-routed (v, g)
 * pair lists for dH (B*V*8 bytes) and their offsets, the per-(b, v) (s, g)
 * records of the staged dE (B*V*8 bytes, S <= 832), plus an fp32 dH
 * accumulator (B*S*D*4) when grad_dtype is bf16 and the vocabulary is
 * processed in more than one L2-sized chunk (and, for S > 832, an fp32 dE
 * carry for the gathered dE's batch-chunk passes).  Pure host arithmetic. */
SPARTON_API size_t sparton_bwd_workspace_bytes(int64_t B, int64_t S, int64_t D, int64_t V,
                                               int grad_dtype);

/*
 * Backward.  Replaces backward_fused (fused.py:215-278) from the saved
 * (Y, I) only.  dH/dE/db are fully overwritten (no accumulation into caller
 * buffers).  db may be NULL or include_bias_grad = 0 (fused.py:221,264) in
 * which case it is written as zeros if non-NULL.  Deterministic: every output
 * element has a single owner that accumulates in the reference's order.
 *   dY : f32 [B, ldDY]    dH : [B*S, D]   dE : [V, D]   db : f32 [V]
 *   grad_dtype : SPARTON_F32 or SPARTON_BF16 for dH and dE.
 *   workspace  : >= sparton_bwd_workspace_bytes(B, S, D, V, grad_dtype) bytes, 16-B aligned.
 */
SPARTON_API int sparton_bwd(const void* H, const void* E, const float* Y, const int32_t* I,
                const float* dY, void* dH, void* dE, float* db,
                int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, int64_t ldDY,
                int include_bias_grad, int grad_dtype,
                void* workspace, size_t workspace_bytes, void* stream);

/*
 * sparton_bwd plus an optional caller-owned cudaEvent_t (dh_ready_event,
 * may be NULL) that is recorded on `stream` as soon as dH is final — before
 * the call's dE/db work (which runs on a library side stream) has joined
 * `stream`.  Lets a caller overlap a consumer of dH (the vocab-sharded
 * head's dH all-reduce) with dE.  Everything else is sparton_bwd.
 */
SPARTON_API int sparton_bwd_ex(const void* H, const void* E, const float* Y, const int32_t* I,
                const float* dY, void* dH, void* dE, float* db,
                int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, int64_t ldDY,
                int include_bias_grad, int grad_dtype,
                void* workspace, size_t workspace_bytes, void* stream, void* dh_ready_event);

/*
 * Backward of the FP8 forward (sparton_fwd_fp8): the same argmax-routed
 * gradients with the e4m3 operands the forward multiplied — H8 [B*S, D] and
 * E8 [V, D] e4m3 bytes with their per-tensor amax (device f32 scalars; the
 * dequantised value is q * amax / 448).  dE = sum_b g * Hdq[b, I], dH =
 * sum_v g * Edq[v] (the straight-through gradient of the FP8 forward), db as
 * sparton_bwd.  Staged tiles and gathers move half the bytes of the bf16
 * backward.  Needs
 * D % 16 == 0 and S <= 832 (the staged dE); workspace as sparton_bwd.
 * No reference counterpart (PAPER.md:375 lists FP8 as future work).
 */
SPARTON_API int sparton_bwd_fp8(const void* H8, const void* E8, const float* amax_h, const float* amax_e,
                const float* Y, const int32_t* I, const float* dY, void* dH, void* dE, float* db,
                int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, int64_t ldDY,
                int include_bias_grad, int grad_dtype,
                void* workspace, size_t workspace_bytes, void* stream, void* dh_ready_event);

/*
 * dH reduction of the vocab-sharded head over NVLink peer memory (SURVEY.md
 * §8e C2): every rank's partial dH (fp32, n elements, n % 4 == 0, 16-B
 * aligned) sits in a buffer all ranks can address.  After the caller's
 * barrier (all partials written), rank `rank` sums its slice of float4 units
 * [rank*c, (rank+1)*c), c = ceil(n/4 / nranks), over the nranks partials in
 * rank order 0..nranks-1 (deterministic, identical on every rank) and stores
 * it to every rank's output buffer — fp32, or bf16 rounded once
 * (out_dtype SPARTON_F32 / SPARTON_BF16); the caller's second barrier
 * publishes the outputs.  The bytes of a reduce-scatter + all-gather in one
 * launch.  parts / outs: host arrays of nranks (1..8) device pointers in rank
 * order (peer-mapped: torch symmetric memory or CUDA IPC).  Replaces no
 * reference function (the reference has no multi-device path).
 */
SPARTON_API int sparton_allreduce_peers(const float* const* parts, void* const* outs, int nranks, int rank,
                                        int out_dtype, int64_t n, void* stream);

/*
 * The same reduction through NVLink SHARP: one multimem.ld_reduce.add.v4.f32
 * per unit on mc_part (the multicast address of the partial buffers — the
 * switch sums the copies) and one multimem.st to mc_out (the multicast
 * address of the output buffers).  Needs an NVLS-capable NVSwitch system
 * (a multicast object of >= 2 GPUs).
 */
SPARTON_API int sparton_allreduce_multimem(const float* mc_part, void* mc_out, int nranks, int rank,
                                           int out_dtype, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif  /* SPARTON_H_ */
