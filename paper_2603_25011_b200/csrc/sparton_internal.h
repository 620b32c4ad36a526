// sparton_internal.h — shared host/device declarations between the C-ABI
// layer (sparton_abi.cu) and the kernels (sparton_fwd.cu, sparton_bwd.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstddef>

#include "../../include/sparton.h"

namespace sparton {

constexpr int kMaxFwdDst = 8;
constexpr int kMaxPeers = 8;   // ranks a peer-memory dH reduction addresses (sparton_coll.cu)
// Sparse-regime thresholds of the backward (percent of the B*V pairs active).
constexpr double kDeSparsePct = 40.0;
constexpr double kDhSparsePct = 12.0;

struct FwdParams {
  const float* bias;
  const uint8_t* mask;
  float* Y;
  int32_t* I;
  // Extra destinations (sparton_fwd_multi): every (b, v) result is also stored
  // to Yx[k] / Ix[k] (same ldY), k < nx — the peers' copies of a sharded
  // head's [B, V] output (P2P stores), fusing the all-gather into the epilogue.
  int nx;
  float* Yx[kMaxFwdDst - 1];
  int32_t* Ix[kMaxFwdDst - 1];
  // mc = 1: Y / I are NVLink SHARP multicast addresses (a symmetric [B, V]
  // buffer bound on every rank): one multimem.st per result reaches every
  // rank's copy, the all-gather done by the switch (nx must be 0).
  int mc;
  int B, S, D, V;
  long long ldY;
  int num_vt;          // number of vocab tiles
  int group_vt;        // vocab tiles per L2 rasterisation group
  long long num_units; // num_vt * B
  int e_evict_last;    // L2 policy for E tiles (experiment switch)
  int sched_bgroups;   // 1: batch-row-per-cluster groups (large B), 0: round-robin units
  int rot;             // per-group rotation of the cluster -> batch-row assignment
  int epi_mode;        // experiment switch: 1 = max-only epilogue (no bias/argmax; wrong I)
  int pack;            // batch rows per 256-position chunk (S = 256/pack in {32, 64, 128}), else 1
  int urows;           // unit rows: B (pack == 1) or ceil(B / pack) batch-row groups
  int n_last;          // UMMA N of a unit's last sequence chunk (multiple of 16, <= 256)
  int fp8;             // 1: H and E are e4m3 (kind::f8f6f4), dequantised by amax_h/448 * amax_e/448;
                       // 2: MXFP8 (kind::mxf8f6f4.block_scale, ue8m0 scales per 32 K elements)
  const float* amax_h; // device scalars (FP8 only)
  const float* amax_e;
};

struct BwdParams {
  const __nv_bfloat16* H;
  const __nv_bfloat16* E;
  const float* Y;
  const int32_t* I;
  const float* dY;
  void* dH;
  void* dE;
  float* db;
  int B, S, D, V;
  long long ldY, ldDY;
  int include_bias_grad;
  int2* pairs;         // workspace: per-b argmax-routed (v, g) lists, B*V entries
  int* offsets;        // workspace: B*nwin*(S+1) per-(b, window, s) list offsets
  float* acc32;        // workspace: fp32 dH accumulator (bf16 output, >1 chunk) or nullptr
  float* dE_acc;       // workspace: fp32 dE carry across batch-chunk passes (bf16 output) or nullptr
  float* db_acc;       // workspace: fp32 db carry across batch-chunk passes
  int bchunk;          // batch rows per dE pass (H chunk kept L2-resident)
  int nwin;            // route windows (RT_WIN vocab rows each)
  int wpc;             // route windows per dH pass (E chunk kept L2-resident)
  int nchunks;         // dH passes
  int2* gi;            // workspace: per-(b, v) (s, g) records, row stride ldGI (staged dE), or nullptr
  long long ldGI;      // even row stride of gi (16-B aligned rows)
  cudaEvent_t dh_ready; // optional: recorded on the caller's stream once dH is final (before dE joins)
  // FP8 backward (sparton_bwd_fp8): H and E are e4m3 bytes (H, E point at
  // them), dequantised by amax/448 (device scalars) once per output element.
  int fp8;
  const float* amax_h;
  const float* amax_e;
  // Sparse regime (SPLADE representations: few active (b, v) pairs).  The
  // route counts the active pairs into stats[0] (zeroed before it); with at
  // most de_sparse_max active pairs dE runs as a per-pair gather (the staged
  // dE and db kernels exit at once), with at most dh_sparse_max dH runs as one
  // pass over the whole vocabulary without the fp32 carry.  Decided on the
  // device: no host synchronisation.  stats == nullptr: dense kernels only.
  unsigned long long* stats;
  long long de_sparse_max;
  long long dh_sparse_max;
};

// Workspace layout for sparton_bwd (byte offsets, 256-B aligned).
struct BwdWorkspace {
  size_t pairs, offsets, db_acc, dE_acc, acc32, gi, stats, total;
  long long ldGI;
  bool de_staged;
  int nwin, wpc, nchunks, bchunk;
};
BwdWorkspace bwd_workspace_layout(long long B, long long S, long long D, long long V, int grad_dtype);

// Development switches (A/B experiments, alternative-path tests).  The shipped
// library reads NO environment variable unless SPARTON_DEV=1 is set, so a
// stray variable cannot change what a production process launches.  Returns
// getenv(name) under the gate, nullptr otherwise.
const char* dev_env(const char* name);

// Records a thread-local error message and returns the status code.
int set_error(int code, const char* msg);
int set_cuda_error(const char* what, cudaError_t e);

// tmSFA / tmSFB: the MXFP8 scale-factor maps (prm.fp8 == 2), else nullptr.
int launch_fwd(const CUtensorMap& tmE, const CUtensorMap& tmH, const CUtensorMap* tmSFA, const CUtensorMap* tmSFB,
               FwdParams prm, int cluster_ctas, int num_sms, cudaStream_t stream);
int launch_quantize_e4m3(const void* x, long long n, void* q, float* amax, cudaStream_t stream);
int fwd_smem_bytes(int cluster_ctas);
int fwd_h_box_rows(int cluster_ctas, int fp8_mode);
// Sequence positions per forward chunk (256; MXFP8: 240) and the short-sequence packing factor.
int fwd_chunk_cols(int fp8_mode);
int fwd_pack(int S, int fp8_mode);
// MXFP8 operands: scale-factor bytes and the quantiser (h_operand: H as
// (B, S, D) laid out per the forward's (unit row, chunk) slots; else E (V, D)).
long long mx_sf_bytes(bool h_operand, long long rows_or_B, long long S, int D);
int launch_quantize_mx(bool h_operand, const void* x, long long rows_or_B, long long S, int D, void* q, void* sf,
                       cudaStream_t stream);
// H viewed as (B*S) x D bf16 with a (64 x rows) box, no swizzle (staged dE tiles).
int encode_bf16_2d_plain(CUtensorMap* map, const void* ptr, long long rows, long long cols, int box_rows,
                         int box_cols);
int launch_bwd(const BwdParams& prm, const CUtensorMap* tmH, int grad_dtype, cudaStream_t stream);
// H viewed as (B*S) x D bytes with a (128 x rows) box, no swizzle (FP8 staged dE tiles).
int encode_u8_2d_plain(CUtensorMap* map, const void* ptr, long long rows, long long cols, int box_rows,
                       int box_cols);
// Rows of H each CTA of a staged-dE cluster loads per batch row (0: staged dE unsupported for S).
int de_staged_rows(int S);
int bwd_max_seq();
// dH reduction over peer memory (sparton_coll.cu): parts/outs are nranks
// device pointers in rank order; n fp32 elements, a multiple of 4.
int launch_allreduce_peers(const float* const* parts, void* const* outs, int nranks, int rank, bool bf16,
                           long long n, cudaStream_t stream);
int launch_allreduce_multimem(const float* mc_part, void* mc_out, int nranks, int rank, bool bf16, long long n,
                              cudaStream_t stream);

}  // namespace sparton
