// sparton_abi.cu — the C-ABI entry points declared in include/sparton.h.
//
// Host-side validation mirrors the reference's error contract
// (reference.py:32-46 shape/dtype checks; fused.py:240-245 backward shape
// checks) but, like backward_fused (fused.py:232-235), never scans values.
// TMA tensor maps are encoded per call through the driver entry point
// obtained from the runtime (no link-time dependency on libcuda, so the
// library loads on GPU-less hosts for symbol checks).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "sparton_internal.h"

namespace sparton {

namespace {
thread_local char g_err[512] = "";

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

struct DevInfo {
  int sms = 0;
  int major = 0;
  int minor = 0;
};

int device_info(DevInfo& out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error("cudaGetDevice", e);
  static DevInfo cache[64];
  static bool have[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && have[dev]) { out = cache[dev]; return SPARTON_OK; }
  DevInfo d;
  if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess)
    return set_cuda_error("cudaDeviceGetAttribute", e);
  if (dev < 64) { cache[dev] = d; have[dev] = true; }
  out = d;
  return SPARTON_OK;
}

int encode_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, int box_rows, int box_cols,
              CUtensorMapSwizzle swz, bool u8) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return set_error(SPARTON_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * (u8 ? 1 : 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (CUresult %d) rows=%lld cols=%lld",
             (int)r, rows, cols);
    return set_error(SPARTON_ECUDA, buf);
  }
  return SPARTON_OK;
}

// Rows of `cols` uint32 (scale-factor chunks), boxes of box_rows rows.
int encode_2d_u32(CUtensorMap* map, const void* ptr, long long rows, int cols, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return set_error(SPARTON_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (scale factors) failed (CUresult %d) rows=%lld", (int)r, rows);
    return set_error(SPARTON_ECUDA, buf);
  }
  return SPARTON_OK;
}

int encode_bf16_2d_swz(CUtensorMap* map, const void* ptr, long long rows, long long cols,
                       int box_rows, int box_cols, CUtensorMapSwizzle swz) {
  return encode_2d(map, ptr, rows, cols, box_rows, box_cols, swz, false);
}


bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int encode_bf16_2d_plain(CUtensorMap* map, const void* ptr, long long rows, long long cols, int box_rows,
                         int box_cols) {
  return encode_bf16_2d_swz(map, ptr, rows, cols, box_rows, box_cols, CU_TENSOR_MAP_SWIZZLE_NONE);
}

const char* dev_env(const char* name) {
  const char* gate = getenv("SPARTON_DEV");
  if (gate == nullptr || gate[0] != '1') return nullptr;
  return getenv(name);
}

int encode_u8_2d_plain(CUtensorMap* map, const void* ptr, long long rows, long long cols, int box_rows,
                       int box_cols) {
  return encode_2d(map, ptr, rows, cols, box_rows, box_cols, CU_TENSOR_MAP_SWIZZLE_NONE, true);
}

int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

int set_cuda_error(const char* what, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return SPARTON_ECUDA;
}

}  // namespace sparton

using namespace sparton;

extern "C" {

int sparton_abi_version(void) { return 100; }

const char* sparton_last_error(void) { return g_err; }

int sparton_device_sm_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  DevInfo d;
  if (device_info(d) != SPARTON_OK) return 0;
  return d.sms;
}

static int check_dims(int64_t B, int64_t S, int64_t D, int64_t V) {
  char buf[200];
  if (B < 1 || S < 1 || D < 1 || V < 1) {
    snprintf(buf, sizeof(buf), "dims must be positive, got B=%lld S=%lld D=%lld V=%lld",
             (long long)B, (long long)S, (long long)D, (long long)V);
    return set_error(SPARTON_EINVAL, buf);
  }
  if (D % 8 != 0) {
    snprintf(buf, sizeof(buf), "D=%lld must be a multiple of 8 (zero-pad the hidden axis)", (long long)D);
    return set_error(SPARTON_EINVAL, buf);
  }
  if (B * S >= (1ll << 31) || V >= (1ll << 31) || B * V >= (1ll << 40) || D > (1 << 20)) {
    snprintf(buf, sizeof(buf), "dims exceed the kernel's index range: B=%lld S=%lld D=%lld V=%lld",
             (long long)B, (long long)S, (long long)D, (long long)V);
    return set_error(SPARTON_EINVAL, buf);
  }
  return SPARTON_OK;
}

static int check_device() {
  DevInfo d;
  int rc = device_info(d);
  if (rc != SPARTON_OK) return rc;
  if (d.major != 10 || d.minor != 0) {
    char buf[128];
    snprintf(buf, sizeof(buf), "sparton kernels are built for sm_100a (B200); device is sm_%d%d",
             d.major, d.minor);
    return set_error(SPARTON_ENOTSUP, buf);
  }
  return SPARTON_OK;
}

// fp8: 0 bf16 operands, 1 e4m3 with per-tensor amax scales, 2 MXFP8 (e4m3
// with the ue8m0 block scales Hsf / Esf of sparton_quantize_mx_{h,e}).
static int fwd_common(const void* H, const void* E, const float* amax_h, const float* amax_e, const float* bias,
                      const uint8_t* mask, float* Y, int32_t* I, int64_t B, int64_t S, int64_t D, int64_t V,
                      int64_t ldY, int cta_group, void* stream, int fp8, int nx = 0,
                      float* const* Yx = nullptr, int32_t* const* Ix = nullptr, const void* Hsf = nullptr,
                      const void* Esf = nullptr, bool multicast = false) {
  int rc = check_dims(B, S, D, V);
  if (rc) return rc;
  if (!H || !E || !bias || !mask || !Y || !I) return set_error(SPARTON_EINVAL, "null pointer argument");
  if (nx < 0 || nx > kMaxFwdDst - 1) return set_error(SPARTON_EINVAL, "ndst must lie in [1, 8]");
  for (int k = 0; k < nx; ++k)
    if (!Yx[k] || !Ix[k]) return set_error(SPARTON_EINVAL, "null destination pointer");
  if (fp8 == 1 && (!amax_h || !amax_e)) return set_error(SPARTON_EINVAL, "null amax pointer");
  if (fp8 == 2 && (!Hsf || !Esf)) return set_error(SPARTON_EINVAL, "null scale-factor pointer");
  if (fp8 == 2 && cta_group != 0 && cta_group != 2)
    return set_error(SPARTON_EINVAL, "MXFP8 runs on CTA pairs (cta_group 0 or 2)");
  if (fp8 == 2 && (!aligned16(Hsf) || !aligned16(Esf)))
    return set_error(SPARTON_EINVAL, "scale factors must be 16-byte aligned");
  if (fp8 && D % 16 != 0)
    return set_error(SPARTON_EINVAL, "e4m3 operands need D to be a multiple of 16 (TMA 16-byte stride)");
  if (!aligned16(H) || !aligned16(E)) return set_error(SPARTON_EINVAL, "H and E must be 16-byte aligned");
  if (ldY < V) return set_error(SPARTON_EINVAL, "ldY must be >= V");
  if (cta_group != 0 && cta_group != 1 && cta_group != 2 && cta_group != 4)
    return set_error(SPARTON_EINVAL, "cta_group must be 0, 1, 2 or 4");
  if ((rc = check_device())) return rc;
  DevInfo d;
  device_info(d);
  int cg = cta_group;
  if (cg == 0) {
    // Default: one CTA pair per cluster.  Two pairs sharing H tiles by TMA
    // multicast (cg = 4) cut L2 traffic but measured slower inside the step
    // (lock-step coupling of the pairs).
    cg = 2;
    if (const char* ev = dev_env("SPARTON_FWD_CLUSTER")) cg = atoi(ev);
    if (cg != 1 && cg != 2 && cg != 4) cg = 2;
    if (fp8 == 2) cg = 2;
  }
  // One 128-byte swizzle row per K step: 64 bf16 or 128 e4m3 columns.
  const int box_cols = fp8 ? 128 : 64;
  CUtensorMap tmE, tmH;
  if ((rc = encode_2d(&tmE, E, V, D, 128, box_cols, CU_TENSOR_MAP_SWIZZLE_128B, fp8))) return rc;
  if ((rc = encode_2d(&tmH, H, B * S, D, fwd_h_box_rows(cg, fp8), box_cols, CU_TENSOR_MAP_SWIZZLE_128B, fp8))) return rc;
  // MX scale factors as rows of 128 uint32 (one 512-B chunk per row).
  CUtensorMap tmSFA, tmSFB;
  if (fp8 == 2) {
    const long long ra = mx_sf_bytes(false, V, 1, (int)D) / 512, rb = mx_sf_bytes(true, B, S, (int)D) / 512;
    if ((rc = encode_2d_u32(&tmSFA, Esf, ra, 128, 1)) || (rc = encode_2d_u32(&tmSFB, Hsf, rb, 128, 2))) return rc;
  }
  FwdParams prm = {};
  prm.bias = bias;
  prm.mask = mask;
  prm.Y = Y;
  prm.I = I;
  prm.B = (int)B;
  prm.S = (int)S;
  prm.D = (int)D;
  prm.V = (int)V;
  prm.ldY = ldY;
  prm.fp8 = fp8;
  prm.nx = nx;
  prm.mc = multicast ? 1 : 0;
  for (int k = 0; k < nx; ++k) {
    prm.Yx[k] = Yx[k];
    prm.Ix[k] = Ix[k];
  }
  prm.amax_h = amax_h;
  prm.amax_e = amax_e;
  {
    const char* ev = dev_env("SPARTON_E_EVICT_LAST");
    // bits 0-1: E policy, bits 2-3: H policy (0 normal, 1 evict_last, 2 evict_first).
    // Both evict_last measured lowest DRAM traffic (profiles/r01_fwd_l2_policy.txt).
    prm.e_evict_last = ev ? atoi(ev) : 5;
  }
  return launch_fwd(tmE, tmH, fp8 == 2 ? &tmSFA : nullptr, fp8 == 2 ? &tmSFB : nullptr, prm, cg, d.sms,
                    static_cast<cudaStream_t>(stream));
}

int sparton_fwd(const void* H, const void* E, const float* bias, const uint8_t* mask, float* Y,
                int32_t* I, int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, int cta_group,
                void* stream) {
  return fwd_common(H, E, nullptr, nullptr, bias, mask, Y, I, B, S, D, V, ldY, cta_group, stream, 0);
}

int sparton_fwd_multi(const void* H, const void* E, const float* bias, const uint8_t* mask, int ndst,
                      float* const* Y_dst, int32_t* const* I_dst, int64_t B, int64_t S, int64_t D, int64_t V,
                      int64_t ldY, int cta_group, void* stream) {
  if (ndst < 1 || ndst > kMaxFwdDst || !Y_dst || !I_dst)
    return set_error(SPARTON_EINVAL, "ndst must lie in [1, 8] with non-null destination arrays");
  return fwd_common(H, E, nullptr, nullptr, bias, mask, Y_dst[0], I_dst[0], B, S, D, V, ldY, cta_group, stream,
                    0, ndst - 1, Y_dst + 1, I_dst + 1);
}

int sparton_fwd_multicast(const void* H, const void* E, const float* bias, const uint8_t* mask, float* Y_mc,
                          int32_t* I_mc, int64_t B, int64_t S, int64_t D, int64_t V, int64_t ldY, int cta_group,
                          void* stream) {
  return fwd_common(H, E, nullptr, nullptr, bias, mask, Y_mc, I_mc, B, S, D, V, ldY, cta_group, stream, 0, 0,
                    nullptr, nullptr, nullptr, nullptr, true);
}

int sparton_fwd_fp8(const void* H8, const void* E8, const float* amax_h, const float* amax_e, const float* bias,
                    const uint8_t* mask, float* Y, int32_t* I, int64_t B, int64_t S, int64_t D, int64_t V,
                    int64_t ldY, int cta_group, void* stream) {
  return fwd_common(H8, E8, amax_h, amax_e, bias, mask, Y, I, B, S, D, V, ldY, cta_group, stream, 1);
}

int64_t sparton_mx_scales_bytes(int64_t B, int64_t S, int64_t D, int64_t V, int operand) {
  if (B < 1 || S < 1 || D < 1 || V < 1 || (operand != SPARTON_MX_H && operand != SPARTON_MX_E)) return 0;
  return operand == SPARTON_MX_H ? mx_sf_bytes(true, B, S, (int)D) : mx_sf_bytes(false, V, 1, (int)D);
}

int sparton_quantize_mx(const void* x, int64_t B, int64_t S, int64_t D, int64_t V, int operand, void* q, void* sf,
                        size_t sf_bytes, void* stream) {
  int rc = check_dims(B, S, D, V);
  if (rc) return rc;
  if (operand != SPARTON_MX_H && operand != SPARTON_MX_E)
    return set_error(SPARTON_EINVAL, "operand must be SPARTON_MX_H or SPARTON_MX_E");
  if (!x || !q || !sf) return set_error(SPARTON_EINVAL, "null pointer argument");
  if (D % 16 != 0) return set_error(SPARTON_EINVAL, "e4m3 operands need D to be a multiple of 16");
  if (!aligned16(x) || !aligned16(q) || !aligned16(sf))
    return set_error(SPARTON_EINVAL, "x, q and sf must be 16-byte aligned");
  if ((int64_t)sf_bytes < sparton_mx_scales_bytes(B, S, D, V, operand))
    return set_error(SPARTON_EINVAL, "scale-factor buffer too small (sparton_mx_scales_bytes)");
  if ((rc = check_device())) return rc;
  const bool h = operand == SPARTON_MX_H;
  return launch_quantize_mx(h, x, h ? B : V, h ? S : 1, (int)D, q, sf, static_cast<cudaStream_t>(stream));
}

int sparton_fwd_mx(const void* Hq, const void* Hsf, const void* Eq, const void* Esf, const float* bias,
                   const uint8_t* mask, float* Y, int32_t* I, int64_t B, int64_t S, int64_t D, int64_t V,
                   int64_t ldY, void* stream) {
  if (D % 16 != 0) return set_error(SPARTON_EINVAL, "e4m3 operands need D to be a multiple of 16");
  return fwd_common(Hq, Eq, nullptr, nullptr, bias, mask, Y, I, B, S, D, V, ldY, 0, stream, 2, 0, nullptr, nullptr,
                    Hsf, Esf);
}

namespace {
int check_allreduce(int nranks, int rank, int out_dtype, int64_t n) {
  if (nranks < 1 || nranks > kMaxPeers) return set_error(SPARTON_EINVAL, "nranks must lie in [1, 8]");
  if (rank < 0 || rank >= nranks) return set_error(SPARTON_EINVAL, "rank must lie in [0, nranks)");
  if (out_dtype != SPARTON_F32 && out_dtype != SPARTON_BF16)
    return set_error(SPARTON_EINVAL, "out_dtype must be SPARTON_F32 or SPARTON_BF16");
  if (n < 0 || n % 4 != 0) return set_error(SPARTON_EINVAL, "n must be a non-negative multiple of 4");
  return SPARTON_OK;
}
}  // namespace

int sparton_allreduce_peers(const float* const* parts, void* const* outs, int nranks, int rank, int out_dtype,
                            int64_t n, void* stream) {
  int rc = check_allreduce(nranks, rank, out_dtype, n);
  if (rc) return rc;
  if (!parts || !outs) return set_error(SPARTON_EINVAL, "null pointer array");
  for (int q = 0; q < nranks; ++q) {
    if (!parts[q] || !outs[q]) return set_error(SPARTON_EINVAL, "null peer pointer");
    if (!aligned16(parts[q]) || (reinterpret_cast<uintptr_t>(outs[q]) & (out_dtype == SPARTON_BF16 ? 7u : 15u)))
      return set_error(SPARTON_EINVAL, "partials must be 16-B aligned, outputs 16-B (fp32) / 8-B (bf16) aligned");
  }
  if ((rc = check_device())) return rc;
  return launch_allreduce_peers(parts, outs, nranks, rank, out_dtype == SPARTON_BF16, n,
                                static_cast<cudaStream_t>(stream));
}

int sparton_allreduce_multimem(const float* mc_part, void* mc_out, int nranks, int rank, int out_dtype, int64_t n,
                               void* stream) {
  int rc = check_allreduce(nranks, rank, out_dtype, n);
  if (rc) return rc;
  if (!mc_part || !mc_out) return set_error(SPARTON_EINVAL, "null multicast address");
  if (!aligned16(mc_part) || (reinterpret_cast<uintptr_t>(mc_out) & (out_dtype == SPARTON_BF16 ? 7u : 15u)))
    return set_error(SPARTON_EINVAL, "multicast addresses must be 16-B (fp32) / 8-B (bf16) aligned");
  if ((rc = check_device())) return rc;
  return launch_allreduce_multimem(mc_part, mc_out, nranks, rank, out_dtype == SPARTON_BF16, n,
                                   static_cast<cudaStream_t>(stream));
}

int sparton_quantize_e4m3(const void* x, int64_t n, void* q, float* amax, void* stream) {
  if (n < 1) return set_error(SPARTON_EINVAL, "n must be positive");
  if (!x || !q || !amax) return set_error(SPARTON_EINVAL, "null pointer argument");
  if (!aligned16(x) || !aligned16(q) || n % 16 != 0)
    return set_error(SPARTON_EINVAL, "x and q must be 16-byte aligned and n a multiple of 16");
  int rc = check_device();
  if (rc) return rc;
  return launch_quantize_e4m3(x, n, q, amax, static_cast<cudaStream_t>(stream));
}

size_t sparton_bwd_workspace_bytes(int64_t B, int64_t S, int64_t D, int64_t V, int grad_dtype) {
  if (B < 1 || S < 1 || D < 1 || V < 1) return 0;
  return bwd_workspace_layout(B, S, D, V, grad_dtype).total;
}

int sparton_bwd(const void* H, const void* E, const float* Y, const int32_t* I, const float* dY,
                void* dH, void* dE, float* db, int64_t B, int64_t S, int64_t D, int64_t V,
                int64_t ldY, int64_t ldDY, int include_bias_grad, int grad_dtype, void* workspace,
                size_t workspace_bytes, void* stream) {
  return sparton_bwd_ex(H, E, Y, I, dY, dH, dE, db, B, S, D, V, ldY, ldDY, include_bias_grad, grad_dtype,
                        workspace, workspace_bytes, stream, nullptr);
}

static int bwd_common(const void* H, const void* E, const float* amax_h, const float* amax_e, const float* Y,
                      const int32_t* I, const float* dY, void* dH, void* dE, float* db, int64_t B, int64_t S,
                      int64_t D, int64_t V, int64_t ldY, int64_t ldDY, int include_bias_grad, int grad_dtype,
                      void* workspace, size_t workspace_bytes, void* stream, void* dh_ready_event, bool fp8) {
  int rc = check_dims(B, S, D, V);
  if (rc) return rc;
  if (!H || !E || !Y || !I || !dY || !dH || !dE || !workspace)
    return set_error(SPARTON_EINVAL, "null pointer argument");
  if (!aligned16(H) || !aligned16(E) || !aligned16(dH) || !aligned16(dE) || !aligned16(workspace))
    return set_error(SPARTON_EINVAL, "H, E, dH, dE and workspace must be 16-byte aligned");
  if (ldY < V || ldDY < V) return set_error(SPARTON_EINVAL, "ldY and ldDY must be >= V");
  if (grad_dtype != SPARTON_F32 && grad_dtype != SPARTON_BF16)
    return set_error(SPARTON_EINVAL, "grad_dtype must be SPARTON_F32 or SPARTON_BF16");
  if (S > bwd_max_seq()) return set_error(SPARTON_EINVAL, "S exceeds the backward's routing limit");
  if (fp8) {
    if (!amax_h || !amax_e) return set_error(SPARTON_EINVAL, "null amax pointer");
    if (D % 16 != 0) return set_error(SPARTON_EINVAL, "e4m3 operands need D to be a multiple of 16");
    if (de_staged_rows((int)S) == 0)
      return set_error(SPARTON_EINVAL, "the FP8 backward supports S <= 832 (staged dE)");
  }
  const BwdWorkspace ws = bwd_workspace_layout(B, S, D, V, grad_dtype);
  const size_t need = ws.total;
  if (workspace_bytes < need) {
    char buf[160];
    snprintf(buf, sizeof(buf), "workspace too small: %zu < %zu bytes", workspace_bytes, need);
    return set_error(SPARTON_EINVAL, buf);
  }
  if ((rc = check_device())) return rc;
  BwdParams p = {};
  p.H = static_cast<const __nv_bfloat16*>(H);
  p.E = static_cast<const __nv_bfloat16*>(E);
  p.Y = Y;
  p.I = I;
  p.dY = dY;
  p.dH = dH;
  p.dE = dE;
  p.db = db;
  p.B = (int)B;
  p.S = (int)S;
  p.D = (int)D;
  p.V = (int)V;
  p.ldY = ldY;
  p.ldDY = ldDY;
  p.include_bias_grad = include_bias_grad;
  char* wsb = static_cast<char*>(workspace);
  p.pairs = reinterpret_cast<int2*>(wsb + ws.pairs);
  p.offsets = reinterpret_cast<int*>(wsb + ws.offsets);
  p.acc32 = ws.acc32 == (size_t)-1 ? nullptr : reinterpret_cast<float*>(wsb + ws.acc32);
  p.dE_acc = ws.dE_acc == (size_t)-1 ? nullptr : reinterpret_cast<float*>(wsb + ws.dE_acc);
  p.db_acc = reinterpret_cast<float*>(wsb + ws.db_acc);
  p.bchunk = ws.bchunk;
  p.nwin = ws.nwin;
  p.wpc = ws.wpc;
  p.nchunks = ws.nchunks;
  p.gi = ws.de_staged ? reinterpret_cast<int2*>(wsb + ws.gi) : nullptr;
  p.ldGI = ws.ldGI;
  p.dh_ready = static_cast<cudaEvent_t>(dh_ready_event);
  p.fp8 = fp8 ? 1 : 0;
  p.amax_h = amax_h;
  p.amax_e = amax_e;
  // Sparse regime (staged-dE shapes, bf16 operands): thresholds in active
  // pairs, as a percentage of B*V (tools/sparse_probe.py measured the
  // crossovers; SPARTON_DE_SPARSE_PCT / SPARTON_DH_SPARSE_PCT override them
  // under the dev gate, a negative value disables the sparse kernel).
  if (ws.de_staged && !fp8) {
    p.stats = reinterpret_cast<unsigned long long*>(wsb + ws.stats);
    double de_pct = kDeSparsePct, dh_pct = kDhSparsePct;
    if (const char* ev = dev_env("SPARTON_DE_SPARSE_PCT")) de_pct = atof(ev);
    if (const char* ev = dev_env("SPARTON_DH_SPARSE_PCT")) dh_pct = atof(ev);
    const double pairs = (double)B * (double)V;
    p.de_sparse_max = de_pct < 0 ? -1 : (long long)(pairs * de_pct / 100.0);
    p.dh_sparse_max = dh_pct < 0 ? -1 : (long long)(pairs * dh_pct / 100.0);
  }
  CUtensorMap tmH;
  if (ws.de_staged) {
    const int rows = de_staged_rows((int)S);
    rc = fp8 ? encode_u8_2d_plain(&tmH, H, B * S, D, rows > 256 ? 256 : rows, 64)
             : encode_bf16_2d_plain(&tmH, H, B * S, D, rows > 256 ? 256 : rows, 64);
    if (rc) return rc;
  }
  return launch_bwd(p, ws.de_staged ? &tmH : nullptr, grad_dtype, static_cast<cudaStream_t>(stream));
}


int sparton_bwd_ex(const void* H, const void* E, const float* Y, const int32_t* I, const float* dY,
                   void* dH, void* dE, float* db, int64_t B, int64_t S, int64_t D, int64_t V,
                   int64_t ldY, int64_t ldDY, int include_bias_grad, int grad_dtype, void* workspace,
                   size_t workspace_bytes, void* stream, void* dh_ready_event) {
  return bwd_common(H, E, nullptr, nullptr, Y, I, dY, dH, dE, db, B, S, D, V, ldY, ldDY, include_bias_grad,
                    grad_dtype, workspace, workspace_bytes, stream, dh_ready_event, false);
}

int sparton_bwd_fp8(const void* H8, const void* E8, const float* amax_h, const float* amax_e, const float* Y,
                    const int32_t* I, const float* dY, void* dH, void* dE, float* db, int64_t B, int64_t S,
                    int64_t D, int64_t V, int64_t ldY, int64_t ldDY, int include_bias_grad, int grad_dtype,
                    void* workspace, size_t workspace_bytes, void* stream, void* dh_ready_event) {
  return bwd_common(H8, E8, amax_h, amax_e, Y, I, dY, dH, dE, db, B, S, D, V, ldY, ldDY, include_bias_grad,
                    grad_dtype, workspace, workspace_bytes, stream, dh_ready_event, true);
}

}  // extern "C"
