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

struct FwdParams {
  const float* bias;
  const uint8_t* mask;
  float* Y;
  int32_t* I;
  int B, S, D, V;
  long long ldY;
  int num_vt;          // number of vocab tiles
  int group_vt;        // vocab tiles per L2 rasterisation group
  long long num_units; // num_vt * B
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
  int* offsets;        // workspace: B*(S+1) list offsets
};

// Records a thread-local error message and returns the status code.
int set_error(int code, const char* msg);
int set_cuda_error(const char* what, cudaError_t e);

int launch_fwd(const CUtensorMap& tmE, const CUtensorMap& tmH, FwdParams prm, int cta_group,
               int num_sms, cudaStream_t stream);
int fwd_smem_bytes(int cta_group);
int launch_bwd(const BwdParams& prm, int grad_dtype, cudaStream_t stream);
size_t bwd_workspace_bytes(long long B, long long S, long long V);
int bwd_max_seq();

}  // namespace sparton
