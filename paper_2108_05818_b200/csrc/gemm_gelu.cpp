// GEMMs with the GELU fused into the cuBLASLt epilogue (model side of the
// GPT step on B200).  The library GEMM is cuBLASLt's (tcgen05 kernels); what
// this file adds is the fusion of the MLP activation into it:
//
//   mode 0 (forward, mlp_in):  u = x · Wᵀ  and  g = gelu(u) in ONE GEMM
//          (CUBLASLT_EPILOGUE_GELU_AUX: D = gelu(acc), aux = acc)
//   mode 1 (backward, mlp_out): du = (dy · W) ⊙ gelu'(u) in ONE GEMM
//          (CUBLASLT_EPILOGUE_DGELU, aux = the saved pre-activation u)
//
// replacing the separate GeluCUDAKernel / GeluBackwardCUDAKernel passes.
// gelu is the tanh approximation (as the model's F.gelu(approximate="tanh")).
// Row-major operands are mapped to cuBLASLt's column-major convention:
//   mode 0: Dᵀ[O,T] = op_T(W stored [K,O]) · xᵀ[K,T]
//   mode 1: Dᵀ[O,T] = Wᵀ-as-stored [O,K] · dyᵀ[K,T]
// Plans (descriptors + heuristic algorithm) are cached per (mode, dtype,
// T, O, K).  The caller provides the workspace; nothing is allocated.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "cs_internal.h"

namespace {

struct Plan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  cublasLtMatmulAlgo_t algo;
  size_t ws_needed = 0;
};

cublasLtHandle_t g_lt = nullptr;
std::mutex g_mu;
std::map<std::tuple<int, int, int64_t, int64_t, int64_t, int64_t>, Plan> g_plans;

int lt_error(const char* what, cublasStatus_t st) {
  cs::set_error("%s: cuBLASLt status %d", what, (int)st);
  return st == CUBLAS_STATUS_SUCCESS ? 0 : -10 - (int)st;
}

#define LT(call, what)                                      \
  do {                                                      \
    cublasStatus_t _st = (call);                            \
    if (_st != CUBLAS_STATUS_SUCCESS) return lt_error(what, _st); \
  } while (0)

int make_plan(int mode, int dtype, int64_t T, int64_t O, int64_t K, int64_t ws_bytes,
              Plan* p) {
  const cudaDataType_t ty = dtype == CS_BF16 ? CUDA_R_16BF : CUDA_R_16F;
  LT(cublasLtMatmulDescCreate(&p->op, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc");
  const cublasOperation_t ta = mode == 1 ? CUBLAS_OP_N : CUBLAS_OP_T;
  const cublasOperation_t tb = CUBLAS_OP_N;
  LT(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)), "transa");
  LT(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)), "transb");
  if (mode != 2) {
    const cublasLtEpilogue_t epi =
        mode == 0 ? CUBLASLT_EPILOGUE_GELU_AUX : CUBLASLT_EPILOGUE_DGELU;
    LT(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)),
       "epilogue");
    const int64_t ld_aux = O;
    LT(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &ld_aux,
                                      sizeof(ld_aux)), "aux ld");
  }
  if (mode != 1) {  // A: W row-major [O,K] = column-major [K,O]
    LT(cublasLtMatrixLayoutCreate(&p->a, ty, K, O, K), "layout a");
  } else {          // A: W row-major [K,O] = column-major [O,K]
    LT(cublasLtMatrixLayoutCreate(&p->a, ty, O, K, O), "layout a");
  }
  LT(cublasLtMatrixLayoutCreate(&p->b, ty, K, T, K), "layout b");  // x / dy row-major [T,K]
  LT(cublasLtMatrixLayoutCreate(&p->d, ty, O, T, O), "layout d");  // out row-major [T,O]
  cublasLtMatmulPreference_t pref;
  LT(cublasLtMatmulPreferenceCreate(&pref), "pref");
  const size_t ws = (size_t)ws_bytes;
  LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws,
                                          sizeof(ws)), "pref ws");
  cublasLtMatmulHeuristicResult_t res;
  int found = 0;
  const cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(g_lt, p->op, p->a, p->b, p->d, p->d,
                                                           pref, 1, &res, &found);
  cublasLtMatmulPreferenceDestroy(pref);
  if (st != CUBLAS_STATUS_SUCCESS || found == 0) {
    cs::set_error("cs_gemm_gelu: no cuBLASLt algorithm for mode %d (%lld x %lld x %lld)", mode,
                  (long long)T, (long long)O, (long long)K);
    return CS_EINVAL;
  }
  p->algo = res.algo;
  p->ws_needed = res.workspaceSize;
  return 0;
}

}  // namespace

extern "C" int cs_gemm_gelu(int mode, const void* w, const void* x, void* out, void* aux,
                            int64_t T, int64_t O, int64_t K, int dtype, void* workspace,
                            int64_t ws_bytes, void* stream) {
  if ((mode != 0 && mode != 1) || !w || !x || !out || !aux || T <= 0 || O <= 0 || K <= 0 ||
      (dtype != CS_FP16 && dtype != CS_BF16) || ws_bytes < 0 || (ws_bytes > 0 && !workspace)) {
    cs::set_error("cs_gemm_gelu: invalid argument");
    return CS_EINVAL;
  }
  Plan* plan;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_lt) LT(cublasLtCreate(&g_lt), "create");
    const auto key = std::make_tuple(mode, dtype, T, O, K, ws_bytes);
    auto it = g_plans.find(key);
    if (it == g_plans.end()) {
      Plan p;
      if (int e = make_plan(mode, dtype, T, O, K, ws_bytes, &p)) return e;
      it = g_plans.emplace(key, p).first;
    }
    plan = &it->second;
  }
  LT(cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux,
                                    sizeof(aux)), "aux ptr");
  const float alpha = 1.0f, beta = 0.0f;
  LT(cublasLtMatmul(g_lt, plan->op, &alpha, w, plan->a, x, plan->b, &beta, out, plan->d, out,
                    plan->d, &plan->algo, workspace, (size_t)ws_bytes,
                    static_cast<cudaStream_t>(stream)), "matmul");
  return 0;  // a library (cuBLASLt) kernel: not counted in cs_launch_count

}

// Residual GEMM: out[T,O] = x[T,K] · W[O,K]ᵀ + res[T,O], with the residual read
// by the GEMM itself (cuBLASLt C ≠ D, beta = 1).  torch.addmm(res, x, Wᵀ)
// first copies res into its output and then accumulates (an extra 2·T·O·2
// bytes per call); here the residual stream stays where it is (the
// LayerNorm backward still needs it) and the sum lands in a new buffer.
extern "C" int cs_gemm_res(const void* w, const void* x, const void* res, void* out, int64_t T,
                           int64_t O, int64_t K, int dtype, void* workspace, int64_t ws_bytes,
                           void* stream) {
  if (!w || !x || !res || !out || T <= 0 || O <= 0 || K <= 0 ||
      (dtype != CS_FP16 && dtype != CS_BF16) || ws_bytes < 0 || (ws_bytes > 0 && !workspace)) {
    cs::set_error("cs_gemm_res: invalid argument");
    return CS_EINVAL;
  }
  Plan* plan;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_lt) LT(cublasLtCreate(&g_lt), "create");
    const auto key = std::make_tuple(2, dtype, T, O, K, ws_bytes);
    auto it = g_plans.find(key);
    if (it == g_plans.end()) {
      Plan p;
      if (int e = make_plan(2, dtype, T, O, K, ws_bytes, &p)) return e;
      it = g_plans.emplace(key, p).first;
    }
    plan = &it->second;
  }
  const float alpha = 1.0f, beta = 1.0f;
  LT(cublasLtMatmul(g_lt, plan->op, &alpha, w, plan->a, x, plan->b, &beta, res, plan->d, out,
                    plan->d, &plan->algo, workspace, (size_t)ws_bytes,
                    static_cast<cudaStream_t>(stream)), "matmul");
  return 0;
}
