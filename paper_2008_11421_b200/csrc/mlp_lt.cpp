// GPT MLP GEMMs with their bias / GELU work in the cuBLASLt epilogue (library
// GEMMs, as the transformer's other GEMMs; what is fused is the elementwise
// work around them):
//
//   forward   f1 = x . W1^T + b1 (the GELU input, written as the epilogue's
//             auxiliary output into the saved slot) and g = gelu_tanh(f1) in
//             one GEMM (CUBLASLT_EPILOGUE_GELU_AUX_BIAS): the separate GELU
//             pass that read f1 and wrote g is gone
//   backward  df1 = (dy . W2) * gelu_tanh'(f1) in the fc2 data-gradient GEMM
//             (CUBLASLT_EPILOGUE_DGELU): replaces the GELU-backward pass.  (The
//             DGELU_BGRAD form would also sum fc1's bias gradient, but only in
//             the output type, bf16; the fp32 sum stays with fc1's weight
//             gradient, which reads df1 anyway.)
//   fc2       y = x2 + g . W2^T + b2 in one GEMM (bias epilogue, beta = 1 on
//             the residual): the layer output is written once, no separate
//             add pass and no intermediate fc2 output
//
// Row-major torch tensors map to column-major cuBLASLt as transposes: the
// row-major [M, N] output is the column-major N x M matrix D with ld = N.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "mlp_lt.hpp"

namespace krt {
namespace {

struct LtState {
  cublasLtHandle_t h = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 64ull << 20;
  std::map<std::tuple<int, int64_t, int64_t, int64_t, int>, cublasLtMatmulAlgo_t> algos;
  std::mutex mu;
};

LtState& lt() {
  static LtState s;
  return s;
}

#define LT_CHECK(x)                                                                          \
  do {                                                                                       \
    cublasStatus_t st_ = (x);                                                                \
    if (st_ != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string(#x) + " failed: " + \
                                                               std::to_string((int)st_));    \
  } while (0)

struct Desc {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  ~Desc() {
    if (op) cublasLtMatmulDescDestroy(op);
    if (a) cublasLtMatrixLayoutDestroy(a);
    if (b) cublasLtMatrixLayoutDestroy(b);
    if (d) cublasLtMatrixLayoutDestroy(d);
  }
};

// D (m x n, col-major, ld m) = op(A) . op(B) with the epilogue; kind tags the
// algorithm cache
void run(int kind, cublasOperation_t ta, cublasOperation_t tb, int64_t m, int64_t n, int64_t k, const void* A,
         int64_t lda, const void* B, int64_t ldb, void* D, cublasLtEpilogue_t epi, const void* bias, int bias_type,
         void* aux, cudaStream_t stream, const void* C = nullptr, cudaDataType_t d_type = CUDA_R_16BF) {
  LtState& s = lt();
  std::lock_guard<std::mutex> lk(s.mu);
  if (!s.h) {
    LT_CHECK(cublasLtCreate(&s.h));
    if (cudaMalloc(&s.ws, s.ws_bytes) != cudaSuccess) throw std::runtime_error("cublasLt workspace: cudaMalloc");
  }
  Desc g;
  LT_CHECK(cublasLtMatmulDescCreate(&g.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
  LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
  LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
  LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias)));
  int32_t bt = bias_type;
  LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)));
  if (aux) {
    LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux)));
    int64_t aux_ld = m;
    LT_CHECK(cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &aux_ld, sizeof(aux_ld)));
    int32_t aux_t = CUDA_R_16BF;
    LT_CHECK(
        cublasLtMatmulDescSetAttribute(g.op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_DATA_TYPE, &aux_t, sizeof(aux_t)));
  }
  const bool tA = ta == CUBLAS_OP_T, tB = tb == CUBLAS_OP_T;
  LT_CHECK(cublasLtMatrixLayoutCreate(&g.a, CUDA_R_16BF, tA ? k : m, tA ? m : k, lda));
  LT_CHECK(cublasLtMatrixLayoutCreate(&g.b, CUDA_R_16BF, tB ? n : k, tB ? k : n, ldb));
  LT_CHECK(cublasLtMatrixLayoutCreate(&g.d, d_type, m, n, m));
  auto key = std::make_tuple(kind, m, n, k, bias_type);
  auto it = s.algos.find(key);
  if (it == s.algos.end()) {
    cublasLtMatmulPreference_t pref;
    LT_CHECK(cublasLtMatmulPreferenceCreate(&pref));
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &s.ws_bytes,
                                         sizeof(s.ws_bytes));
    cublasLtMatmulHeuristicResult_t res{};
    int found = 0;
    cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(s.h, g.op, g.a, g.b, g.d, g.d, pref, 1, &res, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st != CUBLAS_STATUS_SUCCESS || found == 0)
      throw std::runtime_error("cublasLt: no algorithm for the fused epilogue (kind " + std::to_string(kind) +
                               ", m " + std::to_string(m) + ", n " + std::to_string(n) + ", k " +
                               std::to_string(k) + ", bias type " + std::to_string(bias_type) + ")");
    it = s.algos.emplace(key, res.algo).first;
  }
  const float one = 1.f, zero = 0.f;
  LT_CHECK(cublasLtMatmul(s.h, g.op, &one, A, g.a, B, g.b, C ? &one : &zero, C ? C : D, g.d, D, g.d, &it->second,
                          s.ws, s.ws_bytes, stream));
}
}  // namespace

void mlp_fc1_gelu(const void* x, const void* w1, const void* b1, void* f1, void* g, int64_t M, int64_t N, int64_t K,
                  cudaStream_t s) {
  // g^T (N x M) = W1 (K x N col-major, transposed) . x^T (K x M col-major); f1^T as the auxiliary output
  run(0, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, w1, K, x, K, g, CUBLASLT_EPILOGUE_GELU_AUX_BIAS, b1, CUDA_R_16BF, f1, s);
}

void mlp_fc2_dgelu(const void* dy, const void* w2, const void* f1, void* df1, int64_t M, int64_t N, int64_t K,
                   cudaStream_t s) {
  // df1^T (N x M) = W2^T (N x K: W2 [K, N] row-major read column-major) . dy^T (K x M), times gelu' of f1^T
  run(1, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, w2, N, dy, K, df1, CUBLASLT_EPILOGUE_DGELU, nullptr, CUDA_R_16BF,
      const_cast<void*>(f1), s);
}

void mlp_fc2_residual(const void* g, const void* w2, const void* b2, const void* x2, void* y, int64_t M, int64_t N,
                      int64_t K, cudaStream_t s) {
  // y^T (N x M) = W2 (K x N col-major, transposed) . g^T (K x M) + b2 + x2^T
  run(2, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, w2, K, g, K, y, CUBLASLT_EPILOGUE_BIAS, b2, CUDA_R_16BF, nullptr, s, x2);
}

void linear_wgrad_bgrad(const void* dy, const void* x, float* dw, float* db, int64_t M, int64_t N, int64_t K,
                        cudaStream_t s) {
  // dW (row-major [N, K], fp32) = dy^T . x, and db [N] (fp32) = the column sums
  // of dy in the same GEMM: column-major dW^T (K x N) = x^T (K x M, x read
  // column-major) . dy (M x N read as dy^T, transposed); BGRADB sums the B
  // operand (dy) over the reduction dimension M
  run(3, CUBLAS_OP_N, CUBLAS_OP_T, K, N, M, x, K, dy, N, dw, CUBLASLT_EPILOGUE_BGRADB, db, CUDA_R_32F, nullptr, s,
      nullptr, CUDA_R_32F);
}

}  // namespace krt
