// Dense GEMM peak probe on this GPU with cuBLASLt (library GEMMs, measured
// like MEASURED_PEAKS.json's bf16 figure): bf16, fp8 e4m3 (per-tensor scales)
// and NVFP4 (e2m1 with 16-element e4m3 block scales). Gives the fp8 / fp4
// roofline denominators instead of the nominal 2x / 4x of bf16.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a lt_peak.cu -lcublasLt -o lt_peak
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    auto _s = (x);                                                                 \
    if (int(_s) != 0) {                                                            \
      std::fprintf(stderr, "%s:%d: %s = %d\n", __FILE__, __LINE__, #x, int(_s)); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

static double run(cublasLtHandle_t lt, cudaDataType_t ab, int64_t M, int64_t N, int64_t K, int scale_mode) {
  const size_t esz_num = ab == CUDA_R_4F_E2M1 ? 1 : (ab == CUDA_R_16BF ? 4 : 2);  // bytes * 2
  void *A, *B, *D, *ws;
  CK(cudaMalloc(&A, size_t(M) * K * esz_num / 2));
  CK(cudaMalloc(&B, size_t(N) * K * esz_num / 2));
  CK(cudaMalloc(&D, size_t(M) * N * 2));
  const size_t wsz = 64 << 20;
  CK(cudaMalloc(&ws, wsz));
  CK(cudaMemset(A, 0x22, size_t(M) * K * esz_num / 2));
  CK(cudaMemset(B, 0x22, size_t(N) * K * esz_num / 2));
  void *sa = nullptr, *sb = nullptr;
  cublasLtMatmulDesc_t op;
  CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  cublasOperation_t T = CUBLAS_OP_T, Nn = CUBLAS_OP_N;
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &T, sizeof T));
  CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &Nn, sizeof Nn));
  if (ab != CUDA_R_16BF) {
    size_t sbytes_a = 4, sbytes_b = 4;
    if (scale_mode == CUBLASLT_MATMUL_MATRIX_SCALE_VEC16_UE4M3) {  // one e4m3 per 16 elements (padded)
      sbytes_a = size_t((M + 127) / 128 * 128) * ((K / 16 + 3) / 4 * 4);
      sbytes_b = size_t((N + 127) / 128 * 128) * ((K / 16 + 3) / 4 * 4);
      CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_A_SCALE_MODE, &scale_mode, sizeof scale_mode));
      CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_B_SCALE_MODE, &scale_mode, sizeof scale_mode));
    }
    CK(cudaMalloc(&sa, sbytes_a));
    CK(cudaMalloc(&sb, sbytes_b));
    CK(cudaMemset(sa, 0x38, sbytes_a));
    CK(cudaMemset(sb, 0x38, sbytes_b));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_A_SCALE_POINTER, &sa, sizeof sa));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_B_SCALE_POINTER, &sb, sizeof sb));
  }
  cublasLtMatrixLayout_t la, lb, ld;
  CK(cublasLtMatrixLayoutCreate(&la, ab, K, M, K));
  CK(cublasLtMatrixLayoutCreate(&lb, ab, K, N, K));
  CK(cublasLtMatrixLayoutCreate(&ld, CUDA_R_16BF, M, N, M));
  cublasLtMatmulPreference_t pref;
  CK(cublasLtMatmulPreferenceCreate(&pref));
  CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof wsz));
  cublasLtMatmulHeuristicResult_t h[8];
  int n = 0;
  CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, ld, ld, pref, 8, h, &n));
  if (n == 0) {
    std::fprintf(stderr, "no algorithm\n");
    return 0;
  }
  const float alpha = 1.0f, beta = 0.0f;
  double best = 0;
  for (int a = 0; a < n; ++a) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bool ok = true;
    for (int i = 0; i < 3 && ok; ++i)
      ok = cublasLtMatmul(lt, op, &alpha, A, la, B, lb, &beta, D, ld, D, ld, &h[a].algo, ws, wsz, 0) == 0;
    if (!ok) continue;
    const int iters = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i)
      cublasLtMatmul(lt, op, &alpha, A, la, B, lb, &beta, D, ld, D, ld, &h[a].algo, ws, wsz, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * M * N * K * iters / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
  cudaFree(ws);
  if (sa) cudaFree(sa);
  if (sb) cudaFree(sb);
  return best;
}

int main() {
  cublasLtHandle_t lt;
  CK(cublasLtCreate(&lt));
  const int64_t M = 8192, N = 8192, K = 16384;
  std::printf("{\"bf16_tflops\": %.1f, ", run(lt, CUDA_R_16BF, M, N, K, 0));
  std::printf("\"fp8_e4m3_tflops\": %.1f, ", run(lt, CUDA_R_8F_E4M3, M, N, K, 0));
  std::printf("\"nvfp4_tflops\": %.1f, \"shape\": [%lld, %lld, %lld], \"source\": \"cuBLASLt best of the heuristic's algorithms, 20 back-to-back launches, CUDA events\"}\n",
              run(lt, CUDA_R_4F_E2M1, M, N, K, CUBLASLT_MATMUL_MATRIX_SCALE_VEC16_UE4M3), (long long)M,
              (long long)N, (long long)K);
  return 0;
}
