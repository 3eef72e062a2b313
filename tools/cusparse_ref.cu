// cusparse_ref.cu — the library baseline of bench.py's SpMV leg:
// cusparseSpMV on the same FP64 CSR (int32 indices) with an explicit
// algorithm (CUSPARSE_SPMV_CSR_ALG1 / ALG2), timed with CUDA events on the
// caller's stream. Not part of the product (paper_2601_07628_b200 never
// loads it); built by __graft_entry__.build() into tools/_lib/.
#include <cuda_runtime.h>
#include <cusparse.h>

#include <algorithm>
#include <cstdint>
#include <vector>

extern "C" int cusparse_ref_spmv(int64_t m, int64_t n, int64_t nnz, const int32_t* ptr, const int32_t* col,
                                 const double* val, const double* x, double* y, int alg, int reps,
                                 float* median_ms, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cusparseHandle_t h = nullptr;
  if (cusparseCreate(&h) != CUSPARSE_STATUS_SUCCESS) return 1;
  cusparseSetStream(h, s);
  cusparseSpMatDescr_t A = nullptr;
  cusparseDnVecDescr_t vx = nullptr, vy = nullptr;
  int rc = 0;
  void* buf = nullptr;
  size_t bytes = 0;
  const double one = 1.0, zero = 0.0;
  const cusparseSpMVAlg_t a = alg == 2 ? CUSPARSE_SPMV_CSR_ALG2 : CUSPARSE_SPMV_CSR_ALG1;
  std::vector<float> t;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (cusparseCreateCsr(&A, m, n, nnz, (void*)ptr, (void*)col, (void*)val, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                        CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS ||
      cusparseCreateDnVec(&vx, n, (void*)x, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS ||
      cusparseCreateDnVec(&vy, m, (void*)y, CUDA_R_64F) != CUSPARSE_STATUS_SUCCESS) {
    rc = 2;
    goto done;
  }
  if (cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, vx, &zero, vy, CUDA_R_64F, a, &bytes) !=
      CUSPARSE_STATUS_SUCCESS) {
    rc = 3;
    goto done;
  }
  if (bytes && cudaMalloc(&buf, bytes) != cudaSuccess) {
    rc = 4;
    goto done;
  }
  // warm-up (also any one-off analysis of the algorithm)
  if (cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, vx, &zero, vy, CUDA_R_64F, a, buf) !=
      CUSPARSE_STATUS_SUCCESS) {
    rc = 5;
    goto done;
  }
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, s);
    cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, vx, &zero, vy, CUDA_R_64F, a, buf);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  *median_ms = t.empty() ? 0.f : t[t.size() / 2];
done:
  if (buf) cudaFree(buf);
  if (vx) cusparseDestroyDnVec(vx);
  if (vy) cusparseDestroyDnVec(vy);
  if (A) cusparseDestroySpMat(A);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cusparseDestroy(h);
  return rc;
}
