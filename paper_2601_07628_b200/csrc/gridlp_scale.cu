// gridlp_scale.cu — on-device diagonal preconditioning of the LP (north-star
// item 4): Ruiz equilibration and Pock-Chambolle scaling
// of A (cuPDLP's default preconditioner). The reference has no scaling
// (SPEC.md:64), so it is opt-in (SolverConfig.scaling) and the default path
// keeps bit parity. All reductions here are deterministic: maxima are
// order-free (atomicMax on the bit pattern of a non-negative double), sums run
// sequentially along rows of A or of its stored transpose.
#include "../../include/gridlp_b200.h"

#include <cuda_runtime.h>

#include <string>

extern "C" void gridlp_internal_set_error(const char* msg);  // gridlp_b200.cu

namespace {

int kfail(int code, const std::string& m) {
  gridlp_internal_set_error(m.c_str());
  return code;
}

int kcuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return kfail(GRIDLP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GRIDLP_OK;
}

unsigned warps_blocks(int64_t warps) {
  int64_t b = (warps * 32 + 255) / 256;
  if (b < 1) b = 1;
  return (unsigned)(b < 148 * 64 ? b : 148 * 64);
}

unsigned flat_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

// out[r] = max_k |val[k]| over row r (one warp per row; max is order-free)
__global__ void row_absmax_kernel(const int64_t* __restrict__ ptr, const double* __restrict__ val, int64_t m,
                                  double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double mx = 0.0;
    for (int64_t k = ptr[r] + lane; k < ptr[r + 1]; k += 32) mx = fmax(mx, fabs(val[k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) out[r] = mx;
  }
}

// out[r] = sum_k |val[k]|^pw over row r, sequential in entry order (pw = 1 or 2)
__global__ void row_abssum_kernel(const int64_t* __restrict__ ptr, const double* __restrict__ val, int64_t m,
                                  int pw, double* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
      const double a = fabs(val[k]);
      s = __dadd_rn(s, pw == 2 ? __dmul_rn(a, a) : a);
    }
    out[r] = s;
  }
}

// bits[c] = max over entries of column c of the bit pattern of |val|: a
// non-negative double orders like its bit pattern, so the array read back as
// doubles holds the column maxima (order-free, hence deterministic)
__global__ void col_absmax_kernel(const int32_t* __restrict__ col, const double* __restrict__ val, int64_t nnz,
                                  unsigned long long* __restrict__ bits) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    atomicMax(bits + col[k], (unsigned long long)__double_as_longlong(fabs(val[k])));
}

// step[i] = 1 / sqrt(s[i]) (1 when s[i] = 0), d[i] <- d[i] * step[i]
__global__ void update_scale_kernel(const double* __restrict__ s, int64_t n, double* __restrict__ d,
                                    double* __restrict__ step) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = s[i];
    const double f = v > 0.0 ? __ddiv_rn(1.0, __dsqrt_rn(v)) : 1.0;
    step[i] = f;
    d[i] = __dmul_rn(d[i], f);
  }
}

// val[k] <- (dr[row] * val[k]) * dc[col]
__global__ void scale_matrix_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                    double* __restrict__ val, int64_t m, const double* __restrict__ dr,
                                    const double* __restrict__ dc) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double f = dr[r];
    for (int64_t k = ptr[r] + lane; k < ptr[r + 1]; k += 32) val[k] = __dmul_rn(__dmul_rn(f, val[k]), dc[col[k]]);
  }
}

// v[i] <- v[i] * d[i] (mul) or v[i] / d[i] (div); infinities stay infinite
__global__ void scale_vector_kernel(double* __restrict__ v, const double* __restrict__ d, int64_t n, int divide) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = divide ? __ddiv_rn(v[i], d[i]) : __dmul_rn(v[i], d[i]);
}

}  // namespace

extern "C" {

int gridlp_row_absmax(const int64_t* ptr, const double* val, int64_t m, double* out, void* stream) {
  if (m < 0 || (m > 0 && (!ptr || !out))) return kfail(GRIDLP_ERR_ARG, "row_absmax: bad argument");
  if (m == 0) return GRIDLP_OK;
  row_absmax_kernel<<<warps_blocks(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, val, m, out);
  return kcuda(cudaGetLastError(), "row_absmax");
}

int gridlp_row_abssum(const int64_t* ptr, const double* val, int64_t m, int32_t power, double* out, void* stream) {
  if (m < 0 || (m > 0 && (!ptr || !out)) || (power != 1 && power != 2))
    return kfail(GRIDLP_ERR_ARG, "row_abssum: bad argument");
  if (m == 0) return GRIDLP_OK;
  row_abssum_kernel<<<flat_blocks(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, val, m, power, out);
  return kcuda(cudaGetLastError(), "row_abssum");
}

int gridlp_col_absmax(const int32_t* col, const double* val, int64_t nnz, int64_t ncols, double* out,
                      void* stream) {
  if (nnz < 0 || ncols < 0 || (ncols > 0 && !out) || (nnz > 0 && (!col || !val)))
    return kfail(GRIDLP_ERR_ARG, "col_absmax: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = kcuda(cudaMemsetAsync(out, 0, 8 * (size_t)ncols, s), "col_absmax memset");
  if (rc || nnz == 0) return rc;
  col_absmax_kernel<<<flat_blocks(nnz), 256, 0, s>>>(col, val, nnz, reinterpret_cast<unsigned long long*>(out));
  return kcuda(cudaGetLastError(), "col_absmax");
}

int gridlp_update_scale(const double* s, int64_t n, double* d, double* step, void* stream) {
  if (n < 0 || (n > 0 && (!s || !d || !step))) return kfail(GRIDLP_ERR_ARG, "update_scale: bad argument");
  if (n == 0) return GRIDLP_OK;
  update_scale_kernel<<<flat_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(s, n, d, step);
  return kcuda(cudaGetLastError(), "update_scale");
}

int gridlp_scale_matrix(const int64_t* ptr, const int32_t* col, double* val, int64_t m, const double* dr,
                        const double* dc, void* stream) {
  if (m < 0 || (m > 0 && (!ptr || !dr || !dc))) return kfail(GRIDLP_ERR_ARG, "scale_matrix: bad argument");
  if (m == 0) return GRIDLP_OK;
  scale_matrix_kernel<<<warps_blocks(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, col, val, m, dr, dc);
  return kcuda(cudaGetLastError(), "scale_matrix");
}

int gridlp_scale_vector(double* v, const double* d, int64_t n, int32_t divide, void* stream) {
  if (n < 0 || (n > 0 && (!v || !d))) return kfail(GRIDLP_ERR_ARG, "scale_vector: bad argument");
  if (n == 0) return GRIDLP_OK;
  scale_vector_kernel<<<flat_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(v, d, n, divide);
  return kcuda(cudaGetLastError(), "scale_vector");
}

}  // extern "C"
