// gridlp_gen.cu — device generators for the large synthetic LPs of
// BASELINE.json (cfg3 power-law, cfg4 block-angular multi-commodity flow),
// which have no counterpart in the reference's generators.py (SURVEY §8f
// rank 2). Every random quantity is a pure function of (seed, stream,
// global index) — a counter-based hash — so an instance does not depend on
// the grid, the launch shape or the device, and the numpy restatement in
// oracle/synth_oracle.py reproduces it bit for bit at small sizes. All
// floating-point steps are explicit IEEE round-to-nearest operations in the
// same order as the numpy code (no FMA contraction, no libm calls).
#include "../../include/gridlp_b200.h"

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cuda_runtime.h>

#include <string>

extern "C" void gridlp_internal_set_error(const char* msg);  // gridlp_b200.cu

namespace {

int gfail(int code, const std::string& m) {
  gridlp_internal_set_error(m.c_str());
  return code;
}

int gcuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return gfail(GRIDLP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GRIDLP_OK;
}

// splitmix64 finaliser
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// hash(seed, stream, a, b) = mix(mix(mix(seed * 0x100000001B3 + stream) ^ a) ^ b)
__device__ __forceinline__ uint64_t ghash(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed * 0x100000001B3ull + stream) ^ a) ^ b);
}

// uniform in [0, 1) with 53 random bits (exact dyadic)
__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

// ------------------------------------------------------------------ kernels
// Column samples of the power-law rows: entry k of row r draws
// a = 1 + u * kappa, t = a^5 (left-to-right products), c = floor(t) - 1,
// clamped to [0, n) — a continuous power law of exponent 0.8 over columns
// 1..n+1 (kappa = (n+1)^0.2 - 1, computed on the host).
__global__ void powerlaw_sample_kernel(uint64_t seed, const int64_t* __restrict__ alloc_ptr, int64_t m, int64_t n,
                                       double kappa, int32_t* __restrict__ cols) {
  const int64_t total = alloc_ptr[m];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    // row of entry e: binary search in alloc_ptr
    int64_t lo = 0, hi = m;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (alloc_ptr[mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t r = lo, k = e - alloc_ptr[r];
    const double u = u01(ghash(seed, 1, (uint64_t)r, (uint64_t)k));
    const double a = __dadd_rn(1.0, __dmul_rn(u, kappa));
    const double t = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(a, a), a), a), a);
    int64_t c = (int64_t)floor(t) - 1;
    c = c < 0 ? 0 : (c >= n ? n - 1 : c);
    cols[e] = (int32_t)c;
  }
}

// Uniform column samples: entry k of row r draws c = floor(u(seed,1,r,k) * n).
__global__ void uniform_sample_kernel(uint64_t seed, const int64_t* __restrict__ alloc_ptr, int64_t m, int64_t n,
                                      int32_t* __restrict__ cols) {
  const int64_t total = alloc_ptr[m];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (alloc_ptr[mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t c = (int64_t)floor(__dmul_rn(u01(ghash(seed, 1, (uint64_t)lo, (uint64_t)(e - alloc_ptr[lo]))),
                                               (double)n));
    cols[e] = (int32_t)(c < n ? c : n - 1);
  }
}

// Planted optimum, per column j: state u(seed,20,j) < 0.3 -> at the lower
// bound (x* = lo, r* = 0.1 + 0.9 u(seed,21,j)), < 0.4 -> at the upper bound
// (x* = hi, r* = -(0.1 + 0.9 u21)), else interior (x* = lo + (hi - lo)(0.1 +
// 0.8 u(seed,22,j)), r* = 0).
__device__ __forceinline__ void planted_col(uint64_t seed, int64_t j, double lo, double hi, double& x, double& r) {
  const double st = u01(ghash(seed, 20, (uint64_t)j, 0));
  const double w = __dadd_rn(0.1, __dmul_rn(0.9, u01(ghash(seed, 21, (uint64_t)j, 0))));
  if (st < 0.3) { x = lo; r = w; }
  else if (st < 0.4) { x = hi; r = -w; }
  else {
    x = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), __dadd_rn(0.1, __dmul_rn(0.8, u01(ghash(seed, 22, (uint64_t)j, 0))))));
    r = 0.0;
  }
}

// planted dual of row i (state u(seed,23,i): < 0.35 -> 0.5 + u24, < 0.7 -> -(0.5 + u24), else 0)
__device__ __forceinline__ double planted_y(uint64_t seed, int64_t i) {
  const double st = u01(ghash(seed, 23, (uint64_t)i, 0));
  const double yv = __dadd_rn(0.5, u01(ghash(seed, 24, (uint64_t)i, 0)));
  return st < 0.35 ? yv : (st < 0.7 ? -yv : 0.0);
}

// value of matrix entry (r, c): 2 u(seed, 2, r, c) - 1
__device__ __forceinline__ double entry_value(uint64_t seed, int64_t r, int64_t c) {
  return __dsub_rn(__dmul_rn(2.0, u01(ghash(seed, 2, (uint64_t)r, (uint64_t)c))), 1.0);
}

__global__ void planted_cols_kernel(uint64_t seed, int64_t j0, int64_t n, double lo, double hi,
                                    double* __restrict__ x, double* __restrict__ r) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    planted_col(seed, j0 + j, lo, hi, x[j], r[j]);
}

// Planted duals and row bounds around b = A x*: state u(seed,23,i) < 0.35 ->
// lower bound active (y* = 0.5 + u(seed,24,i), lo = b, hi = b + 0.1 + 0.9
// u(seed,25,i)); < 0.7 -> upper active (y* = -(0.5 + u24), hi = b, lo = b -
// (0.1 + 0.9 u25)); else inactive (y* = 0, lo = b - (0.1 + 0.9 u25), hi = b +
// (0.1 + 0.9 u(seed,26,i))).
__global__ void planted_rows_kernel(uint64_t seed, int64_t i0, int64_t m, const double* __restrict__ b,
                                    double* __restrict__ y, double* __restrict__ lo, double* __restrict__ hi) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + q;
    const double st = u01(ghash(seed, 23, (uint64_t)i, 0));
    const double yv = __dadd_rn(0.5, u01(ghash(seed, 24, (uint64_t)i, 0)));
    const double w = __dadd_rn(0.1, __dmul_rn(0.9, u01(ghash(seed, 25, (uint64_t)i, 0))));
    const double bi = b[q];
    if (st < 0.35) { y[q] = yv; lo[q] = bi; hi[q] = __dadd_rn(bi, w); }
    else if (st < 0.7) { y[q] = -yv; hi[q] = bi; lo[q] = __dsub_rn(bi, w); }
    else {
      const double w2 = __dadd_rn(0.1, __dmul_rn(0.9, u01(ghash(seed, 26, (uint64_t)i, 0))));
      y[q] = 0.0; lo[q] = __dsub_rn(bi, w); hi[q] = __dadd_rn(bi, w2);
    }
  }
}

// c = aty + r (the planted reduced cost makes (x*, y*) a KKT point)
__global__ void add_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(a[i], b[i]);
}

// distinct columns of each sorted row that fall in [c0, c1)
__global__ void dedupe_count_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ sorted, int64_t m,
                                    int32_t c0, int32_t c1, int64_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ptr[r], b = ptr[r + 1];
    int64_t cnt = 0;
    for (int64_t k = a; k < b; ++k) {
      const int32_t c = sorted[k];
      cnt += (k == a || c != sorted[k - 1]) && c >= c0 && c < c1;
    }
    counts[r] = cnt;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[m] = 0;
}

// compact them with local column ids c - c0; value of global entry (r0 + r, c)
// is 2 u(seed, 2, r0 + r, c) - 1
__global__ void dedupe_fill_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ sorted, int64_t m,
                                   int64_t r0, int32_t c0, int32_t c1, const int64_t* __restrict__ out_ptr,
                                   uint64_t seed, int32_t* __restrict__ out_cols, double* __restrict__ out_vals) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ptr[r], b = ptr[r + 1];
    int64_t o = out_ptr[r];
    for (int64_t k = a; k < b; ++k) {
      const int32_t c = sorted[k];
      if ((k != a && c == sorted[k - 1]) || c < c0 || c >= c1) continue;
      out_cols[o] = c - c0;
      out_vals[o] = entry_value(seed, r0 + r, c);
      ++o;
    }
  }
}

// constant-count draws of rows r0 .. r0+m-1: entry k of row r is
// floor(u(seed,1,r,k) * n) (the uniform sampler of cfg5, row-major, d per row)
__global__ void band_draws_kernel(uint64_t seed, int64_t r0, int64_t m, int32_t d, int64_t n,
                                  int32_t* __restrict__ cols) {
  const int64_t total = m * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / d, k = e - q * d;
    const int64_t c = (int64_t)floor(__dmul_rn(u01(ghash(seed, 1, (uint64_t)(r0 + q), (uint64_t)k)), (double)n));
    cols[e] = (int32_t)(c < n ? c : n - 1);
  }
}

// b[q] = sum over the distinct columns c of sorted full row r0+q, in column
// order from +0.0, of value(r0+q, c) * x*(c)  (the one-piece A x*)
__global__ void planted_row_dot_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ sorted, int64_t m,
                                       int64_t r0, uint64_t seed, double lo, double hi, double* __restrict__ b) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = ptr[q]; k < ptr[q + 1]; ++k) {
      const int32_t c = sorted[k];
      if (k != ptr[q] && c == sorted[k - 1]) continue;
      double x, r;
      planted_col(seed, c, lo, hi, x, r);
      s = __dadd_rn(s, __dmul_rn(entry_value(seed, r0 + q, c), x));
    }
    b[q] = s;
  }
}

// acc[c] continues the sequential column sum of value * y* with the entries
// of one row chunk, rows ascending (tptr/trows/tvals: the chunk's band block
// transposed; rows local to the chunk starting at global row r0)
__global__ void col_accumulate_kernel(const int32_t* __restrict__ tptr, const int32_t* __restrict__ trows,
                                      const double* __restrict__ tvals, int64_t ncols, int64_t r0, uint64_t seed,
                                      double* __restrict__ acc) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x) {
    double s = acc[c];
    for (int32_t k = tptr[c]; k < tptr[c + 1]; ++k) s = __dadd_rn(s, __dmul_rn(tvals[k], planted_y(seed, r0 + trows[k])));
    acc[c] = s;
  }
}

// out_i = lo + (hi - lo) * u(seed, stream, i0 + i, 0)
__global__ void uniform_kernel(uint64_t seed, uint64_t stream, int64_t i0, int64_t n, double lo, double hi,
                               double* __restrict__ out) {
  const double w = __dsub_rn(hi, lo);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(lo, __dmul_rn(w, u01(ghash(seed, stream, (uint64_t)(i0 + i), 0))));
}

// y_r = sequential sum of the row's products from +0.0 (scipy csr_matvec order)
__global__ void csr_spmv_seq_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ cols,
                                    const double* __restrict__ vals, int64_t m, const double* __restrict__ x,
                                    double* __restrict__ y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) s = __dadd_rn(s, __dmul_rn(vals[k], x[cols[k]]));
    y[r] = s;
  }
}

// Feasible wrapper of the generated rows (generators.py:120-142 pattern):
// a row is ranged with probability `ineq` (u(seed, 5, r) < ineq) and then
// widened by U[0.1, 1) on each side (streams 6, 7); otherwise lo = hi = b.
__global__ void row_bounds_kernel(uint64_t seed, int64_t m, double ineq, const double* __restrict__ b,
                                  double* __restrict__ lo, double* __restrict__ hi) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const double br = b[r];
    if (u01(ghash(seed, 5, (uint64_t)r, 0)) < ineq) {
      const double wl = __dadd_rn(0.1, __dmul_rn(0.9, u01(ghash(seed, 6, (uint64_t)r, 0))));
      const double wh = __dadd_rn(0.1, __dmul_rn(0.9, u01(ghash(seed, 7, (uint64_t)r, 0))));
      lo[r] = __dsub_rn(br, wl);
      hi[r] = __dadd_rn(br, wh);
    } else {
      lo[r] = br;
      hi[r] = br;
    }
  }
}

// Multi-commodity flow rows. Conservation row (k, v), k < K, v < V:
// columns k*E + e for the arcs e incident to v (node adjacency, ascending e),
// +1 for an out-arc, -1 for an in-arc. Coupling row K*V + e: columns k*E + e
// for k = 0..K-1, all +1.
__global__ void mcf_fill_kernel(int64_t K, int64_t V, int64_t E, const int32_t* __restrict__ adj_ptr,
                                const int32_t* __restrict__ adj_arc, const int8_t* __restrict__ adj_sign,
                                const int64_t* __restrict__ row_ptr, int32_t* __restrict__ cols,
                                double* __restrict__ vals) {
  const int64_t m = K * V + E;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = row_ptr[r];
    if (r < K * V) {
      const int64_t k = r / V, v = r - k * V;
      for (int32_t q = adj_ptr[v]; q < adj_ptr[v + 1]; ++q, ++o) {
        cols[o] = (int32_t)(k * E + adj_arc[q]);
        vals[o] = (double)adj_sign[q];
      }
    } else {
      const int64_t e = r - K * V;
      for (int64_t k = 0; k < K; ++k, ++o) {
        cols[o] = (int32_t)(k * E + e);
        vals[o] = 1.0;
      }
    }
  }
}

__global__ void mcf_row_ptr_kernel(int64_t K, int64_t V, int64_t E, const int32_t* __restrict__ adj_ptr,
                                   int64_t* __restrict__ lens) {
  const int64_t m = K * V + E;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= m; r += (int64_t)gridDim.x * blockDim.x) {
    if (r == m) lens[r] = 0;
    else if (r < K * V) { const int64_t v = r % V; lens[r] = adj_ptr[v + 1] - adj_ptr[v]; }
    else lens[r] = K;
  }
}

}  // namespace

extern "C" {

size_t gridlp_gen_workspace_bytes(int64_t max_items, int64_t max_rows) {
  size_t a = 0, b = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, a, (const int32_t*)nullptr, (int32_t*)nullptr,
                                     (int)(max_items < 1 ? 1 : max_items), (int)(max_rows < 1 ? 1 : max_rows),
                                     (const int64_t*)nullptr, (const int64_t*)nullptr);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(max_rows + 1 < 2 ? 2 : max_rows + 1));
  return (a > b ? a : b) + 256;
}

int gridlp_gen_scan64(const int64_t* in, int64_t* out, int64_t n, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1 || !in || !out || n >= (int64_t(1) << 31)) return gfail(GRIDLP_ERR_ARG, "gen_scan64: bad argument");
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int)n);
  if (ws_bytes < need) return gfail(GRIDLP_ERR_WORKSPACE, "gen_scan64: workspace too small");
  return gcuda(cub::DeviceScan::ExclusiveSum(ws, ws_bytes, in, out, (int)n, static_cast<cudaStream_t>(stream)),
               "gen_scan64");
}

int gridlp_gen_powerlaw_sample(uint64_t seed, const int64_t* alloc_ptr, int64_t m, int64_t n, double kappa,
                               int32_t* cols, void* stream) {
  if (m < 0 || n < 1 || n >= (int64_t(1) << 31) || !alloc_ptr || (m > 0 && !cols))
    return gfail(GRIDLP_ERR_ARG, "gen_powerlaw_sample: bad argument");
  if (m == 0) return GRIDLP_OK;
  powerlaw_sample_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, alloc_ptr, m, n, kappa, cols);
  return gcuda(cudaGetLastError(), "gen_powerlaw_sample");
}

int gridlp_gen_uniform_sample(uint64_t seed, const int64_t* alloc_ptr, int64_t m, int64_t n, int32_t* cols,
                              void* stream) {
  if (m < 0 || n < 1 || n >= (int64_t(1) << 31) || !alloc_ptr || (m > 0 && !cols))
    return gfail(GRIDLP_ERR_ARG, "gen_uniform_sample: bad argument");
  if (m == 0) return GRIDLP_OK;
  uniform_sample_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, alloc_ptr, m, n, cols);
  return gcuda(cudaGetLastError(), "gen_uniform_sample");
}

int gridlp_gen_planted_cols(uint64_t seed, int64_t j0, int64_t n, double lo, double hi, double* x, double* r,
                            void* stream) {
  if (n < 0 || j0 < 0 || (n > 0 && (!x || !r)) || !(lo < hi)) return gfail(GRIDLP_ERR_ARG, "gen_planted_cols: bad argument");
  if (n == 0) return GRIDLP_OK;
  planted_cols_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, j0, n, lo, hi, x, r);
  return gcuda(cudaGetLastError(), "gen_planted_cols");
}

int gridlp_gen_planted_rows(uint64_t seed, int64_t i0, int64_t m, const double* b, double* y, double* lo, double* hi,
                            void* stream) {
  if (m < 0 || i0 < 0 || (m > 0 && (!b || !y || !lo || !hi))) return gfail(GRIDLP_ERR_ARG, "gen_planted_rows: bad argument");
  if (m == 0) return GRIDLP_OK;
  planted_rows_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, i0, m, b, y, lo, hi);
  return gcuda(cudaGetLastError(), "gen_planted_rows");
}

int gridlp_gen_band_draws(uint64_t seed, int64_t r0, int64_t m, int32_t d, int64_t n, int32_t* cols, void* stream) {
  if (m < 0 || r0 < 0 || d < 1 || n < 1 || n >= (int64_t(1) << 31) || (m > 0 && !cols))
    return gfail(GRIDLP_ERR_ARG, "gen_band_draws: bad argument");
  if (m == 0) return GRIDLP_OK;
  band_draws_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, r0, m, d, n, cols);
  return gcuda(cudaGetLastError(), "gen_band_draws");
}

int gridlp_gen_planted_row_dot(const int64_t* ptr, const int32_t* sorted, int64_t m, int64_t r0, uint64_t seed,
                               double lo, double hi, double* b, void* stream) {
  if (m < 0 || r0 < 0 || (m > 0 && (!ptr || !b))) return gfail(GRIDLP_ERR_ARG, "gen_planted_row_dot: bad argument");
  if (m == 0) return GRIDLP_OK;
  planted_row_dot_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, sorted, m, r0, seed, lo, hi,
                                                                                     b);
  return gcuda(cudaGetLastError(), "gen_planted_row_dot");
}

int gridlp_gen_col_accumulate(const int32_t* tptr, const int32_t* trows, const double* tvals, int64_t ncols,
                              int64_t r0, uint64_t seed, double* acc, void* stream) {
  if (ncols < 0 || r0 < 0 || (ncols > 0 && (!tptr || !acc))) return gfail(GRIDLP_ERR_ARG, "gen_col_accumulate: bad argument");
  if (ncols == 0) return GRIDLP_OK;
  col_accumulate_kernel<<<grid_for(ncols), 256, 0, static_cast<cudaStream_t>(stream)>>>(tptr, trows, tvals, ncols, r0,
                                                                                        seed, acc);
  return gcuda(cudaGetLastError(), "gen_col_accumulate");
}

int gridlp_gen_add(const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!a || !b || !out))) return gfail(GRIDLP_ERR_ARG, "gen_add: bad argument");
  if (n == 0) return GRIDLP_OK;
  add_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(a, b, n, out);
  return gcuda(cudaGetLastError(), "gen_add");
}

int gridlp_gen_sort_rows(const int64_t* ptr, int64_t m, int64_t items, const int32_t* keys_in, int32_t* keys_out,
                         void* ws, size_t ws_bytes, void* stream) {
  if (m < 0 || items < 0 || items >= (int64_t(1) << 31) || m >= (int64_t(1) << 31) || !ptr)
    return gfail(GRIDLP_ERR_ARG, "gen_sort_rows: bad argument (items and rows must be < 2^31 per call)");
  if (items == 0 || m == 0) return GRIDLP_OK;
  size_t need = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, need, keys_in, keys_out, (int)items, (int)m, ptr, ptr + 1);
  if (ws_bytes < need) return gfail(GRIDLP_ERR_WORKSPACE, "gen_sort_rows: workspace too small");
  return gcuda(cub::DeviceSegmentedSort::SortKeys(ws, ws_bytes, keys_in, keys_out, (int)items, (int)m, ptr, ptr + 1,
                                                  static_cast<cudaStream_t>(stream)),
               "gen_sort_rows");
}

int gridlp_gen_dedupe_count(const int64_t* ptr, const int32_t* sorted, int64_t m, int32_t c0, int32_t c1,
                            int64_t* counts, void* stream) {
  if (m < 0 || !ptr || !counts || c1 < c0) return gfail(GRIDLP_ERR_ARG, "gen_dedupe_count: bad argument");
  dedupe_count_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, sorted, m, c0, c1, counts);
  return gcuda(cudaGetLastError(), "gen_dedupe_count");
}

int gridlp_gen_dedupe_fill(const int64_t* ptr, const int32_t* sorted, int64_t m, int64_t r0, int32_t c0, int32_t c1,
                           const int64_t* out_ptr, uint64_t seed, int32_t* out_cols, double* out_vals, void* stream) {
  if (m < 0 || r0 < 0 || !ptr || !out_ptr || c1 < c0) return gfail(GRIDLP_ERR_ARG, "gen_dedupe_fill: bad argument");
  if (m == 0) return GRIDLP_OK;
  dedupe_fill_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, sorted, m, r0, c0, c1, out_ptr,
                                                                                 seed, out_cols, out_vals);
  return gcuda(cudaGetLastError(), "gen_dedupe_fill");
}

int gridlp_gen_uniform(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n, double lo, double hi, double* out,
                       void* stream) {
  if (n < 0 || i0 < 0 || (n > 0 && !out)) return gfail(GRIDLP_ERR_ARG, "gen_uniform: bad argument");
  if (n == 0) return GRIDLP_OK;
  uniform_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, stream_id, i0, n, lo, hi, out);
  return gcuda(cudaGetLastError(), "gen_uniform");
}

int gridlp_csr_spmv_seq(const int64_t* ptr, const int32_t* cols, const double* vals, int64_t m, const double* x,
                        double* y, void* stream) {
  if (m < 0 || (m > 0 && (!ptr || !y))) return gfail(GRIDLP_ERR_ARG, "csr_spmv_seq: bad argument");
  if (m == 0) return GRIDLP_OK;
  csr_spmv_seq_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(ptr, cols, vals, m, x, y);
  return gcuda(cudaGetLastError(), "csr_spmv_seq");
}

int gridlp_gen_row_bounds(uint64_t seed, int64_t m, double ineq, const double* b, double* lo, double* hi,
                          void* stream) {
  if (m < 0 || (m > 0 && (!b || !lo || !hi))) return gfail(GRIDLP_ERR_ARG, "gen_row_bounds: bad argument");
  if (m == 0) return GRIDLP_OK;
  row_bounds_kernel<<<grid_for(m), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, m, ineq, b, lo, hi);
  return gcuda(cudaGetLastError(), "gen_row_bounds");
}

int gridlp_gen_mcf_row_lengths(int64_t K, int64_t V, int64_t E, const int32_t* adj_ptr, int64_t* lens,
                               void* stream) {
  if (K < 1 || V < 1 || E < 0 || !adj_ptr || !lens || K * E >= (int64_t(1) << 31))
    return gfail(GRIDLP_ERR_ARG, "gen_mcf_row_lengths: bad argument (K*E must be < 2^31)");
  mcf_row_ptr_kernel<<<grid_for(K * V + E + 1), 256, 0, static_cast<cudaStream_t>(stream)>>>(K, V, E, adj_ptr, lens);
  return gcuda(cudaGetLastError(), "gen_mcf_row_lengths");
}

int gridlp_gen_mcf_fill(int64_t K, int64_t V, int64_t E, const int32_t* adj_ptr, const int32_t* adj_arc,
                        const int8_t* adj_sign, const int64_t* row_ptr, int32_t* cols, double* vals, void* stream) {
  if (K < 1 || V < 1 || E < 0 || !adj_ptr || !row_ptr || K * E >= (int64_t(1) << 31))
    return gfail(GRIDLP_ERR_ARG, "gen_mcf_fill: bad argument");
  mcf_fill_kernel<<<grid_for(K * V + E), 256, 0, static_cast<cudaStream_t>(stream)>>>(K, V, E, adj_ptr, adj_arc,
                                                                                     adj_sign, row_ptr, cols, vals);
  return gcuda(cudaGetLastError(), "gen_mcf_fill");
}

}  // extern "C"
