// gridlp_setup.cu — one-off device preprocessing (C ABI, include/gridlp_b200.h):
// block extraction of the permuted matrix, explicit transpose, and the
// SELL-32 warp-window layout of the product kernel. Replaces the host-side
// permute_problem / distribute / slice_block / transpose of the reference
// (partition.py:262-319, sparse_kernels.py:27-58), whose from_coo lexsort is
// the setup hot spot (10.5 s at 20M nnz). Sorting uses CUB (header library);
// every output is deterministic: counts come from exact histograms and every
// sort key is unique inside its segment.
#include "../../include/gridlp_b200.h"

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>

#include <string>

namespace {

}  // namespace
extern "C" void gridlp_internal_set_error(const char* msg);  // gridlp_b200.cu
namespace {

int sfail(int code, const std::string& m) {
  gridlp_internal_set_error(m.c_str());
  return code;
}

int cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return sfail(GRIDLP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GRIDLP_OK;
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Workspace carve-out: [keys int32 x items][vals f64 x items][aux int32 x (segs+1)]
// [aux2 int32 x (segs+1)][cub temp].
struct Ws {
  int32_t* keys;
  double* vals;
  int32_t* aux;
  int32_t* aux2;
  void* cub;
  size_t cub_bytes;
};

size_t cub_bytes_needed(int64_t items, int64_t segs) {
  size_t a = 0, b = 0, c = 0, d = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)(segs + 1));
  cub::DeviceSegmentedSort::SortPairs(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                      (const double*)nullptr, (double*)nullptr, (int)items, (int)segs,
                                      (const int32_t*)nullptr, (const int32_t*)nullptr);
  cub::DeviceSelect::Flagged(nullptr, c, (const int32_t*)nullptr, (const char*)nullptr, (int32_t*)nullptr,
                             (int64_t*)nullptr, (int)segs);
  cub::DeviceScan::ExclusiveSum(nullptr, d, (int64_t*)nullptr, (int64_t*)nullptr, (int)(segs + 1));
  size_t m = a > b ? a : b;
  m = m > c ? m : c;
  return m > d ? m : d;
}

size_t ws_total(int64_t items, int64_t segs) {
  return align_up(4 * (size_t)items) + align_up(8 * (size_t)items) + 2 * align_up(4 * (size_t)(segs + 1)) +
         align_up(cub_bytes_needed(items, segs));
}

Ws carve(void* base, int64_t items, int64_t segs) {
  char* p = static_cast<char*>(base);
  Ws w;
  w.keys = reinterpret_cast<int32_t*>(p);
  p += align_up(4 * (size_t)items);
  w.vals = reinterpret_cast<double*>(p);
  p += align_up(8 * (size_t)items);
  w.aux = reinterpret_cast<int32_t*>(p);
  p += align_up(4 * (size_t)(segs + 1));
  w.aux2 = reinterpret_cast<int32_t*>(p);
  p += align_up(4 * (size_t)(segs + 1));
  w.cub = p;
  w.cub_bytes = align_up(cub_bytes_needed(items, segs));
  return w;
}

// ----------------------------------------------------------------- kernels
// One warp per permuted band row: count the source row's entries whose
// relabelled column falls in [c0, c1).
__global__ void count_kernel(const int64_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                             const int64_t* __restrict__ rows, int64_t nrows, const int32_t* __restrict__ inv_col,
                             int32_t c0, int32_t c1, int32_t* __restrict__ cnt) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w > nrows) return;
  if (w == nrows) {
    if (lane == 0) cnt[nrows] = 0;
    return;
  }
  const int64_t src = rows[w];
  const int64_t a = sptr[src], b = sptr[src + 1];
  int c = 0;
  for (int64_t k = a + lane; k < b; k += 32) {
    const int32_t nc = inv_col[scol[k]];
    c += (nc >= c0 && nc < c1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[w] = c;
}

// One warp per band row: write (local column, value) of the in-band entries
// at out_ptr[row] in source order (sorted afterwards).
__global__ void fill_kernel(const int64_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                            const double* __restrict__ sval, const int64_t* __restrict__ rows, int64_t nrows,
                            const int32_t* __restrict__ inv_col, int32_t c0, int32_t c1,
                            const int32_t* __restrict__ out_ptr, int32_t* __restrict__ keys,
                            double* __restrict__ vals) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int64_t src = rows[w];
  const int64_t a = sptr[src], b = sptr[src + 1];
  int32_t pos = out_ptr[w];
  for (int64_t base = a; base < b; base += 32) {
    const int64_t k = base + lane;
    int32_t nc = -1;
    if (k < b) nc = inv_col[scol[k]];
    const bool in = k < b && nc >= c0 && nc < c1;
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (in) {
      const int off = __popc(m & ((1u << lane) - 1u));
      keys[pos + off] = nc - c0;
      vals[pos + off] = sval[k];
    }
    pos += __popc(m);
  }
}

__global__ void col_hist_kernel(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ cnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[col[k]], 1);
}

// One warp per row: scatter the row's entries into their column buckets
// (slot order inside a bucket is arbitrary; the per-column sort fixes it).
__global__ void transpose_scatter_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                         const double* __restrict__ val, int64_t nrows,
                                         const int32_t* __restrict__ t_ptr, int32_t* __restrict__ fill,
                                         int32_t* __restrict__ keys, double* __restrict__ vals) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  for (int32_t k = ptr[w] + lane; k < ptr[w + 1]; k += 32) {
    const int32_t c = col[k];
    const int32_t p = t_ptr[c] + atomicAdd(&fill[c], 1);
    keys[p] = (int32_t)w;
    vals[p] = val[k];
  }
}

// Row gather + column relabel (internal length-sorted order):
// out row r = in row order[r] with every column index c replaced by
// label[c]; the entries keep their order, so every row sum is unchanged.
__global__ void permute_len_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ order, int64_t nrows,
                                   int32_t* __restrict__ lens) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= nrows; r += (int64_t)gridDim.x * blockDim.x) {
    if (r == nrows) { lens[r] = 0; continue; }
    const int32_t src = order ? order[r] : (int32_t)r;
    lens[r] = ptr[src + 1] - ptr[src];
  }
}

__global__ void permute_fill_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, const int32_t* __restrict__ order,
                                    const int32_t* __restrict__ label, int64_t nrows,
                                    const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_col,
                                    double* __restrict__ out_val) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int32_t src = order ? order[w] : (int32_t)w;
  const int32_t a = ptr[src], n = ptr[src + 1] - a, d = out_ptr[w];
  for (int32_t k = lane; k < n; k += 32) {
    const int32_t c = col[a + k];
    out_col[d + k] = label ? label[c] : c;
    out_val[d + k] = val[a + k];
  }
}

// SELL-32 plan: one warp per 32-row window, lane = row & 31; long rows (length >
// light_row_max) and rows past the end take the last lanes as empty (-1).
__global__ void sell_plan_kernel(const int32_t* __restrict__ ptr, int64_t nrows, int32_t light_row_max,
                                 int32_t* __restrict__ lane_info, int64_t* __restrict__ slice_elems,
                                 int32_t* __restrict__ rank_of, char* __restrict__ long_flag,
                                 int32_t* __restrict__ long_len, int64_t nslices) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nslices) return;
  const int64_t row = s * 32 + lane;
  int len = 0, eff = -2;
  if (row < nrows) {
    len = ptr[row + 1] - ptr[row];
    eff = len <= light_row_max ? len : -1;
    long_flag[row] = len > light_row_max;
    long_len[row] = len > light_row_max ? len : 0;
  }
  // lane = row & 31: the engine's internal length-class order already puts
  // rows of nearly equal length in a slice, so each lane keeps its own row
  // and its sum needs no reshuffle before the epilogue
  int mx = eff > 0 ? eff : 0;
  for (int o = 16; o > 0; o >>= 1) {
    const int e = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = e > mx ? e : mx;
  }
  lane_info[s * 32 + lane] = eff >= 0 ? ((eff << 8) | lane) : -1;
  if (row < nrows) rank_of[row] = lane;
  if (lane == 0) slice_elems[s] = 32 * (int64_t)mx;   // int64: padded entries may pass 2^31
}

__global__ void iota_kernel(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

__global__ void gather_len_kernel(const int32_t* __restrict__ long_rows, const int64_t* __restrict__ count,
                                  const int32_t* __restrict__ ptr, int32_t* __restrict__ hlen) {
  const int64_t n = *count;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    hlen[i] = i < n ? ptr[long_rows[i] + 1] - ptr[long_rows[i]] : 0;
}

__global__ void sizes_kernel(const int64_t* __restrict__ slice_off, int64_t nslices, const int64_t* __restrict__ nh,
                             const int32_t* __restrict__ long_ptr, int64_t* __restrict__ sizes) {
  sizes[0] = slice_off[nslices];
  sizes[1] = *nh;
  sizes[2] = long_ptr[*nh];
}

// SELL fill: one thread per light row writes its entries column-major.
__global__ void sell_fill_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, int64_t nrows, int32_t light_row_max,
                                 const int64_t* __restrict__ slice_off, const int32_t* __restrict__ rank_of,
                                 int32_t* __restrict__ sell_col, double* __restrict__ sell_val) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  const int32_t a = ptr[row], b = ptr[row + 1];
  if (b - a > light_row_max) return;
  const int64_t base = slice_off[row >> 5] + rank_of[row];
  for (int32_t k = a; k < b; ++k) {
    sell_col[base + 32 * (int64_t)(k - a)] = col[k];
    sell_val[base + 32 * (int64_t)(k - a)] = val[k];
  }
}

__global__ void long_fill_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, const int32_t* __restrict__ long_rows,
                                  const int32_t* __restrict__ long_ptr, int64_t nh, int32_t* __restrict__ hcol,
                                  double* __restrict__ hval) {
  for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const int32_t row = long_rows[h];
    const int32_t a = ptr[row], n = ptr[row + 1] - a, d = long_ptr[h];
    for (int32_t j = threadIdx.x; j < n; j += blockDim.x) {
      hcol[d + j] = col[a + j];
      hval[d + j] = val[a + j];
    }
  }
}

unsigned warps_grid(int64_t warps) { return (unsigned)((warps * 32 + 255) / 256); }

}  // namespace

extern "C" {

size_t gridlp_setup_workspace_bytes(int64_t max_items, int64_t max_segments) {
  return ws_total(max_items < 1 ? 1 : max_items, max_segments < 1 ? 1 : max_segments);
}

int gridlp_block_count(const int64_t* src_ptr, const int32_t* src_col, const int64_t* band_rows, int64_t nrows,
                       const int32_t* inv_col, int32_t c0, int32_t c1, int32_t* out_ptr, void* ws,
                       size_t ws_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrows < 0 || !out_ptr || (nrows > 0 && (!src_ptr || !band_rows || !inv_col)))
    return sfail(GRIDLP_ERR_ARG, "block_count: bad argument");
  if (ws_bytes < ws_total(1, nrows)) return sfail(GRIDLP_ERR_WORKSPACE, "block_count: workspace too small");
  Ws w = carve(ws, 1, nrows);
  count_kernel<<<warps_grid(nrows + 1), 256, 0, s>>>(src_ptr, src_col, band_rows, nrows, inv_col, c0, c1, w.aux);
  int rc = cuda_ok(cudaGetLastError(), "block_count");
  if (rc) return rc;
  size_t tb = w.cub_bytes;
  return cuda_ok(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.aux, out_ptr, (int)(nrows + 1), s), "block_count scan");
}

int gridlp_block_fill(const int64_t* src_ptr, const int32_t* src_col, const double* src_val,
                      const int64_t* band_rows, int64_t nrows, const int32_t* inv_col, int32_t c0, int32_t c1,
                      const int32_t* out_ptr, int64_t nnz, int32_t* out_col, double* out_val, void* ws,
                      size_t ws_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrows < 0 || nnz < 0 || (nnz > 0 && (!out_col || !out_val)))
    return sfail(GRIDLP_ERR_ARG, "block_fill: bad argument");
  if (ws_bytes < ws_total(nnz, nrows)) return sfail(GRIDLP_ERR_WORKSPACE, "block_fill: workspace too small");
  if (nnz == 0 || nrows == 0) return GRIDLP_OK;
  Ws w = carve(ws, nnz, nrows);
  fill_kernel<<<warps_grid(nrows), 256, 0, s>>>(src_ptr, src_col, src_val, band_rows, nrows, inv_col, c0, c1,
                                                out_ptr, w.keys, w.vals);
  int rc = cuda_ok(cudaGetLastError(), "block_fill");
  if (rc) return rc;
  size_t tb = w.cub_bytes;
  return cuda_ok(cub::DeviceSegmentedSort::SortPairs(w.cub, tb, w.keys, out_col, w.vals, out_val, (int)nnz,
                                                     (int)nrows, out_ptr, out_ptr + 1, s),
                 "block_fill sort");
}

int gridlp_csr_transpose(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows, int64_t ncols,
                         int64_t nnz, int32_t* t_ptr, int32_t* t_col, double* t_val, void* ws, size_t ws_bytes,
                         void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrows < 0 || ncols < 0 || nnz < 0 || !t_ptr) return sfail(GRIDLP_ERR_ARG, "csr_transpose: bad argument");
  if (ws_bytes < ws_total(nnz, ncols)) return sfail(GRIDLP_ERR_WORKSPACE, "csr_transpose: workspace too small");
  Ws w = carve(ws, nnz < 1 ? 1 : nnz, ncols);
  int rc = cuda_ok(cudaMemsetAsync(w.aux, 0, 4 * (size_t)(ncols + 1), s), "csr_transpose memset");
  if (rc) return rc;
  if (nnz > 0) {
    col_hist_kernel<<<1184, 256, 0, s>>>(col, nnz, w.aux);
    if ((rc = cuda_ok(cudaGetLastError(), "csr_transpose hist"))) return rc;
  }
  size_t tb = w.cub_bytes;
  if ((rc = cuda_ok(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.aux, t_ptr, (int)(ncols + 1), s), "transpose scan")))
    return rc;
  if (nnz == 0) return GRIDLP_OK;
  if ((rc = cuda_ok(cudaMemsetAsync(w.aux2, 0, 4 * (size_t)(ncols + 1), s), "csr_transpose memset2"))) return rc;
  transpose_scatter_kernel<<<warps_grid(nrows), 256, 0, s>>>(ptr, col, val, nrows, t_ptr, w.aux2, w.keys, w.vals);
  if ((rc = cuda_ok(cudaGetLastError(), "csr_transpose scatter"))) return rc;
  tb = w.cub_bytes;
  return cuda_ok(cub::DeviceSegmentedSort::SortPairs(w.cub, tb, w.keys, t_col, w.vals, t_val, (int)nnz, (int)ncols,
                                                     t_ptr, t_ptr + 1, s),
                 "csr_transpose sort");
}

int gridlp_col_counts(const int32_t* col, int64_t nnz, int64_t ncols, int32_t* counts, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nnz < 0 || ncols < 0 || (ncols > 0 && !counts) || (nnz > 0 && !col))
    return sfail(GRIDLP_ERR_ARG, "col_counts: bad argument");
  int rc = cuda_ok(cudaMemsetAsync(counts, 0, 4 * (size_t)ncols, s), "col_counts memset");
  if (rc || nnz == 0) return rc;
  col_hist_kernel<<<1184, 256, 0, s>>>(col, nnz, counts);
  return cuda_ok(cudaGetLastError(), "col_counts");
}

int gridlp_csr_permute(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows,
                       const int32_t* row_order, const int32_t* col_label, int32_t* out_ptr, int32_t* out_col,
                       double* out_val, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrows < 0 || !out_ptr || (nrows > 0 && !ptr)) return sfail(GRIDLP_ERR_ARG, "csr_permute: bad argument");
  if (ws_bytes < ws_total(1, nrows)) return sfail(GRIDLP_ERR_WORKSPACE, "csr_permute: workspace too small");
  Ws w = carve(ws, 1, nrows);
  permute_len_kernel<<<warps_grid((nrows + 32) / 32 + 1), 256, 0, s>>>(ptr, row_order, nrows, w.aux);
  int rc = cuda_ok(cudaGetLastError(), "csr_permute lens");
  if (rc) return rc;
  size_t tb = w.cub_bytes;
  if ((rc = cuda_ok(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.aux, out_ptr, (int)(nrows + 1), s), "permute scan")))
    return rc;
  if (nrows == 0) return GRIDLP_OK;
  permute_fill_kernel<<<warps_grid(nrows), 256, 0, s>>>(ptr, col, val, row_order, col_label, nrows, out_ptr, out_col,
                                                       out_val);
  return cuda_ok(cudaGetLastError(), "csr_permute fill");
}

int gridlp_sell_plan(const int32_t* ptr, int64_t nrows, int32_t light_row_max, int32_t* lane_info,
                     int64_t* slice_off, int32_t* rank_of, int32_t* long_rows, int32_t* long_ptr,
                     int64_t* sizes, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nslices = (nrows + 31) / 32;
  if (nrows < 0 || !slice_off || !sizes || (nrows > 0 && (!ptr || !lane_info || !rank_of || !long_rows || !long_ptr)))
    return sfail(GRIDLP_ERR_ARG, "sell_plan: bad argument");
  // aux: slice elements [nslices+1]; keys: long-row lengths [nrows+1]; vals: flags (char) + count
  if (ws_bytes < ws_total(nrows + 8, nrows + nslices + 2)) return sfail(GRIDLP_ERR_WORKSPACE, "sell_plan: workspace too small");
  Ws w = carve(ws, nrows + 8, nrows + nslices + 2);
  char* flags = reinterpret_cast<char*>(w.vals);
  int64_t* nsel = reinterpret_cast<int64_t*>(w.vals + (nrows + 7) / 8 + 1);
  // per-slice padded entry counts, scanned in int64 (a block's padded SELL
  // entries may pass 2^31 even when its nonzeros do not)
  int64_t* elems = reinterpret_cast<int64_t*>(w.vals + (nrows + 7) / 8 + 2);
  int32_t* hlen = w.keys;
  int32_t* ids = w.aux2;
  int rc;
  if ((rc = cuda_ok(cudaMemsetAsync(elems, 0, 8 * (size_t)(nslices + 1), s), "sell_plan memset"))) return rc;
  if (nslices > 0) {
    sell_plan_kernel<<<warps_grid(nslices), 256, 0, s>>>(ptr, nrows, light_row_max, lane_info, elems, rank_of, flags,
                                                         hlen, nslices);
    if ((rc = cuda_ok(cudaGetLastError(), "sell_plan"))) return rc;
  }
  size_t tb = w.cub_bytes;
  if ((rc = cuda_ok(cub::DeviceScan::ExclusiveSum(w.cub, tb, elems, slice_off, (int)(nslices + 1), s), "plan scan")))
    return rc;
  if ((rc = cuda_ok(cudaMemsetAsync(nsel, 0, 8, s), "sell_plan memset2"))) return rc;
  if (nrows > 0) {
    iota_kernel<<<1184, 256, 0, s>>>(ids, nrows);
    tb = w.cub_bytes;
    if ((rc = cuda_ok(cub::DeviceSelect::Flagged(w.cub, tb, ids, flags, long_rows, nsel, (int)nrows, s), "select")))
      return rc;
  }
  gather_len_kernel<<<64, 256, 0, s>>>(long_rows, nsel, ptr, hlen);
  if ((rc = cuda_ok(cudaGetLastError(), "sell_plan lens"))) return rc;
  tb = w.cub_bytes;
  // long_ptr has room for nrows + 1 entries; scan the first (#long + 1) — bounded by nrows + 1
  if ((rc = cuda_ok(cub::DeviceScan::ExclusiveSum(w.cub, tb, hlen, long_ptr, (int)(nrows + 1), s), "long scan")))
    return rc;
  sizes_kernel<<<1, 1, 0, s>>>(slice_off, nslices, nsel, long_ptr, sizes);
  return cuda_ok(cudaGetLastError(), "sell_plan sizes");
}

int gridlp_sell_fill(const int32_t* ptr, const int32_t* col, const double* val, int64_t nrows, int32_t light_row_max,
                     const int64_t* slice_off, const int32_t* rank_of, const int32_t* long_rows,
                     const int32_t* long_ptr, int64_t num_long, int32_t* sell_col, double* sell_val,
                     int64_t sell_elems, int32_t* long_col, double* long_val, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nrows < 0 || sell_elems < 0 || (sell_elems > 0 && (!sell_col || !sell_val)))
    return sfail(GRIDLP_ERR_ARG, "sell_fill: bad argument");
  int rc;
  if (sell_elems > 0) {
    if ((rc = cuda_ok(cudaMemsetAsync(sell_col, 0, 4 * (size_t)sell_elems, s), "sell_fill memset"))) return rc;
    if ((rc = cuda_ok(cudaMemsetAsync(sell_val, 0, 8 * (size_t)sell_elems, s), "sell_fill memset"))) return rc;
  }
  if (nrows > 0) {
    sell_fill_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(ptr, col, val, nrows, light_row_max, slice_off,
                                                                    rank_of, sell_col, sell_val);
    if ((rc = cuda_ok(cudaGetLastError(), "sell_fill"))) return rc;
  }
  if (num_long > 0) {
    long_fill_kernel<<<(unsigned)(num_long < 1184 ? num_long : 1184), 256, 0, s>>>(ptr, col, val, long_rows,
                                                                                    long_ptr, num_long, long_col,
                                                                                    long_val);
    if ((rc = cuda_ok(cudaGetLastError(), "long_fill"))) return rc;
  }
  return GRIDLP_OK;
}

}  // extern "C"
