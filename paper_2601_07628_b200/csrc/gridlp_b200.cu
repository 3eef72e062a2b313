// gridlp_b200.cu — sm_100a kernels + C ABI for the distributed-PDHG hot path.
//
// Design:
//  * Sparse products run over a tile directory of each CSR block. A light
//    tile (<= 256 rows, <= 4096 nnz) is processed by one 256-thread CTA in
//    two phases: (a) all threads stream values/column indices (coalesced,
//    L2 evict-first) and gather the dense vector (L2 evict-last), writing
//    the rounded products val*x into shared memory — this balances the
//    gathers over the CTA regardless of row lengths; (b) one thread per row
//    adds its products left to right from +0.0 and applies the fused PDHG
//    epilogue. Because each product is rounded and then added in index
//    order, the row sum is bit-identical to scipy's csr_matvec — the
//    reference's kernel (sparse_kernels.py:18-24). A heavy tile (one row
//    longer than exact_row_max) is tree-summed by the whole CTA.
//  * The epilogue's per-row vector reads (x, c, bounds, anchor) are issued
//    before phase (a) so their DRAM latency overlaps the gathers.
//  * No FMA contraction anywhere: every multiply/add/divide is an explicit
//    __d*_rn so each numpy expression of the reference is reproduced
//    operation for operation.
//  * Reductions are deterministic: fixed warp-shuffle tree per CTA, one
//    slot per CTA, then one fixed-order final pass.
#include "../../include/gridlp_b200.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

namespace {

constexpr int TPB = 256;
constexpr int WARPS = TPB / 32;
constexpr int CAP = GRIDLP_TILE_NNZ_CAP;
constexpr int UNROLL = 8;
constexpr int64_t ROWS_MAX_BLOCKS = 1184;  // 8 x 148 SMs

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GRIDLP_OK;
}

// ---------------------------------------------------------------- device math
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// numpy.maximum for float64: NaN-propagating, returns b on ties (incl. ±0).
__device__ __forceinline__ double np_maximum(double a, double b) {
  return (isnan(a) || a > b) ? a : b;
}
// numpy.clip(x, lo, hi) = _NPY_MIN(_NPY_MAX(x, lo), hi) (numpy clip.cpp).
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
  double t = isnan(x) ? x : (x > lo ? x : lo);
  return isnan(t) ? t : (t < hi ? t : hi);
}

// Halpern weights, bit-identical to the Python float expressions
// (1.0 + gamma) * (k + 1.0) / (k + 2.0) and 1.0 / (k + 2.0)
// (pdhg_engine.py:187-188).
__device__ __forceinline__ void halpern_weights(double gamma, int64_t k, double& wm, double& wa) {
  const double kd = (double)k;
  const double k2 = dadd(kd, 2.0);
  wm = ddiv(dmul(dadd(1.0, gamma), dadd(kd, 1.0)), k2);
  wa = ddiv(1.0, k2);
}
// (w_map * mapped - gamma * current) + w_anchor * anchor (pdhg_engine.py:189)
__device__ __forceinline__ double halpern_mix(double t, double cur, double anc, double wm,
                                              double gamma, double wa) {
  return dadd(dsub(dmul(wm, t), dmul(gamma, cur)), dmul(wa, anc));
}

// ------------------------------------------------------------ cache policies
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// ------------------------------------------------ async copies (TMA, LDGSTS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}
// 1D bulk copy global -> shared through the TMA unit (SASS UBLKCP), completion
// signalled on `bar`, L2 evict-first policy for the streamed matrix.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 8-byte LDGSTS gather with an L2 evict-last policy (the dense vector stays
// resident in L2 across iterations).
__device__ __forceinline__ void cp_async8(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;"
               ::"r"(smem_u32(dst)), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------- deterministic sums
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum NR per-thread accumulators over the CTA; result valid in thread 0.
template <int NR>
__device__ __forceinline__ void block_sum(double (&acc)[NR], double (*scratch)[WARPS]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    double v = warp_sum(acc[q]);
    if (lane == 0) scratch[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      double s = scratch[q][0];
#pragma unroll
      for (int w = 1; w < WARPS; ++w) s = dadd(s, scratch[q][w]);
      acc[q] = s;
    }
  }
}

// --------------------------------------------------------------- epilogues
// Each op: NRED reduction slots; load(r) fetches the row's operands (issued
// early); row(r, sum, data, acc) applies the epilogue.

struct Empty {};

template <bool SUMSQ>
struct OpStore {
  static constexpr int NRED = SUMSQ ? 1 : 0;
  double* out;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double s, const Data&, double* acc) const {
    out[r] = s;
    if (SUMSQ) acc[0] = dadd(acc[0], dmul(s, s));
  }
};

struct OpPrimal {
  static constexpr int NRED = 0;
  double* x;
  double* xbar;
  const double* x0;
  const double* c;
  const double* lo;
  const double* hi;
  const gridlp_step_t* step;
  int32_t iter;
  bool halpern;
  double tau, gamma, wm, wa;
  struct Data { double x, c, lo, hi, x0; };
  __device__ void prepare() {
    tau = step->tau;
    gamma = step->gamma;
    halpern_weights(gamma, step->inner_k + iter, wm, wa);
  }
  __device__ Data load(int64_t r) const {
    Data d;
    d.x = x[r]; d.c = c[r]; d.lo = lo[r]; d.hi = hi[r];
    d.x0 = halpern ? x0[r] : 0.0;
    return d;
  }
  __device__ void row(int64_t r, double aty, const Data& d, double*) const {
    const double xh = np_clip(dsub(d.x, dmul(tau, dsub(d.c, aty))), d.lo, d.hi);
    xbar[r] = dsub(dmul(2.0, xh), d.x);
    x[r] = halpern ? halpern_mix(xh, d.x, d.x0, wm, gamma, wa) : xh;
  }
};

// v = y/sigma - z; sigma * (v - clip(v, -hi, -lo))  (pdhg_engine.py:176-181)
__device__ __forceinline__ double dual_map(double y, double z, double sigma, double lo, double hi) {
  const double v = dsub(ddiv(y, sigma), z);
  return dmul(sigma, dsub(v, np_clip(v, -hi, -lo)));
}

struct OpDual {
  static constexpr int NRED = 0;
  double* y;
  const double* y0;
  const double* lo;
  const double* hi;
  const gridlp_step_t* step;
  int32_t iter;
  bool halpern;
  double sigma, gamma, wm, wa;
  struct Data { double y, lo, hi, y0; };
  __device__ void prepare() {
    sigma = step->sigma;
    gamma = step->gamma;
    halpern_weights(gamma, step->inner_k + iter, wm, wa);
  }
  __device__ Data load(int64_t r) const {
    Data d;
    d.y = y[r]; d.lo = lo[r]; d.hi = hi[r];
    d.y0 = halpern ? y0[r] : 0.0;
    return d;
  }
  __device__ void row(int64_t r, double z, const Data& d, double*) const {
    const double yh = dual_map(d.y, z, sigma, d.lo, d.hi);
    y[r] = halpern ? halpern_mix(yh, d.y, d.y0, wm, gamma, wa) : yh;
  }
};

struct OpKktRows {
  static constexpr int NRED = 4;
  const double* y;
  const double* lo;
  const double* hi;
  double* ax;
  struct Data { double y, lo, hi; };
  __device__ void prepare() {}
  __device__ Data load(int64_t r) const { return {y[r], lo[r], hi[r]}; }
  __device__ void row(int64_t r, double s, const Data& d, double* acc) const {
    if (ax) ax[r] = s;
    // range_violation (pdhg_engine.py:206-208)
    const double rv = dsub(np_maximum(dsub(s, d.hi), 0.0), np_maximum(dsub(d.lo, s), 0.0));
    acc[0] = dadd(acc[0], dmul(rv, rv));
    // bound_penalty(-y) (pdhg_engine.py:192-203)
    const double v = -d.y;
    const double pos = np_maximum(v, 0.0);
    const double neg = np_maximum(-v, 0.0);
    const bool fu = isfinite(d.hi), fl = isfinite(d.lo);
    if (fu) acc[1] = dadd(acc[1], dmul(d.hi, pos));
    else if (pos > 0.0) acc[3] = dadd(acc[3], 1.0);
    if (fl) acc[2] = dadd(acc[2], dmul(d.lo, neg));
    else if (neg > 0.0) acc[3] = dadd(acc[3], 1.0);
  }
};

struct OpKktCols {
  static constexpr int NRED = 4;
  const double* x;
  const double* c;
  const double* lo;
  const double* hi;
  double* xpb;
  const gridlp_step_t* step;
  double tau;
  struct Data { double x, c, lo, hi; };
  __device__ void prepare() { tau = step->tau; }
  __device__ Data load(int64_t r) const { return {x[r], c[r], lo[r], hi[r]}; }
  __device__ void row(int64_t r, double aty, const Data& d, double* acc) const {
    // pdhg_engine.py:325-336
    const double shifted = dsub(d.x, dmul(tau, dsub(d.c, aty)));
    const double xp = np_clip(shifted, d.lo, d.hi);
    const double rd = ddiv(dsub(xp, d.x), tau);
    const double rc = ddiv(dsub(xp, shifted), tau);
    const double dx = dsub(d.x, xp);
    acc[0] = dadd(acc[0], dmul(rd, rd));
    acc[1] = dadd(acc[1], dmul(d.c, d.x));
    acc[2] = dadd(acc[2], dmul(rc, d.x));
    acc[3] = dadd(acc[3], dmul(dx, dx));
    if (xpb) xpb[r] = dsub(dmul(2.0, xp), d.x);
  }
};

struct OpProbe {
  static constexpr int NRED = 2;
  const double* y;
  const double* lo;
  const double* hi;
  const double* ax;
  double* dy_out;
  const gridlp_step_t* step;
  double sigma;
  struct Data { double y, lo, hi, ax; };
  __device__ void prepare() { sigma = step->sigma; }
  __device__ Data load(int64_t r) const { return {y[r], lo[r], hi[r], ax ? ax[r] : 0.0}; }
  __device__ void row(int64_t r, double z, const Data& d, double* acc) const {
    const double yp = dual_map(d.y, z, sigma, d.lo, d.hi);
    const double dy = dsub(d.y, yp);
    acc[0] = dadd(acc[0], dmul(dy, dy));
    if (ax) acc[1] = dadd(acc[1], dmul(dmul(0.5, dsub(d.ax, z)), dy));
    if (dy_out) dy_out[r] = dy;
  }
};

struct OpHalfDiffDot {
  static constexpr int NRED = 1;
  const double* a;
  const double* b;
  const double* d;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double* acc) const {
    acc[0] = dadd(acc[0], dmul(dmul(0.5, dsub(a[r], b[r])), d[r]));
  }
};

struct OpAnchor {
  static constexpr int NRED = 1;
  double* v;
  double* anchor;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double* acc) const {
    const double cur = v[r];
    const double e = dsub(cur, anchor[r]);
    acc[0] = dadd(acc[0], dmul(e, e));
    anchor[r] = cur;
  }
};

struct OpDot {
  static constexpr int NRED = 1;
  const double* a;
  const double* b;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double* acc) const {
    acc[0] = dadd(acc[0], dmul(a[r], b[r]));
  }
};

struct OpDiv {
  static constexpr int NRED = 0;
  const double* in;
  double* out;
  double divisor;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double*) const { out[r] = ddiv(in[r], divisor); }
};

struct OpInitPrimal {
  static constexpr int NRED = 0;
  double* x;
  double* anchor;
  const double* lo;
  const double* hi;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double*) const {
    const double v = np_clip(0.0, lo[r], hi[r]);
    x[r] = v;
    anchor[r] = v;
  }
};

// ------------------------------------------------------------------ kernels
template <int NR>
struct AccN { double v[NR > 0 ? NR : 1]; };

template <class Op>
__device__ __forceinline__ void store_partials(double (&acc)[Op::NRED > 0 ? Op::NRED : 1],
                                               double* partials) {
  if constexpr (Op::NRED > 0) {
    __shared__ double scratch[Op::NRED][WARPS];
    block_sum<Op::NRED>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < Op::NRED; ++q) partials[(int64_t)blockIdx.x * GRIDLP_MAX_RED + q] = acc[q];
    }
  }
}

// Sparse-product + fused-epilogue kernel over a tile directory, one CTA per
// tile. LEAN (variant 2) trades the early epilogue prefetch and the 8-deep
// unroll for <= 32 registers, so 8 CTAs (64 warps) stay resident per SM and
// keep the gather stream saturated.
template <class Op, int U, int MINB, bool LEAN>
__global__ void __launch_bounds__(TPB, MINB) tile_kernel(gridlp_csr_t A, const double* __restrict__ g,
                                                         Op op, double* __restrict__ partials) {
  extern __shared__ double prod[];
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;

  const int tid = threadIdx.x;
  const int64_t t = blockIdx.x;
  const int r0 = A.tile_ptr[t];
  const int r1 = A.tile_ptr[t + 1];
  const int p0 = A.row_ptr[r0];
  const int p1 = A.row_ptr[r1];
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int* __restrict__ col = A.col_idx;
  const double* __restrict__ val = A.values;

  if (r1 - r0 == 1 && p1 - p0 > A.exact_row_max) {
    // heavy row: CTA-wide strided products, deterministic tree sum
    typename Op::Data d{};
    if (tid == 0) d = op.load(r0);
    double s = 0.0;
    for (int k = p0 + tid; k < p1; k += TPB)
      s = dadd(s, dmul(ld_stream(val + k, pf), ld_gather(g + ld_stream(col + k, pf), pl)));
    double tmp[1] = {s};
    __shared__ double hscratch[1][WARPS];
    block_sum<1>(tmp, hscratch);
    if (tid == 0) op.row(r0, tmp[0], d, acc);
    __syncthreads();
  } else {
    const int r = r0 + tid;
    const bool mine = r < r1;
    typename Op::Data d{};
    int a = 0, b = 0;
    if (mine && !LEAN) {
      d = op.load(r);
      a = A.row_ptr[r] - p0;
      b = A.row_ptr[r + 1] - p0;
    }
    // phase (a): balanced gathers, rounded products into shared memory
    for (int base = p0 + tid; base < p1; base += TPB * U) {
      int cidx[U];
      double v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * TPB;
        cidx[u] = k < p1 ? ld_stream(col + k, pf) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * TPB;
        v[u] = k < p1 ? ld_stream(val + k, pf) : 0.0;
        xv[u] = k < p1 ? ld_gather(g + cidx[u], pl) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * TPB;
        if (k < p1) prod[k - p0] = dmul(v[u], xv[u]);
      }
    }
    if (mine && LEAN) {
      d = op.load(r);
      a = A.row_ptr[r] - p0;
      b = A.row_ptr[r + 1] - p0;
    }
    __syncthreads();
    // phase (b): sequential row sums (scipy csr_matvec order) + epilogue
    if (mine) {
      double s = 0.0;
      for (int k = a; k < b; ++k) s = dadd(s, prod[k]);
      op.row(r, s, d, acc);
    }
  }
  store_partials<Op>(acc, partials);
}

// One CTA per tile with the matrix stream staged by the TMA unit
// (variants 3/4): thread 0 issues two 1D bulk copies (values, column
// indices) into shared memory, so the LSU/L1 path carries only the gathers
// and the epilogue vectors. Gathers read the staged column indices and the
// rounded products overwrite the staged values in place; row sums as above.
template <class Op, int U, int MINB>
__global__ void __launch_bounds__(TPB, MINB) tile_kernel_tma(gridlp_csr_t A, const double* __restrict__ g,
                                                             Op op, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int cap = A.tile_nnz_cap;
  double* sv = reinterpret_cast<double*>(smem_raw);
  int* sc = reinterpret_cast<int*>(smem_raw + (size_t)(cap + 4) * 8);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + (size_t)(cap + 4) * 8 + (size_t)(cap + 8) * 4);
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  const int tid = threadIdx.x;
  const int64_t t = blockIdx.x;
  const int r0 = A.tile_ptr[t];
  const int r1 = A.tile_ptr[t + 1];
  const int p0 = A.row_ptr[r0];
  const int p1 = A.row_ptr[r1];
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();

  if (r1 - r0 == 1 && p1 - p0 > A.exact_row_max) {
    typename Op::Data d{};
    if (tid == 0) d = op.load(r0);
    double s = 0.0;
    for (int k = p0 + tid; k < p1; k += TPB)
      s = dadd(s, dmul(ld_stream(A.values + k, pf), ld_gather(g + ld_stream(A.col_idx + k, pf), pl)));
    double tmp[1] = {s};
    __shared__ double hscratch[1][WARPS];
    block_sum<1>(tmp, hscratch);
    if (tid == 0) op.row(r0, tmp[0], d, acc);
    __syncthreads();
  } else {
    const int nnz = p1 - p0;
    if (tid == 0) {
      const int va = p0 & ~1, vb = (p1 + 1) & ~1;
      const int ca = p0 & ~3, cb = (p1 + 3) & ~3;
      const uint32_t vbytes = (uint32_t)(vb - va) * 8u, cbytes = (uint32_t)(cb - ca) * 4u;
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(bar, vbytes + cbytes);
      if (vbytes) tma_bulk_g2s(sv, A.values + va, vbytes, bar, pf);
      if (cbytes) tma_bulk_g2s(sc, A.col_idx + ca, cbytes, bar, pf);
    }
    const int r = r0 + tid;
    const bool mine = r < r1;
    typename Op::Data d{};
    int a = 0, b = 0;
    if (mine) {
      d = op.load(r);
      a = A.row_ptr[r] - p0;
      b = A.row_ptr[r + 1] - p0;
    }
    __syncthreads();            // barrier initialised before anyone waits on it
    mbar_wait(bar, 0);
    double* v = sv + (p0 & 1);
    const int* c = sc + (p0 & 3);
    for (int base = tid; base < nnz; base += TPB * U) {
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * TPB;
        xv[u] = k < nnz ? ld_gather(g + c[k], pl) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * TPB;
        if (k < nnz) v[k] = dmul(v[k], xv[u]);
      }
    }
    __syncthreads();
    if (mine) {
      double sum = 0.0;
      for (int k = a; k < b; ++k) sum = dadd(sum, v[k]);
      op.row(r, sum, d, acc);
    }
  }
  store_partials<Op>(acc, partials);
}

// SELL-32 window kernel (variant 6). One CTA = one window of 256 rows =
// 8 warps = 8 slices. Each lane owns one light row of its slice and walks
// the row's entries in their original order: the column index and value of
// step j are 32 consecutive elements across the warp (fully coalesced), the
// gather of x is one 8-byte load, and the sum lives in a register — no
// shared-memory staging of products, no bank conflicts, no phase barrier.
// Sums are parked in shared memory by window-local row and the epilogue
// then runs in natural row order (coalesced vector traffic). Blocks past the
// windows tree-sum one heavy row each (compact CSR).
template <class Op, int U, int MINB, bool EARLY>
__global__ void __launch_bounds__(TPB, MINB) sell_kernel(gridlp_csr_t A, const double* __restrict__ g, Op op,
                                                         double* __restrict__ partials) {
  __shared__ double sums[TPB];
  __shared__ int have[TPB];
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  const int tid = threadIdx.x;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int64_t w = blockIdx.x;
  if (w >= A.num_windows) {
    const int64_t h = w - A.num_windows;
    const int row = A.heavy_rows[h];
    const int p0 = A.heavy_ptr[h], p1 = A.heavy_ptr[h + 1];
    typename Op::Data d{};
    if (tid == 0) d = op.load(row);
    double s = 0.0;
    for (int k = p0 + tid; k < p1; k += TPB)
      s = dadd(s, dmul(ld_stream(A.heavy_vals + k, pf), ld_gather(g + ld_stream(A.heavy_cols + k, pf), pl)));
    double tmp[1] = {s};
    __shared__ double hscratch[1][WARPS];
    block_sum<1>(tmp, hscratch);
    if (tid == 0) op.row(row, tmp[0], d, acc);
    __syncthreads();
  } else {
    const int64_t r = w * TPB + tid;
    const bool in_range = r < A.num_rows;
    typename Op::Data d{};
    if (EARLY && in_range) d = op.load(r);   // natural-order epilogue operands, issued first
    have[tid] = 0;
    const int lane = tid & 31;
    const int64_t slice = w * WARPS + (tid >> 5);
    const int info = A.lane_info[slice * 32 + lane];
    __syncthreads();
    if (info >= 0) {
      const int len = info >> 8;
      const int64_t base = (int64_t)A.slice_off[slice] + lane;
      const int* __restrict__ cp = A.sell_cols + base;
      const double* __restrict__ vp = A.sell_vals + base;
      double s = 0.0;
      for (int j = 0; j < len; j += U) {
        int c[U];
        double v[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = j + u < len;
          c[u] = ok ? ld_stream(cp + 32 * (j + u), pf) : 0;
          v[u] = ok ? ld_stream(vp + 32 * (j + u), pf) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (j + u < len) ? ld_gather(g + c[u], pl) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j + u < len) s = dadd(s, dmul(v[u], x[u]));
      }
      sums[info & 255] = s;
      have[info & 255] = 1;
    }
    if (!EARLY && in_range) d = op.load(r);
    __syncthreads();
    if (in_range && have[tid]) op.row(r, sums[tid], d, acc);
  }
  store_partials<Op>(acc, partials);
}

// Warp-window SELL kernel (variant 9): the window is ONE warp (32 rows,
// sorted by length inside the slice), so there is no CTA-wide barrier — each
// warp parks its 32 sums in shared memory, __syncwarp()s and runs the
// natural-order epilogue of its own 32 rows. CTAs are WPB warps; heavy rows
// (compact CSR) are tree-summed by the blocks past the windows.
template <class Op, int U, int WPB, bool EARLY, int MINB>
__global__ void __launch_bounds__(WPB * 32, MINB) sell32_kernel(gridlp_csr_t A, const double* __restrict__ g, Op op,
                                                          double* __restrict__ partials) {
  __shared__ double sums[WPB][32];
  __shared__ int have[WPB][32];
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  constexpr int NT = WPB * 32;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int64_t nblk_win = (A.num_windows + WPB - 1) / WPB;
  if ((int64_t)blockIdx.x >= nblk_win) {
    const int64_t h = blockIdx.x - nblk_win;
    const int row = A.heavy_rows[h];
    const int p0 = A.heavy_ptr[h], p1 = A.heavy_ptr[h + 1];
    typename Op::Data d{};
    if (tid == 0) d = op.load(row);
    double s = 0.0;
    for (int k = p0 + tid; k < p1; k += NT)
      s = dadd(s, dmul(ld_stream(A.heavy_vals + k, pf), ld_gather(g + ld_stream(A.heavy_cols + k, pf), pl)));
    s = warp_sum(s);
    __shared__ double hs[WPB];
    if (lane == 0) hs[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double t = hs[0];
      for (int w = 1; w < WPB; ++w) t = dadd(t, hs[w]);
      op.row(row, t, d, acc);
    }
  } else {
    const int64_t slice = (int64_t)blockIdx.x * WPB + warp;
    if (slice < A.num_windows) {
      const int64_t r = slice * 32 + lane;
      const bool in_range = r < A.num_rows;
      typename Op::Data d{};
      if (EARLY && in_range) d = op.load(r);
      have[warp][lane] = 0;
      const int info = A.lane_info[slice * 32 + lane];
      __syncwarp();
      if (info >= 0) {
        const int len = info >> 8;
        const int64_t base = (int64_t)A.slice_off[slice] + lane;
        const int* __restrict__ cp = A.sell_cols + base;
        const double* __restrict__ vp = A.sell_vals + base;
        double s = 0.0;
        for (int j = 0; j < len; j += U) {
          int c[U];
          double v[U], x[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const bool ok = j + u < len;
            c[u] = ok ? ld_stream(cp + 32 * (j + u), pf) : 0;
            v[u] = ok ? ld_stream(vp + 32 * (j + u), pf) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) x[u] = (j + u < len) ? ld_gather(g + c[u], pl) : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j + u < len) s = dadd(s, dmul(v[u], x[u]));
        }
        sums[warp][info & 31] = s;
        have[warp][info & 31] = 1;
      }
      if (!EARLY && in_range) d = op.load(r);
      __syncwarp();
      if (in_range && have[warp][lane]) op.row(r, sums[warp][lane], d, acc);
    }
  }
  if constexpr (Op::NRED > 0) {
    // deterministic: warp tree, then warps in order
    __shared__ double rs[Op::NRED][WPB];
#pragma unroll
    for (int q = 0; q < Op::NRED; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) rs[q][warp] = v;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < Op::NRED; ++q) {
        double t = rs[q][0];
        for (int w = 1; w < WPB; ++w) t = dadd(t, rs[q][w]);
        partials[(int64_t)blockIdx.x * GRIDLP_MAX_RED + q] = t;
      }
    }
  }
}

// Persistent, TMA-pipelined product + epilogue kernel (variant 0).
// Each CTA walks its light tiles (round-robin over light_tiles) with a
// two-slot pipeline: while tile i is gathered and summed, the TMA unit
// streams tile i+1's values and column indices into the other slot. The
// gathers of the dense vector are 8-byte LDGSTS (cp.async) straight into
// shared memory, so every gather of a tile is in flight at once without
// holding registers. Row sums are the same sequential +0.0-seeded sums as
// the one-CTA-per-tile kernel (bit-identical to scipy). Heavy tiles follow,
// tree-summed by the whole CTA. Reduction partials are per CTA, in a fixed
// tile order, hence deterministic.
struct PipeLayout {
  int cap;
  __host__ __device__ size_t vals_bytes() const { return (size_t)(cap + 4) * 8; }
  __host__ __device__ size_t cols_bytes() const { return (size_t)(cap + 8) * 4; }
  __host__ __device__ size_t slot_bytes() const { return vals_bytes() + cols_bytes(); }
  __host__ __device__ size_t total() const { return 2 * slot_bytes() + (size_t)cap * 8 + 64; }
};

template <class Op>
__global__ void __launch_bounds__(TPB) tile_kernel_pipe(gridlp_csr_t A, const double* __restrict__ g,
                                                        Op op, double* __restrict__ partials) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const PipeLayout L{A.tile_nnz_cap};
  double* xbuf = reinterpret_cast<double*>(smem_raw + 2 * L.slot_bytes());
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 2 * L.slot_bytes() + (size_t)L.cap * 8);
  auto slot_vals = [&](int s) { return reinterpret_cast<double*>(smem_raw + s * L.slot_bytes()); };
  auto slot_cols = [&](int s) {
    return reinterpret_cast<int*>(smem_raw + s * L.slot_bytes() + L.vals_bytes());
  };

  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  const int tid = threadIdx.x;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int* __restrict__ rp = A.row_ptr;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // stage the streams of light tile #idx (in this CTA's sequence) into slot s
  auto issue = [&](int64_t idx, int s) {
    const int t = A.light_tiles[idx];
    const int p0 = rp[A.tile_ptr[t]];
    const int p1 = rp[A.tile_ptr[t + 1]];
    const int va = p0 & ~1, vb = (p1 + 1) & ~1;
    const int ca = p0 & ~3, cb = (p1 + 3) & ~3;
    const uint32_t vbytes = (uint32_t)(vb - va) * 8u, cbytes = (uint32_t)(cb - ca) * 4u;
    fence_proxy_async();
    mbar_expect_tx(&bars[s], vbytes + cbytes);
    if (vbytes) tma_bulk_g2s(slot_vals(s), A.values + va, vbytes, &bars[s], pf);
    if (cbytes) tma_bulk_g2s(slot_cols(s), A.col_idx + ca, cbytes, &bars[s], pf);
  };

  const int64_t stride = gridDim.x;
  int64_t i = blockIdx.x;
  uint32_t phase[2] = {0u, 0u};
  if (i < A.num_light && tid == 0) issue(i, 0);
  for (int it = 0; i < A.num_light; ++it, i += stride) {
    const int s = it & 1;
    const int t = A.light_tiles[i];
    const int r0 = A.tile_ptr[t];
    const int r1 = A.tile_ptr[t + 1];
    const int p0 = rp[r0];
    const int p1 = rp[r1];
    const int nnz = p1 - p0;
    const int r = r0 + tid;
    const bool mine = r < r1;
    typename Op::Data d{};
    int a = 0, b = 0;
    if (mine) {
      d = op.load(r);                   // epilogue operands: in flight during the gathers
      a = rp[r] - p0;
      b = rp[r + 1] - p0;
    }
    if (tid == 0 && i + stride < A.num_light) issue(i + stride, s ^ 1);
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1u;
    const double* sv = slot_vals(s) + (p0 & 1);
    const int* sc = slot_cols(s) + (p0 & 3);
    for (int k = tid; k < nnz; k += TPB) cp_async8(&xbuf[k], g + sc[k], pl);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int k = tid; k < nnz; k += TPB) xbuf[k] = dmul(sv[k], xbuf[k]);
    __syncthreads();
    if (mine) {
      double sum = 0.0;
      for (int k = a; k < b; ++k) sum = dadd(sum, xbuf[k]);
      op.row(r, sum, d, acc);
    }
    __syncthreads();
  }

  for (int64_t h = blockIdx.x; h < A.num_heavy; h += stride) {
    const int t = A.heavy_tiles[h];
    const int row = A.tile_ptr[t];
    const int p0 = rp[row], p1 = rp[row + 1];
    typename Op::Data d{};
    if (tid == 0) d = op.load(row);
    double sum = 0.0;
    for (int k = p0 + tid; k < p1; k += TPB)
      sum = dadd(sum, dmul(ld_stream(A.values + k, pf), ld_gather(g + ld_stream(A.col_idx + k, pf), pl)));
    double tmp[1] = {sum};
    __shared__ double hscratch[1][WARPS];
    block_sum<1>(tmp, hscratch);
    if (tid == 0) op.row(row, tmp[0], d, acc);
    __syncthreads();
  }
  store_partials<Op>(acc, partials);
}

// Row-wise epilogue over ascending-order sums of partial vectors.
template <class Op>
__global__ void __launch_bounds__(TPB) rows_kernel(gridlp_src_t src, int64_t n, Op op,
                                                   double* __restrict__ partials) {
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  op.prepare();
  const int np = src.nparts;
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
    const typename Op::Data d = op.load(r);
    double s = 0.0;
    if (np > 0) {
      s = src.parts[0][r];
      for (int q = 1; q < np; ++q) s = dadd(s, src.parts[q][r]);
    }
    op.row(r, s, d, acc);
  }
  store_partials<Op>(acc, partials);
}

// Fixed-order final reduction of per-CTA slots.
__global__ void __launch_bounds__(TPB) reduce_kernel(const double* __restrict__ partials,
                                                     int64_t nslots, int nred,
                                                     double* __restrict__ out) {
  __shared__ double scratch[GRIDLP_MAX_RED][WARPS];
  double acc[GRIDLP_MAX_RED];
#pragma unroll
  for (int q = 0; q < GRIDLP_MAX_RED; ++q) acc[q] = 0.0;
  for (int64_t s = threadIdx.x; s < nslots; s += TPB) {
#pragma unroll
    for (int q = 0; q < GRIDLP_MAX_RED; ++q)
      if (q < nred) acc[q] = dadd(acc[q], partials[s * GRIDLP_MAX_RED + q]);
  }
  block_sum<GRIDLP_MAX_RED>(acc, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < nred; ++q) out[q] = acc[q];
}

__global__ void step_advance_kernel(gridlp_step_t* st, int64_t delta) {
  if (threadIdx.x == 0 && blockIdx.x == 0) st->inner_k += delta;
}

// ------------------------------------------------------------------ host side
int64_t rows_blocks(int64_t n) {
  int64_t b = (n + TPB - 1) / TPB;
  if (b < 1) b = 1;
  return b < ROWS_MAX_BLOCKS ? b : ROWS_MAX_BLOCKS;
}

int check_csr(const gridlp_csr_t* A) {
  if (!A) return fail(GRIDLP_ERR_ARG, "null matrix");
  if (A->num_rows < 0 || A->num_cols < 0 || A->nnz < 0 || A->num_tiles < 0)
    return fail(GRIDLP_ERR_ARG, "negative matrix dimension");
  if (A->nnz >= (int64_t(1) << 31)) return fail(GRIDLP_ERR_ARG, "block nnz must be < 2^31");
  if (A->tile_nnz_cap < 64 || A->tile_nnz_cap > CAP || (A->tile_nnz_cap & 7))
    return fail(GRIDLP_ERR_ARG, "tile_nnz_cap must be a multiple of 8 in [64, TILE_NNZ_CAP]");
  if (A->exact_row_max < 0 || A->exact_row_max > A->tile_nnz_cap / 2)
    return fail(GRIDLP_ERR_ARG, "exact_row_max must be in [0, tile_nnz_cap/2]");
  if (A->variant < 0 || A->variant > 10) return fail(GRIDLP_ERR_ARG, "unknown kernel variant");
  if (A->variant >= 6) {
    const int win = A->variant >= 9 ? 32 : TPB;
    if (A->num_rows > 0 &&
        (!A->slice_off || !A->lane_info || A->num_windows != (A->num_rows + win - 1) / win))
      return fail(GRIDLP_ERR_ARG, "SELL layout missing or inconsistent");
    if (A->num_heavy_rows > 0 && (!A->heavy_rows || !A->heavy_ptr || !A->heavy_cols || !A->heavy_vals))
      return fail(GRIDLP_ERR_ARG, "missing heavy-row CSR");
    if (A->nnz > 0 && (!A->sell_cols || !A->sell_vals)) return fail(GRIDLP_ERR_ARG, "missing SELL arrays");
    return GRIDLP_OK;
  }
  if (A->num_light + A->num_heavy != A->num_tiles)
    return fail(GRIDLP_ERR_ARG, "light + heavy tiles must cover the tile directory");
  if (A->num_tiles > 0 && ((A->num_light > 0 && !A->light_tiles) || (A->num_heavy > 0 && !A->heavy_tiles)))
    return fail(GRIDLP_ERR_ARG, "missing light/heavy tile lists");
  if (A->num_rows > 0 && (!A->row_ptr || !A->tile_ptr || A->num_tiles < 1))
    return fail(GRIDLP_ERR_ARG, "missing row_ptr/tile_ptr");
  if (A->nnz > 0 && (!A->col_idx || !A->values)) return fail(GRIDLP_ERR_ARG, "missing col_idx/values");
  return GRIDLP_OK;
}

int64_t src_rows(const gridlp_src_t* src) { return src->A ? src->A->num_rows : src->num_rows; }

// CTAs of the persistent kernel: SMs x resident CTAs (cached per op type and
// shared-memory size).
template <class Op>
int pipe_grid(size_t smem) {
  static size_t cached_smem = 0;
  static int cached = 0;
  if (cached > 0 && cached_smem == smem) return cached;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (cudaFuncSetAttribute(tile_kernel_pipe<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_kernel_pipe<Op>, TPB, smem) != cudaSuccess)
    return -1;
  if (per_sm < 1) per_sm = 1;
  cached = sms * per_sm;
  cached_smem = smem;
  return cached;
}

template <class Op>
int launch_op(const gridlp_src_t* src, Op op, const gridlp_red_t* red, void* stream,
              const char* name) {
  if (!src) return fail(GRIDLP_ERR_ARG, std::string(name) + ": null source");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = src_rows(src);
  int64_t slots;
  if (src->A) {
    int rc = check_csr(src->A);
    if (rc) return rc;
    if (src->A->num_rows > 0 && src->A->nnz > 0 && !src->gather)
      return fail(GRIDLP_ERR_ARG, std::string(name) + ": missing gather vector");
    slots = src->A->num_rows <= 0 ? 0
            : (src->A->variant >= 9 ? (src->A->num_windows + 1) / 2 + src->A->num_heavy_rows
               : src->A->variant >= 6 ? src->A->num_windows + src->A->num_heavy_rows : src->A->num_tiles);
  } else {
    if (src->nparts < 0 || src->nparts > GRIDLP_MAX_PARTS)
      return fail(GRIDLP_ERR_ARG, std::string(name) + ": nparts out of range");
    for (int q = 0; q < src->nparts; ++q)
      if (!src->parts[q] && n > 0) return fail(GRIDLP_ERR_ARG, std::string(name) + ": null part");
    slots = n > 0 ? rows_blocks(n) : 0;
  }
  double* partials = nullptr;
  if (Op::NRED > 0) {
    if (!red || !red->out) return fail(GRIDLP_ERR_ARG, std::string(name) + ": reduction output required");
    if (slots > 0) {
      if (!red->partials || red->capacity < slots)
        return fail(GRIDLP_ERR_WORKSPACE, std::string(name) + ": reduction workspace too small (need " +
                                              std::to_string(slots) + " slots)");
      partials = red->partials;
    }
  }
  if (slots > 0) {
    if (src->A && src->A->variant == 0) {
      const size_t smem = PipeLayout{src->A->tile_nnz_cap}.total();
      int grid = pipe_grid<Op>(smem);
      if (grid <= 0) return fail(GRIDLP_ERR_CUDA, std::string(name) + ": occupancy query failed");
      if (grid > slots) grid = (int)slots;
      slots = grid;
      tile_kernel_pipe<Op><<<(unsigned)grid, TPB, smem, s>>>(*src->A, src->gather, op, partials);
    } else if (src->A) {
      const gridlp_csr_t& M = *src->A;
      const size_t sm_prod = M.tile_nnz_cap * sizeof(double);
      const size_t sm_tma = (size_t)(M.tile_nnz_cap + 4) * 8 + (size_t)(M.tile_nnz_cap + 8) * 4 + 16;
      const unsigned nb = (unsigned)slots;
      switch (M.variant) {
        case 2: tile_kernel<Op, 4, 8, true><<<nb, TPB, sm_prod, s>>>(M, src->gather, op, partials); break;
        case 3: tile_kernel_tma<Op, 4, 8><<<nb, TPB, sm_tma, s>>>(M, src->gather, op, partials); break;
        case 4: tile_kernel_tma<Op, 8, 5><<<nb, TPB, sm_tma, s>>>(M, src->gather, op, partials); break;
        case 5: tile_kernel<Op, 4, 6, false><<<nb, TPB, sm_prod, s>>>(M, src->gather, op, partials); break;
        case 9: case 10: {
          const int64_t nwb = (M.num_windows + 1) / 2;
          const unsigned nb9 = (unsigned)(nwb + M.num_heavy_rows);
          slots = nb9;
          if (!nb9) break;
          if (M.variant == 9) sell32_kernel<Op, 4, 2, false, 32><<<nb9, 64, 0, s>>>(M, src->gather, op, partials);
          else sell32_kernel<Op, 4, 2, true, 21><<<nb9, 64, 0, s>>>(M, src->gather, op, partials);
          break;
        }
        case 6: case 7: case 8: {
          const unsigned nsell = (unsigned)(M.num_windows + M.num_heavy_rows);
          slots = nsell;
          if (!nsell) break;
          if (M.variant == 6) sell_kernel<Op, 4, 8, false><<<nsell, TPB, 0, s>>>(M, src->gather, op, partials);
          else if (M.variant == 7) sell_kernel<Op, 8, 6, false><<<nsell, TPB, 0, s>>>(M, src->gather, op, partials);
          else sell_kernel<Op, 4, 5, true><<<nsell, TPB, 0, s>>>(M, src->gather, op, partials);
          break;
        }
        default: tile_kernel<Op, UNROLL, 5, false><<<nb, TPB, sm_prod, s>>>(M, src->gather, op, partials); break;
      }
    } else {
      rows_kernel<Op><<<(unsigned)slots, TPB, 0, s>>>(*src, n, op, partials);
    }
    int rc = check_launch(name);
    if (rc) return rc;
  }
  if (Op::NRED > 0) {
    reduce_kernel<<<1, TPB, 0, s>>>(partials, slots, Op::NRED, red->out);
    int rc = check_launch(name);
    if (rc) return rc;
  }
  return GRIDLP_OK;
}

gridlp_src_t rows_src(int64_t n) {
  gridlp_src_t s;
  std::memset(&s, 0, sizeof(s));
  s.num_rows = n;
  return s;
}

struct KernelAttrInit {
  KernelAttrInit() {}
};

}  // namespace

// ===================================================================== C ABI
extern "C" {

int gridlp_abi_version(void) { return GRIDLP_ABI_VERSION; }

const char* gridlp_last_error(void) { return g_err.c_str(); }

// not part of the header: lets the setup translation unit share the error slot
void gridlp_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

int gridlp_device_info(int device, int32_t* sm_count, int64_t* l2_bytes) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("device_info: ") + cudaGetErrorString(e));
  if (sm_count) *sm_count = v;
  e = cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("device_info: ") + cudaGetErrorString(e));
  if (l2_bytes) *l2_bytes = v;
  return GRIDLP_OK;
}

int64_t gridlp_op_slots(const gridlp_src_t* src) {
  if (!src) return 0;
  if (src->A && src->A->variant >= 9) return (src->A->num_windows + 1) / 2 + src->A->num_heavy_rows;
  if (src->A && src->A->variant >= 6) return src->A->num_windows + src->A->num_heavy_rows;
  if (src->A) return src->A->num_rows > 0 ? src->A->num_tiles : 0;
  return src->num_rows > 0 ? rows_blocks(src->num_rows) : 0;
}

int gridlp_op_store(const gridlp_src_t* src, double* out, uint32_t flags, const gridlp_red_t* red,
                    void* stream) {
  if (!src) return fail(GRIDLP_ERR_ARG, "op_store: null source");
  if (!out && src_rows(src) > 0) return fail(GRIDLP_ERR_ARG, "op_store: null output");
  if (flags & GRIDLP_F_SUMSQ) return launch_op(src, OpStore<true>{out}, red, stream, "op_store");
  return launch_op(src, OpStore<false>{out}, red, stream, "op_store");
}

int gridlp_op_primal(const gridlp_src_t* src, const gridlp_primal_t* pv, const gridlp_step_t* d_step,
                     int32_t iter, uint32_t flags, void* stream) {
  if (!pv || !d_step) return fail(GRIDLP_ERR_ARG, "op_primal: null argument");
  if (src && src_rows(src) != pv->n) return fail(GRIDLP_ERR_ARG, "op_primal: length mismatch");
  OpPrimal op{};
  op.x = pv->x; op.xbar = pv->x_bar; op.x0 = pv->x_anchor; op.c = pv->c; op.lo = pv->lo; op.hi = pv->hi;
  op.step = d_step; op.iter = iter; op.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  return launch_op(src, op, nullptr, stream, "op_primal");
}

int gridlp_op_dual(const gridlp_src_t* src, const gridlp_dual_t* dv, const gridlp_step_t* d_step,
                   int32_t iter, uint32_t flags, void* stream) {
  if (!dv || !d_step) return fail(GRIDLP_ERR_ARG, "op_dual: null argument");
  if (src && src_rows(src) != dv->m) return fail(GRIDLP_ERR_ARG, "op_dual: length mismatch");
  OpDual op{};
  op.y = dv->y; op.y0 = dv->y_anchor; op.lo = dv->lo; op.hi = dv->hi;
  op.step = d_step; op.iter = iter; op.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  return launch_op(src, op, nullptr, stream, "op_dual");
}

int gridlp_op_kkt_rows(const gridlp_src_t* src, const gridlp_dual_t* dv, double* ax,
                       const gridlp_red_t* red, void* stream) {
  if (!dv) return fail(GRIDLP_ERR_ARG, "op_kkt_rows: null argument");
  if (src && src_rows(src) != dv->m) return fail(GRIDLP_ERR_ARG, "op_kkt_rows: length mismatch");
  OpKktRows op{dv->y, dv->lo, dv->hi, ax};
  return launch_op(src, op, red, stream, "op_kkt_rows");
}

int gridlp_op_kkt_cols(const gridlp_src_t* src, const gridlp_primal_t* pv, double* x_probe_bar,
                       const gridlp_step_t* d_step, const gridlp_red_t* red, void* stream) {
  if (!pv || !d_step) return fail(GRIDLP_ERR_ARG, "op_kkt_cols: null argument");
  if (src && src_rows(src) != pv->n) return fail(GRIDLP_ERR_ARG, "op_kkt_cols: length mismatch");
  OpKktCols op{};
  op.x = pv->x; op.c = pv->c; op.lo = pv->lo; op.hi = pv->hi; op.xpb = x_probe_bar; op.step = d_step;
  return launch_op(src, op, red, stream, "op_kkt_cols");
}

int gridlp_op_probe(const gridlp_src_t* src, const gridlp_dual_t* dv, const double* ax, double* dy_out,
                    const gridlp_step_t* d_step, const gridlp_red_t* red, void* stream) {
  if (!dv || !d_step) return fail(GRIDLP_ERR_ARG, "op_probe: null argument");
  if (src && src_rows(src) != dv->m) return fail(GRIDLP_ERR_ARG, "op_probe: length mismatch");
  OpProbe op{};
  op.y = dv->y; op.lo = dv->lo; op.hi = dv->hi; op.ax = ax; op.dy_out = dy_out; op.step = d_step;
  return launch_op(src, op, red, stream, "op_probe");
}

int gridlp_op_halfdiff_dot(const double* a, const double* b, const double* d, int64_t n,
                           const gridlp_red_t* red, void* stream) {
  if (n < 0 || (n > 0 && (!a || !b || !d))) return fail(GRIDLP_ERR_ARG, "op_halfdiff_dot: bad argument");
  gridlp_src_t src = rows_src(n);
  return launch_op(&src, OpHalfDiffDot{a, b, d}, red, stream, "op_halfdiff_dot");
}

int gridlp_op_anchor(double* v, double* anchor, int64_t n, const gridlp_red_t* red, void* stream) {
  if (n < 0 || (n > 0 && (!v || !anchor))) return fail(GRIDLP_ERR_ARG, "op_anchor: bad argument");
  gridlp_src_t src = rows_src(n);
  return launch_op(&src, OpAnchor{v, anchor}, red, stream, "op_anchor");
}

int gridlp_op_dot(const double* a, const double* b, int64_t n, const gridlp_red_t* red, void* stream) {
  if (n < 0 || (n > 0 && (!a || !b))) return fail(GRIDLP_ERR_ARG, "op_dot: bad argument");
  gridlp_src_t src = rows_src(n);
  return launch_op(&src, OpDot{a, b}, red, stream, "op_dot");
}

int gridlp_op_div(const double* in, double* out, int64_t n, double divisor, void* stream) {
  if (n < 0 || (n > 0 && (!in || !out))) return fail(GRIDLP_ERR_ARG, "op_div: bad argument");
  gridlp_src_t src = rows_src(n);
  return launch_op(&src, OpDiv{in, out, divisor}, nullptr, stream, "op_div");
}

int gridlp_op_init_primal(const gridlp_primal_t* pv, void* stream) {
  if (!pv) return fail(GRIDLP_ERR_ARG, "op_init_primal: null argument");
  gridlp_src_t src = rows_src(pv->n);
  return launch_op(&src, OpInitPrimal{pv->x, pv->x_anchor, pv->lo, pv->hi}, nullptr, stream,
                   "op_init_primal");
}

int gridlp_op_step_advance(gridlp_step_t* d_step, int64_t delta, void* stream) {
  if (!d_step) return fail(GRIDLP_ERR_ARG, "op_step_advance: null step");
  step_advance_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(d_step, delta);
  return check_launch("op_step_advance");
}

}  // extern "C"
