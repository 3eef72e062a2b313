// gridlp_b200.cu — sm_100a kernels + C ABI for the distributed-PDHG hot path.
//
// Design:
//  * Sparse products run over a SELL-32 layout of each CSR block: 32
//    consecutive rows form a slice owned by one warp, lanes ordered by row
//    length; entry j of lane l sits at slice_off[s] + 32 j + l in the row's
//    original order. A warp step therefore reads 32 consecutive column
//    indices and values (coalesced, L2 evict-first), gathers 32 entries of
//    the dense vector (L2 evict-last) and each lane adds its product to a
//    register sum left to right from +0.0 — bit-identical to scipy's
//    csr_matvec, the reference's kernel (sparse_kernels.py:18-24). The
//    fused PDHG epilogue then runs in natural row order.
//  * Rows longer than light_row_max live in a compact CSR. Up to
//    exact_row_max entries one warp owns the row: 32 products per step,
//    added to a single running sum in entry order through warp shuffles
//    (still bit-identical to scipy). Longer rows are cut into chunks of
//    GRIDLP_HEAVY_CHUNK entries; one CTA per chunk tree-sums its part and
//    the last chunk CTA of a row to arrive adds the chunk sums in chunk order
//    (deterministic) and applies the epilogue. The heavy and long kernels
//    are launched before the SELL kernel so long rows do not form a tail.
//  * No FMA contraction anywhere: every multiply/add/divide is an explicit
//    __d*_rn so each numpy expression of the reference is reproduced
//    operation for operation.
//  * Reductions are deterministic: fixed warp-shuffle tree per CTA, one
//    slot per CTA, then one fixed-order final pass.
#include "../../include/gridlp_b200.h"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace {

constexpr int TPB = 256;
constexpr int WARPS = TPB / 32;
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
// Bounds-checked build (-DGRIDLP_CHECKED, native.build(checked=True),
// tests/test_gpu_bounds.py): every gather index, SELL lane extent, long-row
// range and written row is verified in the kernel; a violation prints where
// and traps. The product build compiles the checks away.
#ifdef GRIDLP_CHECKED
#define GRIDLP_CHECK(cond, what)                                                                      \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("GRIDLP_CHECK failed: %s at %s:%d (block %d, thread %d)\n", what, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                      \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define GRIDLP_CHECK(cond, what) \
  do {                           \
  } while (0)
#endif

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
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
  float v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// ------------------------------------------------------- value codecs
// gridlp_csr_t.val_codec (GRIDLP_VALS_*): how a block's values are stored.
// Every codec rebuilds the exact FP64 value before the same dmul, so the
// products are those of FP64 storage bit for bit; only the stream bytes
// change (12 / 8 / 4 B per nonzero).
template <int VC> struct Vals;
template <> struct Vals<GRIDLP_VALS_F64> {
  using T = double;
  static __device__ __forceinline__ T ld(const void* p, int64_t k, uint64_t pol) {
    return ld_stream(static_cast<const double*>(p) + k, pol);
  }
  static __device__ __forceinline__ T zero() { return 0.0; }
  static __device__ __forceinline__ double val(T v, int) { return v; }
  static __device__ __forceinline__ int col(int c) { return c; }
};
template <> struct Vals<GRIDLP_VALS_F32> {
  using T = float;
  static __device__ __forceinline__ T ld(const void* p, int64_t k, uint64_t pol) {
    return ld_stream(static_cast<const float*>(p) + k, pol);
  }
  static __device__ __forceinline__ T zero() { return 0.0f; }
  static __device__ __forceinline__ double val(T v, int) { return (double)v; }   // exact widening
  static __device__ __forceinline__ int col(int c) { return c; }
};
template <> struct Vals<GRIDLP_VALS_UNIT> {
  struct T {};
  static __device__ __forceinline__ T ld(const void*, int64_t, uint64_t) { return T{}; }
  static __device__ __forceinline__ T zero() { return T{}; }
  static __device__ __forceinline__ double val(T, int c) { return c < 0 ? -1.0 : 1.0; }   // sign bit
  static __device__ __forceinline__ int col(int c) { return c & 0x7fffffff; }
};

// column-band carry: coherent (the kernel may rewrite the row), first to leave L2
__device__ __forceinline__ double ld_carry(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// (Gathers allocate in L1: with L1::no_allocate cfg3 ran 3144 vs 2174 us per
// iteration and cfg4 4859 vs 4168 — the hot columns of power-law and MCF
// matrices hit in L1; profiles/r2/ab_gather_l1_noalloc_cfg*.json. A minimum
// shared-memory carveout (largest L1) gave cfg3 -0.9 %, cfg2 / cfg4 no
// change: ab_l1_carveout_cfg*.json; not applied.)

// coherent read-once load (the thread rewrites the element later), first to leave L2
__device__ __forceinline__ double ld_once(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// Gathers are L2 evict_last (a warp-uniform policy descriptor). A per-column
// policy split (hot prefix evict_last, rest evict_first: gridlp_csr_t
// .hot_cols in round 2) was measured without gain on cfg3 and cost ~10
// instructions per gather (a per-lane descriptor moved into a uniform
// register), so it was removed; hot_cols is reserved.

// ------------------------------------------- programmatic dependent launch
// The heavy-chunk, long-row and SELL kernels of one product touch disjoint
// rows, so each lets the next one start as soon as SM slots free up
// (launch_dependents at entry) and waits for its predecessor only at its very
// end (wait), so the last kernel's completion still implies the whole
// product's. The first kernel of a product is launched normally, after the
// producer of its gather vector.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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

template <bool SUMSQ, bool STREAM = false>
struct OpStore {
  static constexpr int NRED = SUMSQ ? 1 : 0;
  double* out;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double s, const Data&, double* acc) const {
    if (STREAM)
      __stcs(out + r, s);   // running sums of a column band: read once by the next band
    else
      out[r] = s;
    if (SUMSQ) acc[0] = dadd(acc[0], dmul(s, s));
  }
};

// Partial row sums written into every group member's receive slot (peer
// exchange); the product's last CTA fences and signals the members.
struct OpPeerStore {
  static constexpr int NRED = 0;
  gridlp_peer_t pe;
  double* local;                     // optional local copy of the partial (block-local cross terms)
  int64_t base;                      // (parity * G + my_slot) * len
  int32_t total_ctas;
  using Data = Empty;
  __device__ void prepare() { base = ((int64_t)(*pe.epoch & 1u) * pe.group_size + pe.my_slot) * pe.len; }
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double s, const Data&, double*) const {
    for (int q = 0; q < pe.group_size; ++q) pe.dst[q][base + r] = s;
    if (local) local[r] = s;
  }
  // called by every CTA after its rows are written
  __device__ void cta_done() const {
    __threadfence_system();           // every thread's peer stores before the CTA's arrival
    __syncthreads();
    if (threadIdx.x == 0) {
      if (atomicAdd(pe.cta_count, 1u) == (uint32_t)total_ctas - 1u) {
        *pe.cta_count = 0u;
        __threadfence_system();
        for (int q = 0; q < pe.group_size; ++q) atomicAdd_system(pe.flag[q], 1u);
      }
    }
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
  bool uniform_bounds;     // every variable has the bounds lo[0], hi[0] (GRIDLP_F_UNIFORM_BOUNDS)
  double tau, gamma, wm, wa, lo0, hi0;
  uint64_t pf;
  struct Data { double x, c, lo, hi, x0; };
  __device__ void prepare() {
    tau = step->tau;
    gamma = step->gamma;
    halpern_weights(gamma, step->inner_k + iter, wm, wa);
    pf = policy_evict_first();
    if (uniform_bounds) {
      lo0 = lo[0];
      hi0 = hi[0];
    }
  }
  // read-once operands and the x rewrite leave L2 first; x_bar keeps the
  // normal policy: it is the next product's gather vector
  __device__ Data load(int64_t r) const {
    Data d;
    d.x = ld_once(x + r, pf); d.c = ld_stream(c + r, pf);
    if (uniform_bounds) {
      d.lo = lo0;
      d.hi = hi0;
    } else {
      d.lo = ld_stream(lo + r, pf);
      d.hi = ld_stream(hi + r, pf);
    }
    d.x0 = halpern ? ld_stream(x0 + r, pf) : 0.0;
    return d;
  }
  __device__ void row(int64_t r, double aty, const Data& d, double*) const {
    const double xh = np_clip(dsub(d.x, dmul(tau, dsub(d.c, aty))), d.lo, d.hi);
    xbar[r] = dsub(dmul(2.0, xh), d.x);
    st_hint(x + r, halpern ? halpern_mix(xh, d.x, d.x0, wm, gamma, wa) : xh, pf);
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
  uint64_t pf;
  struct Data { double y, lo, hi, y0; };
  __device__ void prepare() {
    sigma = step->sigma;
    gamma = step->gamma;
    halpern_weights(gamma, step->inner_k + iter, wm, wa);
    pf = policy_evict_first();
  }
  // y is the next product's gather vector (normal policy); bounds and
  // anchor are read once
  __device__ Data load(int64_t r) const {
    Data d;
    d.y = y[r]; d.lo = ld_stream(lo + r, pf); d.hi = ld_stream(hi + r, pf);
    d.y0 = halpern ? ld_stream(y0 + r, pf) : 0.0;
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
  const double* dr;        // row scale of a scaled LP (NULL: unscaled)
  struct Data { double y, lo, hi; };
  __device__ void prepare() {}
  __device__ Data load(int64_t r) const { return {y[r], lo[r], hi[r]}; }
  __device__ void row(int64_t r, double s, const Data& ds, double* acc) const {
    if (ax) ax[r] = s;
    Data d = ds;
    if (dr) {
      // original LP: A x = s / Dr, bounds / Dr, y = Dr y~
      const double w = dr[r];
      s = ddiv(s, w);
      d.lo = ddiv(d.lo, w);
      d.hi = ddiv(d.hi, w);
      d.y = dmul(d.y, w);
    }
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
  const double* dc;        // column scale of a scaled LP (NULL: unscaled)
  double tau;
  struct Data { double x, c, lo, hi; };
  __device__ void prepare() { tau = step->tau; }
  __device__ Data load(int64_t r) const { return {x[r], c[r], lo[r], hi[r]}; }
  __device__ void row(int64_t r, double aty, const Data& d, double* acc) const {
    // pdhg_engine.py:325-336
    const double shifted = dsub(d.x, dmul(tau, dsub(d.c, aty)));
    const double xp = np_clip(shifted, d.lo, d.hi);
    const double dx = dsub(d.x, xp);
    if (!dc) {
      const double rd = ddiv(dsub(xp, d.x), tau);
      const double rc = ddiv(dsub(xp, shifted), tau);
      acc[0] = dadd(acc[0], dmul(rd, rd));
      acc[1] = dadd(acc[1], dmul(d.c, d.x));
      acc[2] = dadd(acc[2], dmul(rc, d.x));
    } else {
      // the same evaluation on the ORIGINAL LP at x = Dc x~ (A^T y = aty / Dc,
      // c = c~ / Dc, bounds * Dc), same step tau; restart terms below stay scaled
      const double w = dc[r];
      const double xo = dmul(d.x, w);
      const double co = ddiv(d.c, w);
      const double sh = dsub(xo, dmul(tau, dsub(co, ddiv(aty, w))));
      const double xpo = np_clip(sh, dmul(d.lo, w), dmul(d.hi, w));
      const double rd = ddiv(dsub(xpo, xo), tau);
      const double rc = ddiv(dsub(xpo, sh), tau);
      acc[0] = dadd(acc[0], dmul(rd, rd));
      acc[1] = dadd(acc[1], dmul(co, xo));
      acc[2] = dadd(acc[2], dmul(rc, xo));
    }
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

struct OpDivNorm {
  static constexpr int NRED = 0;
  const double* in;
  double* out;
  const double* sumsq;
  using Data = Empty;
  __device__ void prepare() {}
  __device__ Data load(int64_t) const { return {}; }
  __device__ void row(int64_t r, double, const Data&, double*) const {
    out[r] = ddiv(in[r], __dsqrt_rn(*sumsq));
  }
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

template <class T, class = void>
struct HasCtaDone : std::false_type {};
template <class T>
struct HasCtaDone<T, std::void_t<decltype(std::declval<const T&>().cta_done())>> : std::true_type {};

template <class Op>
__device__ __forceinline__ void product_cta_done(const Op& op) {
  if constexpr (HasCtaDone<Op>::value) op.cta_done();
}

#ifndef GRIDLP_PEER_WAIT_NS
#define GRIDLP_PEER_WAIT_NS (120ull * 1000000000ull)   // default peer-wait bound: 120 s
#endif
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifndef GRIDLP_SELL_WPB
#define GRIDLP_SELL_WPB 2
#endif
constexpr int SELL_WPB = GRIDLP_SELL_WPB;   // warps (slices) per CTA
constexpr int SELL_NT = SELL_WPB * 32;
constexpr int SELL_U = 4;            // steps in flight per lane
constexpr int SELL_MINB = 48 / SELL_WPB;   // 48 warps per SM at <= 42 registers (no spills with the hinted epilogues)
#ifndef GRIDLP_HEAVY_U
#define GRIDLP_HEAVY_U SELL_U        // heavy-chunk kernel: loads in flight per thread
#endif
#ifndef LONG_U
#define LONG_U 2                     // long-row kernel: 64-entry blocks (registers -> occupancy)
#endif

// A product row's epilogue. With `terms` (canonical reductions, launch_op)
// the row's reduction terms are stored per row (terms[q * n + r]) and summed
// later in a fixed row order independent of which kernel / CTA owned the
// row; otherwise they accumulate into the thread's partials.
template <class Op>
__device__ __forceinline__ void emit_row(const Op& op, int64_t r, double s, const typename Op::Data& d,
                                         double* acc, double* __restrict__ terms, int64_t n) {
  GRIDLP_CHECK(r >= 0 && r < n, "row index outside the block");
  if constexpr (Op::NRED > 0) {
    if (terms) {
      double t[Op::NRED];
#pragma unroll
      for (int q = 0; q < Op::NRED; ++q) t[q] = 0.0;
      op.row(r, s, d, t);
#pragma unroll
      for (int q = 0; q < Op::NRED; ++q) terms[(int64_t)q * n + r] = t[q];
      return;
    }
  }
  op.row(r, s, d, acc);
}

// Deterministic per-CTA reduction of a WPB-warp CTA: warp tree, then warps
// in order, one slot per CTA.
template <class Op, int WPB>
__device__ __forceinline__ void cta_partials_n(double (&acc)[Op::NRED > 0 ? Op::NRED : 1], double* partials) {
  if constexpr (Op::NRED > 0) {
    if (!partials) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double rs[Op::NRED][WPB];
#pragma unroll
    for (int q = 0; q < Op::NRED; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) rs[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < Op::NRED; ++q) {
        double t = rs[q][0];
        for (int w = 1; w < WPB; ++w) t = dadd(t, rs[q][w]);
        partials[(int64_t)blockIdx.x * GRIDLP_MAX_RED + q] = t;
      }
    }
  }
}
template <class Op>
__device__ __forceinline__ void cta_partials(double (&acc)[Op::NRED > 0 ? Op::NRED : 1], double* partials) {
  cta_partials_n<Op, SELL_WPB>(acc, partials);
}

// Heavy rows, one CTA per chunk of GRIDLP_HEAVY_CHUNK entries: strided
// per-thread sums, warp tree, warps in order; the last-arriving chunk CTA of
// a row adds the chunk sums in chunk order (deterministic) and applies the
// fused epilogue. Launched before the slice kernel of the same product; its
// reduction partials occupy slots [0, num_chunks).
template <class Op, int VC>
__global__ void __launch_bounds__(SELL_NT) heavy_chunk_kernel(gridlp_csr_t A, const double* __restrict__ g, Op op,
                                                              double* __restrict__ partials, double* __restrict__ terms,
                                                              int cross_wait) {
  constexpr int U = GRIDLP_HEAVY_U;
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  if (cross_wait) pdl_wait();     // chained to the previous product (see launch_op)
  pdl_launch_dependents();
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t c = blockIdx.x;
  const int h = A.chunk_row[c];
  const int c0 = A.chunk_first[h];
  const int nch = A.chunk_first[h + 1] - c0;
  const int64_t p0 = (int64_t)A.long_ptr[h] + (c - c0) * (int64_t)GRIDLP_HEAVY_CHUNK;
  const int64_t pe = A.long_ptr[h + 1];
  const int64_t p1 = p0 + GRIDLP_HEAVY_CHUNK < pe ? p0 + GRIDLP_HEAVY_CHUNK : pe;
  GRIDLP_CHECK(h >= 0 && h < A.num_long_rows && c0 >= 0 && c - c0 < nch && p0 < pe && pe <= A.nnz,
               "heavy chunk outside its row / the block");
  using V = Vals<VC>;
  double s = 0.0;
  for (int64_t k0 = p0 + tid; k0 < p1; k0 += (int64_t)SELL_NT * U) {
    int cc[U];
    typename V::T vv[U];
    double xx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * SELL_NT;
      cc[u] = k < p1 ? ld_stream(A.long_cols + k, pf) : 0;
      vv[u] = k < p1 ? V::ld(A.long_vals, k, pf) : V::zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cu = V::col(cc[u]);
      GRIDLP_CHECK(k0 + (int64_t)u * SELL_NT >= p1 || (cu >= 0 && cu < A.num_cols), "heavy-row gather index");
      xx[u] = k0 + (int64_t)u * SELL_NT < p1 ? ld_gather(g + cu, pl) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + (int64_t)u * SELL_NT < p1) s = dadd(s, dmul(V::val(vv[u], cc[u]), xx[u]));
  }
  s = warp_sum(s);
  __shared__ double hs[SELL_WPB];
  if (lane == 0) hs[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double t = hs[0];
#pragma unroll
    for (int w = 1; w < SELL_WPB; ++w) t = dadd(t, hs[w]);
    bool last = true;
    if (nch > 1) {
      // last-arriving chunk CTA of the row adds the chunk sums in chunk order
      A.chunk_sums[c] = t;
      __threadfence();
      last = atomicAdd(&A.chunk_done[h], 1) == nch - 1;
      if (last) {
        __threadfence();
        t = __ldcg(A.chunk_sums + c0);
        for (int q = 1; q < nch; ++q) t = dadd(t, __ldcg(A.chunk_sums + c0 + q));
        A.chunk_done[h] = 0;   // self-reset for the next launch (stream-ordered)
      }
    }
    if (last) {
      const int row = A.long_rows[h];
      const typename Op::Data d = op.load(row);
      emit_row(op, row, t, d, acc, terms, A.num_rows);
    }
  }
  cta_partials<Op>(acc, partials);
  product_cta_done(op);
  pdl_wait();
}

// Long exact rows (light_row_max < length <= exact_row_max), one warp per
// row, longest rows first (exact_long is sorted by length). The row is
// walked in blocks of 32*U entries: the warp streams the block's values and
// column indices (coalesced), gathers x and forms the rounded products in
// parallel, parks them in shared memory, and lane 0 adds them to the running
// sum in entry order — the sequential +0.0-seeded sum of scipy's
// csr_matvec. The next block's gathers and the block after's streams are in
// flight while lane 0 runs the add chain, so a row costs about one FP64
// add latency per entry. Reduction partials follow the heavy kernel's.
template <class Op, int VC>
__global__ void __launch_bounds__(SELL_NT) long_row_kernel(gridlp_csr_t A, const double* __restrict__ g, Op op,
                                                           double* __restrict__ partials, double* __restrict__ terms,
                                                           int cross_wait) {
  constexpr int U = LONG_U;
  constexpr int B = 32 * U;
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  __shared__ double prod[SELL_WPB][B];
  if (cross_wait) pdl_wait();
  pdl_launch_dependents();
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * SELL_WPB + warp;
  if (q < A.num_exact_long) {
    const int h = A.exact_long[q];
    const int64_t p0 = A.long_ptr[h];
    const int len = A.long_ptr[h + 1] - A.long_ptr[h];
    GRIDLP_CHECK(h >= 0 && h < A.num_long_rows && len >= 0 && p0 + len <= A.nnz, "long row outside the block");
    using V = Vals<VC>;
    const int* __restrict__ cp = A.long_cols + p0;
    const int64_t vp = p0;   // value index base (codec-typed loads)
    int ca[U], cb[U];
    typename V::T va[U], vb[U];
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = 32 * u + lane, k2 = B + 32 * u + lane;
      ca[u] = k < len ? ld_stream(cp + k, pf) : 0;
      va[u] = k < len ? V::ld(A.long_vals, vp + k, pf) : V::zero();
      cb[u] = k2 < len ? ld_stream(cp + k2, pf) : 0;
      vb[u] = k2 < len ? V::ld(A.long_vals, vp + k2, pf) : V::zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cu = V::col(ca[u]);
      GRIDLP_CHECK(32 * u + lane >= len || (cu >= 0 && cu < A.num_cols), "long-row gather index");
      x[u] = 32 * u + lane < len ? ld_gather(g + cu, pl) : 0.0;
    }
    double s = A.carry ? ld_carry(A.carry + A.long_rows[h], pf) : 0.0;   // column bands: continue the chain
    for (int j0 = 0; j0 < len; j0 += B) {
      double p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) p[u] = dmul(V::val(va[u], ca[u]), x[u]);
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; ++u) prod[warp][32 * u + lane] = p[u];
      __syncwarp();
      // in flight during the add chain: gathers of block j0+B, streams of block j0+2B
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cu = V::col(cb[u]);
        GRIDLP_CHECK(j0 + B + 32 * u + lane >= len || (cu >= 0 && cu < A.num_cols), "long-row gather index");
        x[u] = j0 + B + 32 * u + lane < len ? ld_gather(g + cu, pl) : 0.0;
        ca[u] = cb[u];
        va[u] = vb[u];
        const int k = j0 + 2 * B + 32 * u + lane;
        cb[u] = k < len ? ld_stream(cp + k, pf) : 0;
        vb[u] = k < len ? V::ld(A.long_vals, vp + k, pf) : V::zero();
      }
      if (lane == 0) {
        const int cnt = len - j0 < B ? len - j0 : B;
#pragma unroll 16
        for (int t = 0; t < cnt; ++t) s = dadd(s, prod[warp][t]);
      }
    }
    if (lane == 0) {
      const int row = A.long_rows[h];
      const typename Op::Data d = op.load(row);
      emit_row(op, row, s, d, acc, terms, A.num_rows);
    }
  }
  cta_partials<Op>(acc, partials);
  product_cta_done(op);
  pdl_wait();
}

// Product + fused epilogue over the light rows of a SELL-32 block: each CTA
// owns SELL_WPB slices; its reduction partials follow the heavy and long
// kernels' in the slot array. Lane l of a slice's warp owns row 32 s + l,
// sums it in a register and applies the epilogue to it directly — no shared
// memory and no barrier on the light path.
template <class Op, int VC>
__global__ void __launch_bounds__(SELL_NT, SELL_MINB) sell32_kernel(gridlp_csr_t A, const double* __restrict__ g,
                                                                   Op op, double* __restrict__ partials,
                                                                   double* __restrict__ terms, int cross_wait) {
  constexpr int U = SELL_U;
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  if (cross_wait) pdl_wait();
  // the next product's first kernel may start on SM slots this one frees; it
  // waits for this grid's completion before touching anything it writes
  pdl_launch_dependents();
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  op.prepare();
  const uint64_t pf = policy_evict_first();
  const uint64_t pl = policy_evict_last();
  const int64_t slice = (int64_t)blockIdx.x * SELL_WPB + warp;
  if (slice < A.num_slices) {
    // lane = row & 31 (sell_plan): the lane's sum is its own row's
    const int64_t r = slice * 32 + lane;
    const int info = A.lane_info[slice * 32 + lane];
    if (info >= 0) {
      const int len = info >> 8;
      using V = Vals<VC>;
      const int64_t base = A.slice_off[slice] + lane;
      GRIDLP_CHECK((info & 31) == lane && (len == 0 || base + 32 * (int64_t)(len - 1) < A.slice_off[slice + 1]),
                   "SELL lane outside its slice");
      const int* __restrict__ cp = A.sell_cols + base;
      double s = A.carry ? ld_carry(A.carry + r, pf) : 0.0;   // column bands: continue the chain
      for (int j = 0; j < len; j += U) {
        int c[U];
        typename V::T v[U];
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = j + u < len;
          c[u] = ok ? ld_stream(cp + 32 * (j + u), pf) : 0;
          v[u] = ok ? V::ld(A.sell_vals, base + 32 * (j + u), pf) : V::zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int cu = V::col(c[u]);
          GRIDLP_CHECK(j + u >= len || (cu >= 0 && cu < A.num_cols), "SELL gather index");
          x[u] = (j + u < len) ? ld_gather(g + cu, pl) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j + u < len) s = dadd(s, dmul(V::val(v[u], c[u]), x[u]));
      }
      // epilogue operands are loaded after the sums: issuing them first costs
      // registers (occupancy) and measured slower (profiles/r1, variant 10)
      const typename Op::Data d = op.load(r);
      emit_row(op, r, s, d, acc, terms, A.num_rows);
    }
  }
  cta_partials<Op>(acc, partials);
  product_cta_done(op);
  pdl_wait();
}

// Software-pipelined SELL lanes: the same lane-owns-row sum as
// sell32_kernel, but the column/value streams of step block j+U are issued
// before the gathers of block j are consumed, so each block costs one memory
// round trip (the gathers) instead of two (streams, then the gathers that
// depend on them). More registers (fewer warps per SM): it pays on long
// lanes whose streams miss L2 (power-law rows), not on short ones.
#ifndef GRIDLP_PIPE_MINB
#define GRIDLP_PIPE_MINB (40 / GRIDLP_SELL_WPB)   // 40 warps per SM at <= 51 registers
#endif
#ifndef GRIDLP_PIPE_U
#define GRIDLP_PIPE_U SELL_U
#endif
constexpr int PIPE_MINB = GRIDLP_PIPE_MINB;
// WPB warps (slices) per CTA: SELL_WPB, or 4 for GRIDLP_CSR_WIDE_CTAS blocks
template <class Op, int VC, int WPB = SELL_WPB>
__global__ void __launch_bounds__(WPB * 32, 40 / WPB) sell32_pipe_kernel(gridlp_csr_t A, const double* __restrict__ g,
                                                                        Op op, double* __restrict__ partials,
                                                                        double* __restrict__ terms, int cross_wait) {
  constexpr int U = GRIDLP_PIPE_U;
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t slice = (int64_t)blockIdx.x * WPB + warp;
  using V = Vals<VC>;
  const uint64_t pf = policy_evict_first();
  int info = -1, len = 0;
  const int* __restrict__ cp = nullptr;
  int64_t vb = 0;   // value index base (codec-typed loads)
  int c[U];
  typename V::T v[U];
  if (slice < A.num_slices) {
    info = A.lane_info[slice * 32 + lane];
    len = info >= 0 ? info >> 8 : 0;
    const int64_t base = A.slice_off[slice] + lane;
    GRIDLP_CHECK(info < 0 || ((info & 31) == lane && (len == 0 || base + 32 * (int64_t)(len - 1) <
                                                                      A.slice_off[slice + 1])),
                 "SELL lane outside its slice");
    cp = A.sell_cols + base;
    vb = base;
  }
  // the first block's streams are constant matrix data: issued before the
  // wait on a chained predecessor product
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = u < len;
    c[u] = ok ? ld_stream(cp + 32 * u, pf) : 0;
    v[u] = ok ? V::ld(A.sell_vals, vb + 32 * u, pf) : V::zero();
  }
  if (cross_wait) pdl_wait();
  pdl_launch_dependents();
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  op.prepare();
  const uint64_t pl = policy_evict_last();
  if (info >= 0) {
    const int64_t r = slice * 32 + lane;
    double s = A.carry ? ld_carry(A.carry + r, pf) : 0.0;   // column bands: continue the chain
    for (int j = 0; j < len; j += U) {
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cu = V::col(c[u]);
        GRIDLP_CHECK(j + u >= len || (cu >= 0 && cu < A.num_cols), "SELL gather index");
        x[u] = (j + u < len) ? ld_gather(g + cu, pl) : 0.0;
      }
      int cn[U];
      typename V::T vn[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = j + U + u;
        const bool ok = k < len;
        cn[u] = ok ? ld_stream(cp + 32 * k, pf) : 0;
        vn[u] = ok ? V::ld(A.sell_vals, vb + 32 * k, pf) : V::zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j + u < len) s = dadd(s, dmul(V::val(v[u], c[u]), x[u]));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = cn[u];
        v[u] = vn[u];
      }
    }
    const typename Op::Data d = op.load(r);
    emit_row(op, r, s, d, acc, terms, A.num_rows);
  }
  cta_partials_n<Op, WPB>(acc, partials);
  product_cta_done(op);
  pdl_wait();
}

// ----------------------------------------- persistent kernel (launch-bound LPs)
// A whole chunk of iterations in ONE cooperative launch: every warp of a
// co-resident grid walks the SELL slices (lane = row, sequential sum) and the
// exact long rows (warp per row, entry-order add chain by lane 0) of the
// primal product, grid barrier, then the dual product, grid barrier, for
// n_iters iterations. Per-row arithmetic is that of sell32 / long_row, so
// the iterates are the graph path's bit for bit; what goes is the per-kernel
// launch and drain (two products of ~20k nonzeros per iteration at
// BASELINE configs[0] are a few µs of launch each). Vectors rewritten inside
// the launch are read through L2 (ld.global.cg), never the incoherent L1 /
// read-only paths. Heavy (chunked) rows are not supported: the caller falls
// back to gridlp_pdhg_iterate.
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ void grid_barrier(unsigned int* count, volatile unsigned int* gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1u) {
      *count = 0u;
      __threadfence();
      *gen = g + 1u;
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// light slices [lbeg, lend) with stride lstep (this CTA's range, warp-strided),
// then (longs) the exact long rows strided over every warp of the grid
template <class Op>
__device__ __forceinline__ void persistent_product(const gridlp_csr_t& A, const double* __restrict__ g, const Op& op,
                                                   int64_t gw, int64_t W, double* prod, int64_t lbeg, int64_t lend,
                                                   int64_t lstep, bool longs) {
  const int lane = threadIdx.x & 31;
  double acc[1] = {0.0};
  for (int64_t slice = lbeg; slice < lend; slice += lstep) {
    const int64_t r = slice * 32 + lane;
    const int info = A.lane_info[r];
    if (info < 0) continue;
    const int len = info >> 8;
    const int64_t base = A.slice_off[slice] + lane;
    double s = A.carry ? ld_cg(A.carry + r) : 0.0;
    for (int j = 0; j < len; j += SELL_U) {
      int c[SELL_U];
      double v[SELL_U], x[SELL_U];
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) {
        const bool ok = j + u < len;
        c[u] = ok ? A.sell_cols[base + 32 * (j + u)] : 0;
        v[u] = ok ? A.sell_vals[base + 32 * (j + u)] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SELL_U; ++u) x[u] = (j + u < len) ? ld_cg(g + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < SELL_U; ++u)
        if (j + u < len) s = dadd(s, dmul(v[u], x[u]));
    }
    const typename Op::Data d = op.load(r);
    op.row(r, s, d, acc);
  }
  // exact long rows: warp per row, products parked in shared memory, lane 0
  // adds them in entry order (long_row_kernel's chain)
  for (int64_t q = gw; longs && q < A.num_exact_long; q += W) {
    const int h = A.exact_long[q];
    const int64_t p0 = A.long_ptr[h];
    const int len = A.long_ptr[h + 1] - A.long_ptr[h];
    double s = A.carry ? ld_cg(A.carry + A.long_rows[h]) : 0.0;
    for (int j0 = 0; j0 < len; j0 += 32) {
      const int k = j0 + lane;
      const double pv = k < len ? dmul(A.long_vals[p0 + k], ld_cg(g + A.long_cols[p0 + k])) : 0.0;
      __syncwarp();
      prod[lane] = pv;
      __syncwarp();
      if (lane == 0) {
        const int cnt = len - j0 < 32 ? len - j0 : 32;
        for (int t = 0; t < cnt; ++t) s = dadd(s, prod[t]);
      }
    }
    if (lane == 0) {
      const int row = A.long_rows[h];
      const typename Op::Data d = op.load(row);
      op.row(row, s, d, acc);
    }
    __syncwarp();
  }
}

// coherent epilogue loads for the persistent kernel (x, y, x_bar rewritten in-launch)
struct OpPrimalCg : OpPrimal {
  __device__ Data load(int64_t r) const {
    Data d;
    d.x = ld_cg(x + r); d.c = c[r]; d.lo = lo[r]; d.hi = hi[r];
    d.x0 = halpern ? x0[r] : 0.0;
    return d;
  }
};
struct OpDualCg : OpDual {
  __device__ Data load(int64_t r) const {
    Data d;
    d.y = ld_cg(y + r); d.lo = lo[r]; d.hi = hi[r];
    d.y0 = halpern ? y0[r] : 0.0;
    return d;
  }
};

constexpr int PERSIST_TPB = 256;
constexpr int PERSIST_WARPS = PERSIST_TPB / 32;
constexpr int PERSIST_U = 8;          // gathers in flight per lane (indices come from shared memory)

// One CTA's contiguous range of light slices of one product, resident in
// shared memory for the whole launch when it fits: SELL indices and values,
// lane_info, the slice offsets, and the epilogue operands of its rows (the
// iterate itself, x or y, lives there too and is written back at the end).
struct SmemSlices {
  int64_t s0, s1;                     // slice range
  int64_t e0;                         // slice_off[s0]
  const int* cols;
  const double* vals;
  const int* info;                    // lane_info[32 (s - s0) + lane]
  const int64_t* off;                 // slice_off[s] - e0, s in [s0, s1]
  double* v[5];                       // per-row operands (op specific), row = 32 (s - s0) + lane
};

__device__ __forceinline__ void persist_range(int64_t nslices, int64_t& s0, int64_t& s1) {
  s0 = nslices * blockIdx.x / gridDim.x;
  s1 = nslices * (blockIdx.x + 1) / gridDim.x;
}

// bytes of shared memory a CTA's range needs (nv per-row operands)
__device__ __forceinline__ int64_t smem_need(const gridlp_csr_t& A, int64_t s0, int64_t s1, int nv) {
  const int64_t ent = A.slice_off[s1] - A.slice_off[s0];
  const int64_t rows = 32 * (s1 - s0);
  return 12 * ent + 4 * rows + 8 * (s1 - s0 + 1) + 8 * nv * rows + 64;
}

// carve + fill (all threads); returns the bytes used
__device__ int64_t smem_stage(const gridlp_csr_t& A, int64_t s0, int64_t s1, unsigned char* base, int nv,
                              const double* const* src, SmemSlices& S) {
  const int64_t e0 = A.slice_off[s0];
  const int64_t ent = A.slice_off[s1] - e0;
  const int64_t rows = 32 * (s1 - s0);
  unsigned char* p = base;
  double* vals = reinterpret_cast<double*>(p);
  p += 8 * ent;
  for (int q = 0; q < nv; ++q) {
    S.v[q] = reinterpret_cast<double*>(p);
    p += 8 * rows;
  }
  int64_t* off = reinterpret_cast<int64_t*>(p);
  p += 8 * (s1 - s0 + 1);
  int* cols = reinterpret_cast<int*>(p);
  p += 4 * ent;
  int* info = reinterpret_cast<int*>(p);
  p += 4 * rows;
  for (int64_t k = threadIdx.x; k < ent; k += blockDim.x) {
    vals[k] = A.sell_vals[e0 + k];
    cols[k] = A.sell_cols[e0 + k];
  }
  for (int64_t k = threadIdx.x; k <= s1 - s0; k += blockDim.x) off[k] = A.slice_off[s0 + k] - e0;
  for (int64_t k = threadIdx.x; k < rows; k += blockDim.x) {
    const int64_t r = 32 * s0 + k;
    info[k] = A.lane_info[r];
    for (int q = 0; q < nv; ++q) S.v[q][k] = (src[q] && r < A.num_rows) ? src[q][r] : 0.0;
  }
  S.s0 = s0; S.s1 = s1; S.e0 = e0; S.cols = cols; S.vals = vals; S.info = info; S.off = off;
  return (int64_t)(p - base);
}

// sequential sum of one lane's row from the staged slice (sell32's order)
__device__ __forceinline__ double smem_row_sum(const SmemSlices& S, int64_t ls, int lane, int len,
                                               const double* __restrict__ g, double s) {
  const int64_t base = S.off[ls] + lane;
  for (int j = 0; j < len; j += PERSIST_U) {
    double x[PERSIST_U];
#pragma unroll
    for (int u = 0; u < PERSIST_U; ++u) x[u] = (j + u < len) ? ld_cg(g + S.cols[base + 32 * (j + u)]) : 0.0;
#pragma unroll
    for (int u = 0; u < PERSIST_U; ++u)
      if (j + u < len) s = dadd(s, dmul(S.vals[base + 32 * (j + u)], x[u]));
  }
  return s;
}

__global__ void __launch_bounds__(PERSIST_TPB) persistent_iterate_kernel(gridlp_csr_t AT, gridlp_csr_t A,
                                                                        OpPrimalCg pop, OpDualCg dop, int32_t n_iters,
                                                                        unsigned int* bar, gridlp_step_t* step,
                                                                        int64_t smem_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double prod[PERSIST_WARPS][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * PERSIST_WARPS;
  const int64_t gw = (int64_t)blockIdx.x * PERSIST_WARPS + warp;
  volatile unsigned int* gen = bar + 1;
  // this CTA's light slices of both products, staged in shared memory when
  // they fit (uniform per CTA); rows of long / heavy-free exact long rows stay
  // in global memory (warp per row, strided over the grid)
  int64_t ps0, ps1, ds0, ds1;
  persist_range(AT.num_slices, ps0, ps1);
  persist_range(A.num_slices, ds0, ds1);
  // primal operands: x, c, lo, hi, x0; dual: y, lo, hi, y0
  const bool staged = smem_need(AT, ps0, ps1, 5) + smem_need(A, ds0, ds1, 4) <= smem_bytes;
  SmemSlices P{}, D{};
  if (staged) {
    const double* psrc[5] = {pop.x, pop.c, pop.lo, pop.hi, pop.halpern ? pop.x0 : nullptr};
    const double* dsrc[4] = {dop.y, dop.lo, dop.hi, dop.halpern ? dop.y0 : nullptr};
    const int64_t used = smem_stage(AT, ps0, ps1, smem, 5, psrc, P);
    smem_stage(A, ds0, ds1, smem + ((used + 15) & ~int64_t(15)), 4, dsrc, D);
    __syncthreads();
  }
  for (int32_t t = 0; t < n_iters; ++t) {
    OpPrimalCg p = pop;
    p.iter = t;
    p.prepare();
    if (staged) {
      for (int64_t ls = warp; ls < ps1 - ps0; ls += PERSIST_WARPS) {
        const int64_t k = 32 * ls + lane;
        const int info = P.info[k];
        if (info < 0) continue;
        const int64_t r = 32 * (ps0 + ls) + lane;
        const double aty = smem_row_sum(P, ls, lane, info >> 8, dop.y, AT.carry ? ld_cg(AT.carry + r) : 0.0);
        // OpPrimal::row on the staged operands (x kept in shared memory)
        const double xv = P.v[0][k];
        const double xh = np_clip(dsub(xv, dmul(p.tau, dsub(P.v[1][k], aty))), P.v[2][k], P.v[3][k]);
        p.xbar[r] = dsub(dmul(2.0, xh), xv);
        P.v[0][k] = p.halpern ? halpern_mix(xh, xv, P.v[4][k], p.wm, p.gamma, p.wa) : xh;
      }
    } else {
      persistent_product(AT, (const double*)dop.y, p, gw, W, prod[warp], ps0 + warp, ps1, PERSIST_WARPS,
                         false);                                              // K1 gathers y
    }
    persistent_product(AT, (const double*)dop.y, p, gw, W, prod[warp], 0, 0, 1, true);    // exact long rows
    grid_barrier(bar, gen, gridDim.x);
    OpDualCg d = dop;
    d.iter = t;
    d.prepare();
    if (staged) {
      for (int64_t ls = warp; ls < ds1 - ds0; ls += PERSIST_WARPS) {
        const int64_t k = 32 * ls + lane;
        const int info = D.info[k];
        if (info < 0) continue;
        const int64_t r = 32 * (ds0 + ls) + lane;
        const double z = smem_row_sum(D, ls, lane, info >> 8, pop.xbar, A.carry ? ld_cg(A.carry + r) : 0.0);
        const double yv = D.v[0][k];
        const double yh = dual_map(yv, z, d.sigma, D.v[1][k], D.v[2][k]);
        const double yn = d.halpern ? halpern_mix(yh, yv, D.v[3][k], d.wm, d.gamma, d.wa) : yh;
        D.v[0][k] = yn;
        d.y[r] = yn;                    // the next primal product gathers y
      }
    } else {
      persistent_product(A, (const double*)pop.xbar, d, gw, W, prod[warp], ds0 + warp, ds1, PERSIST_WARPS,
                         false);                                              // K2 gathers x_bar
    }
    persistent_product(A, (const double*)pop.xbar, d, gw, W, prod[warp], 0, 0, 1, true);
    grid_barrier(bar, gen, gridDim.x);
  }
  if (staged) {
    // the primal iterate lived in shared memory: write it back
    for (int64_t k = threadIdx.x; k < 32 * (ps1 - ps0); k += blockDim.x) {
      const int64_t r = 32 * ps0 + k;
      if (r < AT.num_rows && P.info[k] >= 0) pop.x[r] = P.v[0][k];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) step->inner_k += n_iters;
}

// ------------------------------------------------ cluster kernel (tiny LPs)
// For LPs whose vectors and matrix fit in one thread-block cluster's shared
// memory (BASELINE configs[0]: 2k x 4k, 20k nonzeros), a chunk of iterations
// runs in ONE cluster launch with no global-memory round trip per product:
// every CTA holds a replica of x_bar and y, and its contiguous range of both
// matrices' SELL slices with the row operands; a product's gathers read the
// local replica, the owner lane of a row broadcasts its new x_bar / y entry
// into every CTA's replica through distributed shared memory, and a hardware
// cluster barrier (release / acquire) separates the products. Per-row
// arithmetic is sell32's (sequential sums, the same epilogue functions), so
// iterates are the graph path's bit for bit.
namespace cg = cooperative_groups;
constexpr int CLUSTER_CTAS = 8;      // portable cluster size (16 measured: 4.68 µs/iteration on cfg1)
constexpr int CLUSTER_TPB = 512;
constexpr int CLUSTER_WARPS = CLUSTER_TPB / 32;

// a lane's sequential row sum from shared memory: indices, then the replica
// values, PERSIST_U entries at a time in flight, then the in-order add chain
__device__ __forceinline__ double cluster_row_sum(const SmemSlices& S, int64_t base, int len, const double* rep) {
  double s = 0.0;
  for (int j = 0; j < len; j += PERSIST_U) {
    int c[PERSIST_U];
    double x[PERSIST_U], v[PERSIST_U];
#pragma unroll
    for (int u = 0; u < PERSIST_U; ++u) c[u] = (j + u < len) ? S.cols[base + 32 * (j + u)] : 0;
#pragma unroll
    for (int u = 0; u < PERSIST_U; ++u) {
      x[u] = rep[c[u]];
      v[u] = (j + u < len) ? S.vals[base + 32 * (j + u)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PERSIST_U; ++u)
      if (j + u < len) s = dadd(s, dmul(v[u], x[u]));
  }
  return s;
}

// slice ranges of the CTAs, balanced by SELL entries (host: cluster_plan)
struct ClusterPlan {
  int64_t pb[CLUSTER_CTAS + 1];       // primal product (A^T) slice boundaries
  int64_t db[CLUSTER_CTAS + 1];       // dual product (A) slice boundaries
};

// The KKT / restart-probe pass fused into the cluster launch (gridlp_pdhg_iterate_cluster
// with a gridlp_cluster_kkt_t): the three products of the pass read the same
// shared-memory slices; each row's reduction terms go to the caller's term
// buffers in the layout of gridlp_red_t.terms, reduced afterwards by
// gridlp_reduce_terms exactly as the unfused ops reduce them.
struct ClusterKkt {
  int32_t mode;            // 0 none, 1 KKT rows + cols, 2 + restart probe
  double* t_rows;          // [4 m]
  double* t_cols;          // [4 n]
  double* t_probe;         // [2 m]
  double* ax;              // [m]  A x (the probe's cross term)
  double* xpb;             // [n]  x_probe_bar
  const double* dr;        // scale vectors of a scaled LP (or NULL)
  const double* dc;
};

__global__ void __cluster_dims__(CLUSTER_CTAS, 1, 1) __launch_bounds__(CLUSTER_TPB)
    cluster_iterate_kernel(gridlp_csr_t AT, gridlp_csr_t A, OpPrimal pop, OpDual dop, int32_t n_iters,
                           gridlp_step_t* step, ClusterPlan plan, ClusterKkt kkt) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = AT.num_rows, m = A.num_rows;
  double* xbar_r = reinterpret_cast<double*>(smem);             // replica [n]
  double* y_r = xbar_r + n;                                      // replica [m]
  unsigned char* rest = reinterpret_cast<unsigned char*>(y_r + m);
  const int64_t ps0 = plan.pb[rank], ps1 = plan.pb[rank + 1], ds0 = plan.db[rank], ds1 = plan.db[rank + 1];
  SmemSlices P{}, D{};
  const double* psrc[5] = {pop.x, pop.c, pop.lo, pop.hi, pop.halpern ? pop.x0 : nullptr};
  const double* dsrc[4] = {dop.y, dop.lo, dop.hi, dop.halpern ? dop.y0 : nullptr};
  const int64_t used = smem_stage(AT, ps0, ps1, rest, 5, psrc, P);
  smem_stage(A, ds0, ds1, rest + ((used + 15) & ~int64_t(15)), 4, dsrc, D);
  for (int64_t k = threadIdx.x; k < m; k += CLUSTER_TPB) y_r[k] = dop.y[k];
  // remote replicas of every CTA in the cluster
  double* xbar_at[CLUSTER_CTAS];
  double* y_at[CLUSTER_CTAS];
#pragma unroll
  for (int q = 0; q < CLUSTER_CTAS; ++q) {
    xbar_at[q] = cluster.map_shared_rank(xbar_r, q);
    y_at[q] = cluster.map_shared_rank(y_r, q);
  }
  cluster.sync();
  for (int32_t t = 0; t < n_iters; ++t) {
    OpPrimal p = pop;
    p.iter = t;
    p.prepare();
    for (int64_t ls = warp; ls < ps1 - ps0; ls += CLUSTER_WARPS) {
      const int64_t k = 32 * ls + lane;
      const int info = P.info[k];
      if (info < 0) continue;
      const int len = info >> 8;
      const int64_t base = P.off[ls] + lane;
      const double aty = cluster_row_sum(P, base, len, y_r);
      const int64_t r = 32 * (ps0 + ls) + lane;
      const double xv = P.v[0][k];
      const double xh = np_clip(dsub(xv, dmul(p.tau, dsub(P.v[1][k], aty))), P.v[2][k], P.v[3][k]);
      const double xb = dsub(dmul(2.0, xh), xv);
      P.v[0][k] = p.halpern ? halpern_mix(xh, xv, P.v[4][k], p.wm, p.gamma, p.wa) : xh;
#pragma unroll
      for (int q = 0; q < CLUSTER_CTAS; ++q) xbar_at[q][r] = xb;
    }
    cluster.sync();
    OpDual d = dop;
    d.iter = t;
    d.prepare();
    for (int64_t ls = warp; ls < ds1 - ds0; ls += CLUSTER_WARPS) {
      const int64_t k = 32 * ls + lane;
      const int info = D.info[k];
      if (info < 0) continue;
      const int len = info >> 8;
      const int64_t base = D.off[ls] + lane;
      const double z = cluster_row_sum(D, base, len, xbar_r);
      const int64_t r = 32 * (ds0 + ls) + lane;
      const double yv = D.v[0][k];
      const double yh = dual_map(yv, z, d.sigma, D.v[1][k], D.v[2][k]);
      const double yn = d.halpern ? halpern_mix(yh, yv, D.v[3][k], d.wm, d.gamma, d.wa) : yh;
      D.v[0][k] = yn;
#pragma unroll
      for (int q = 0; q < CLUSTER_CTAS; ++q) y_at[q][r] = yn;
    }
    cluster.sync();
  }
  // owners write the iterates back (x_bar for completeness: the next chunk
  // recomputes it before use)
  for (int64_t k = threadIdx.x; k < 32 * (ps1 - ps0); k += CLUSTER_TPB) {
    const int64_t r = 32 * ps0 + k;
    if (r < n && P.info[k] >= 0) {
      pop.x[r] = P.v[0][k];
      pop.xbar[r] = xbar_r[r];
    }
  }
  for (int64_t k = threadIdx.x; k < 32 * (ds1 - ds0); k += CLUSTER_TPB) {
    const int64_t r = 32 * ds0 + k;
    if (r < m && D.info[k] >= 0) dop.y[r] = D.v[0][k];
  }
  if (kkt.mode > 0) {
    // x into the x_bar replicas (x_bar was written back above); the y
    // replicas already hold the final y
    cluster.sync();
    for (int64_t ls = warp; ls < ps1 - ps0; ls += CLUSTER_WARPS) {
      const int64_t k = 32 * ls + lane;
      if (P.info[k] < 0) continue;
      const int64_t r = 32 * (ps0 + ls) + lane;
#pragma unroll
      for (int q = 0; q < CLUSTER_CTAS; ++q) xbar_at[q][r] = P.v[0][k];
    }
    cluster.sync();
    // KKT rows: A x, range violation and bound penalty per row (OpKktRows)
    OpKktRows kr{dop.y, dop.lo, dop.hi, kkt.ax, kkt.dr};
    for (int64_t ls = warp; ls < ds1 - ds0; ls += CLUSTER_WARPS) {
      const int64_t k = 32 * ls + lane;
      const int info = D.info[k];
      if (info < 0) continue;
      const int64_t r = 32 * (ds0 + ls) + lane;
      const double sx = cluster_row_sum(D, D.off[ls] + lane, info >> 8, xbar_r);
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      kr.row(r, sx, OpKktRows::Data{D.v[0][k], D.v[1][k], D.v[2][k]}, t);
#pragma unroll
      for (int q = 0; q < 4; ++q) kkt.t_rows[(int64_t)q * m + r] = t[q];
    }
    // KKT cols: A^T y, the projected-gradient terms and x_probe_bar (OpKktCols)
    OpKktCols kc{};
    kc.x = pop.x; kc.c = pop.c; kc.lo = pop.lo; kc.hi = pop.hi; kc.xpb = kkt.xpb; kc.step = step; kc.dc = kkt.dc;
    kc.prepare();
    for (int64_t ls = warp; ls < ps1 - ps0; ls += CLUSTER_WARPS) {
      const int64_t k = 32 * ls + lane;
      const int info = P.info[k];
      if (info < 0) continue;
      const int64_t r = 32 * (ps0 + ls) + lane;
      const double aty = cluster_row_sum(P, P.off[ls] + lane, info >> 8, y_r);
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      kc.row(r, aty, OpKktCols::Data{P.v[0][k], P.v[1][k], P.v[2][k], P.v[3][k]}, t);
#pragma unroll
      for (int q = 0; q < 4; ++q) kkt.t_cols[(int64_t)q * n + r] = t[q];
    }
    if (kkt.mode > 1) {
      cluster.sync();                           // every CTA is done reading the x replica
      for (int64_t ls = warp; ls < ps1 - ps0; ls += CLUSTER_WARPS) {
        const int64_t k = 32 * ls + lane;
        if (P.info[k] < 0) continue;
        const int64_t r = 32 * (ps0 + ls) + lane;
        const double v = kkt.xpb[r];            // this thread's own write above
#pragma unroll
        for (int q = 0; q < CLUSTER_CTAS; ++q) xbar_at[q][r] = v;
      }
      cluster.sync();
      // restart probe: A x_probe_bar, the dual map and its norms (OpProbe)
      OpProbe pr{};
      pr.y = dop.y; pr.lo = dop.lo; pr.hi = dop.hi; pr.ax = kkt.ax; pr.dy_out = nullptr; pr.step = step;
      pr.prepare();
      for (int64_t ls = warp; ls < ds1 - ds0; ls += CLUSTER_WARPS) {
        const int64_t k = 32 * ls + lane;
        const int info = D.info[k];
        if (info < 0) continue;
        const int64_t r = 32 * (ds0 + ls) + lane;
        const double z = cluster_row_sum(D, D.off[ls] + lane, info >> 8, xbar_r);
        double t[2] = {0.0, 0.0};
        pr.row(r, z, OpProbe::Data{D.v[0][k], D.v[1][k], D.v[2][k], kkt.ax[r]}, t);
        kkt.t_probe[r] = t[0];
        kkt.t_probe[m + r] = t[1];
      }
    }
    cluster.sync();                             // no CTA leaves while others read its replicas
  }
  if (rank == 0 && threadIdx.x == 0) step->inner_k += n_iters;
}

// Row-wise epilogue over ascending-order sums of partial vectors.
template <class Op>
__global__ void __launch_bounds__(TPB) rows_kernel(gridlp_src_t src, int64_t n, Op op,
                                                   double* __restrict__ partials, gridlp_peer_t pe) {
  constexpr int NR = Op::NRED > 0 ? Op::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  op.prepare();
  if (src.peer) {
    // peer exchange (pe = *src.peer, passed by value): wait for the G
    // members' partials of this exchange, then add the slots in ascending order
    const uint32_t e = *pe.epoch;
    if (threadIdx.x == 0) {
      const uint32_t target = (e + 1u) * (uint32_t)pe.group_size;
      const uint64_t limit = pe.timeout_ns > 0 ? (uint64_t)pe.timeout_ns : GRIDLP_PEER_WAIT_NS;
      const uint64_t t0 = global_ns();
      uint32_t v;
      while (true) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pe.my_flag) : "memory");
        if ((int32_t)(v - target) >= 0) break;
        // a member that never arrives within collective_timeout_seconds is a
        // dead or diverged peer: fail the launch (cudaErrorLaunchFailure, the
        // host maps it to CollectiveTimeout) instead of hanging the device
        if (global_ns() - t0 > limit) __trap();
        __nanosleep(256);
      }
    }
    __syncthreads();
    const double* __restrict__ slots = pe.recv + (int64_t)(e & 1u) * pe.group_size * pe.len;
    for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
      const typename Op::Data d = op.load(r);
      double s = __ldcv(slots + r);
      for (int q = 1; q < pe.group_size; ++q) s = dadd(s, __ldcv(slots + (int64_t)q * pe.len + r));
      op.row(r, s, d, acc);
    }
    store_partials<Op>(acc, partials);
    return;
  }
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

__global__ void epoch_advance_kernel(uint32_t* epoch) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *epoch += 1u;
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

// Canonical reduction of per-row terms (emit_row): the same grid-stride row
// partition and tree as rows_kernel, so a fused product's reductions do not
// depend on its layout (row classes, light_row_max, column bands) and equal
// those of the partial-sum path for the same rows.
template <int NR>
__global__ void __launch_bounds__(TPB) terms_reduce_kernel(const double* __restrict__ terms, int64_t n,
                                                           double* __restrict__ partials) {
  double acc[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) acc[q] = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * TPB + threadIdx.x; r < n; r += (int64_t)gridDim.x * TPB) {
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = dadd(acc[q], terms[(int64_t)q * n + r]);
  }
  __shared__ double scratch[NR][WARPS];
  block_sum<NR>(acc, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NR; ++q) partials[(int64_t)blockIdx.x * GRIDLP_MAX_RED + q] = acc[q];
  }
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
  if (A->num_rows < 0 || A->num_cols < 0 || A->nnz < 0 || A->num_slices < 0 || A->num_long_rows < 0 ||
      A->num_chunks < 0 || A->num_exact_long < 0 || A->num_exact_long > A->num_long_rows)
    return fail(GRIDLP_ERR_ARG, "negative or inconsistent matrix dimension");
  if (A->nnz >= (int64_t(1) << 31)) return fail(GRIDLP_ERR_ARG, "block nnz must be < 2^31");
  if (A->light_row_max < 0 || A->exact_row_max < A->light_row_max || A->exact_row_max > GRIDLP_ROW_MAX_LIMIT)
    return fail(GRIDLP_ERR_ARG, "need 0 <= light_row_max <= exact_row_max <= GRIDLP_ROW_MAX_LIMIT");
  if (A->num_exact_long > 0 && !A->exact_long) return fail(GRIDLP_ERR_ARG, "missing exact_long");
  if (A->num_slices != (A->num_rows + 31) / 32) return fail(GRIDLP_ERR_ARG, "num_slices must be ceil(rows/32)");
  if (A->num_rows > 0 && (!A->slice_off || !A->lane_info)) return fail(GRIDLP_ERR_ARG, "missing SELL slices");
  if (A->val_codec < GRIDLP_VALS_F64 || A->val_codec > GRIDLP_VALS_UNIT)
    return fail(GRIDLP_ERR_ARG, "unknown val_codec");
  const bool need_vals = A->val_codec != GRIDLP_VALS_UNIT;
  if (A->nnz > 0 && (!A->sell_cols || (need_vals && !A->sell_vals)))
    return fail(GRIDLP_ERR_ARG, "missing SELL arrays");
  if (A->num_long_rows > 0 && (!A->long_rows || !A->long_ptr || !A->long_cols || (need_vals && !A->long_vals)))
    return fail(GRIDLP_ERR_ARG, "missing long-row CSR");
  if (A->num_chunks > 0 && (!A->chunk_first || !A->chunk_row || !A->chunk_sums || !A->chunk_done))
    return fail(GRIDLP_ERR_ARG, "missing heavy-row chunk directory");
  return GRIDLP_OK;
}

int64_t long_blocks(const gridlp_csr_t* A) { return (A->num_exact_long + SELL_WPB - 1) / SELL_WPB; }

// ---- light-row kernel variant (gridlp_set_tuning "sell_variant"):
//  0 = sell32_kernel, 1 = sell32_pipe_kernel (streams one step block ahead).
// (Requesting the epilogue operands before the gathers was measured slower
// in an interleaved A/B: profiles/r2/ab_sell_variant_cfg*.json.)
// (TMA-staged streams with persistent warps were measured 1.9-2.3x slower on
// cfg2 / cfg3 and removed: profiles/r2/ncu_cfg2_tma_8x2_dual_rejected.md.)
int g_sell_variant = 1;
int g_chain_products = 1;           // pdhg_iterate: programmatic launch between products
int g_wide_ctas = 1;                // honour GRIDLP_CSR_WIDE_CTAS (0: always SELL_WPB-warp CTAs)

int64_t light_blocks(const gridlp_csr_t* A) {
  return A->num_slices > 0 ? (A->num_slices + SELL_WPB - 1) / SELL_WPB : 0;
}

// CTAs (= reduction slots) of one product
int64_t sell_blocks(const gridlp_csr_t* A) {
  return A->num_rows > 0 ? A->num_chunks + long_blocks(A) + light_blocks(A) : 0;
}

int64_t src_rows(const gridlp_src_t* src) { return src->A ? src->A->num_rows : src->num_rows; }

// Launch one of a product's kernels. `programmatic` marks a programmatic
// dependency on the previous kernel in the stream: a sibling of the same
// product (disjoint rows; the kernel waits for it only at its end), or —
// with cross_wait — the last kernel of the previous product, which the
// kernel waits for before its first dependent access.
template <class K, class Op>
cudaError_t launch_part(K kern, int64_t blocks, int threads, int smem, bool programmatic, int cross_wait,
                        cudaStream_t s, const gridlp_csr_t& M, const double* gather, Op op, double* partials,
                        double* terms) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  if (programmatic) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, M, gather, op, partials, terms, cross_wait);
}

template <class Op, int VC>
cudaError_t launch_light(int64_t blocks, bool programmatic, int cross_wait, cudaStream_t s, const gridlp_csr_t& M,
                         const double* gather, Op op, double* partials, double* terms) {
  if constexpr (Op::NRED == 0 && !HasCtaDone<Op>::value) {
    // main-loop products over blocks of very short rows: 4-warp CTAs (not for
    // ops that count their CTAs, e.g. the peer store's arrival protocol)
    if (g_sell_variant == 1 && g_wide_ctas && (M.launch_flags & GRIDLP_CSR_WIDE_CTAS) && SELL_WPB < 4) {
      return launch_part(&sell32_pipe_kernel<Op, VC, 4>, (M.num_slices + 3) / 4, 128, 0, programmatic, cross_wait,
                         s, M, gather, op, partials, terms);
    }
  }
  if (g_sell_variant == 1)
    return launch_part(&sell32_pipe_kernel<Op, VC>, blocks, SELL_NT, 0, programmatic, cross_wait, s, M, gather, op,
                       partials, terms);
  return launch_part(&sell32_kernel<Op, VC>, blocks, SELL_NT, 0, programmatic, cross_wait, s, M, gather, op,
                     partials, terms);
}

// The up-to-three kernels of one product over block M (heavy chunks, exact
// long rows, SELL lanes), for value codec VC.
template <class Op, int VC>
cudaError_t launch_product(const gridlp_csr_t& M, int64_t slots, bool cross, cudaStream_t s, const double* gather,
                           Op op, double* kpartials, double* terms) {
  const int64_t nlong = long_blocks(&M);
  const int64_t nlight = slots - M.num_chunks - nlong;
  bool prev = cross;           // programmatic edge to the previous kernel
  int cw = cross ? 1 : 0;      // the first kernel launched waits for the previous product
  cudaError_t e = cudaSuccess;
  if (M.num_chunks > 0) {
    e = launch_part(&heavy_chunk_kernel<Op, VC>, M.num_chunks, SELL_NT, 0, prev, cw, s, M, gather, op, kpartials,
                    terms);
    prev = true;
    cw = 0;
  }
  if (e == cudaSuccess && nlong > 0) {
    e = launch_part(&long_row_kernel<Op, VC>, nlong, SELL_NT, 0, prev, cw, s, M, gather, op,
                    kpartials ? kpartials + M.num_chunks * GRIDLP_MAX_RED : nullptr, terms);
    prev = true;
    cw = 0;
  }
  if (e == cudaSuccess && nlight > 0)
    e = launch_light<Op, VC>(nlight, prev, cw, s, M, gather, op,
                             kpartials ? kpartials + (M.num_chunks + nlong) * GRIDLP_MAX_RED : nullptr, terms);
  return e;
}

// One op. `cross`: the product's first kernel is chained to the previous
// product on the stream by programmatic dependent launch (pdhg_iterate only:
// there the previous kernel is always the last kernel of a product).
template <class Op>
int launch_op(const gridlp_src_t* src, Op op, const gridlp_red_t* red, void* stream,
              const char* name, bool cross = false) {
  if (!src) return fail(GRIDLP_ERR_ARG, std::string(name) + ": null source");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = src_rows(src);
  int64_t slots;
  if (src->A) {
    int rc = check_csr(src->A);
    if (rc) return rc;
    if (src->A->num_rows > 0 && src->A->nnz > 0 && !src->gather)
      return fail(GRIDLP_ERR_ARG, std::string(name) + ": missing gather vector");
    slots = sell_blocks(src->A);
  } else {
    if (src->peer) {
      const gridlp_peer_t* pe = src->peer;
      if (pe->group_size < 1 || pe->group_size > GRIDLP_MAX_PARTS || !pe->recv || !pe->my_flag || !pe->epoch ||
          pe->len != n)
        return fail(GRIDLP_ERR_ARG, std::string(name) + ": inconsistent peer source");
    }
    if (src->nparts < 0 || src->nparts > GRIDLP_MAX_PARTS)
      return fail(GRIDLP_ERR_ARG, std::string(name) + ": nparts out of range");
    for (int q = 0; q < src->nparts; ++q)
      if (!src->parts[q] && n > 0) return fail(GRIDLP_ERR_ARG, std::string(name) + ": null part");
    slots = n > 0 ? rows_blocks(n) : 0;
  }
  double* partials = nullptr;
  double* terms = nullptr;
  int64_t red_slots = slots;
  if (Op::NRED > 0) {
    if (!red || !red->out) return fail(GRIDLP_ERR_ARG, std::string(name) + ": reduction output required");
    // canonical reductions for fused products when the caller passes a
    // per-row term buffer (see gridlp_red_t)
    if (src->A && n > 0 && red->terms && red->terms_capacity >= n * Op::NRED && red->partials &&
        red->capacity >= rows_blocks(n)) {
      terms = red->terms;
      red_slots = rows_blocks(n);
      partials = red->partials;
    } else if (slots > 0) {
      if (!red->partials || red->capacity < slots)
        return fail(GRIDLP_ERR_WORKSPACE, std::string(name) + ": reduction workspace too small (need " +
                                              std::to_string(slots) + " slots)");
      partials = red->partials;
    }
  }
  double* kpartials = terms ? nullptr : partials;   // product kernels' CTA partials
  if (slots > 0) {
    if (src->A) {
      const gridlp_csr_t& M = *src->A;
      cudaError_t e;
      if (M.val_codec == GRIDLP_VALS_UNIT)
        e = launch_product<Op, GRIDLP_VALS_UNIT>(M, slots, cross, s, src->gather, op, kpartials, terms);
      else if (M.val_codec == GRIDLP_VALS_F32)
        e = launch_product<Op, GRIDLP_VALS_F32>(M, slots, cross, s, src->gather, op, kpartials, terms);
      else
        e = launch_product<Op, GRIDLP_VALS_F64>(M, slots, cross, s, src->gather, op, kpartials, terms);
      if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
    } else
      rows_kernel<Op><<<(unsigned)slots, TPB, 0, s>>>(*src, n, op, partials,
                                                      src->peer ? *src->peer : gridlp_peer_t{});
    int rc = check_launch(name);
    if (rc) return rc;
  }
  if (Op::NRED > 0) {
    if (terms) {
      terms_reduce_kernel<(Op::NRED > 0 ? Op::NRED : 1)><<<(unsigned)red_slots, TPB, 0, s>>>(terms, n, partials);
      int rc = check_launch(name);
      if (rc) return rc;
    }
    reduce_kernel<<<1, TPB, 0, s>>>(partials, red_slots, Op::NRED, red->out);
    int rc = check_launch(name);
    if (rc) return rc;
  }
  if (!src->A && src->peer) {
    epoch_advance_kernel<<<1, 32, 0, s>>>(src->peer->epoch);
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

}  // namespace

// ===================================================================== C ABI
extern "C" {

int gridlp_abi_version(void) { return GRIDLP_ABI_VERSION; }

int gridlp_build_flags(void) {
#ifdef GRIDLP_CHECKED
  return GRIDLP_BUILD_CHECKED;
#else
  return 0;
#endif
}

const char* gridlp_last_error(void) { return g_err.c_str(); }

// not part of the header: lets the setup translation unit share the error slot
void gridlp_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

int gridlp_enable_peer_access(int peer_device) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("enable_peer_access: ") + cudaGetErrorString(e));
  if (peer_device == dev) return GRIDLP_OK;
  int can = 0;
  e = cudaDeviceCanAccessPeer(&can, dev, peer_device);
  if (e != cudaSuccess || !can) return fail(GRIDLP_ERR_CUDA, "enable_peer_access: no P2P path between the devices");
  e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return GRIDLP_OK;
  }
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("enable_peer_access: ") + cudaGetErrorString(e));
  return GRIDLP_OK;
}

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

int gridlp_set_tuning(const char* key, int64_t value) {
  if (!key) return fail(GRIDLP_ERR_ARG, "set_tuning: null key");
  const std::string k(key);
  if (k == "sell_variant") {
    if (value < 0 || value > 1) return fail(GRIDLP_ERR_ARG, "set_tuning: sell_variant must be 0 or 1");
    g_sell_variant = (int)value;
  } else if (k == "chain_products") {
    g_chain_products = value != 0;
  } else if (k == "wide_ctas") {
    g_wide_ctas = value != 0;
  } else {
    return fail(GRIDLP_ERR_ARG, "set_tuning: unknown key " + k);
  }
  return GRIDLP_OK;
}

int64_t gridlp_get_tuning(const char* key) {
  if (!key) return -1;
  const std::string k(key);
  if (k == "sell_variant") return g_sell_variant;
  if (k == "chain_products") return g_chain_products;
  if (k == "wide_ctas") return g_wide_ctas;
  return -1;
}

int64_t gridlp_op_slots(const gridlp_src_t* src) {
  if (!src) return 0;
  if (src->A) return sell_blocks(src->A);
  return src->num_rows > 0 ? rows_blocks(src->num_rows) : 0;
}

int gridlp_op_store(const gridlp_src_t* src, double* out, uint32_t flags, const gridlp_red_t* red,
                    void* stream) {
  if (!src) return fail(GRIDLP_ERR_ARG, "op_store: null source");
  if (!out && src_rows(src) > 0) return fail(GRIDLP_ERR_ARG, "op_store: null output");
  if (flags & GRIDLP_F_SUMSQ) return launch_op(src, OpStore<true>{out}, red, stream, "op_store");
  if (flags & GRIDLP_F_STREAM) return launch_op(src, OpStore<false, true>{out}, red, stream, "op_store");
  return launch_op(src, OpStore<false>{out}, red, stream, "op_store");
}

int gridlp_op_store_peer(const gridlp_src_t* src, const gridlp_peer_t* peer, double* local_out, void* stream) {
  if (!src || !src->A || !peer) return fail(GRIDLP_ERR_ARG, "op_store_peer: needs a product source and a peer");
  if (peer->group_size < 1 || peer->group_size > GRIDLP_MAX_PARTS || peer->my_slot < 0 ||
      peer->my_slot >= peer->group_size || peer->len != src->A->num_rows || !peer->epoch || !peer->cta_count)
    return fail(GRIDLP_ERR_ARG, "op_store_peer: inconsistent peer description");
  for (int q = 0; q < peer->group_size; ++q)
    if (!peer->dst[q] || !peer->flag[q]) return fail(GRIDLP_ERR_ARG, "op_store_peer: null member buffer");
  OpPeerStore op{};
  op.pe = *peer;
  op.local = local_out;
  op.total_ctas = (int32_t)sell_blocks(src->A);
  if (op.total_ctas == 0) {
    // no CTA would signal: signal from a one-thread kernel instead
    // (an empty block still takes part in the exchange)
    return fail(GRIDLP_ERR_ARG, "op_store_peer: empty block (no rows)");
  }
  return launch_op(src, op, nullptr, stream, "op_store_peer");
}

}  // extern "C"

namespace {
int op_primal(const gridlp_src_t* src, const gridlp_primal_t* pv, const gridlp_step_t* d_step, int32_t iter,
              uint32_t flags, void* stream, bool cross) {
  if (!pv || !d_step) return fail(GRIDLP_ERR_ARG, "op_primal: null argument");
  if (src && src_rows(src) != pv->n) return fail(GRIDLP_ERR_ARG, "op_primal: length mismatch");
  OpPrimal op{};
  op.x = pv->x; op.xbar = pv->x_bar; op.x0 = pv->x_anchor; op.c = pv->c; op.lo = pv->lo; op.hi = pv->hi;
  op.step = d_step; op.iter = iter; op.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  op.uniform_bounds = (flags & GRIDLP_F_UNIFORM_BOUNDS) != 0 && pv->n > 0;
  return launch_op(src, op, nullptr, stream, "op_primal", cross);
}

int op_dual(const gridlp_src_t* src, const gridlp_dual_t* dv, const gridlp_step_t* d_step, int32_t iter,
            uint32_t flags, void* stream, bool cross) {
  if (!dv || !d_step) return fail(GRIDLP_ERR_ARG, "op_dual: null argument");
  if (src && src_rows(src) != dv->m) return fail(GRIDLP_ERR_ARG, "op_dual: length mismatch");
  OpDual op{};
  op.y = dv->y; op.y0 = dv->y_anchor; op.lo = dv->lo; op.hi = dv->hi;
  op.step = d_step; op.iter = iter; op.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  return launch_op(src, op, nullptr, stream, "op_dual", cross);
}
}  // namespace

extern "C" {

int gridlp_op_primal(const gridlp_src_t* src, const gridlp_primal_t* pv, const gridlp_step_t* d_step,
                     int32_t iter, uint32_t flags, void* stream) {
  return op_primal(src, pv, d_step, iter, flags, stream, false);
}

int gridlp_op_dual(const gridlp_src_t* src, const gridlp_dual_t* dv, const gridlp_step_t* d_step,
                   int32_t iter, uint32_t flags, void* stream) {
  return op_dual(src, dv, d_step, iter, flags, stream, false);
}

int gridlp_op_kkt_rows(const gridlp_src_t* src, const gridlp_dual_t* dv, double* ax,
                       const gridlp_red_t* red, void* stream) {
  if (!dv) return fail(GRIDLP_ERR_ARG, "op_kkt_rows: null argument");
  if (src && src_rows(src) != dv->m) return fail(GRIDLP_ERR_ARG, "op_kkt_rows: length mismatch");
  OpKktRows op{dv->y, dv->lo, dv->hi, ax, dv->scale};
  return launch_op(src, op, red, stream, "op_kkt_rows");
}

int gridlp_op_kkt_cols(const gridlp_src_t* src, const gridlp_primal_t* pv, double* x_probe_bar,
                       const gridlp_step_t* d_step, const gridlp_red_t* red, void* stream) {
  if (!pv || !d_step) return fail(GRIDLP_ERR_ARG, "op_kkt_cols: null argument");
  if (src && src_rows(src) != pv->n) return fail(GRIDLP_ERR_ARG, "op_kkt_cols: length mismatch");
  OpKktCols op{};
  op.x = pv->x; op.c = pv->c; op.lo = pv->lo; op.hi = pv->hi; op.xpb = x_probe_bar; op.step = d_step;
  op.dc = pv->scale;
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

int gridlp_op_div_norm(const double* in, double* out, int64_t n, const double* sumsq, void* stream) {
  if (n < 0 || !sumsq || (n > 0 && (!in || !out))) return fail(GRIDLP_ERR_ARG, "op_div_norm: bad argument");
  gridlp_src_t src = rows_src(n);
  return launch_op(&src, OpDivNorm{in, out, sumsq}, nullptr, stream, "op_div_norm");
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

int gridlp_pdhg_iterate(const gridlp_src_t* primal_src, const gridlp_primal_t* pv, const gridlp_src_t* dual_src,
                        const gridlp_dual_t* dv, gridlp_step_t* d_step, int32_t n_iters, uint32_t flags,
                        void* stream) {
  if (!primal_src || !dual_src || !pv || !dv || !d_step || n_iters < 0)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate: bad argument");
  if (!primal_src->A || !dual_src->A)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate: needs fused sources (single-block axes)");
  // every product after the first is chained to its predecessor by
  // programmatic dependent launch (launch_op `cross`): its CTAs take SM slots
  // as the predecessor's tail frees them, stage their matrix streams, and
  // wait for the predecessor's completion before the first gather
  const bool chain = g_chain_products && primal_src->A->num_rows > 0 && primal_src->A->nnz > 0 &&
                     dual_src->A->num_rows > 0 && dual_src->A->nnz > 0;
  for (int32_t t = 0; t < n_iters; ++t) {
    int rc = op_primal(primal_src, pv, d_step, t, flags, stream, chain && t > 0);
    if (rc) return rc;
    rc = op_dual(dual_src, dv, d_step, t, flags, stream, chain);
    if (rc) return rc;
  }
  return n_iters > 0 ? gridlp_op_step_advance(d_step, n_iters, stream) : GRIDLP_OK;
}

int gridlp_cluster_plan(const gridlp_src_t* primal_src, const gridlp_src_t* dual_src, int64_t* plan,
                        int64_t plan_len) {
  if (!primal_src || !dual_src || !plan || plan_len < GRIDLP_CLUSTER_PLAN_LEN)
    return fail(GRIDLP_ERR_ARG, "cluster_plan: bad argument");
  const gridlp_csr_t* AT = primal_src->A;
  const gridlp_csr_t* A = dual_src->A;
  if (!AT || !A) return fail(GRIDLP_ERR_ARG, "cluster_plan: needs fused sources");
  int rc = check_csr(AT);
  if (!rc) rc = check_csr(A);
  if (rc) return rc;
  if (AT->num_cols != A->num_rows || A->num_cols != AT->num_rows)
    return fail(GRIDLP_ERR_ARG, "cluster_plan: A and A^T shapes disagree");
  if (AT->num_long_rows > 0 || A->num_long_rows > 0 || AT->carry || A->carry)
    return fail(GRIDLP_ERR_UNSUPPORTED, "cluster_plan: long rows / column bands need the graph path");
  if (AT->val_codec != GRIDLP_VALS_F64 || A->val_codec != GRIDLP_VALS_F64)
    return fail(GRIDLP_ERR_UNSUPPORTED, "cluster_plan: compact value codecs need the graph path");
  const int64_t n = AT->num_rows, m = A->num_rows;
  constexpr int64_t SMEM_MAX = 227 * 1024;
  if (8 * (n + m) + 12 * (AT->nnz + A->nnz) / CLUSTER_CTAS > SMEM_MAX || AT->num_slices > (1 << 16) ||
      A->num_slices > (1 << 16))
    return fail(GRIDLP_ERR_UNSUPPORTED, "cluster_plan: LP does not fit one cluster's shared memory");
  // entry-balanced slice ranges per CTA and the exact shared memory of the
  // largest CTA, from the slice offsets (synchronous D2H, a few KB)
  std::vector<int64_t> po(AT->num_slices + 1), dofs(A->num_slices + 1);
  if (cudaMemcpy(po.data(), AT->slice_off, 8 * po.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(dofs.data(), A->slice_off, 8 * dofs.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(GRIDLP_ERR_CUDA, "cluster_plan: slice offsets");
  auto balance = [](const std::vector<int64_t>& off, int64_t* b) {
    const int64_t ns = (int64_t)off.size() - 1;
    const int64_t total = off[ns] + 64 * ns;
    int64_t s = 0;
    b[0] = 0;
    for (int q = 1; q < CLUSTER_CTAS; ++q) {
      const int64_t target = total * q / CLUSTER_CTAS;
      while (s < ns && off[s] + 64 * s < target) ++s;
      b[q] = s;
    }
    b[CLUSTER_CTAS] = ns;
  };
  int64_t* pb = plan;
  int64_t* db = plan + CLUSTER_CTAS + 1;
  balance(po, pb);
  balance(dofs, db);
  auto need = [](const std::vector<int64_t>& off, int64_t s0, int64_t s1, int nv) {
    const int64_t rows = 32 * (s1 - s0);
    return 12 * (off[s1] - off[s0]) + 4 * rows + 8 * (s1 - s0 + 1) + 8 * nv * rows + 64;
  };
  int64_t mx = 0;
  for (int q = 0; q < CLUSTER_CTAS; ++q) {
    const int64_t x = need(po, pb[q], pb[q + 1], 5);
    const int64_t y = need(dofs, db[q], db[q + 1], 4);
    mx = std::max(mx, ((x + 15) & ~int64_t(15)) + y);
  }
  const int64_t smem = 8 * (n + m) + mx + 64;
  plan[2 * (CLUSTER_CTAS + 1)] = smem;
  if (smem > SMEM_MAX) return fail(GRIDLP_ERR_UNSUPPORTED, "cluster_plan: LP does not fit one cluster's shared memory");
  return GRIDLP_OK;
}

int gridlp_pdhg_iterate_cluster(const gridlp_src_t* primal_src, const gridlp_primal_t* pv, const gridlp_src_t* dual_src,
                                const gridlp_dual_t* dv, gridlp_step_t* d_step, int32_t n_iters, uint32_t flags,
                                const int64_t* plan, const gridlp_cluster_kkt_t* kkt_pass, void* stream) {
  if (!primal_src || !dual_src || !pv || !dv || !d_step || n_iters < 0 || !plan)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate_cluster: bad argument");
  const gridlp_csr_t* AT = primal_src->A;
  const gridlp_csr_t* A = dual_src->A;
  if (!AT || !A || AT->num_rows != pv->n || A->num_rows != dv->m)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate_cluster: needs fused sources of matching lengths");
  const int64_t smem = plan[2 * (CLUSTER_CTAS + 1)];
  if (smem <= 0 || smem > 227 * 1024) return fail(GRIDLP_ERR_ARG, "pdhg_iterate_cluster: plan from gridlp_cluster_plan");
  ClusterKkt kk{};
  if (kkt_pass && kkt_pass->mode > 0) {
    if (kkt_pass->mode > 2 || !kkt_pass->t_rows || !kkt_pass->t_cols || !kkt_pass->ax || !kkt_pass->xpb ||
        (kkt_pass->mode > 1 && !kkt_pass->t_probe))
      return fail(GRIDLP_ERR_ARG, "pdhg_iterate_cluster: incomplete KKT pass buffers");
    kk.mode = kkt_pass->mode;
    kk.t_rows = kkt_pass->t_rows; kk.t_cols = kkt_pass->t_cols; kk.t_probe = kkt_pass->t_probe;
    kk.ax = kkt_pass->ax; kk.xpb = kkt_pass->xpb; kk.dr = dv->scale; kk.dc = pv->scale;
  }
  if (n_iters == 0 && kk.mode == 0) return GRIDLP_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cluster_iterate_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cluster_iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  ClusterPlan cp;
  for (int q = 0; q <= CLUSTER_CTAS; ++q) {
    cp.pb[q] = plan[q];
    cp.db[q] = plan[CLUSTER_CTAS + 1 + q];
  }
  OpPrimal pop{};
  pop.x = pv->x; pop.xbar = pv->x_bar; pop.x0 = pv->x_anchor; pop.c = pv->c; pop.lo = pv->lo; pop.hi = pv->hi;
  pop.step = d_step; pop.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  OpDual dop{};
  dop.y = dv->y; dop.y0 = dv->y_anchor; dop.lo = dv->lo; dop.hi = dv->hi;
  dop.step = d_step; dop.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CLUSTER_CTAS);
  cfg.blockDim = dim3(CLUSTER_TPB);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_iterate_kernel, *AT, *A, pop, dop, n_iters, d_step, cp, kk);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("pdhg_iterate_cluster: ") + cudaGetErrorString(e));
  return GRIDLP_OK;
}

int gridlp_reduce_terms(const double* terms, int64_t n, int32_t nred, const gridlp_red_t* red, void* stream) {
  if (n < 0 || (nred != 1 && nred != 2 && nred != 4) || !red || !red->out || (n > 0 && !terms))
    return fail(GRIDLP_ERR_ARG, "reduce_terms: bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t slots = rows_blocks(n);
  if (n > 0) {
    if (!red->partials || red->capacity < slots) return fail(GRIDLP_ERR_WORKSPACE, "reduce_terms: workspace too small");
    switch (nred) {
      case 1: terms_reduce_kernel<1><<<(unsigned)slots, TPB, 0, s>>>(terms, n, red->partials); break;
      case 2: terms_reduce_kernel<2><<<(unsigned)slots, TPB, 0, s>>>(terms, n, red->partials); break;
      default: terms_reduce_kernel<4><<<(unsigned)slots, TPB, 0, s>>>(terms, n, red->partials); break;
    }
    int rc = check_launch("reduce_terms");
    if (rc) return rc;
  }
  reduce_kernel<<<1, TPB, 0, s>>>(red->partials, n > 0 ? slots : 0, nred, red->out);
  return check_launch("reduce_terms");
}

int gridlp_iterate_graph_create(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                                const gridlp_src_t* dual_src, const gridlp_dual_t* dv, gridlp_step_t* d_step,
                                int32_t n_iters, uint32_t flags, void** graph_exec) {
  if (!graph_exec || n_iters < 1) return fail(GRIDLP_ERR_ARG, "iterate_graph_create: bad argument");
  *graph_exec = nullptr;
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("iterate_graph_create: ") + cudaGetErrorString(e));
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(cs);
    return fail(GRIDLP_ERR_CUDA, std::string("iterate_graph_create: ") + cudaGetErrorString(e));
  }
  const int rc = gridlp_pdhg_iterate(primal_src, pv, dual_src, dv, d_step, n_iters, flags, cs);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess || !g)
    return fail(GRIDLP_ERR_CUDA, std::string("iterate_graph_create: ") + cudaGetErrorString(e));
  cudaGraphExec_t ge = nullptr;
  e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("iterate_graph_create: ") + cudaGetErrorString(e));
  *graph_exec = ge;
  return GRIDLP_OK;
}

int gridlp_graph_launch(void* graph_exec, void* stream) {
  if (!graph_exec) return fail(GRIDLP_ERR_ARG, "graph_launch: null graph");
  cudaError_t e = cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("graph_launch: ") + cudaGetErrorString(e));
  return GRIDLP_OK;
}

int gridlp_graph_destroy(void* graph_exec) {
  if (graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec));
  return GRIDLP_OK;
}

// ------------------------------------------------ device-side main loop
}  // extern "C"

namespace {

struct LoopCtx {
  cudaGraph_t parent = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t stream = nullptr;
  bool capturing = false;
};

// Python's max(a, b): a unless b > a (NaN a stays, NaN b never wins)
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }

// One thread: the host's per-pass logic of PdhgEngine.step / _kkt on the
// pass's slots (single block: every axis sum is the single term), in the
// same IEEE operations and order. Sets the WHILE condition.
__global__ void loop_decide_kernel(const double* __restrict__ slots, gridlp_loop_t* L, double* __restrict__ ring,
                                   cudaGraphConditionalHandle h) {
  const int64_t p = L->passes;
  const int64_t K = L->kkt_interval;
  const int64_t total = L->total + K;
  const int64_t inner_k = L->inner_k + K;
  const double* kr = slots + (int64_t)L->slot_rows * GRIDLP_MAX_RED;
  const double* kc = slots + (int64_t)L->slot_cols * GRIDLP_MAX_RED;
  const double* pr = slots + (int64_t)L->slot_probe * GRIDLP_MAX_RED;
  const bool restarts = L->restarts != 0;
  double* rec = ring + p * GRIDLP_LOOP_REC;
  for (int q = 0; q < 4; ++q) {
    rec[q] = kr[q];
    rec[4 + q] = kc[q];
  }
  rec[8] = restarts ? pr[0] : 0.0;
  rec[9] = restarts ? pr[1] : 0.0;
  rec[10] = 0.0;
  // _kkt: report (pdhg_engine.py:192-216, solver_driver)
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const double pen = kr[3] > 0.0 ? inf : dsub(kr[1], kr[2]);
  const double obj_p = kc[1];
  const double obj_d = dadd(-pen, kc[2]);
  const double r_p = ddiv(__dsqrt_rn(kr[0]), dadd(1.0, L->bnorm));
  const double r_d = ddiv(__dsqrt_rn(kc[0]), dadd(1.0, L->cnorm));
  double r_g;
  if (!isfinite(obj_d) || !isfinite(obj_p))
    r_g = inf;
  else
    r_g = ddiv(fabs(dsub(obj_p, obj_d)), dadd(1.0, py_max(fabs(obj_p), fabs(obj_d))));
  bool stop = !isfinite(r_p) || !isfinite(r_d) || isnan(dadd(obj_p, L->obj_const));   // _broken
  double overall = r_p;                                   // Report.overall = max(r_p, r_d, r_gap)
  if (r_d > overall) overall = r_d;
  if (r_g > overall) overall = r_g;
  if (!stop && overall <= L->tolerance) stop = true;      // optimal
  if (!stop && restarts) {
    const double eta = L->eta, om = L->omega;
    const double value = dadd(dadd(dmul(ddiv(om, eta), kc[3]), ddiv(pr[0], dmul(eta, om))), dmul(2.0, pr[1]));
    const double fp = __dsqrt_rn(py_max(value, 0.0));
    rec[10] = fp;
    const double base = L->has_base ? L->base_fp : fp;
    bool r = false;                                       // restart_decision (pdhg_engine.py:262-282)
    if (fp <= dmul(L->beta_sufficient, base))
      r = true;
    else if (L->has_prev && fp <= dmul(L->beta_necessary, base) && fp > L->prev_fp)
      r = true;
    if (!r) r = (double)inner_k >= dmul(L->beta_artificial, (double)total);
    if (r) {
      stop = true;                                        // the host applies the restart
    } else {
      L->base_fp = base;
      L->has_base = 1;
      L->prev_fp = fp;
      L->has_prev = 1;
    }
  }
  if (!stop && total + K > L->max_iterations) stop = true;   // the next interval would pass the limit
  if (!stop && p + 1 >= L->max_passes) stop = true;          // ring full
  rec[11] = stop ? 1.0 : 0.0;
  L->passes = p + 1;
  L->stopped = stop ? 1 : 0;
  if (!stop) {
    L->total = total;
    L->inner_k = inner_k;
  }
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}

}  // namespace

extern "C" {

int gridlp_loop_graph_begin(void* stream, void** ctx) {
  if (!ctx) return fail(GRIDLP_ERR_ARG, "loop_graph_begin: null ctx");
  *ctx = nullptr;
  auto* c = new LoopCtx;
  c->stream = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaGraphCreate(&c->parent, 0);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&c->handle, c->parent, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node = nullptr;
  if (e == cudaSuccess) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = c->handle;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    e = cudaGraphAddNode(&node, c->parent, nullptr, 0, &np);
    if (e == cudaSuccess) c->body = np.conditional.phGraph_out[0];
  }
  if (e == cudaSuccess)
    e = cudaStreamBeginCaptureToGraph(c->stream, c->body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    if (c->parent) cudaGraphDestroy(c->parent);
    delete c;
    return fail(GRIDLP_ERR_CUDA, std::string("loop_graph_begin: ") + cudaGetErrorString(e));
  }
  c->capturing = true;
  *ctx = c;
  return GRIDLP_OK;
}

int gridlp_loop_graph_decide(void* ctx, const double* slots, gridlp_loop_t* d_loop, double* d_ring) {
  auto* c = static_cast<LoopCtx*>(ctx);
  if (!c || !c->capturing || !slots || !d_loop || !d_ring) return fail(GRIDLP_ERR_ARG, "loop_graph_decide: bad argument");
  loop_decide_kernel<<<1, 1, 0, c->stream>>>(slots, d_loop, d_ring, c->handle);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("loop_graph_decide: ") + cudaGetErrorString(e));
  return GRIDLP_OK;
}

int gridlp_loop_graph_abort(void* ctx) {
  auto* c = static_cast<LoopCtx*>(ctx);
  if (!c) return GRIDLP_OK;
  if (c->capturing) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->stream, &g);
    cudaGetLastError();
  }
  if (c->parent) cudaGraphDestroy(c->parent);
  delete c;
  return GRIDLP_OK;
}

int gridlp_loop_graph_end(void* ctx, void** graph_exec) {
  auto* c = static_cast<LoopCtx*>(ctx);
  if (!c || !graph_exec) return fail(GRIDLP_ERR_ARG, "loop_graph_end: bad argument");
  *graph_exec = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  c->capturing = false;
  cudaGraphExec_t ge = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, c->parent, 0);
  cudaGraphDestroy(c->parent);
  delete c;
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GRIDLP_ERR_CUDA, std::string("loop_graph_end: ") + cudaGetErrorString(e));
  }
  *graph_exec = ge;
  return GRIDLP_OK;
}

size_t gridlp_persistent_scratch_bytes(void) { return 64; }

int gridlp_pdhg_iterate_persistent(const gridlp_src_t* primal_src, const gridlp_primal_t* pv,
                                   const gridlp_src_t* dual_src, const gridlp_dual_t* dv, gridlp_step_t* d_step,
                                   int32_t n_iters, uint32_t flags, void* scratch, void* stream) {
  if (!primal_src || !dual_src || !pv || !dv || !d_step || n_iters < 0 || !scratch)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate_persistent: bad argument");
  const gridlp_csr_t* AT = primal_src->A;
  const gridlp_csr_t* A = dual_src->A;
  if (!AT || !A) return fail(GRIDLP_ERR_ARG, "pdhg_iterate_persistent: needs fused sources");
  int rc = check_csr(AT);
  if (!rc) rc = check_csr(A);
  if (rc) return rc;
  if (AT->num_chunks > 0 || A->num_chunks > 0)
    return fail(GRIDLP_ERR_UNSUPPORTED, "pdhg_iterate_persistent: heavy (chunked) rows need the graph path");
  if (AT->val_codec != GRIDLP_VALS_F64 || A->val_codec != GRIDLP_VALS_F64)
    return fail(GRIDLP_ERR_UNSUPPORTED, "pdhg_iterate_persistent: compact value codecs need the graph path");
  if (AT->num_rows != pv->n || A->num_rows != dv->m)
    return fail(GRIDLP_ERR_ARG, "pdhg_iterate_persistent: length mismatch");
  if (n_iters == 0) return GRIDLP_OK;
  // one CTA per SM with up to PERSIST_SMEM of shared memory: each CTA stages
  // its slice range of both matrices there when it fits
  constexpr int PERSIST_SMEM = 200 * 1024;
  static int blocks_per_sm = 0, sms = 0;
  if (!blocks_per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(persistent_iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PERSIST_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, persistent_iterate_kernel, PERSIST_TPB,
                                                  PERSIST_SMEM);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  // enough warps for the larger product's slices (one slice per warp), never
  // more than co-resident
  const int64_t work = std::max(std::max(AT->num_slices, A->num_slices), std::max(AT->num_exact_long,
                                                                                  A->num_exact_long));
  int64_t want = (work + PERSIST_WARPS - 1) / PERSIST_WARPS;
  const int64_t cap = (int64_t)blocks_per_sm * sms;
  const int nblocks = (int)std::max<int64_t>(1, std::min(want, cap));
  int64_t smem_bytes = PERSIST_SMEM;
  OpPrimalCg pop{};
  pop.x = pv->x; pop.xbar = pv->x_bar; pop.x0 = pv->x_anchor; pop.c = pv->c; pop.lo = pv->lo; pop.hi = pv->hi;
  pop.step = d_step; pop.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  OpDualCg dop{};
  dop.y = dv->y; dop.y0 = dv->y_anchor; dop.lo = dv->lo; dop.hi = dv->hi;
  dop.step = d_step; dop.halpern = (flags & GRIDLP_F_HALPERN) != 0;
  gridlp_csr_t at = *AT, a = *A;
  unsigned int* bar = static_cast<unsigned int*>(scratch);
  void* args[] = {&at, &a, &pop, &dop, &n_iters, &bar, &d_step, &smem_bytes};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)persistent_iterate_kernel, dim3(nblocks),
                                              dim3(PERSIST_TPB), args, PERSIST_SMEM,
                                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(GRIDLP_ERR_CUDA, std::string("pdhg_iterate_persistent: ") + cudaGetErrorString(e));
  return GRIDLP_OK;
}

}  // extern "C"
