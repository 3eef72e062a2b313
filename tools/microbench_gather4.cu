// Random FP64 gathers through the TMA unit (cp.async.bulk.tensor 2D
// tile::gather4, sm_100a) vs plain ld.global gathers: is the 255 G/s
// L1->L2 request ceiling of profiles/r1/microbench_gather.log also the TMA
// path's ceiling?  x is viewed as an (n/2) x 2 tensor of doubles; one
// gather4 fetches four 16-byte rows (the wanted element and its neighbour).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb4 tools/microbench_gather4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(su32(b)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}

constexpr int WARPS = 4;

// each warp round = 128 indices: lane l gathers idx[round*128 + 4l .. +4]
template <int STAGES>
__global__ void __launch_bounds__(WARPS * 32) k_tma(const __grid_constant__ CUtensorMap tm, const int4* __restrict__ idx,
                                                    long rounds, double* out, int* err) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[WARPS][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wbuf = reinterpret_cast<double*>(sm) + (size_t)warp * STAGES * 512;  // 128-B slot per lane (TMA dst alignment)
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long gw = (long)blockIdx.x * WARPS + warp, nw = (long)gridDim.x * WARPS;
  auto issue = [&](long r, int s) {
    if (lane == 0) mbar_expect_tx(&bars[warp][s], 32 * 64);
    __syncwarp();
    int4 c = idx[r * 32 + lane];
    gather4(wbuf + s * 512 + lane * 16, &tm, &bars[warp][s], 0, c.x >> 1, c.y >> 1, c.z >> 1, c.w >> 1);
  };
  for (int s = 0; s < STAGES; ++s) {
    long r = gw + s * nw;
    if (r < rounds) issue(r, s);
  }
  double acc = 0.0;
  for (long k = 0;; ++k) {
    long r = gw + k * nw;
    if (r >= rounds) break;
    int s = (int)(k % STAGES);
    uint32_t ph = (uint32_t)((k / STAGES) & 1);
    long spin = 0;
    while (!mbar_try_wait(&bars[warp][s], ph)) {
      if (++spin > 20000000) {
        atomicExch(err, 1);
        return;
      }
    }
    int4 c = idx[r * 32 + lane];
    const double* b = wbuf + s * 512 + lane * 16;
    acc += b[0 + (c.x & 1)] + b[2 + (c.y & 1)] + b[4 + (c.z & 1)] + b[6 + (c.w & 1)];
    __syncwarp();
    long rn = gw + (k + STAGES) * nw;
    if (rn < rounds) issue(rn, s);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int U>
__global__ void __launch_bounds__(WARPS * 32) k_ld(const double* __restrict__ x, const int4* __restrict__ idx,
                                                   long rounds, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long gw = (long)blockIdx.x * WARPS + warp, nw = (long)gridDim.x * WARPS;
  double acc = 0.0;
  long r = gw;
  for (; r + (U - 1) * nw < rounds; r += U * nw) {
    int4 c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = idx[(r + u * nw) * 32 + lane];
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u][0] = __ldg(x + c[u].x);
      v[u][1] = __ldg(x + c[u].y);
      v[u][2] = __ldg(x + c[u].z);
      v[u][3] = __ldg(x + c[u].w);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u][0] + v[u][1] + v[u][2] + v[u][3];
  }
  for (; r < rounds; r += nw) {
    int4 c = idx[r * 32 + lane];
    acc += __ldg(x + c.x) + __ldg(x + c.y) + __ldg(x + c.z) + __ldg(x + c.w);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long G = 20'000'000;  // gathers (cfg2 nnz)
  const long rounds = G / 128;
  std::mt19937_64 rng(7);
  for (long n : {2'000'000L, 8'000'000L}) {
    std::vector<int> hidx(G);
    for (auto& v : hidx) v = (int)(rng() % n);
    std::vector<double> hx(n);
    for (long i = 0; i < n; ++i) hx[i] = (double)(i % 1000) * 0.001;
    double *x, *out;
    int *idx, *err;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&idx, G * 4));
    CK(cudaMalloc(&out, 64L << 20));
    CK(cudaMalloc(&err, 4));
    CK(cudaMemset(err, 0, 4));
    CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hidx.data(), G * 4, cudaMemcpyHostToDevice));
    double want = 0;
    for (long i = 0; i < G; ++i) want += hx[hidx[i]];

    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t gstride[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)cr);
      return 1;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto sum_out = [&](int nthreads) {
      std::vector<double> h(nthreads);
      cudaMemcpy(h.data(), out, nthreads * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      for (double v : h) s += v;
      return s;
    };
    for (int cps : {2, 4, 8}) {
      int grid = sms * cps;
      // plain loads
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(out, 0, 64L << 20));
        cudaEventRecord(e0);
        k_ld<4><<<grid, WARPS * 32>>>(x, (const int4*)idx, rounds, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("n=%ldM grid=%d ld.global U4: %.1f us %.0f Ggath/s  sum rel err %.1e\n", n / 1000000, grid,
                        ms * 1e3, G / (ms * 1e-3) / 1e9, (sum_out(grid * WARPS * 32) - want) / want);
      }
      // TMA gather4
      const int STAGES = 4;
      size_t smem = (size_t)WARPS * STAGES * 512 * 8;
      CK(cudaFuncSetAttribute(k_tma<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(out, 0, 64L << 20));
        cudaEventRecord(e0);
        k_tma<STAGES><<<grid, WARPS * 32, smem>>>(tm, (const int4*)idx, rounds, out, err);
        cudaEventRecord(e1);
        cudaError_t ce = cudaEventSynchronize(e1);
        if (ce != cudaSuccess) {
          printf("tma kernel error %s\n", cudaGetErrorString(ce));
          return 1;
        }
        int herr = 0;
        cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep)
          printf("n=%ldM grid=%d TMA gather4 x%d stages: %.1f us %.0f Ggath/s  sum rel err %.1e  timeout=%d\n",
                 n / 1000000, grid, STAGES, ms * 1e3, G / (ms * 1e-3) / 1e9,
                 (sum_out(grid * WARPS * 32) - want) / want, herr);
        if (herr) return 2;
      }
    }
    cudaFree(x);
    cudaFree(idx);
    cudaFree(out);
    cudaFree(err);
  }
  return 0;
}
