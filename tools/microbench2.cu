// Microbenchmarks for alternatives to the L1->L2 request port that bounds the
// random 8-byte gather of the FP64 CSR product:
//   smem   : gather from the CTA's own shared memory (x window in SMEM)
//   dsmem  : gather from a cluster's distributed shared memory (CS CTAs)
//   bulk16 : one 16-byte cp.async.bulk (TMA engine) per gather into SMEM
//   mixed  : half the gathers via LDG, half via cp.async.bulk
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench2 tools/microbench2.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));               \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int WIN = 24576;  // doubles per CTA window (192 KB)

__device__ __forceinline__ int ldcs(const int* p) { return __ldcs(p); }

// idx values are < WIN (local) or < CS*WIN (cluster)
template <int U>
__global__ void __launch_bounds__(1024, 1) k_smem(const int* __restrict__ idx, long n, double* out) {
  extern __shared__ double win[];
  for (int i = threadIdx.x; i < WIN; i += blockDim.x) win[i] = i * 0.5;
  __syncthreads();
  double s = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (i + u * stride < n) ? ldcs(idx + i + u * stride) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) s += win[c[u]];
  }
  if (s == 12345.678) out[0] = s;
}

template <int U, int CS>
__global__ void __launch_bounds__(1024, 1) k_dsmem(const int* __restrict__ idx, long n, double* out) {
  extern __shared__ double win[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < WIN; i += blockDim.x) win[i] = i * 0.5;
  cl.sync();
  double s = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (i + u * stride < n) ? ldcs(idx + i + u * stride) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned r = (unsigned)c[u] / WIN;
      const double* p = cl.map_shared_rank(win, r);
      s += p[c[u] - r * WIN];
    }
  }
  cl.sync();
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One 16-byte bulk copy per gather (TMA engine), U per lane in flight.
template <int U>
__global__ void __launch_bounds__(256) k_bulk16(const int* __restrict__ idx, const double* __restrict__ x, long n,
                                                double* out) {
  __shared__ __align__(16) double buf[8][32 * U * 2];
  __shared__ __align__(8) uint64_t bar[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  double s = 0;
  uint32_t phase = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (i + u * stride < n) ? ldcs(idx + i + u * stride) : 0;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w])), "r"(32 * U * 16)
                   : "memory");
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* src = x + (c[u] & ~1);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
              smem_u32(&buf[w][(u * 32 + lane) * 2])),
          "l"(src), "r"(smem_u32(&bar[w]))
          : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar[w])), "r"(phase)
          : "memory");
    phase ^= 1;
#pragma unroll
    for (int u = 0; u < U; ++u) s += buf[w][(u * 32 + lane) * 2 + (c[u] & 1)];
    __syncwarp();
  }
  if (s == 12345.678) out[0] = s;
}

// Half of each warp's gathers via LDG, half via 16-byte bulk copies.
template <int U>
__global__ void __launch_bounds__(256) k_mixed(const int* __restrict__ idx, const double* __restrict__ x, long n,
                                               double* out) {
  __shared__ __align__(16) double buf[8][32 * U * 2];
  __shared__ __align__(8) uint64_t bar[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;");
  double s = 0;
  uint32_t phase = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U * 2) {
    int c[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = (i + u * stride < n) ? ldcs(idx + i + u * stride) : 0;
      d[u] = (i + (U + u) * stride < n) ? ldcs(idx + i + (U + u) * stride) : 0;
    }
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w])), "r"(32 * U * 16)
                   : "memory");
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
              smem_u32(&buf[w][(u * 32 + lane) * 2])),
          "l"(x + (d[u] & ~1)), "r"(smem_u32(&bar[w]))
          : "memory");
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + c[u]);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar[w])), "r"(phase)
          : "memory");
    phase ^= 1;
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u] + buf[w][(u * 32 + lane) * 2 + (d[u] & 1)];
    __syncwarp();
  }
  if (s == 12345.678) out[0] = s;
}

template <class F>
float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

template <int CS>
void run_dsmem(const int* idx, long N, double* out, int sms) {
  auto kern = k_dsmem<4, CS>;
  const size_t smem = WIN * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (CS > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int tpb : {512, 1024}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(tpb);
    cfg.dynamicSmemBytes = smem;
    int nclusters = 0;
    cfg.gridDim = dim3(CS);
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters <= 0) {
      printf("dsmem CS=%d tpb=%d: occupancy query failed\n", CS, tpb);
      cudaGetLastError();
      continue;
    }
    cfg.gridDim = dim3(nclusters * CS);
    float ms = timeit([&] { CK(cudaLaunchKernelEx(&cfg, kern, idx, N, out)); });
    printf("dsmem CS=%2d tpb=%4d clusters=%3d (%d CTAs): %.1f us  %.0f Ggath/s\n", CS, tpb, nclusters,
           nclusters * CS, ms * 1e3, N / ms / 1e6);
  }
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long N = 20'000'000;
  double *x, *out;
  int* idx;
  CK(cudaMalloc(&idx, N * 4));
  CK(cudaMalloc(&x, 2'000'000L * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, 2'000'000L * 8));
  std::vector<int> h(N);
  std::mt19937 rng(1);
  // local SMEM
  for (long i = 0; i < N; ++i) h[i] = rng() % WIN;
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, WIN * 8));
  for (int tpb : {512, 1024}) {
    float ms = timeit([&] { k_smem<4><<<sms, tpb, WIN * 8>>>(idx, N, out); });
    printf("smem tpb=%4d: %.1f us  %.0f Ggath/s\n", tpb, ms * 1e3, N / ms / 1e6);
  }
  // DSMEM at several cluster sizes: idx over CS windows
  for (int cs : {2, 4, 8, 16}) {
    for (long i = 0; i < N; ++i) h[i] = rng() % (cs * WIN);
    CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
    if (cs == 2) run_dsmem<2>(idx, N, out, sms);
    if (cs == 4) run_dsmem<4>(idx, N, out, sms);
    if (cs == 8) run_dsmem<8>(idx, N, out, sms);
    if (cs == 16) run_dsmem<16>(idx, N, out, sms);
  }
  // TMA 16-byte bulk gathers from a 2M-double vector (L2-resident)
  for (long i = 0; i < N; ++i) h[i] = rng() % 2'000'000;
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  for (int bps : {4, 8}) {
    int grid = sms * bps;
    float b2 = timeit([&] { k_bulk16<2><<<grid, 256>>>(idx, x, N, out); });
    float b4 = timeit([&] { k_bulk16<4><<<grid, 256>>>(idx, x, N, out); });
    float m2 = timeit([&] { k_mixed<2><<<grid, 256>>>(idx, x, N, out); });
    float m4 = timeit([&] { k_mixed<4><<<grid, 256>>>(idx, x, N, out); });
    printf("grid=%d bulk16 U2 %.1f us (%.0f G/s) U4 %.1f us (%.0f G/s) | mixed U2 %.1f us (%.0f G/s) U4 %.1f us (%.0f G/s)\n",
           grid, b2 * 1e3, N / b2 / 1e6, b4 * 1e3, N / b4 / 1e6, m2 * 1e3, N / m2 / 1e6, m4 * 1e3, N / m4 / 1e6);
  }
  return 0;
}
