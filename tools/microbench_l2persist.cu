// Does an L2 set-aside (persisting access-policy window over the hottest
// prefix of the gathered vector) lift the gather rate of a vector larger
// than L2? Zipf(0.8) 8-byte gathers (the cfg3 column law, hottest first)
// over 160 MB and 80 MB vectors, uniform over 96 / 128 MB; window W MB over
// the vector's prefix (W = 0: no window), gathers plain (`ld.global.nc`) or
// L2 evict_last-hinted. Indices streamed evict-first, as the SELL streams.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_l2persist tools/microbench_l2persist.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int U, bool HINT>
__global__ void k_gather(const int* __restrict__ idx, const double* __restrict__ x, long n, double* out) {
  const uint64_t pl = pol_last(), pf = pol_first();
  double s = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int* p = idx + i + u * stride;
      int v = 0;
      if (i + u * stride < n) asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pf));
      c[u] = v;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (HINT)
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[u]) : "l"(x + c[u]), "l"(pl));
      else
        asm("ld.global.nc.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + c[u]));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0, maxp = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
  printf("{\"max_persisting_l2_mb\": %.1f}\n", maxp / 1048576.0);
  const long n = 100000000;
  int* d_idx;
  double *d_x, *d_out;
  CK(cudaMalloc(&d_idx, n * sizeof(int)));
  CK(cudaMalloc(&d_x, 512l << 20));
  CK(cudaMalloc(&d_out, 8));
  CK(cudaMemset(d_x, 0, 512l << 20));
  std::vector<int> h(n);
  std::mt19937_64 rng(1);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct Case { int law; int mb; };
  const Case cases[] = {{1, 160}, {1, 80}, {0, 96}, {0, 128}};
  const int wins[] = {0, 16, 32, 48, 64, 80, 96};
  for (const Case& cs : cases) {
    const long V = (long)cs.mb * (1l << 20) / 8;
    if (cs.law == 0) {
      std::uniform_int_distribution<long> u(0, V - 1);
      for (long i = 0; i < n; ++i) h[i] = (int)u(rng);
    } else {
      std::uniform_real_distribution<double> u(0.0, 1.0);
      const double k = std::pow((double)V + 1.0, 0.2) - 1.0;
      for (long i = 0; i < n; ++i) {
        const double j = std::pow(1.0 + u(rng) * k, 5.0) - 1.0;
        long jj = (long)j;
        h[i] = (int)(jj < V ? jj : V - 1);
      }
    }
    CK(cudaMemcpy(d_idx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    for (int w : wins) {
      if ((long)w << 20 > maxp || w > cs.mb) continue;
      for (int hint = 0; hint < 2; ++hint) {
        cudaStreamAttrValue attr = {};
        CK(cudaCtxResetPersistingL2Cache());
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)w << 20));
        attr.accessPolicyWindow.base_ptr = d_x;
        attr.accessPolicyWindow.num_bytes = (size_t)w << 20;
        attr.accessPolicyWindow.hitRatio = w ? 1.0f : 0.0f;
        attr.accessPolicyWindow.hitProp = w ? cudaAccessPropertyPersisting : cudaAccessPropertyNormal;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
        auto launch = [&]() {
          if (hint) k_gather<8, true><<<sms * 16, 128, 0, st>>>(d_idx, d_x, n, d_out);
          else k_gather<8, false><<<sms * 16, 128, 0, st>>>(d_idx, d_x, n, d_out);
        };
        launch();
        CK(cudaStreamSynchronize(st));
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
          CK(cudaEventRecord(a, st));
          launch();
          CK(cudaEventRecord(b, st));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          best = ms < best ? ms : best;
        }
        printf("{\"law\": \"%s\", \"vector_mb\": %d, \"window_mb\": %d, \"hint_evict_last\": %d, \"ms\": %.3f, "
               "\"G_gathers_per_s\": %.1f}\n",
               cs.law ? "zipf0.8" : "uniform", cs.mb, w, hint, best, n / (best * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
  }
  return 0;
}
