// Random 8-byte gathers over a vector of V MB (indices streamed, int32):
// uniform indices and Zipf(0.8)-weighted indices (the column-degree law of
// the cfg3 power-law LP, heaviest columns first as in the engine's
// length-class order). Measures the gather rate the L2 / DRAM can sustain
// for each vector size — the ceiling of a product whose gathered vector
// outgrows L2 (cfg3: x̄ 160 MB, y 80 MB).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_l2 tools/microbench_l2.cu
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

template <int U>
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
    for (int u = 0; u < U; ++u) asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[u]) : "l"(x + c[u]), "l"(pl));
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long n = 100000000;  // gathers per launch (cfg3: ~195M per product)
  int* d_idx;
  double *d_x, *d_out;
  CK(cudaMalloc(&d_idx, n * sizeof(int)));
  CK(cudaMalloc(&d_x, 512l << 20));
  CK(cudaMalloc(&d_out, 8));
  CK(cudaMemset(d_x, 0, 512l << 20));
  std::vector<int> h(n);
  std::mt19937_64 rng(1);
  const int mbs[] = {8, 16, 32, 40, 48, 64, 80, 96, 128, 160, 256};
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int law = 0; law < 2; ++law) {
    for (int mb : mbs) {
      const long V = (long)mb * (1l << 20) / 8;
      if (law == 0) {
        std::uniform_int_distribution<long> u(0, V - 1);
        for (long i = 0; i < n; ++i) h[i] = (int)u(rng);
      } else {
        // Zipf(0.8) by inverse CDF of w_j ~ (j+1)^-0.8: F(j) ~ ((j+1)^0.2 - 1) / ((V+1)^0.2 - 1)
        std::uniform_real_distribution<double> u(0.0, 1.0);
        const double k = std::pow((double)V + 1.0, 0.2) - 1.0;
        for (long i = 0; i < n; ++i) {
          const double j = std::pow(1.0 + u(rng) * k, 5.0) - 1.0;
          long jj = (long)j;
          h[i] = (int)(jj < V ? jj : V - 1);
        }
      }
      CK(cudaMemcpy(d_idx, h.data(), n * sizeof(int), cudaMemcpyHostToDevice));
      k_gather<8><<<sms * 16, 128>>>(d_idx, d_x, n, d_out);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        k_gather<8><<<sms * 16, 128>>>(d_idx, d_x, n, d_out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
      }
      printf("{\"law\": \"%s\", \"vector_mb\": %d, \"gathers\": %ld, \"ms\": %.3f, \"G_gathers_per_s\": %.1f}\n",
             law ? "zipf0.8" : "uniform", mb, n, best, n / (best * 1e-3) / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}
