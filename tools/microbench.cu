// Microbenchmarks that bound the FP64 CSR product on this B200:
//   stream  : coalesced read of N doubles (DRAM ceiling for the matrix stream)
//   gather  : idx streamed (int32, coalesced) + x[idx] gathered (8 B random,
//             x L2-resident) — the product's irreducible random access
//   spmv-like: idx + val streamed, x gathered, sum per thread
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void k_stream(const double* __restrict__ a, long n, double* out) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) s += __ldcs(a + i);
  if (s == 12345.678) out[0] = s;
}

template <int U>
__global__ void k_gather(const int* __restrict__ idx, const double* __restrict__ x, long n, double* out) {
  double s = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (i + u * stride < n) ? __ldcs(idx + i + u * stride) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 12345.678) out[0] = s;
}

template <int U>
__global__ void k_spmvlike(const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ x,
                           long n, double* out) {
  double s = 0;
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    int c[U];
    double a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool ok = i + u * stride < n;
      c[u] = ok ? __ldcs(idx + i + u * stride) : 0;
      a[u] = ok ? __ldcs(val + i + u * stride) : 0.0;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s += a[u] * v[u];
  }
  if (s == 12345.678) out[0] = s;
}

template <class F>
float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long N = 20'000'000;
  std::vector<long> xsizes = {1'000'000, 2'000'000, 8'000'000, 20'000'000};
  double *val, *x, *out, *big;
  int* idx;
  const long BIG = 64'000'000;
  CK(cudaMalloc(&val, N * 8)); CK(cudaMalloc(&idx, N * 4)); CK(cudaMalloc(&x, 20'000'000L * 8));
  CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&big, BIG * 8));
  CK(cudaMemset(val, 0, N * 8)); CK(cudaMemset(x, 0, 20'000'000L * 8)); CK(cudaMemset(big, 0, BIG * 8));
  std::vector<int> h(N);
  float ms = timeit([&] { k_stream<<<sms * 8, 256>>>(big, BIG, out); });
  printf("stream  %ld doubles: %.3f ms  %.1f GB/s\n", BIG, ms, BIG * 8 / ms / 1e6);
  for (long xs : xsizes) {
    std::mt19937 rng(1);
    for (long i = 0; i < N; ++i) h[i] = rng() % xs;
    CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
    for (int tpb : {256, 512}) {
      for (int bps : {4, 8}) {
        int grid = sms * bps * 256 / tpb;
        float g4 = timeit([&] { k_gather<4><<<grid, tpb>>>(idx, x, N, out); });
        float g8 = timeit([&] { k_gather<8><<<grid, tpb>>>(idx, x, N, out); });
        float s4 = timeit([&] { k_spmvlike<4><<<grid, tpb>>>(idx, val, x, N, out); });
        float s8 = timeit([&] { k_spmvlike<8><<<grid, tpb>>>(idx, val, x, N, out); });
        printf("x=%ldM tpb=%d grid=%d | gather U4 %.1f us (%.0f Ggath/s) U8 %.1f us | spmv-like U4 %.1f us (%.0f GB/s stream) U8 %.1f us (%.0f GB/s)\n",
               xs / 1000000, tpb, grid, g4 * 1e3, N / g4 / 1e6, g8 * 1e3, s4 * 1e3, N * 12 / s4 / 1e6, s8 * 1e3,
               N * 12 / s8 / 1e6);
      }
    }
  }
  // sorted (coalesced) gather for comparison
  for (long i = 0; i < N; ++i) h[i] = (int)(i % 2'000'000);
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  float sc = timeit([&] { k_spmvlike<8><<<sms * 8, 256>>>(idx, val, x, N, out); });
  printf("spmv-like sequential idx: %.1f us (%.0f GB/s stream)\n", sc * 1e3, N * 12 / sc / 1e6);
  return 0;
}
