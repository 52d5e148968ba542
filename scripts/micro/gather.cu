// Microbenchmark: random 32-byte record gathers from a 1 GiB table.
// Measures device time per gather under different L2 fetch settings / PTX
// cache hints; run under ncu to read dram__sectors_read per gather.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) Rec { double a, b, c, d; };

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int MODE>
__global__ void gather(const Rec* __restrict__ tab, uint64_t n, double* out, int iters) {
  double acc = 0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const uint64_t k = mix(tid * 1315423911ull + it) & (n - 1);
    const Rec* p = tab + k;
    double a, b, c, d;
    if (MODE == 0) {
      const Rec r = *p; a = r.a; b = r.b; c = r.c; d = r.d;
    } else if (MODE == 1) {
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
      asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2+16];" : "=d"(c), "=d"(d) : "l"(p));
    } else {
      asm volatile("ld.global.nc.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
      asm volatile("ld.global.nc.L2::64B.v2.f64 {%0,%1}, [%2+16];" : "=d"(c), "=d"(d) : "l"(p));
    }
    acc += a + b + c + d;
  }
  out[tid] = acc;
}

int main(int argc, char** argv) {
  const uint64_t n = 1ull << 25;  // 32M records x 32 B = 1 GiB
  Rec* tab; double* out;
  cudaMalloc(&tab, n * sizeof(Rec));
  cudaMemset(tab, 0, n * sizeof(Rec));
  const int blocks = 148 * 8, threads = 256, iters = 64;
  cudaMalloc(&out, (size_t)blocks * threads * 8);
  const int lim = argc > 1 ? atoi(argv[1]) : -1;
  if (lim >= 0) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lim);
    size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("set limit %d -> %s, now %zu\n", lim, cudaGetErrorString(e), v);
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) gather<0><<<blocks, threads>>>(tab, n, out, iters);
      if (mode == 1) gather<1><<<blocks, threads>>>(tab, n, out, iters);
      if (mode == 2) gather<2><<<blocks, threads>>>(tab, n, out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double g = (double)blocks * threads * iters;
      if (rep) printf("mode %d: %.3f ms, %.2f Ggather/s, %.0f GB/s at 32B, %.0f GB/s at 64B\n", mode, ms,
                      g / ms / 1e6, g * 32 / ms / 1e6, g * 64 / ms / 1e6);
    }
  }
  return 0;
}
