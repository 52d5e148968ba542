// Microbenchmark: random-access reads from a 1 GiB table (>> 126 MB L2).
// Measures random-read throughput at access sizes 8/16/32/64/128 B and the
// cost of a dependent pair (8 B index -> 32 B record, the cut-point lookup
// followed by the ancestor gather).  Run it under ncu with
// dram__bytes_read.sum to see the DRAM bytes fetched per access.
//   ./gather [l2_fetch_limit]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

// BYTES-sized random reads, ILP independent accesses per thread per round.
template <int BYTES, int ILP>
__global__ void __launch_bounds__(256) rand_read(const uint4* __restrict__ tab, uint64_t bytes, double* out,
                                                 int rounds) {
  constexpr int V = BYTES >= 16 ? BYTES / 16 : 1;
  const uint64_t n = bytes / (BYTES >= 16 ? BYTES : 16);
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < rounds; ++it) {
    uint4 v[ILP][V];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      const uint64_t e = mix(tid * 0x9E3779B97F4A7C15ull + it * ILP + k) % n;
      const uint4* p = tab + e * V;
      if (BYTES == 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        v[k][0] = make_uint4(w.x, w.y, 0, 0);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) v[k][c] = p[c];
      }
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k)
#pragma unroll
      for (int c = 0; c < V; ++c) acc += v[k][c].x ^ v[k][c].w;
  }
  out[tid] = (double)acc;
}

// Dependent pair: 8 B index read at a random position, then a 32 B record
// at the index it holds (both random).
template <int ILP>
__global__ void __launch_bounds__(256) dep_pair(const uint32_t* __restrict__ idx, const uint4* __restrict__ rec,
                                                uint64_t n, double* out, int rounds) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < rounds; ++it) {
    uint2 ix[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      const uint64_t e = mix(tid * 0x9E3779B97F4A7C15ull + it * ILP + k) & (n - 1);
      ix[k] = *reinterpret_cast<const uint2*>(idx + 2 * e);
    }
    uint4 a[ILP], b[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      const uint4* p = rec + 2 * (uint64_t)(ix[k].x & (n - 1));
      a[k] = p[0];
      b[k] = p[1];
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc += a[k].x ^ b[k].w;
  }
  out[tid] = (double)acc;
}


// 32-byte random reads with an explicit PTX load flavour (cache operator /
// L1 policy): 0 = ld.global (default), 1 = ld.global.cg (L2 only),
// 2 = ld.global.cs (streaming), 3 = ld.global.L1::no_allocate,
// 4 = ld.global.nc (texture path), 5 = ld.global.lu, 6 = ld.global.cv
template <int FLAVOUR, int ILP>
__global__ void __launch_bounds__(256) rand32_flavour(const uint4* __restrict__ tab, uint64_t n32, double* out,
                                                      int rounds) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < rounds; ++it) {
    uint32_t v[ILP][8];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      const uint64_t e = mix(tid * 0x9E3779B97F4A7C15ull + it * ILP + k) % n32;
      const uint4* p = tab + 2 * e;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t* d = &v[k][4 * h];
        const uint4* q = p + h;
        if (FLAVOUR == 0)
          asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else if (FLAVOUR == 1)
          asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else if (FLAVOUR == 2)
          asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else if (FLAVOUR == 3)
          asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else if (FLAVOUR == 4)
          asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else if (FLAVOUR == 5)
          asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
        else
          asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "l"(q));
      }
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc += v[k][0] ^ v[k][7];
  }
  out[tid] = (double)acc;
}

// Random 32-byte writes (scatter), for the write-side cost.
__global__ void __launch_bounds__(256) rand32_write(uint4* tab, uint64_t n32, int rounds) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < rounds * 4; ++it) {
    const uint64_t e = mix(tid * 0x9E3779B97F4A7C15ull + it) % n32;
    tab[2 * e] = make_uint4((uint32_t)tid, it, 1, 2);
    tab[2 * e + 1] = make_uint4(3, 4, 5, 6);
  }
}

__global__ void fill(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)mix(i);
}

template <typename F>
void timeit(const char* name, double accesses, double bytes_each, F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %8.3f ms  %7.2f Gaccess/s  %7.0f GB/s useful\n", name, ms, accesses / ms / 1e6,
         accesses * bytes_each / ms / 1e6);
}

int main(int argc, char** argv) {
  const uint64_t bytes = 1ull << 30;
  uint4* tab;
  double* out;
  cudaMalloc(&tab, bytes);
  fill<<<148 * 8, 256>>>((uint32_t*)tab, bytes / 4);
  const int blocks = 148 * 8, threads = 256, rounds = 16;
  cudaMalloc(&out, (size_t)blocks * threads * 8);
  if (argc > 1) {
    const int lim = atoi(argv[1]);
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lim);
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit %d -> %s, now %zu\n", lim, cudaGetErrorString(e), v);
  }
  const double th = (double)blocks * threads * rounds;
#define RR(B, I)                                                                                   \
  timeit("rand_read " #B "B ilp" #I, th * I, B,                                                    \
         [&] { rand_read<B, I><<<blocks, threads>>>(tab, bytes, out, rounds); })
  RR(8, 4); RR(8, 8);
  RR(16, 4); RR(16, 8);
  RR(32, 4); RR(32, 8);
  RR(64, 4);
  RR(128, 2);
  const uint64_t n = bytes / 32;
  timeit("dep_pair 8B->32B ilp4", th * 4, 40,
         [&] { dep_pair<4><<<blocks, threads>>>((const uint32_t*)tab, tab, n, out, rounds); });
  timeit("dep_pair 8B->32B ilp8", th * 8, 40,
         [&] { dep_pair<8><<<blocks, threads>>>((const uint32_t*)tab, tab, n, out, rounds); });
  const uint64_t n32 = bytes / 32;
#define FL(F)                                                                                      \
  timeit("rand32 flavour " #F " ilp8", th * 8, 32,                                                \
         [&] { rand32_flavour<F, 8><<<blocks, threads>>>(tab, n32, out, rounds); })
  FL(0); FL(1); FL(2); FL(3); FL(4); FL(5); FL(6);
  timeit("rand32 write", th * 4, 32, [&] { rand32_write<<<blocks, threads>>>(tab, n32, rounds); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
