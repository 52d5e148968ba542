// Markstein-style division check (K4's q = s / total): with y = RN(1/b)
// and q0 = RN(a y), r = fma(-q0, b, a) is exact and q = fma(r, y, q0) is
// RN(a / b).  Compared against IEEE a / b on the GPU for random and
// adversarial (b with all-ones significand, a near b, a near 0) pairs in
// K4's domain: b = total in [1, 2^29), a = prefix sum in [0, b].
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false div_check.cu -o div_check
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
template <typename T>
__global__ void check(uint64_t seed, int64_t per_thread, unsigned long long* bad, unsigned long long* count) {
  const uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long nb = 0;
  for (int64_t it = 0; it < per_thread; ++it) {
    const uint64_t h1 = mix(seed ^ (id * 0x9E3779B97F4A7C15ull + it)), h2 = mix(h1 + 0x1234567ull);
    T b, a;
    const int kind = (int)(h2 & 7);
    // b: total in [1, 2^29); kind 1 forces an all-ones significand
    const double eb = (double)(h1 % 29);
    double bb = ldexp(1.0 + (double)(h1 >> 11) * 0x1p-53, (int)eb);
    if (kind == 1) bb = ldexp(2.0 - 0x1p-52, (int)eb);
    b = (T)bb;
    // a in [0, b]: uniform fraction, near b, near 0, exact multiples
    const double f = (double)(h2 >> 11) * 0x1p-53;
    if (kind == 2) a = b - (T)ldexp(f, -40) * b;
    else if (kind == 3) a = (T)ldexp(f, -(int)(h2 % 900)) * b;
    else if (kind == 4) a = b;
    else a = (T)f * b;
    const T y = (T)1 / b;
    const T q0 = a * y;
    const T r = fma(-q0, b, a);
    const T q = fma(r, y, q0);
    const T ref = a / b;
    if (!(q == ref) && !(q != q && ref != ref)) {
      if (nb < 4 && id < 2) printf("mismatch a=%a b=%a q=%a ref=%a\n", (double)a, (double)b, (double)q, (double)ref);
      ++nb;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(count, (unsigned long long)per_thread);
}

int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  for (int prec = 0; prec < 2; ++prec) {
    cudaMemset(d, 0, 16);
    if (prec == 0) check<double><<<148 * 16, 256>>>(7, 8192, d, d + 1);
    else check<float><<<148 * 16, 256>>>(9, 8192, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s: %llu mismatches in %llu divisions\n", prec == 0 ? "fp64" : "fp32", h[0], h[1]);
  }
  return 0;
}
