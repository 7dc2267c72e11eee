// Microbenchmark (not product code): shared-memory atomic throughput on B200,
// to size the K2 histogram design. Prints atomics/clk/SM for several patterns.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(unsigned long long* out, int iters, int bins) {
  extern __shared__ unsigned long long h64[];
  unsigned* h32 = (unsigned*)h64;
  for (int i = threadIdx.x; i < bins; i += blockDim.x) h64[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    int b = (MODE == 2 || MODE == 3) ? ((threadIdx.x * 37 + i * 101) % bins)
            : MODE == 4 ? ((threadIdx.x + i * 64) % bins)          // lane-distinct banks
            : MODE == 5 ? ((threadIdx.x & ~31) + i * 8) % bins      // whole warp on one address
            : (x >> 8) % bins;
    if (MODE == 0 || MODE == 2) atomicAdd(&h64[b], (unsigned long long)(x & 7));
    else atomicAdd(&h32[b], x & 7);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0 + h64[0] * 0;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 4096 * 8);
  int iters = 4096;
  for (int mode = 1; mode < 6; mode += (mode == 1 ? 2 : 1)) for (int bins : {4096, 16384}) for (int thr : {256, 1024}) {
    size_t sm = bins * 8;
    void (*f)(unsigned long long*, int, int) = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f<<<148, thr, sm>>>(d, iters, bins);
    cudaEventRecord(a);
    f<<<148 * 2, thr, sm>>>(d, iters, bins);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double tot = 148.0 * 2 * thr * iters;
    printf("mode=%d(%s,%s) bins=%5d thr=%4d: %.2f Gatom/s, %.1f atom/clk/SM (clk64 per block %llu) err=%s\n", mode,
           (mode == 0 || mode == 2) ? "u64" : "u32", mode >= 2 ? "strided" : "random", bins, thr, tot / ms / 1e6,
           tot / (ms * 1e-3 * 1.9e9) / 148, cyc, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
