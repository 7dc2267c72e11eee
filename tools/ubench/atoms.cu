// Shared-memory atomic throughput on this GPU (diagnostic for K2's roofline):
// every CTA (1024 threads, one per SM) adds into a 48 KB smem histogram with
//   mode 0: conflict-free addresses (lane l -> bank l),
//   mode 1: pseudo-random addresses (hash of (thread, iteration)),
//   mode 2: all lanes of a warp on one word,
//   mode 3: pseudo-random addresses, the returned old values used (ATOMS with a result),
//   mode 4: as 3 with the old values OR-ed after a bias (K2's checked packed add).
// Prints warp-atomic instructions/s and lane-updates per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu && ./atoms
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k(int mode, int iters, unsigned *out) {
    __shared__ unsigned h[12288];
    for (int i = threadIdx.x; i < 12288; i += 1024) h[i] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned a;
        if (mode == 0) a = (warp * 32 + lane + it * 1024) % 12288;
        else if (mode == 1 || mode >= 3) { x = x * 1664525u + 1013904223u; a = (x >> 8) % 12288; }
        else a = (warp * 97 + it) % 12288;
        if (mode == 3) acc += atomicAdd(h + a, 1u);
        else if (mode == 4) acc |= atomicAdd(h + a, 1u) + 1u + 0x40004000u;
        else atomicAdd(h + a, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 || acc == 0x12345678u) out[blockIdx.x] = h[0] + acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned *out;
    cudaMalloc(&out, sms * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int mode = 0; mode < 5; ++mode) {
        k<<<sms, 1024>>>(mode, 64, out);
        cudaEventRecord(a);
        k<<<sms, 1024>>>(mode, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double lanes = (double)sms * 1024 * iters, warps = lanes / 32;
        const double clocks = ms * 1e-3 * clk * 1e3;
        printf("{\"mode\": \"%s\", \"ms\": %.3f, \"warp_atoms_per_s\": %.4g, \"lane_updates_per_clk_per_sm\": %.3f, "
               "\"warp_atoms_per_clk_per_sm\": %.4f, \"clock_khz\": %d}\n",
               mode == 0 ? "conflict-free" : mode == 1 ? "random" : mode == 2 ? "one word per warp"
               : mode == 3 ? "random, result used" : "random, checked (result biased and OR-ed)", ms, warps / (ms * 1e-3),
               lanes / clocks / sms, warps / clocks / sms, clk);
    }
    return 0;
}
