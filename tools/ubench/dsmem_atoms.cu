// Distributed-shared-memory atomic throughput on this GPU (diagnostic for a
// cluster-wide K2 histogram): a thread-block cluster of C CTAs
// (1024 threads each, one per SM) holds one histogram of C x NB words, CTA r owning
// words [r*NB, (r+1)*NB); every thread adds into pseudo-random words of the whole
// cluster histogram with
//   mode 0: red.shared::cluster.add.u32 (no result),
//   mode 1: atom.shared::cluster.add.u32 with the result biased and OR-ed (K2's checked add),
//   mode 2: red on the CTA's own words only (local baseline through the same code).
// Prints lane updates per clock per SM for C = 1, 2, 4, 8, 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_atoms dsmem_atoms.cu && ./dsmem_atoms
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NB = 48 * 1024;  // words per CTA (192 KB)

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(1024, 1) k(int mode, int iters, unsigned *out) {
    extern __shared__ __align__(16) unsigned h[];
    for (int i = threadIdx.x; i < NB; i += 1024) h[i] = 0;
    const unsigned C = cluster_size(), me = cluster_rank();
    cluster_sync();
    const unsigned base = (unsigned)__cvta_generic_to_shared(h);
    unsigned x = (threadIdx.x + 1024u * blockIdx.x) * 2654435761u + 12345u, acc = 0;
    const unsigned total = C * NB;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const unsigned a = (x >> 4) % total;
        const unsigned r = mode == 2 ? me : a / NB, w = a % NB;
        unsigned remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(base + 4u * w), "r"(r));
        if (mode == 1) {
            unsigned old;
            asm volatile("atom.relaxed.cluster.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(remote), "r"(1u) : "memory");
            acc |= old + 1u + 0x40004000u;
        } else {
            asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(remote), "r"(1u) : "memory");
        }
    }
    cluster_sync();
    if (threadIdx.x == 0 || acc == 0x12345678u) out[blockIdx.x] = h[0] + acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned *out;
    cudaMalloc(&out, 1024 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = NB * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 2048;
    for (int C = 1; C <= 16; C *= 2) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(C);
        int nclusters = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
        if (e != cudaSuccess || nclusters <= 0) {
            printf("{\"cluster\": %d, \"error\": \"%s\", \"max_active_clusters\": %d}\n", C, cudaGetErrorString(e), nclusters);
            cudaGetLastError();
            continue;
        }
        cfg.gridDim = dim3(nclusters * C);
        for (int mode = 0; mode < 3; ++mode) {
            e = cudaLaunchKernelEx(&cfg, k, mode, 32, out);
            cudaEventRecord(a);
            e = cudaLaunchKernelEx(&cfg, k, mode, iters, out);
            cudaEventRecord(b);
            cudaError_t e2 = cudaEventSynchronize(b);
            if (e != cudaSuccess || e2 != cudaSuccess) {
                printf("{\"cluster\": %d, \"mode\": %d, \"error\": \"%s / %s\"}\n", C, mode, cudaGetErrorString(e), cudaGetErrorString(e2));
                cudaGetLastError();
                continue;
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double ctas = (double)nclusters * C;
            const double lanes = ctas * 1024 * iters;
            const double clocks = ms * 1e-3 * clk * 1e3;
            printf("{\"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"mode\": \"%s\", \"ms\": %.3f, "
                   "\"lane_updates_per_clk_per_sm\": %.3f, \"lane_updates_per_s_gpu\": %.4g, \"clock_khz\": %d}\n",
                   C, nclusters, (int)ctas,
                   mode == 0 ? "random over the cluster, red" : mode == 1 ? "random over the cluster, atom checked"
                                                                          : "own CTA only, red (mapa path)",
                   ms, lanes / clocks / ctas, lanes / (ms * 1e-3), clk);
        }
    }
    return 0;
}
