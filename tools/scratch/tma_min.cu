// Minimal cp.async.bulk.tensor check (diagnostics)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, unsigned char *out, int xb, int yb, int mode, int cx, int cy) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)) : "memory");
    if (mode != 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(xb*yb) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(sa(buf)), "l"(&tm), "r"(cx), "r"(cy), "r"(0), "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" :: "r"(sa(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < xb*yb; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char **argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  int cx = argc > 2 ? atoi(argv[2]) : -1, cy = argc > 3 ? atoi(argv[3]) : -1;
  void *p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  int W = 128, H = 96; unsigned char *img, *out;
  cudaMalloc(&img, W*H); cudaMalloc(&out, 4096);
  unsigned char h[128*96]; for (int i = 0; i < W*H; ++i) h[i] = i % 251; cudaMemcpy(img, h, W*H, cudaMemcpyHostToDevice);
  CUtensorMap tm; cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}, str[2] = {(cuuint64_t)W, (cuuint64_t)W*H};
  cuuint32_t box[3] = {80, 34, 1}, es[3] = {1,1,1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128, 80*34>>>(tm, out, 80, 34, mode, cx, cy);
  printf("launch %s sync %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(cudaDeviceSynchronize()));
  unsigned char o[80*34]; cudaMemcpy(o, out, 80*34, cudaMemcpyDeviceToHost);
  printf("o[0]=%d (oob 0) o[81]=%d (want %d)\n", o[0], o[81], h[0]);
  return 0;
}
