// How do concurrent cp.async.bulk copies overlap?  One thread issues N copies of `bytes` at once
// (each on its own mbarrier), then waits for all; cycles per batch vs N.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint8_t* src, uint32_t bytes, int n, int reps, unsigned long long* cyc, int nthr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int t = threadIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    for (int i = t; i < n; i += nthr) {  // copies issued by nthr threads
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)i * bytes)),
                   "l"(src + ((size_t)(r * 16 + i) % 64) * bytes), "r"(bytes), "r"(sa(&bar[i]))
                   : "memory");
    }
    for (int i = 0; i < n; i++)
      asm volatile(
          "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}\n" ::"r"(
              sa(&bar[i])),
          "r"((uint32_t)(r & 1)));
    __syncthreads();
  }
  if (t == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 1, 64 << 20);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long h[256];
  for (int grid : {1, 148})
    for (int nthr : {1, 32})
      for (uint32_t bytes : {4096u, 16384u})
        for (int n : {1, 2, 4, 8, 12}) {
          if (bytes * n > 200 * 1024) continue;
          const int reps = 200;
          k<<<grid, 32, bytes * n>>>(buf, bytes, n, reps, cyc, nthr);
          cudaDeviceSynchronize();
          cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
          double avg = 0;
          for (int i = 0; i < grid; i++) avg += h[i];
          avg /= grid;
          printf("grid=%3d issuers=%2d bytes=%5u n=%2d : %.0f clk/batch  %.1f B/clk/SM\n", grid, nthr, bytes, n,
                 avg / reps, (double)bytes * n * reps / avg);
        }
  return 0;
}
