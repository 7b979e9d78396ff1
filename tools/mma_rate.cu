// Microbenchmark: back-to-back tcgen05.mma.cta_group::1.kind::i8 (M = 128, K = 32 bytes) issue
// rate per SM for N = 64 / 128 / 256, operands in shared memory (no-swizzle K-major), with and
// without a tcgen05.commit after every MMA.  One CTA per SM, one issuing warp.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2601_14980_b200/csrc/umma.cuh"
using namespace pcb;

__global__ void k(int N, int n_mma, int commit_each, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  for (int o = threadIdx.x * 16; o < 128 * 1024; o += blockDim.x * 16) *reinterpret_cast<uint4*>(sm + o) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 32) umma::tmem_alloc<512>(&tb);
  if (threadIdx.x == 0) umma::mbar_init(&bar, 1);
  umma::fence_async_smem();
  umma::tmem_fence_before();
  __syncthreads();
  umma::tmem_fence_after();
  const uint32_t tm = tb;
  if (threadIdx.x < 32) {
    const uint64_t ad = umma::desc_kmajor(umma::smem_u32(sm), 128);
    const uint64_t bd = umma::desc_kmajor(umma::smem_u32(sm + 65536), N);
    const uint32_t idesc = umma::idesc_i8(128, N);
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; i++) {
      asm volatile(
          "{\n\t.reg .pred p, e;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "elect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + (i & 1) * 256),
          "l"(ad + (uint64_t)((i & 7) * 256)), "l"(bd), "r"(idesc), "r"((uint32_t)(i & 7)));
      if (commit_each) {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                umma::smem_u32(&bar))
            : "memory");
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            umma::smem_u32(&bar))
        : "memory");
    // wait for the final commit: phase (number of commits - 1) & 1
    const uint32_t ncommit = (commit_each ? n_mma : 0) + 1;
    umma::mbar_wait(&bar, (ncommit - 1) & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  umma::tmem_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8 * 256);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  unsigned long long h[256];
  for (int grid : {148})
    for (int ce : {1})
      for (int N : {64, 96, 128, 144, 160, 192, 224, 256}) {
        const int n = 4096;
        k<<<grid, 128, 160 * 1024>>>(N, n, ce, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < grid; i++) avg += h[i];
        avg /= grid;
        printf("grid %3d commit_each %d N %3d: %.1f clk/MMA  (%.0f int8 MAC/clk/SM) err %d\n", grid, ce, N, avg / n,
               128.0 * N * 32 * n / avg, (int)e);
      }
  return 0;
}
