// Microbenchmark: tcgen05.mma.cta_group::1.kind::i8 (M = 128, K = 32 bytes) issue cost per MMA
// for repeating N patterns, e.g. {256, 32} (the K = 72 chunking: 64 + 8 primes) against
// {160, 128} / {144, 144} (two near-even chunks).  One CTA per SM, one issuing warp, no commit
// between MMAs.  Prints clk per pattern and useful int8 MAC/clk/SM.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2601_14980_b200/csrc/umma.cuh"
using namespace pcb;

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

// one or two MMAs per repetition (n1 == 0: one), operands in registers, fully unrolled body
__global__ void k(int n0, int n1, int reps, unsigned long long* cyc) {
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
    const uint64_t b0 = umma::desc_kmajor(umma::smem_u32(sm + 65536), n0);
    const uint64_t b1 = umma::desc_kmajor(umma::smem_u32(sm + 65536), n1 ? n1 : 32);
    const uint32_t i0 = umma::idesc_i8(128, n0), i1 = umma::idesc_i8(128, n1 ? n1 : 32);
    const uint64_t ad = umma::desc_kmajor(umma::smem_u32(sm), 128);
    const long long t0 = clock64();
    if (n1) {
      for (int i = 0; i < reps; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          mma(tm, ad + (uint64_t)(u * 256), b0, i0, (uint32_t)(i + u));
          mma(tm + 256, ad + (uint64_t)(u * 256), b1, i1, (uint32_t)(i + u));
        }
      }
    } else {
      for (int i = 0; i < reps; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; u++) mma(tm + (u & 1) * 256, ad + (uint64_t)(u * 256), b0, i0, (uint32_t)(i + u));
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            umma::smem_u32(&bar))
        : "memory");
    umma::mbar_wait(&bar, 0);
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
  std::vector<std::vector<int>> pats = {{32}, {64}, {96}, {128}, {144}, {160}, {176}, {192}, {208}, {224}, {256},
                                        {256, 32}, {160, 128}, {144, 144}, {192, 96}, {176, 112}, {256, 64},
                                        {256, 192}, {224, 224}, {256, 128}, {192, 192}};
  unsigned long long h[256];
  for (auto& p : pats) {
    const int reps = 4096;
    const int grid = 148;
    k<<<grid, 128, 160 * 1024>>>(p[0], p.size() > 1 ? p[1] : 0, reps, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; i++) avg += h[i];
    avg /= grid;
    int ncols = 0;
    printf("N = {");
    for (size_t j = 0; j < p.size(); j++) { printf("%s%d", j ? "," : "", p[j]); ncols += p[j]; }
    printf("}: %.1f clk per pattern (%.1f per MMA), %.0f int8 MAC/clk/SM, err %d\n", avg / reps,
           avg / reps / p.size(), 128.0 * ncols * 32 * reps / avg, (int)e);
  }
  return 0;
}
