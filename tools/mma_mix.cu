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

__global__ void k(const int* pat, int np, int reps, unsigned long long* cyc) {
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
    uint64_t bd[8];
    uint32_t id[8];
    for (int j = 0; j < np; j++) {
      bd[j] = umma::desc_kmajor(umma::smem_u32(sm + 65536), pat[j]);
      id[j] = umma::idesc_i8(128, pat[j]);
    }
    const uint64_t ad = umma::desc_kmajor(umma::smem_u32(sm), 128);
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
#pragma unroll 1
      for (int j = 0; j < np; j++) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + (j & 1) * 256),
            "l"(ad + (uint64_t)((i & 7) * 256)), "l"(bd[j]), "r"(id[j]), "r"((uint32_t)(i & 7)));
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
  int* dpat;
  cudaMalloc(&cyc, 8 * 256);
  cudaMalloc(&dpat, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  std::vector<std::vector<int>> pats = {{32}, {64}, {96}, {128}, {144}, {160}, {176}, {192}, {208}, {224}, {256},
                                        {256, 32}, {160, 128}, {144, 144}, {192, 96}, {176, 112}, {256, 64},
                                        {256, 192}, {224, 224}, {256, 128}, {192, 192}};
  unsigned long long h[256];
  for (auto& p : pats) {
    cudaMemcpy(dpat, p.data(), p.size() * 4, cudaMemcpyHostToDevice);
    const int reps = 2048;
    const int grid = 148;
    k<<<grid, 128, 160 * 1024>>>(dpat, (int)p.size(), reps, cyc);
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
