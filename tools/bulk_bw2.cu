// Microbenchmark: cp.async.bulk global -> shared throughput per SM as a function of copy size
// and of the number of ISSUING WARPS (each warp keeps `inflight` copies in flight in its own
// slots).  All SMs stream the same L2-resident 256 KB window (like the W stream of rnsx.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw2 bulk_bw2.cu && ./bulk_bw2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, size_t span, uint32_t bytes, int inflight, int iters,
                            unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[64];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight * nw; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = clock64();
  if ((threadIdx.x & 31) == 0) {
    const size_t nchunk = span / bytes;
    uint32_t ph = 0;
    for (int it = 0; it < iters + inflight; it++) {
      const int slot = w * inflight + it % inflight;
      if (it >= inflight) {
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}\n" ::"r"(
                sa(&bar[slot])),
            "r"((ph >> (it % inflight)) & 1));
        ph ^= 1u << (it % inflight);
      }
      if (it < iters) {
        const uint8_t* s = src + (size_t)((it * nw + w + blockIdx.x * 7) % nchunk) * bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[slot])), "r"(bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + (size_t)slot * bytes)),
                     "l"(s), "r"(bytes), "r"(sa(&bar[slot]))
                     : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 1, 64 << 20);
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * 8);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long h[1024];
  for (uint32_t bytes : {4096u, 8192u, 16384u, 32768u})
    for (int nw : {1, 2, 4})
      for (int inflight : {2, 4, 8}) {
        if ((size_t)bytes * inflight * nw > 192 * 1024 || inflight * nw > 64) continue;
        const int iters = 256;  // per warp
        bulk_kernel<<<nsm, 32 * nw, bytes * inflight * nw>>>(buf, 256 * 1024, bytes, inflight, iters, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < nsm; i++) avg += h[i];
        avg /= nsm;
        printf("bytes=%6u warps=%d inflight/warp=%d : %.1f B/clk/SM (%.0f clk per copy per SM) err=%d\n", bytes, nw,
               inflight, (double)bytes * iters * nw / avg, avg / (iters * nw), (int)e);
      }
  return 0;
}
