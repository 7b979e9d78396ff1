// Microbenchmark: cp.async.bulk (global -> shared, mbarrier complete_tx) throughput per SM.
// One CTA per SM; one elected thread keeps `inflight` copies of `bytes` each in flight over a
// ring of slots, streaming a `span`-byte window of a global buffer (shared by all SMs, or a
// private window per SM).  Also: a plain LDG.128 -> STS copy loop by 4 warps for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw bulk_bw.cu && ./bulk_bw
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* src, size_t span, int priv, uint32_t bytes, int inflight, int iters,
                            unsigned long long* cyc, int spin) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; i++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (priv ? (size_t)blockIdx.x * span : 0);
  const size_t nchunk = span / bytes;
  const long long t0 = clock64();
  uint32_t ph[32] = {};
  for (int it = 0; it < iters + inflight; it++) {
    const int slot = it % inflight;
    if (it >= inflight) {  // wait for the copy issued inflight iterations ago
      if (spin)
        asm volatile(
            "{\n\t.reg .pred P;\nS_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra S_%=;\n\t}\n" ::"r"(
                sa(&bar[slot])),
            "r"(ph[slot]));
      else
        asm volatile(
            "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}\n" ::"r"(
                sa(&bar[slot])),
            "r"(ph[slot]));
      ph[slot] ^= 1;
    }
    if (it < iters) {
      const uint8_t* s = base + (size_t)((it + blockIdx.x * 7) % nchunk) * bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[slot])), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)slot * bytes)),
                   "l"(s), "r"(bytes), "r"(sa(&bar[slot]))
                   : "memory");
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}

__global__ void ldg_kernel(const uint8_t* src, size_t span, int priv, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint8_t* base = src + (priv ? (size_t)blockIdx.x * span : 0);
  const size_t n16 = span / 16;
  const long long t0 = clock64();
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; it++) {  // each iteration: 128 threads x 8 x 16 B = 16 KB
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; k++)
      v[k] = reinterpret_cast<const uint4*>(base)[((size_t)it * 1024 + k * 128 + threadIdx.x + blockIdx.x * 97) % n16];
#pragma unroll
    for (int k = 0; k < 8; k++) reinterpret_cast<uint4*>(sm)[(k * 128 + threadIdx.x) % 4096] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  if (acc.x == 12345) cyc[0] = 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t span = 1 << 20;
  uint8_t* buf;
  cudaMalloc(&buf, span * nsm);
  cudaMemset(buf, 1, span * nsm);
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * 8);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ldg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long h[1024];
  for (int spin = 0; spin < 2; spin++)
  for (int priv = 0; priv < 1; priv++)
    for (uint32_t bytes : {4096u, 16384u, 32768u, 65536u})
      for (int inflight : {2, 3, 6, 12}) {
        if ((size_t)bytes * inflight > 200 * 1024) continue;
        const int iters = (int)((64ull << 20) / nsm / bytes) + 16;
        bulk_kernel<<<nsm, 32, bytes * inflight>>>(buf, priv ? span : 256 * 1024, priv, bytes, inflight, iters, cyc, spin);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        double avg = 0;
        for (int i = 0; i < nsm; i++) { mx = h[i] > mx ? h[i] : mx; avg += h[i]; }
        avg /= nsm;
        printf("bulk spin=%d bytes=%6u inflight=%2d : %.1f B/clk/SM (avg cyc %.0f) err=%d\n", spin, bytes, inflight,
               (double)bytes * iters / avg, avg, (int)e);
      }
  for (int priv = 0; priv < 2; priv++) {
    const int iters = (int)((64ull << 20) / nsm / 16384);
    ldg_kernel<<<nsm, 128, 64 * 1024>>>(buf, priv ? span : 256 * 1024, priv, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nsm; i++) avg += h[i];
    avg /= nsm;
    printf("ldg  priv=%d 128 thr x 8 x 16B : %.1f B/clk/SM\n", priv, 16384.0 * iters / avg);
  }
  return 0;
}
