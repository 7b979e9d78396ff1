// imad_peak.cu — integer-multiply roofline microbenchmark (the denominator of roofline.frac).
//
// "P_MAC32 is the peak MAC32/s from an IMAD microbenchmark: independent
// IMAD.WIDE.U32 and IMAD.LO/IMAD.HI chains on all SMs, at the clocks seen under load."
// Two kernels, each with 8 independent accumulator chains per thread, grid = 148 x 8 CTAs:
//   * wide : a MAC32 is one `IMAD.WIDE.U32` (64-bit accumulate)             -> 1 MAC32/instr
//   * lohi : a MAC32 is `IMAD` (lo) + `IMAD.HI.U32` (hi) into two accumulators -> 1 MAC32/2 instr
// The reported peak is the larger of the two (a larger denominator is the conservative choice).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) imad_wide_kernel(uint64_t* out, uint32_t a0, uint32_t b0, int iters) {
  uint64_t acc[kChains];
  uint32_t a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) {
    acc[c] = threadIdx.x + c;
    a[c] = a0 + 7u * c + threadIdx.x;
  }
  const uint32_t b = b0 ^ blockIdx.x;
#pragma unroll 1
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int c = 0; c < kChains; c++) {
        // acc = a*b + acc  (64-bit): one IMAD.WIDE.U32
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"(a[c]), "r"(b));
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s ^= acc[c];
  if (s == 0x123456789abcdefull) out[0] = s;  // keep the work alive
}

__global__ void __launch_bounds__(256) imad_lohi_kernel(uint64_t* out, uint32_t a0, uint32_t b0, int iters) {
  uint32_t lo[kChains], hi[kChains], a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) {
    lo[c] = threadIdx.x + c;
    hi[c] = c;
    a[c] = a0 + 7u * c + threadIdx.x;
  }
  const uint32_t b = b0 ^ blockIdx.x;
#pragma unroll 1
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int c = 0; c < kChains; c++) {
        asm volatile("mad.lo.u32 %0, %2, %3, %0;\n\tmad.hi.u32 %1, %2, %3, %1;"
                     : "+r"(lo[c]), "+r"(hi[c]) : "r"(a[c]), "r"(b));
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s ^= lo[c] ^ hi[c];
  if (s == 0x12345678u) out[0] = s;
}

}  // namespace

extern "C" {

// Runs one kernel (kind 0 = wide, 1 = lo/hi) on the current device and returns the achieved
// MAC32/s (CUDA-event timed, after one warm-up launch).  Returns < 0 on CUDA error.
double pcb_imad_peak(int kind, int iters, float* ms_out) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = nsm * 8, threads = 256;
  uint64_t* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    if (kind == 0)
      imad_wide_kernel<<<blocks, threads>>>(out, 0x9e3779b9u, 0x7f4a7c15u, iters);
    else
      imad_lohi_kernel<<<blocks, threads>>>(out, 0x9e3779b9u, 0x7f4a7c15u, iters);
  };
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -2.0;
  if (ms_out) *ms_out = ms;
  const double macs = (double)blocks * threads * iters * 16.0 * kChains;
  return macs / (ms * 1e-3);
}

}  // extern "C"
