// Throughput of the wide multiply-add forms on one B200 (all SMs, high occupancy):
//  mode 0: IMAD.WIDE.U32  (no carry), 64-bit accumulate, b uniform
//  mode 1: IMAD.WIDE.U32  (no carry), b per-thread (vector register)
//  mode 2: IMAD.WIDE.U32.X carry chains (4 independent chains of 8 pairs), b uniform
//  mode 3: IMAD.WIDE.U32.X carry chains, b per-thread
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t* out, uint32_t b0, int iters) {
  uint32_t b = (MODE & 1) ? (b0 ^ (threadIdx.x * 0x9e3779b9u)) : b0;
  uint32_t lo[8], hi[8], a[8];
#pragma unroll
  for (int c = 0; c < 8; c++) { lo[c] = threadIdx.x + c; hi[c] = c; a[c] = 0x9e3779b9u * (c + 1) + threadIdx.x; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      if (MODE < 2) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
          uint64_t acc = ((uint64_t)hi[c] << 32) | lo[c];
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a[c]), "r"(b));
          lo[c] = (uint32_t)acc; hi[c] = (uint32_t)(acc >> 32);
        }
      } else {
        // 2 independent chains of 4 pairs each (chain = mad.lo.cc ... madc.hi)
#pragma unroll
        for (int ch = 0; ch < 2; ch++) {
          asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(lo[4*ch]), "+r"(hi[4*ch]) : "r"(a[4*ch]), "r"(b));
#pragma unroll
          for (int c = 1; c < 4; c++)
            asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(lo[4*ch+c]), "+r"(hi[4*ch+c]) : "r"(a[4*ch+c]), "r"(b));
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; c++) s ^= lo[c] ^ hi[c];
  if (s == 12345) out[0] = s;
}
template <int MODE> void run(const char* name) {
  uint32_t* o; cudaMalloc(&o, 4);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int iters = 2000, blocks = nsm * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, 256>>>(o, 0x7f4a7c15u, iters);
  cudaEventRecord(e0); k<MODE><<<blocks, 256>>>(o, 0x7f4a7c15u, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double macs = (double)blocks * 256 * iters * 16 * 8;
  printf("%-40s %.2f TMAC32/s\n", name, macs / (ms * 1e-3) / 1e12);
}
int main() {
  run<0>("IMAD.WIDE       b uniform");
  run<1>("IMAD.WIDE       b vector");
  run<2>("IMAD.WIDE.X chains b uniform");
  run<3>("IMAD.WIDE.X chains b vector");
  return 0;
}
