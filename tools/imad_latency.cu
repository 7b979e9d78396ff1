// Microbenchmark: dependent latency / per-warp throughput of IMAD.WIDE.U32.X carry chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_latency imad_latency.cu
#include <cstdio>
#include <cstdint>
template <int CH>
__global__ void k(uint32_t* out, uint32_t b, int iters, long long* cyc) {
  uint32_t lo[CH], hi[CH], a[CH];
  for (int c = 0; c < CH; c++) { lo[c] = threadIdx.x + c; hi[c] = c; a[c] = 0x9e3779b9u * (c + 1); }
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 32; u++) {
#pragma unroll
      for (int c = 0; c < CH; c++)
        asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(lo[c]), "+r"(hi[c]) : "r"(a[c]), "r"(b));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int c = 0; c < CH; c++) s ^= lo[c] ^ hi[c];
  if (s == 12345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH> void run(int warps) {
  uint32_t* o; long long* c; cudaMalloc(&o, 4); cudaMalloc(&c, 8);
  int iters = 200;
  k<CH><<<1, 32 * warps>>>(o, 0x7f4a7c15u, iters, c);
  k<CH><<<1, 32 * warps>>>(o, 0x7f4a7c15u, iters, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * 32.0);
  printf("chains=%d warps_per_block=%d  cycles per chain-step %.2f  -> cycles per IMAD.WIDE issue (per warp) %.2f\n", CH, warps, per, per / CH);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1);
  run<1>(4); run<4>(4); run<1>(8); run<4>(8); run<2>(16);
  return 0;
}
