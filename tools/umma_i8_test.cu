// Standalone check of the tcgen05 int8 MMA path used by the RNS base extension:
//   D[128 x N] (s32, TMEM) = A[128 x K] (u8, smem, K-major) * B[N x K]^T (u8, smem, K-major)
// with hand-built shared-memory / instruction descriptors (no swizzle, chunk-major layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_i8_test tools/umma_i8_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2601_14980_b200/csrc/umma.cuh"

constexpr int M = 128, K = 288, N = 288, NH = 144;

__global__ void __launch_bounds__(128, 1) k_test(const uint8_t* A, const uint8_t* B, int32_t* D) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sA = sm;                       // M*K
  uint8_t* sB = sm + M * K;               // N*K
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  // global (row-major) -> smem canonical chunk-major layout
  for (int idx = tid; idx < M * K / 16; idx += blockDim.x) {
    const int r = idx / (K / 16), c = idx % (K / 16);
    *(uint4*)(sA + pcb::umma::kmajor_off(r, c * 16, M)) = *(const uint4*)(A + (size_t)r * K + c * 16);
  }
  for (int idx = tid; idx < N * K / 16; idx += blockDim.x) {
    const int r = idx / (K / 16), c = idx % (K / 16);
    *(uint4*)(sB + pcb::umma::kmajor_off(r, c * 16, N)) = *(const uint4*)(B + (size_t)r * K + c * 16);
  }
  if (tid < 32) pcb::umma::tmem_alloc<512>(&tbase);
  if (tid == 0) pcb::umma::mbar_init(&mbar, 1);
  pcb::umma::fence_async_smem();
  pcb::umma::tmem_fence_before();
  __syncthreads();
  pcb::umma::tmem_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t a0 = pcb::umma::smem_u32(sA), b0 = pcb::umma::smem_u32(sB);
    const uint32_t idesc = pcb::umma::idesc_i8(M, NH);
    for (int h = 0; h < N / NH; h++)
      for (int s = 0; s < K / 32; s++) {
        const uint64_t da = pcb::umma::desc_kmajor(a0 + s * 2 * M * 16, M);
        const uint64_t db = pcb::umma::desc_kmajor(b0 + s * 2 * N * 16 + (h * NH / 8) * 128, N);
        pcb::umma::mma_i8(tm + h * NH, da, db, idesc, s > 0);
      }
    pcb::umma::commit(&mbar);
  }
  pcb::umma::mbar_wait(&mbar, 0);
  pcb::umma::tmem_fence_after();
  const int warp = tid >> 5, lane = tid & 31;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    pcb::umma::tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
    pcb::umma::tmem_wait_ld();
    for (int j = 0; j < 16; j++) D[(size_t)row * N + c0 + j] = (int32_t)v[j];
  }
  pcb::umma::tmem_fence_before();
  __syncthreads();
  if (tid < 32) pcb::umma::tmem_dealloc<512>(tm);
}

int main() {
  std::vector<uint8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = (uint8_t)rand();
  for (auto& x : B) x = (uint8_t)rand();
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, (size_t)M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = (M + N) * K;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_test<<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<int32_t> D((size_t)M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; i++)
    for (int j = 0; j < N; j++) {
      int64_t s = 0;
      for (int k = 0; k < K; k++) s += (int)A[i * K + k] * (int)B[j * K + k];
      if (s != D[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %d want %lld\n", i, j, D[(size_t)i * N + j], (long long)s);
        bad++;
      }
    }
  printf("umma_i8_test: %ld mismatches of %d\n", bad, M * N);
  return bad != 0;
}
