// modexp.cu — batched fixed-exponent modular exponentiation  y_i = x_i^e mod m.
//
// The generic primitive behind every Paillier half-exponentiation; exported on its own as
// pcb_modexp_batch (the batched counterpart of the reference's ModArith::pow /
// pow_mod, /root/reference/proj/src/paillier.cpp:26-30, bignat.cpp:295-321) and used by the
// tests to pin the Montgomery core against Python's pow() on random odd moduli.
#include <cstdint>
#include <cuda_runtime.h>

#include "bigops.cuh"
#include "mont.cuh"
#include "pcb_internal.h"

namespace pcb {

template <int S>
struct ModexpParams {
  ModCtx<S> mod;
  const uint32_t* x;      // count x x_limbs (AoS), x < 2^(32 x_limbs), x_limbs <= S
  uint32_t* y;            // count x S (AoS)
  const uint8_t* ops;     // exponent op stream (build_ops)
  uint4* tab;             // per-thread odd-power tables
  int nsched, ntab, x_limbs, count, exp_is_zero;
};

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) modexp_kernel(const __grid_constant__ ModexpParams<S> P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr bool AR = S <= 64;
  smod_fill<S>(smem, P.mod.m);
  __syncthreads();
  const SMod<S> M{smem_addr(smem), P.mod.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + S;
  const Slot<S> Acc{smem_addr(slots + warp * (64 * S) + lane * 4)};
  const Slot<S> Op{smem_addr(slots + warp * (64 * S) + 32 * S + lane * 4)};
  const uint32_t nthr = gridDim.x * blockDim.x;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  GTable<S> tab{P.tab, nthr, g};
  for (int i = g; i < P.count; i += nthr) {
    uint32_t X[S];
    if (P.exp_is_zero) {
      // x^0 = 1 mod m (0 when m == 1: exp_is_zero == 2)
#pragma unroll
      for (int j = 0; j < S; j++) X[j] = 0;
      X[0] = P.exp_is_zero == 1 ? 1u : 0u;
    } else {
      Acc.store_global(P.x + (size_t)i * P.x_limbs, P.x_limbs);
      Op.store_const(P.mod.r2);
      mont_mul_ss<S, AR>(X, Acc, Op, M);  // x R mod m (also reduces x)
      Acc.store(X);
      mont_pow<S, AR>(Acc, Op, tab, P.ntab, P.ops, P.nsched, M);
      Op.store_small(1);
      mont_mul_ss<S, AR>(X, Acc, Op, M);  // out of Montgomery form
    }
    uint4* dst = reinterpret_cast<uint4*>(P.y + (size_t)i * S);
#pragma unroll
    for (int c = 0; c < S / 4; c++) dst[c] = make_uint4(X[4 * c], X[4 * c + 1], X[4 * c + 2], X[4 * c + 3]);
  }
}

template <int S>
static pcb_status launch_modexp(const uint32_t* m, const uint32_t* r2, uint32_t minv, const uint32_t* sched_d,
                                int nsched, int ntab, bool exp_zero, const uint32_t* x_d, uint32_t x_limbs,
                                size_t count, uint32_t* y_d, cudaStream_t st) {
  ModexpParams<S> P{};
  for (int j = 0; j < S; j++) {
    P.mod.m[j] = m[j];
    P.mod.r2[j] = r2[j];
  }
  P.mod.minv = minv;
  P.x = x_d;
  P.y = y_d;
  P.ops = (const uint8_t*)sched_d;
  P.nsched = nsched;
  P.ntab = ntab;
  P.x_limbs = (int)x_limbs;
  P.count = (int)count;
  P.exp_is_zero = exp_zero ? (m[0] == 1 && [&] { for (int j = 1; j < S; j++) if (m[j]) return false; return true; }() ? 2 : 1) : 0;
  const size_t smem = (size_t)kThreadsPerBlock * S * 8 + S * 4;
  int blocks = 0;
  if (auto e = occupancy_grid(modexp_kernel<S>, smem, &blocks)) return e;
  const uint32_t nthr = (uint32_t)blocks * kThreadsPerBlock;
  uint4* tab = nullptr;
  if (auto e = scratch_alloc((size_t)nthr * ntab * S * 4, (void**)&tab, st)) return e;
  P.tab = tab;
  modexp_kernel<S><<<blocks, kThreadsPerBlock, smem, st>>>(P);
  return cuda_check(cudaGetLastError());
}

pcb_status modexp_dispatch(int S, const uint32_t* m, const uint32_t* r2, uint32_t minv, const uint32_t* sched_d,
                           int nsched, int ntab, bool exp_zero, const uint32_t* x_d, uint32_t x_limbs, size_t count,
                           uint32_t* y_d, cudaStream_t st) {
  switch (S) {
    case 32: return launch_modexp<32>(m, r2, minv, sched_d, nsched, ntab, exp_zero, x_d, x_limbs, count, y_d, st);
    case 64: return launch_modexp<64>(m, r2, minv, sched_d, nsched, ntab, exp_zero, x_d, x_limbs, count, y_d, st);
    case 96: return launch_modexp<96>(m, r2, minv, sched_d, nsched, ntab, exp_zero, x_d, x_limbs, count, y_d, st);
    default: return PCB_E_SHAPE;
  }
}

}  // namespace pcb
