// side.cu — the hot kernel: one CRT half (one modulus) of a batch of Paillier exponentiations.
//
//   ENC  y = (1 + m n mod m2) * r^e mod m2        e = n mod phi(m2)   (paillier.cpp:339-342:
//                                                  g_power_half x half_pow, binomial g)
//   DEC  y = c^e mod m2                            e = p - 1           (the c^(p-1) form of the
//                                                  CRT decryption, paillier.cpp:357-358)
//   POW  y = x^e mod m2                            generic batched ModArith::pow
//
// Structure: a warp-uniform step machine wrapped around exactly ONE Montgomery product site.
// With a single site and a single modulus per kernel, ptxas keeps the modulus limbs in uniform
// registers (operands of IMAD.WIDE.U32.X, no vector registers, no loads in the inner loop) and
// the accumulator + multiplicand fit the register file.  Every step is  R = Acc * B * R^-1
// (A = the Acc slot, B = the Acc slot for squarings or the Op slot otherwise); the prologue /
// epilogue of each step only moves data between registers, smem slots and global memory.
#include <cstdint>
#include <cuda_runtime.h>

#include "bigops.cuh"
#include "mont.cuh"
#include "paillier_params.cuh"
#include "pcb_internal.h"

namespace pcb {

enum SideMode : int { kSideEnc = 0, kSideDec = 1, kSidePow = 2 };

template <int S>
struct SideArgs {
  ModCtx<S> mod;          // m2 (p^2, q^2 or any odd modulus)
  uint32_t c1[S];         // ENC: n R mod m2      DEC: R^3 mod m2
  const uint8_t* ops;     // exponent op stream (mont_pow format)
  int nops, ntab;
  uint4* tab;             // per-thread odd-power table + 1 park entry
  const uint32_t* x;      // ENC: r (x_limbs)   DEC: c (x_limbs = 2L)   POW: x
  int x_limbs;
  const uint32_t* m;      // ENC: plaintexts (m_limbs)
  int m_limbs;
  const int32_t* skip;    // per-element status from validation (nullable): != 0 => skip
  uint32_t* y;            // count x S (AoS), plain residues
  int count, mode;
};

#ifndef PCB_SIDE_AREG_MAX
#define PCB_SIDE_AREG_MAX 64  // largest S that keeps the multiplicand in registers
#endif
#ifndef PCB_SIDE_MINB
#define PCB_SIDE_MINB 1
#endif
template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock, PCB_SIDE_MINB) side_kernel(const __grid_constant__ SideArgs<S> P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr bool AR = S <= PCB_SIDE_AREG_MAX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Slot<S> Acc{smem_addr(smem + warp * (64 * S) + lane * 4)};
  const Slot<S> Op{smem_addr(smem + warp * (64 * S) + 32 * S + lane * 4)};
  const uint32_t nthr = gridDim.x * blockDim.x;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const GTable<S> tab{P.tab, nthr, g};
  const PMod<S> M(P.mod);
  const int park = P.ntab;
  // step plan (uniform):  [pre0] pre1 | x^2 | table (ntab-1) | main (nops-1) | final
  const int npre = P.mode == kSidePow ? 1 : 2;
  const int s_x2 = npre, s_tab = s_x2 + 1, s_main = s_tab + (P.ntab - 1), s_fin = s_main + (P.nops - 1);
  const int nsteps = s_fin + 1;

  for (int i = g; i < P.count; i += nthr) {
    if (P.skip && P.skip[i] != 0) continue;
    const uint32_t* xs = P.x + (size_t)i * P.x_limbs;
#pragma unroll 1
    for (int s = 0; s < nsteps; s++) {
      // ---- prologue: stage A in Acc and B in Op (or B = Acc for squarings) -----------------
      bool b_is_acc = false;
      if (s < npre) {
        const bool first = s == 0 && npre == 2;
        if (P.mode == kSideEnc) {
          if (first) {  // A = m, B = n R          -> m n
            Acc.store_global(P.m + (size_t)i * P.m_limbs, P.m_limbs);
            Op.store_const(P.c1);
          } else {      // A = r, B = R^2          -> r R
            Acc.store_global(xs, P.x_limbs);
            Op.store_const(P.mod.r2);
          }
        } else if (P.mode == kSideDec) {
          if (first) {  // A = c_hi, B = R^3       -> c_hi R^2
            Acc.store_global(xs + S, P.x_limbs - S);
            Op.store_const(P.c1);
          } else {      // A = c_lo, B = R^2       -> c_lo R
            Acc.store_global(xs, P.x_limbs < S ? P.x_limbs : S);
            Op.store_const(P.mod.r2);
          }
        } else {        // POW: A = x, B = R^2
          Acc.store_global(xs, P.x_limbs);
          Op.store_const(P.mod.r2);
        }
      } else if (s == s_x2) {
        b_is_acc = true;  // x^2
      } else if (s < s_main) {
        // table build: Acc = x^(2e-1), Op = x^2
      } else if (s < s_fin) {
        const uint8_t op = P.ops[s - s_main + 1];
        if (op == kOpSquare)
          b_is_acc = true;
        else
          tab.to_slot(op, Op);
      } else {  // final
        if (P.mode == kSideEnc)
          tab.to_slot(park, Op);  // (1 + m n), plain  -> result plain
        else
          Op.store_small(1);      // out of Montgomery form
      }
      // ---- the single Montgomery product site --------------------------------------------
      uint32_t R[S];
      mont_mul_ss<S, AR, PMod<S>, S / 2>(R, Acc, b_is_acc ? Acc : Op, M);  // fully unrolled rows
      // ---- epilogue -------------------------------------------------------------------------
      if (s < npre) {
        const bool first = s == 0 && npre == 2;
        if (first) {
          if (P.mode == kSideEnc) {
            uint32_t one[S];
#pragma unroll
            for (int j = 0; j < S; j++) one[j] = j == 0;
            // 1 + m n mod m2 (g_power_half, paillier.cpp:263): add with carry, then reduce
            uint32_t T[S + 1];
            asm volatile("add.cc.u32 %0, %1, 1;" : "=r"(T[0]) : "r"(R[0]));
#pragma unroll
            for (int j = 1; j < S; j++) asm volatile("addc.cc.u32 %0, %1, 0;" : "=r"(T[j]) : "r"(R[j]));
            asm volatile("addc.u32 %0, 0, 0;" : "=r"(T[S]));
            cond_sub<S, PMod<S>>(T, M);
#pragma unroll
            for (int j = 0; j < S; j++) R[j] = T[j];
            (void)one;
          }
          tab.put(park, R);
        } else {
          if (P.mode == kSideDec) {  // c R = c_lo R + c_hi R^2
            uint32_t H[S];
            tab.get(park, H);
            uint32_t T[S + 1];
            asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(T[0]) : "r"(R[0]), "r"(H[0]));
#pragma unroll
            for (int j = 1; j < S; j++) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(T[j]) : "r"(R[j]), "r"(H[j]));
            asm volatile("addc.u32 %0, 0, 0;" : "=r"(T[S]));
            cond_sub<S, PMod<S>>(T, M);
#pragma unroll
            for (int j = 0; j < S; j++) R[j] = T[j];
          }
          Acc.store(R);
          tab.put(0, R);  // x
        }
      } else if (s == s_x2) {
        Op.store(R);  // x^2 ; Acc still holds x
      } else if (s < s_main) {
        Acc.store(R);
        tab.put(s - s_tab + 1, R);
        if (s == s_main - 1) tab.to_slot(P.ops[0], Acc);  // seed the accumulator
      } else if (s < s_fin) {
        Acc.store(R);
      } else {
        uint4* dst = reinterpret_cast<uint4*>(P.y + (size_t)i * S);
#pragma unroll
        for (int c = 0; c < S / 4; c++) dst[c] = make_uint4(R[4 * c], R[4 * c + 1], R[4 * c + 2], R[4 * c + 3]);
      }
      if (P.ntab == 1 && s == s_x2) tab.to_slot(P.ops[0], Acc);  // degenerate table (w = 1)
    }
  }
}

// Canonical algorithmic MAC32 of one element: MM(k) = 2 s^2 + s,
// EXP(k, e) = (e + ceil(e/4)) MM(k); one CRT half of Enc = EXP(|n|, |n|) + 2 MM(|n|),
// of Dec = EXP(|n|, |n|/2) + 2 MM(|n|).  `ebits_canon` is the canonical exponent width.
static double canon_mac32(int S, int ebits_canon) {
  const double mm = 2.0 * S * S + S;
  return ((double)ebits_canon + (double)((ebits_canon + 3) / 4)) * mm + 2.0 * mm;
}

template <int S>
pcb_status launch_side(const ModCtx<S>& mod, const uint32_t* c1, const uint8_t* ops, int nops, int ntab, int mode,
                       const uint32_t* x, int x_limbs, const uint32_t* m, int m_limbs, const int32_t* skip,
                       size_t count, uint32_t* y, cudaStream_t st, int ebits_canon) {
  SideArgs<S> P;
  P.mod = mod;
  for (int j = 0; j < S; j++) P.c1[j] = c1 ? c1[j] : 0u;
  P.ops = ops;
  P.nops = nops;
  P.ntab = ntab;
  P.x = x;
  P.x_limbs = x_limbs;
  P.m = m;
  P.m_limbs = m_limbs;
  P.skip = skip;
  P.y = y;
  P.count = (int)count;
  P.mode = mode;
  const size_t smem = (size_t)kThreadsPerBlock * S * 8;
  int blocks = 0;
  if (auto e = item_grid(side_kernel<S>, smem, count, &blocks)) return e;
  const size_t nthr = (size_t)blocks * kThreadsPerBlock;
  if (auto e = scratch_alloc(nthr * (ntab + 1) * S * 4, (void**)&P.tab, st)) return e;
  ProfMark pm;
  if (prof_enabled()) pm = prof_start(st);
  side_kernel<S><<<blocks, kThreadsPerBlock, smem, st>>>(P);
  count_launch();
  // ebits_canon < 0: a stage whose canonical work is accounted on another launch
  if (prof_enabled()) prof_stop(pm, st, ebits_canon < 0 ? 0.0 : canon_mac32(S, ebits_canon) * (double)count);
  scratch_free(P.tab, st);
  return cuda_check(cudaGetLastError());
}

#define PCB_SIDE(S)                                                                                               \
  template pcb_status launch_side<S>(const ModCtx<S>&, const uint32_t*, const uint8_t*, int, int, int,          \
                                     const uint32_t*, int, const uint32_t*, int, const int32_t*, size_t, uint32_t*, \
                                     cudaStream_t, int);
PCB_SIDE(32)
PCB_SIDE(64)

}  // namespace pcb
