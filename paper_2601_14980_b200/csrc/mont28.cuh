// mont28.cuh — carry-free batched Montgomery arithmetic in radix 2^r (r = 28 / 27).
//
// Why: on B200 a carry-chained IMAD.WIDE.U32.X issues at HALF the rate of a plain
// IMAD.WIDE.U32 (measured 9.27 vs 17.40 TMAC32/s, tools/imad_modes.cu, profiles/r01_imad_modes.txt),
// so a 32-bit-limb CIOS with carry chains (mont.cuh) tops out at ~53% of the IMAD roofline.
// Here every limb holds r < 32 bits and every partial product is accumulated into a 64-bit
// lazy accumulator with a plain IMAD.WIDE (no carry in/out):
//   * one CIOS row adds b*A_j + q*M_j to accumulator j; an accumulator lives N rows, so it
//     absorbs at most 2N products < 2^(2r):  2N * 2^(2r) < 2^64  (r = 28: N <= 127);
//   * the division by 2^r per row moves accumulators down one slot (register renaming in the
//     fully unrolled row loop) plus ONE carry (acc0 >> r) into the next slot;
//   * R = 2^(rN) > 4m, so outputs stay < 2m without a conditional subtraction per product
//     (lazy reduction); one normalisation pass (ALU pipe) per product restores r-bit limbs.
// All independent accumulators of a row give ptxas an ILP of ~N instead of one carry chain.
//
// Layout: TPI consecutive lanes cooperate on one residue (TPI = 1, 2, 4); lane t of a group owns
// limbs [tK, (t+1)K), K = N / TPI, for the accumulator, the multiplicand (registers) and the
// modulus (block-shared memory).  Row digits b_i come from a shared-memory slot in which digit
// i of group g sits at word (i * G + g), G = 32 / TPI  (conflict-free, lanes of a group
// broadcast).  Every exact algorithm yields the same residues as the reference's
// WordBarrett/pow_mod (bignat.cpp:273-321), so results stay bit-identical.
#pragma once
#include <cstdint>

// Row unroll of mm(): -1 = K rows (one register rotation, default), 0 = all N rows, r > 0 = r
// rows where r divides N (else K).
#ifndef PCB_R28_ROWS
#define PCB_R28_ROWS -1
#endif

namespace pcb {
namespace r28 {

__device__ __forceinline__ uint32_t lds32v(uint32_t a) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64v(uint32_t a) {
  uint2 v;
  asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32v(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// acc += a * b  (IMAD.WIDE.U32, no carry flags; free to schedule)
__device__ __forceinline__ void madw(uint64_t& acc, uint32_t a, uint32_t b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

template <int RB, int N, int TPI>
struct Cfg {
  static constexpr int K = N / TPI;
  static constexpr int G = 32 / TPI;
  static constexpr uint32_t MASK = (1u << RB) - 1u;
  static_assert(N % TPI == 0 && K % 2 == 0, "limb split");
  static_assert(2.0 * N * (double)(1ull << (2 * RB)) < 18446744073709551616.0, "lazy accumulator bound");
};

// Per-lane view of one residue slot in shared memory (digits of one group).
template <int RB, int N, int TPI>
struct DSlot {
  uint32_t a;  // byte address of digit 0 of this group
  __device__ __forceinline__ uint32_t digit(int i) const { return lds32v(a + i * Cfg<RB, N, TPI>::G * 4); }
  __device__ __forceinline__ void set(int i, uint32_t v) const { sts32v(a + i * Cfg<RB, N, TPI>::G * 4, v); }
  // lane t stores its K limbs
  __device__ __forceinline__ void store(const uint32_t (&x)[Cfg<RB, N, TPI>::K], int t) const {
    constexpr int K = Cfg<RB, N, TPI>::K;
#pragma unroll
    for (int j = 0; j < K; j++) set(t * K + j, x[j]);
  }
  __device__ __forceinline__ void load(uint32_t (&x)[Cfg<RB, N, TPI>::K], int t) const {
    constexpr int K = Cfg<RB, N, TPI>::K;
#pragma unroll
    for (int j = 0; j < K; j++) x[j] = digit(t * K + j);
  }
};

// R (lane's K limbs, normalised, value < 2m) = A * B * 2^(-rN) mod m (lazy).
//   A: lane's K limbs (registers), limbs < 2^r; B: digits in a DSlot, < 2^r; A, B < 2m.
//   mlane: shared byte address of this lane's K modulus limbs (8-byte aligned); minv = -m^-1 mod 2^r.
template <int RB, int N, int TPI>
__device__ __forceinline__ void mm(uint32_t (&R)[N / TPI], const uint32_t (&A)[N / TPI],
                                   const DSlot<RB, N, TPI>& B, uint32_t mlane, uint32_t minv, int t) {
  using C = Cfg<RB, N, TPI>;
  constexpr int K = C::K;
  uint64_t T[K];
#pragma unroll
  for (int j = 0; j < K; j++) T[j] = 0;
  // Rows are unrolled K at a time: the one-slot shift per row rotates the accumulator's register
  // names with period K, so a K-row body needs no moves, while the code stays 1/TPI of a full
  // unroll (a fully unrolled 152-row product is ~460 KB of SASS and stalls on instruction fetch).
  constexpr int RU = PCB_R28_ROWS == 0 ? N : ((PCB_R28_ROWS > 0 && N % PCB_R28_ROWS == 0) ? PCB_R28_ROWS : K);
  static_assert(N % RU == 0, "row unroll must divide N");
#pragma unroll 1
  for (int i0 = 0; i0 < N; i0 += RU) {
#pragma unroll
  for (int ii = 0; ii < RU; ii++) {
    const int i = i0 + ii;
    const uint32_t b = B.digit(i);
#pragma unroll
    for (int j = 0; j < K; j++) madw(T[j], A[j], b);
    uint32_t q = ((uint32_t)T[0] * minv) & C::MASK;
    if constexpr (TPI > 1) q = __shfl_sync(0xffffffffu, q, 0, TPI);
#pragma unroll
    for (int j = 0; j < K; j += 2) {
      const uint2 m2 = lds64v(mlane + j * 4);
      madw(T[j], m2.x, q);
      madw(T[j + 1], m2.y, q);
    }
    // divide by 2^r: lane 0's slot 0 is now 0 mod 2^r; every other slot moves down one place
    if constexpr (TPI == 1) {
      const uint64_t c0 = T[0] >> RB;
#pragma unroll
      for (int j = 0; j < K - 1; j++) T[j] = T[j + 1];
      T[K - 1] = 0;
      T[0] += c0;
    } else {
      const uint64_t lo = T[0];
      uint64_t in = __shfl_down_sync(0xffffffffu, lo, 1, TPI);
      if (t == TPI - 1) in = 0;
      const uint64_t c0 = (t == 0) ? (lo >> RB) : 0ull;
#pragma unroll
      for (int j = 0; j < K - 1; j++) T[j] = T[j + 1];
      T[K - 1] = in;
      T[0] += c0;
    }
  }
  }
  // normalise to r-bit limbs (ALU pipe); carries across lanes in TPI-1 rounds
  uint64_t c = 0;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const uint64_t v = T[j] + c;
    R[j] = (uint32_t)v & C::MASK;
    c = v >> RB;
  }
  if constexpr (TPI > 1) {
#pragma unroll
    for (int rnd = 0; rnd < TPI - 1; rnd++) {
      uint64_t cin = __shfl_up_sync(0xffffffffu, c, 1, TPI);
      if (t == 0) cin = 0;
      c = cin;
#pragma unroll
      for (int j = 0; j < K; j++) {
        const uint64_t v = (uint64_t)R[j] + c;
        R[j] = (uint32_t)v & C::MASK;
        c = v >> RB;
      }
    }
  }
}

// ---- conversions between 32-bit words and radix-2^r limbs (prologue/epilogue only) --------
// lane's K limbs of the value held in `w` (nw 32-bit words, LE) starting at limb `first`
template <int RB, int K>
__device__ __forceinline__ void words_to_limbs(uint32_t (&x)[K], const uint32_t* w, int nw, int first) {
  constexpr uint32_t MASK = (1u << RB) - 1u;
#pragma unroll
  for (int j = 0; j < K; j++) {
    const int bit = (first + j) * RB;
    const int wd = bit >> 5, sh = bit & 31;
    const uint32_t lo = wd < nw ? w[wd] : 0u;
    const uint32_t hi = wd + 1 < nw ? w[wd + 1] : 0u;
    x[j] = (uint32_t)((((uint64_t)hi << 32) | lo) >> sh) & MASK;
  }
}

// limbs (N in smem slot, any lane may read all) -> 32-bit word k
template <int RB, int N, int TPI>
__device__ __forceinline__ uint32_t limbs_word(const DSlot<RB, N, TPI>& s, int k) {
  const int bit = 32 * k;
  const int l0 = bit / RB, sh = bit - l0 * RB;
  uint64_t acc = 0;
  int got = -sh;
#pragma unroll 1
  for (int l = l0; l < N && got < 32; l++) {
    const uint64_t v = s.digit(l);
    if (got < 0)
      acc |= v >> (-got);
    else
      acc |= v << got;
    got += RB;
  }
  return (uint32_t)acc;
}

}  // namespace r28
}  // namespace pcb
