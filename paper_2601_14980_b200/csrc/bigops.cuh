// bigops.cuh — small fixed-width helpers around the Montgomery core (mont.cuh): loads,
// comparisons, modular add/sub, plain products.  All straight-line, register resident.
#pragma once
#include <cstdint>

#include "mont.cuh"

namespace pcb {

template <int S>
__device__ __forceinline__ void load_zext(uint32_t (&X)[S], const uint32_t* __restrict__ src, int nl) {
#pragma unroll
  for (int j = 0; j < S; j++) X[j] = j < nl ? src[j] : 0u;
}

template <int S>
__device__ __forceinline__ void zero(uint32_t (&X)[S]) {
#pragma unroll
  for (int j = 0; j < S; j++) X[j] = 0u;
}

template <int S>
__device__ __forceinline__ bool is_zero(const uint32_t (&X)[S]) {
  uint32_t o = 0;
#pragma unroll
  for (int j = 0; j < S; j++) o |= X[j];
  return o == 0;
}

// X < C  (C in constant bank or registers, S limbs)
template <int S>
__device__ __forceinline__ bool lt(const uint32_t (&X)[S], const uint32_t* __restrict__ C) {
  uint32_t d, hi;
  asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(X[0]), "r"(C[0]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(X[j]), "r"(C[j]));
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(hi));
  (void)d;
  return hi != 0;  // borrow out  <=>  X < C
}

// a < b for little-endian word arrays in memory (a: na words, b: nb words), scanning from the top.
__device__ __forceinline__ bool lt_words(const uint32_t* a, int na, const uint32_t* b, int nb) {
  const int n = na > nb ? na : nb;
  for (int j = n - 1; j >= 0; j--) {
    const uint32_t x = j < na ? a[j] : 0u, y = j < nb ? b[j] : 0u;
    if (x != y) return x < y;
  }
  return false;
}
__device__ __forceinline__ bool is_zero_words(const uint32_t* a, int na) {
  uint32_t o = 0;
  for (int j = 0; j < na; j++) o |= a[j];
  return o == 0;
}

// X = (X + Y) mod M for X, Y < M
template <int S, class MA>
__device__ __forceinline__ void mod_add(uint32_t (&X)[S], const uint32_t (&Y)[S], const MA& M) {
  uint32_t T[S + 1];
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(T[0]) : "r"(X[0]), "r"(Y[0]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(T[j]) : "r"(X[j]), "r"(Y[j]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(T[S]));
  cond_sub<S, MA>(T, M);
#pragma unroll
  for (int j = 0; j < S; j++) X[j] = T[j];
}

// X = (X - Y) mod M for X, Y < M
template <int S, class MA>
__device__ __forceinline__ void mod_sub(uint32_t (&X)[S], const uint32_t (&Y)[S], const MA& M) {
  uint32_t br;
  asm volatile("sub.cc.u32 %0, %0, %1;" : "+r"(X[0]) : "r"(Y[0]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("subc.cc.u32 %0, %0, %1;" : "+r"(X[j]) : "r"(Y[j]));
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(br));
  // add back M & br
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 e = M.ev4(c), o = M.od4(c);
    const uint32_t mm[8] = {e.x, o.x, e.y, o.y, e.z, o.z, e.w, o.w};
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (c == 0 && u == 0)
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(X[0]) : "r"(mm[0] & br));
      else
        asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(X[8 * c + u]) : "r"(mm[u] & br));
    }
  }
  asm volatile("addc.u32 %0, %0, 0;" : "+r"(br));  // consume carry (value unused)
}

// X += 1 mod M  (X < M)
template <int S, class MA>
__device__ __forceinline__ void mod_inc(uint32_t (&X)[S], const MA& M) {
  uint32_t T[S + 1];
  asm volatile("add.cc.u32 %0, %1, 1;" : "=r"(T[0]) : "r"(X[0]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("addc.cc.u32 %0, %1, 0;" : "=r"(T[j]) : "r"(X[j]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(T[S]));
  cond_sub<S, MA>(T, M);
#pragma unroll
  for (int j = 0; j < S; j++) X[j] = T[j];
}

// out[0..2N) = X + Y*C  with X (N limbs, registers), Y digits in slot `Ys` (N limbs),
// C an SMod (N limbs).  Low words are written back into the slot positions of the consumed
// digits; returns the high N words in H.  (Garner recombination c = c_p + p^2 t.)
template <int N>
__device__ __forceinline__ void mul_add_smod(uint32_t (&H)[N], const uint32_t (&X)[N], const Slot<N>& Ys,
                                             const SMod<N>& C) {
  uint32_t T[N + 2];
#pragma unroll
  for (int j = 0; j < N; j++) T[j] = X[j];
  T[N] = 0;
  T[N + 1] = 0;
#pragma unroll 1
  for (int i = 0; i < N; i++) {
    const uint32_t b = Ys.digit(i);
    uint32_t top;
#pragma unroll
    for (int c = 0; c < N / 8; c++) {
      const uint4 m = C.ev4(c);
      if (c == 0)
        mac_first(T[0], T[1], m.x, b);
      else
        mac_next(T[8 * c + 0], T[8 * c + 1], m.x, b);
      mac_next(T[8 * c + 2], T[8 * c + 3], m.y, b);
      mac_next(T[8 * c + 4], T[8 * c + 5], m.z, b);
      mac_next(T[8 * c + 6], T[8 * c + 7], m.w, b);
    }
    addc_cc(T[N]);
    top = carry_word();
#pragma unroll
    for (int c = 0; c < N / 8; c++) {
      const uint4 m = C.od4(c);
      if (c == 0)
        mac_first(T[1], T[2], m.x, b);
      else
        mac_next(T[8 * c + 1], T[8 * c + 2], m.x, b);
      mac_next(T[8 * c + 3], T[8 * c + 4], m.y, b);
      mac_next(T[8 * c + 5], T[8 * c + 6], m.z, b);
      mac_next(T[8 * c + 7], T[8 * c + 8], m.w, b);
    }
    addc_nc(top);
    Ys.set_digit(i, T[0]);  // finished low word i
#pragma unroll
    for (int j = 0; j < N; j++) T[j] = T[j + 1];
    T[N] = top;
  }
#pragma unroll
  for (int j = 0; j < N; j++) H[j] = T[j];
}

// Column (product-scanning) accumulator: 96 bits.
struct Col96 {
  uint64_t lo = 0;
  uint32_t hi = 0;
  __device__ __forceinline__ void add(uint64_t p) {
    lo += p;
    hi += (lo < p) ? 1u : 0u;
  }
  __device__ __forceinline__ uint32_t pop() {  // emit low word, shift right 32
    const uint32_t w = (uint32_t)lo;
    lo = (lo >> 32) | ((uint64_t)hi << 32);
    hi = 0;
    return w;
  }
};

// Truncated product  U = A * C mod 2^(32N)  (A registers, C constant bank).
template <int N>
__device__ __forceinline__ void mul_lo(uint32_t (&U)[N], const uint32_t (&A)[N], const uint32_t* __restrict__ C) {
  Col96 acc;
#pragma unroll
  for (int k = 0; k < N; k++) {
#pragma unroll
    for (int i = 0; i <= k; i++) acc.add((uint64_t)A[i] * C[k - i]);
    U[k] = acc.pop();
  }
}

// Does  U * C == X  hold exactly?  (U, C: N limbs; X: 2N limbs)  Used to verify the exact
// division of the L function.  Product scanning: no 2N-word temporary.
template <int N>
__device__ __forceinline__ bool mul_eq(const uint32_t (&U)[N], const uint32_t* __restrict__ C,
                                       const uint32_t (&X)[2 * N]) {
  Col96 acc;
  uint32_t d = 0;
#pragma unroll
  for (int k = 0; k < 2 * N - 1; k++) {
#pragma unroll
    for (int i = (k < N ? 0 : k - N + 1); i <= (k < N ? k : N - 1); i++) acc.add((uint64_t)U[i] * C[k - i]);
    d |= acc.pop() ^ X[k];
  }
  d |= acc.pop() ^ X[2 * N - 1];
  return d == 0;
}

}  // namespace pcb
