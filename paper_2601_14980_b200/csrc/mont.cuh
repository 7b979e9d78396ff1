// mont.cuh — batched Montgomery arithmetic for sm_100a (one big-integer residue per thread).
//
// Replaces the reference's WordBarrett::mul_mod / pow_mod inner loop
// (/root/reference/proj/src/bignat.cpp:273-321, used by Paillier::half_pow paillier.cpp:275-305)
// with a CIOS Montgomery product on 32-bit limbs.  Any exact modular algorithm yields the same
// residues, so the results are bit-identical to the reference.
//
// Hardware mapping (B200, sm_100a):
//   * every 32x32->64 multiply-accumulate is ONE `IMAD.WIDE.U32(.X)`: ptxas fuses the PTX pair
//     `mad{c}.lo.cc.u32 / madc.hi.cc.u32` acting on an aligned 64-bit register pair into a single
//     wide multiply-add with a predicate carry in/out (checked with cuobjdump);
//   * the accumulator is kept as two arrays E ("even") and O ("odd") whose register pairs never
//     overlap: products b*A[2k] land on E pairs, b*A[2k+1] on O pairs.  The per-row division by
//     2^32 is free: E and O swap roles every row, and the remaining two-word shift of the array
//     that becomes "odd" is fused into the next row's multiply-add (destination pair != addend
//     pair), so the inner loop has no register moves at all;
//   * the modulus is part of a __grid_constant__ kernel parameter: its limbs are uniform
//     (constant-bank / uniform-register) operands, costing no vector registers;
//   * row digits b_i (and, for wide moduli, the multiplicand A) come from a per-thread shared
//     memory slot laid out in warp-interleaved 16-byte chunks (conflict-free LDS.128/STS.128);
//   * the exponent is batch-uniform (r^n, c^(p-1) ...): the window schedule is one byte stream
//     read by all threads — no divergence, no per-element exponent traffic.
#pragma once
#include <cstdint>

namespace pcb {

// ------------------------------------------------------------------------------------------
// Carry-chain primitives.  `asm volatile` keeps the PTX order of each chain (the CC flag is an
// implicit dependency NVVM does not see); ptxas still schedules independent chains freely.
// ------------------------------------------------------------------------------------------
// {hi:lo} += a*b (no carry in), CC out
__device__ __forceinline__ void mac_first(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
  asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
               : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// {hi:lo} += a*b + CC, CC out
__device__ __forceinline__ void mac_next(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
  asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
               : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// {dhi:dlo} = a*b + {shi:slo} + CC, CC out   (the fused two-word shift)
__device__ __forceinline__ void mac_shift(uint32_t& dlo, uint32_t& dhi, uint32_t a, uint32_t b, uint32_t slo,
                                          uint32_t shi) {
  asm volatile("madc.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.cc.u32 %1, %2, %3, %5;"
               : "=r"(dlo), "=r"(dhi) : "r"(a), "r"(b), "r"(slo), "r"(shi));
}
__device__ __forceinline__ void add_cc(uint32_t& x, uint32_t y) { asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(x) : "r"(y)); }
__device__ __forceinline__ void addc_cc(uint32_t& x) { asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(x)); }
__device__ __forceinline__ void addc_nc(uint32_t& x) { asm volatile("addc.u32 %0, %0, 0;" : "+r"(x)); }
__device__ __forceinline__ uint32_t carry_word() {
  uint32_t r;
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(r));
  return r;
}

// ------------------------------------------------------------------------------------------
// Per-modulus constants (host-computed, passed by value inside a __grid_constant__ param).
// ------------------------------------------------------------------------------------------
template <int S>
struct ModCtx {
  uint32_t m[S];    // modulus, little-endian u32 limbs, zero padded (odd, m < 2^(32S))
  uint32_t r2[S];   // R^2 mod m, R = 2^(32S)
  uint32_t minv;    // -m^(-1) mod 2^32
  uint32_t pad_[3];
};

// ------------------------------------------------------------------------------------------
// Shared-memory operand slots.  A slot holds S words of one thread in the warp-interleaved
// chunked layout:  chunk c (16 B) of lane l lives at  warp_base + c*128 + l*4  (words).
// Chunks [0, S/8) hold the even-indexed limbs (A0,A2,A4,A6 | A8,...), chunks [S/8, S/4) the
// odd-indexed limbs, so the even/odd product chains each read whole 16-byte chunks.
// The per-thread global-memory power tables use the same chunk order (thread-major inside a
// chunk => a warp's chunk access is one contiguous 512-byte segment).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
struct Slot {
  uint32_t a;  // shared-window byte address of this lane's chunk 0 (= warp_base + lane*16)
  __device__ __forceinline__ uint4 chunk(int c) const { return lds128(a + c * 512); }
  __device__ __forceinline__ void set_chunk(int c, uint4 v) const { sts128(a + c * 512, v); }
  __device__ __forceinline__ uint32_t digit_addr(int i) const {
    const int c = (i & 1) ? (S / 8 + (i >> 3)) : (i >> 3);
    return a + c * 512 + ((i >> 1) & 3) * 4;
  }
  __device__ __forceinline__ uint32_t digit(int i) const { return lds32(digit_addr(i)); }
  __device__ __forceinline__ void set_digit(int i, uint32_t v) const { sts32(digit_addr(i), v); }
  // even digit 2t / odd digit 2t+1
  __device__ __forceinline__ uint32_t digit_ev(int t) const { return lds32(a + (t >> 2) * 512 + (t & 3) * 4); }
  __device__ __forceinline__ uint32_t digit_od(int t) const { return lds32(a + (S / 8 + (t >> 2)) * 512 + (t & 3) * 4); }
  template <int N>
  __device__ __forceinline__ void store(const uint32_t (&x)[N]) const {
    static_assert(N >= S, "store width");
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      set_chunk(c, make_uint4(x[8 * c], x[8 * c + 2], x[8 * c + 4], x[8 * c + 6]));
      set_chunk(S / 8 + c, make_uint4(x[8 * c + 1], x[8 * c + 3], x[8 * c + 5], x[8 * c + 7]));
    }
  }
  __device__ __forceinline__ void store_const(const uint32_t* x) const {
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      set_chunk(c, make_uint4(x[8 * c], x[8 * c + 2], x[8 * c + 4], x[8 * c + 6]));
      set_chunk(S / 8 + c, make_uint4(x[8 * c + 1], x[8 * c + 3], x[8 * c + 5], x[8 * c + 7]));
    }
  }
  // global AoS limbs (nl <= S valid, rest zero)
  __device__ __forceinline__ void store_global(const uint32_t* __restrict__ src, int nl) const {
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      const int j = 8 * c;
      set_chunk(c, make_uint4(j < nl ? src[j] : 0u, j + 2 < nl ? src[j + 2] : 0u, j + 4 < nl ? src[j + 4] : 0u,
                              j + 6 < nl ? src[j + 6] : 0u));
      set_chunk(S / 8 + c, make_uint4(j + 1 < nl ? src[j + 1] : 0u, j + 3 < nl ? src[j + 3] : 0u,
                                      j + 5 < nl ? src[j + 5] : 0u, j + 7 < nl ? src[j + 7] : 0u));
    }
  }
  __device__ __forceinline__ void store_small(uint32_t w0) const {  // value w0 < 2^32
    set_chunk(0, make_uint4(w0, 0, 0, 0));
#pragma unroll
    for (int c = 1; c < S / 4; c++) set_chunk(c, make_uint4(0, 0, 0, 0));
  }
  template <int N>
  __device__ __forceinline__ void load(uint32_t (&x)[N]) const {
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      uint4 e = chunk(c), o = chunk(S / 8 + c);
      x[8 * c] = e.x; x[8 * c + 2] = e.y; x[8 * c + 4] = e.z; x[8 * c + 6] = e.w;
      x[8 * c + 1] = o.x; x[8 * c + 3] = o.y; x[8 * c + 5] = o.z; x[8 * c + 7] = o.w;
    }
  }
};

// Block-shared copy of a modulus in the same even/odd split layout (one 16-byte chunk per
// 4 limbs, no lane interleave): every lane reads the same address => broadcast LDS.128.
// Loaded once per block; the asm volatile loads stop ptxas from hoisting the S limbs into
// vector registers (which would not fit next to the accumulator at S >= 64).
template <int S>
struct SMod {
  uint32_t a;      // shared byte address: chunks [0,S/8) even limbs, [S/8,S/4) odd limbs
  uint32_t minv;
  __device__ __forceinline__ uint4 ev4(int c) const { return lds128(a + c * 16); }
  __device__ __forceinline__ uint4 od4(int c) const { return lds128(a + (S / 8 + c) * 16); }
  __device__ __forceinline__ uint32_t limb(int j) const {
    return lds32(a + ((j & 1) ? (S / 8 + (j >> 3)) : (j >> 3)) * 16 + ((j >> 1) & 3) * 4);
  }
};

// Modulus read straight from a __grid_constant__ kernel parameter: with a single product
// site per kernel, ptxas keeps these limbs in uniform registers (IMAD.WIDE UR operands).
template <int S>
struct PMod {
  const ModCtx<S>& k;
  uint32_t minv;
  __device__ __forceinline__ explicit PMod(const ModCtx<S>& c) : k(c), minv(c.minv) {}
  __device__ __forceinline__ uint4 ev4(int c) const { return make_uint4(k.m[8 * c], k.m[8 * c + 2], k.m[8 * c + 4], k.m[8 * c + 6]); }
  __device__ __forceinline__ uint4 od4(int c) const { return make_uint4(k.m[8 * c + 1], k.m[8 * c + 3], k.m[8 * c + 5], k.m[8 * c + 7]); }
};

// Cooperative fill of an SMod by the threads of a block (call __syncthreads() after).
template <int S>
__device__ __forceinline__ void smod_fill(uint32_t* dst, const uint32_t* m) {
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    const int c = (j & 1) ? (S / 8 + (j >> 3)) : (j >> 3);
    dst[c * 4 + ((j >> 1) & 3)] = m[j];
  }
}

// Per-thread table in global memory: entry e, chunk c of global thread g at
//   tab[((e * (S/4) + c) * nthreads + g)]   (uint4 units)
template <int S>
struct GTable {
  uint4* tab;
  uint32_t nthr, g;
  __device__ __forceinline__ uint4* at(int e, int c) const { return tab + ((size_t)(e * (S / 4) + c) * nthr + g); }
  template <int N>
  __device__ __forceinline__ void put(int e, const uint32_t (&x)[N]) const {
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      *at(e, c) = make_uint4(x[8 * c], x[8 * c + 2], x[8 * c + 4], x[8 * c + 6]);
      *at(e, S / 8 + c) = make_uint4(x[8 * c + 1], x[8 * c + 3], x[8 * c + 5], x[8 * c + 7]);
    }
  }
  template <int N>
  __device__ __forceinline__ void get(int e, uint32_t (&x)[N]) const {
#pragma unroll
    for (int c = 0; c < S / 8; c++) {
      uint4 ev = *at(e, c), od = *at(e, S / 8 + c);
      x[8 * c] = ev.x; x[8 * c + 2] = ev.y; x[8 * c + 4] = ev.z; x[8 * c + 6] = ev.w;
      x[8 * c + 1] = od.x; x[8 * c + 3] = od.y; x[8 * c + 5] = od.z; x[8 * c + 7] = od.w;
    }
  }
  __device__ __forceinline__ void to_slot(int e, const Slot<S>& s) const {
    uint4 v[S / 4];
#pragma unroll
    for (int c = 0; c < S / 4; c++) v[c] = *at(e, c);
#pragma unroll
    for (int c = 0; c < S / 4; c++) s.set_chunk(c, v[c]);
  }
};

// ------------------------------------------------------------------------------------------
// Operand accessors.  ev4(c) = (A[8c], A[8c+2], A[8c+4], A[8c+6]);  od4(c) = the odd limbs.
// ------------------------------------------------------------------------------------------
template <int S>
struct ARegs {  // multiplicand in registers
  const uint32_t (&A)[S];
  __device__ __forceinline__ uint4 ev4(int c) const { return make_uint4(A[8 * c], A[8 * c + 2], A[8 * c + 4], A[8 * c + 6]); }
  __device__ __forceinline__ uint4 od4(int c) const { return make_uint4(A[8 * c + 1], A[8 * c + 3], A[8 * c + 5], A[8 * c + 7]); }
};
template <int S>
struct ASlot {  // multiplicand streamed from this thread's shared-memory slot
  Slot<S> s;
  __device__ __forceinline__ uint4 ev4(int c) const { return s.chunk(c); }
  __device__ __forceinline__ uint4 od4(int c) const { return s.chunk(S / 8 + c); }
};
__device__ __forceinline__ uint4 lds128v(uint32_t a) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
// Streamed multiplicand that ptxas may not CSE across rows (volatile): keeps A out of the
// register file (2S+4 live registers in the core instead of 3S+4).
template <int S>
struct ASlotV {
  uint32_t a;
  __device__ __forceinline__ uint4 ev4(int c) const { return lds128v(a + c * 512); }
  __device__ __forceinline__ uint4 od4(int c) const { return lds128v(a + (S / 8 + c) * 512); }
};

// ------------------------------------------------------------------------------------------
// One CIOS row on the split accumulator.
//   Er: "even" role — word j at weight j (j < S).
//   Or: "odd" role with a pending two-word shift — Or[j] at weight j-1 (j = 1..S+1).
// Computes  V <- (V + b*A + q*M) / 2^32,  q = (V + b*A)_0 * minv mod 2^32, after which the roles
// swap: Or holds the new even words, Er the new odd words (again pending a two-word shift).
// ------------------------------------------------------------------------------------------
template <int S, class AA, class MA>
__device__ __forceinline__ void mont_row(uint32_t (&Er)[S + 2], uint32_t (&Or)[S + 2], const AA& A, uint32_t b,
                                         const MA& M) {
  // weight-0 word of the odd role joins the even role; its carry enters the odd chain
  add_cc(Er[0], Or[1]);
  // odd products, fused shift:  (Or[2k], Or[2k+1]) = b*A[2k+1] + (Or[2k+2], Or[2k+3]) + cc
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 a = A.od4(c);
    mac_shift(Or[8 * c + 0], Or[8 * c + 1], a.x, b, Or[8 * c + 2], Or[8 * c + 3]);
    mac_shift(Or[8 * c + 2], Or[8 * c + 3], a.y, b, Or[8 * c + 4], Or[8 * c + 5]);
    mac_shift(Or[8 * c + 4], Or[8 * c + 5], a.z, b, Or[8 * c + 6], Or[8 * c + 7]);
    mac_shift(Or[8 * c + 6], Or[8 * c + 7], a.w, b, Or[8 * c + 8], Or[8 * c + 9]);
  }
  uint32_t co = carry_word();
  // even products
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 a = A.ev4(c);
    if (c == 0)
      mac_first(Er[0], Er[1], a.x, b);
    else
      mac_next(Er[8 * c + 0], Er[8 * c + 1], a.x, b);
    mac_next(Er[8 * c + 2], Er[8 * c + 3], a.y, b);
    mac_next(Er[8 * c + 4], Er[8 * c + 5], a.z, b);
    mac_next(Er[8 * c + 6], Er[8 * c + 7], a.w, b);
  }
  uint32_t ce = carry_word();
  const uint32_t q = Er[0] * M.minv;
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 m = M.ev4(c);
    if (c == 0)
      mac_first(Er[0], Er[1], m.x, q);
    else
      mac_next(Er[8 * c + 0], Er[8 * c + 1], m.x, q);
    mac_next(Er[8 * c + 2], Er[8 * c + 3], m.y, q);
    mac_next(Er[8 * c + 4], Er[8 * c + 5], m.z, q);
    mac_next(Er[8 * c + 6], Er[8 * c + 7], m.w, q);
  }
  addc_nc(ce);
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 m = M.od4(c);
    if (c == 0)
      mac_first(Or[0], Or[1], m.x, q);
    else
      mac_next(Or[8 * c + 0], Or[8 * c + 1], m.x, q);
    mac_next(Or[8 * c + 2], Or[8 * c + 3], m.y, q);
    mac_next(Or[8 * c + 4], Or[8 * c + 5], m.z, q);
    mac_next(Or[8 * c + 6], Or[8 * c + 7], m.w, q);
  }
  addc_nc(co);
  // Er becomes the odd role: its words 2..S+1 carry weights 1..S of the next row
  Er[S] = ce;
  Er[S + 1] = co;
}

// If T (S+1 words, T < 2m) >= m then T -= m.  Two borrow chains, no extra S-word temporary.
template <int S, class MA>
__device__ __forceinline__ void cond_sub(uint32_t (&T)[S + 1], const MA& M) {
  uint32_t d, hi;
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 e = M.ev4(c), o = M.od4(c);
    const uint32_t mm[8] = {e.x, o.x, e.y, o.y, e.z, o.z, e.w, o.w};
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (c == 0 && u == 0)
        asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(T[0]), "r"(mm[0]));
      else
        asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(T[8 * c + u]), "r"(mm[u]));
    }
  }
  asm volatile("subc.u32 %0, %1, 0;" : "=r"(hi) : "r"(T[S]));
  // hi == 0xffffffff  <=>  T < m  (keep);  hi == 0  <=>  T >= m  (subtract)
  const uint32_t mask = ~hi;
#pragma unroll
  for (int c = 0; c < S / 8; c++) {
    const uint4 e = M.ev4(c), o = M.od4(c);
    const uint32_t mm[8] = {e.x, o.x, e.y, o.y, e.z, o.z, e.w, o.w};
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (c == 0 && u == 0)
        asm volatile("sub.cc.u32 %0, %0, %1;" : "+r"(T[0]) : "r"(mm[0] & mask));
      else
        asm volatile("subc.cc.u32 %0, %0, %1;" : "+r"(T[8 * c + u]) : "r"(mm[u] & mask));
    }
  }
  asm volatile("subc.u32 %0, %0, 0;" : "+r"(T[S]));
  (void)d;
}

// Row pairs per loop iteration.  The hot side kernel unrolls all S/2 row pairs (no loop
// back-edge => ptxas renames the shifted accumulator freely instead of emitting register
// moves; measured +14% on 2048-bit modexp); cold kernels keep 1 for code size.
#ifndef PCB_ROW_UNROLL
#define PCB_ROW_UNROLL 1
#endif
constexpr int kRowUnroll = PCB_ROW_UNROLL;

// R = A * B * 2^(-32S) mod m, fully reduced.  B digits from a smem slot.
// Preconditions: A < 2^(32S), B < m  (then the CIOS bound gives V < 2m before cond_sub).
template <int S, class AA, class MA, int U = kRowUnroll>
__device__ __forceinline__ void mont_mul_core(uint32_t (&R)[S], const AA& A, const Slot<S>& B, const MA& M) {
  uint32_t X[S + 2], Y[S + 2];
#pragma unroll
  for (int j = 0; j < S + 2; j++) {
    X[j] = 0;
    Y[j] = 0;
  }
#pragma unroll U
  for (int t = 0; t < S / 2; t++) {
    const uint32_t b0 = B.digit_ev(t), b1 = B.digit_od(t);
    mont_row<S, AA, MA>(X, Y, A, b0, M);  // X even-role, Y odd-role
    mont_row<S, AA, MA>(Y, X, A, b1, M);  // roles swapped back
  }
  // V = sum X[j] 2^(32j) + sum_{i>=1} Y[i] 2^(32(i-1))
  uint32_t T[S + 1];
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(T[0]) : "r"(X[0]), "r"(Y[1]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(T[j]) : "r"(X[j]), "r"(Y[j + 1]));
  asm volatile("addc.u32 %0, %1, 0;" : "=r"(T[S]) : "r"(Y[S + 1]));
  cond_sub<S, MA>(T, M);
#pragma unroll
  for (int j = 0; j < S; j++) R[j] = T[j];
}

// Register multiplicand.
template <int S, class MA>
__device__ __forceinline__ void mont_mul(uint32_t (&R)[S], const uint32_t (&A)[S], const Slot<S>& B, const MA& M) {
  mont_mul_core<S, ARegs<S>, MA>(R, ARegs<S>{A}, B, M);
}

// Slot form:  R (registers) = A(slot) * B(slot) * R^-1 mod m.
//   AREG = true : A is copied into registers first (3S+4 live registers in the core);
//   AREG = false: A is streamed from shared memory by both product chains (2S+4 registers).
template <int S, bool AREG, class MA, int U = kRowUnroll>
__device__ __forceinline__ void mont_mul_ss(uint32_t (&R)[S], const Slot<S>& A, const Slot<S>& B, const MA& M) {
  if constexpr (AREG) {
    uint32_t Ar[S];
    A.load(Ar);
    mont_mul_core<S, ARegs<S>, MA, U>(R, ARegs<S>{Ar}, B, M);
  } else {
    mont_mul_core<S, ASlotV<S>, MA, U>(R, ASlotV<S>{A.a}, B, M);
  }
}

// ------------------------------------------------------------------------------------------
// Fixed-exponent sliding-window exponentiation (warp-uniform op stream).
// ops[0] = index of the odd power that seeds the accumulator; then one byte per Montgomery
// product: kOpSquare, or a table index t (multiply by x^(2t+1)).  Built on the host
// (build_ops in abi.cu).  The odd-power table lives in per-thread global memory.
// Acc holds x (Montgomery form) on entry and x^e (Montgomery form) on exit; Op is scratch.
// ------------------------------------------------------------------------------------------
constexpr uint8_t kOpSquare = 0xff;

template <int S>
__device__ __forceinline__ void slot_to_tab(const GTable<S>& tab, int e, const Slot<S>& s) {
#pragma unroll
  for (int c = 0; c < S / 4; c++) *tab.at(e, c) = s.chunk(c);
}

template <int S, bool AREG, class MA>
__device__ __forceinline__ void mont_pow(const Slot<S>& Acc, const Slot<S>& Op, const GTable<S>& tab, int ntab,
                                         const uint8_t* __restrict__ ops, int nops, const MA& M) {
  slot_to_tab(tab, 0, Acc);  // x
  {
    uint32_t R[S];
    mont_mul_ss<S, AREG, MA>(R, Acc, Acc, M);  // x^2
    Op.store(R);
  }
#pragma unroll 1
  for (int e = 1; e < ntab; e++) {  // x^(2e+1) = x^(2e-1) * x^2
    uint32_t R[S];
    mont_mul_ss<S, AREG, MA>(R, Acc, Op, M);
    Acc.store(R);
    tab.put(e, R);
  }
  tab.to_slot((int)ops[0], Acc);
#pragma unroll 1
  for (int s = 1; s < nops; s++) {
    const uint8_t op = ops[s];
    const bool sq = op == kOpSquare;
    if (!sq) tab.to_slot(op, Op);
    uint32_t R[S];
    mont_mul_ss<S, AREG, MA>(R, Acc, sq ? Acc : Op, M);
    Acc.store(R);
  }
}

}  // namespace pcb
