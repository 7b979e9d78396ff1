// rns.cu — batched modular exponentiation mod p^2 / q^2 in a residue number system, with the
// two base extensions of every Montgomery product on the int8 tensor cores (tcgen05.mma
// kind::i8, int32 accumulation in TMEM).
//
// Why: the CIOS carry-chain core (mont.cuh) is bounded by the half-rate IMAD.WIDE.X (9.27
// TMAC32/s).  In RNS a product is O(k) independent 32-bit modmuls; its O(k^2) part is two
// base extensions, each a product with a FIXED k x k matrix — a batch x k GEMM.  Split into
// bytes (4 on each side) it is exact on the int8 tensor cores.
//
// Algorithm (Bajard-Imbert RNS Montgomery, restated and checked in oracle/rns_oracle.py):
//   bases B, B' of K = 72 primes < 2^30;  per-prime lazy Montgomery residues x~ = x 2^32 mod m;
//   MM(x, y) = x y M^-1 mod N  (lazy, < (2K+2) N):
//     t~ = REDC(x~ y~);  xi = REDC(t~ C1)  (B)          -> GEMM 1 (A = bytes of xi)
//     qh' = REDC(V1)   r~' = REDC(t~' C2) + REDC(qh' C3)  xi' = REDC(r~' C4)  (B')
//     beta = floor(sum xi'/m' + 2^-20)                  -> GEMM 2 (A = bytes of xi', beta)
//     r~ = REDC(V2)  (B, exact extension)
//   Results are exact residues mod N after the final conversion (rns_out_kernel), so Enc/Dec
//   stay bit-identical to the reference (paillier.cpp:275-361).
//
// CTA = 256 threads = one tile of 128 elements (TMEM lane = element); thread (e, h) owns the B
// residues [36h, 36h+36) and the B' residues [36h, 36h+36) of element e = 32 (warp%4) + lane.
// Shared memory: W1 (288 x 288 B), W2 (288 x 320 B), the A tile (128 x 320 B), all in the
// no-swizzle K-major core-matrix layout of umma.cuh.  One thread issues the MMAs.
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "host/hbn.hpp"
#include "mont.cuh"
#include "pcb_internal.h"
#include "rns.h"
#include "umma.cuh"

namespace pcb {

namespace {

constexpr int K = kRnsK;            // primes per base
constexpr int HK = K / 2;           // residues per thread per base
constexpr int K1 = 4 * K;           // GEMM 1 reduction bytes (288)
constexpr int K2 = kRnsK2;          // GEMM 2 reduction bytes (4(K+1) padded to 32: 320)
constexpr int NOUT = 4 * K;         // GEMM output columns (byte class b, prime) = 288
constexpr int NH = NOUT / 2;        // MMA N per instruction (144)
constexpr int TILE = 128;
constexpr int NTHR = 256;
constexpr uint32_t SM_W1 = 0;
constexpr uint32_t SM_W2 = SM_W1 + NOUT * K1;
constexpr uint32_t SM_A = SM_W2 + NOUT * K2;
constexpr uint32_t SM_S = SM_A + TILE * K2;
constexpr uint32_t SM_BYTES = SM_S + 2 * TILE * 8;
static_assert(SM_BYTES <= 227 * 1024, "shared memory");

__device__ __forceinline__ uint32_t redc(uint64_t T, uint32_t m, uint32_t minv) {
  const uint32_t u = (uint32_t)T * minv;
  return (uint32_t)((T + (uint64_t)u * m) >> 32);
}
__device__ __forceinline__ uint32_t mulr(uint32_t a, uint32_t b, uint32_t m, uint32_t minv) {
  return redc((uint64_t)a * b, m, minv);
}

struct RnsArgs {
  RnsConsts c;                  // per-modulus constants (rns.h)
  const uint8_t* wimg;          // W1 image then W2 image (shared-memory layout), NOUT*(K1+K2) B
  const uint8_t* ops;
  int nops, ntab;
  uint32_t* tab;                // per-thread table: thread g, entry e at (g * (ntab + 2) + e) * K
  const uint32_t* x;            // ENC: r   DEC: c (2S words)   POW: x
  int x_words;
  const uint32_t* m;            // ENC: plaintexts
  int m_words;
  uint32_t* out;                // count x K: B' residues (lazy Montgomery) of the result
  int count, mode, S;
};

// x (nw words, LE) -> this thread's lazy Montgomery residues (B part then B' part):
//   acc~ <- acc~ 2^32 + w 2^32 (mod m) per word, from the top word down
template <int h>
__device__ __forceinline__ void to_rns(uint32_t (&X)[K], const uint32_t* w, int nw, const RnsConsts& C) {
#pragma unroll
  for (int q = 0; q < K; q++) {
    const int pi = q < HK ? h * HK + q : K + h * HK + (q - HK);
    const uint32_t m = C.mod[pi], mi = C.minv[pi], Q = C.q64[pi];
    uint32_t acc = 0;
#pragma unroll 1
    for (int t = nw - 1; t >= 0; t--) {
      uint32_t v = mulr(acc, Q, m, mi) + mulr(w[t], Q, m, mi);
      if (v >= 2 * m) v -= 2 * m;
      acc = v;
    }
    X[q] = acc;
  }
}

}  // namespace

// One RNS Montgomery product for the whole tile: X <- MM(X, Y).  All 256 threads; h (the
// thread's residue half) is a template parameter so every per-prime constant is a
// compile-time offset into the __grid_constant__ parameter (a constant-bank operand).
template <int h>
__device__ __forceinline__ void rns_mm(uint32_t (&X)[K], const uint32_t (&Y)[K], const RnsArgs& P, uint8_t* sm,
                                       uint32_t tm, uint64_t* mbar, uint32_t& phase, int e, int warp) {
  const RnsConsts& C = P.c;
  uint8_t* sA = sm + SM_A;
  double* sS = reinterpret_cast<double*>(sm + SM_S);
  const uint32_t tl = tm + ((uint32_t)((warp & 3) * 32) << 16);
  // ---- 1. t = x y (both bases); xi (B) -> A tile --------------------------------------------
  uint32_t Tp[HK];
#pragma unroll
  for (int q = 0; q < HK; q += 4) {
    uint32_t xi[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int i = h * HK + q + u;
      const uint32_t t = mulr(X[q + u], Y[q + u], C.mod[i], C.minv[i]);
      xi[u] = mulr(t, C.c1[i], C.mod[i], C.minv[i]);
    }
    const int chunk = (h * HK + q) / 4;
    *reinterpret_cast<uint4*>(sA + umma::kmajor_off(e, chunk * 16, TILE)) = make_uint4(xi[0], xi[1], xi[2], xi[3]);
  }
#pragma unroll
  for (int q = 0; q < HK; q++) {
    const int j = K + h * HK + q;
    Tp[q] = mulr(X[HK + q], Y[HK + q], C.mod[j], C.minv[j]);
  }
  umma::fence_async_smem();
  umma::tmem_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    umma::tmem_fence_after();
    const uint32_t a0 = umma::smem_u32(sA), w1 = umma::smem_u32(sm + SM_W1);
    const uint32_t idesc = umma::idesc_i8(TILE, NH);
#pragma unroll 1
    for (int hh = 0; hh < 2; hh++)
#pragma unroll 1
      for (int s = 0; s < K1 / 32; s++)
        umma::mma_i8(tm + hh * NH, umma::desc_kmajor(a0 + s * 2 * TILE * 16, TILE),
                     umma::desc_kmajor(w1 + s * 2 * NOUT * 16 + (hh * NH / 8) * 128, NOUT), idesc, s > 0);
    umma::commit(mbar);
  }
  umma::mbar_wait(mbar, phase);
  phase ^= 1;
  umma::tmem_fence_after();
  // ---- 3. qh', r~' (new B' residues), xi' (B') -> A tile, partial beta sum ------------------
  double sp = 0.0;
#pragma unroll
  for (int g = 0; g < HK; g += 12) {
    uint32_t d[4][12];
#pragma unroll
    for (int b = 0; b < 4; b++) {
      uint32_t v8[8], v4[4];
      const uint32_t col = b * K + h * HK + g;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v8[0]), "=r"(v8[1]), "=r"(v8[2]), "=r"(v8[3]), "=r"(v8[4]), "=r"(v8[5]), "=r"(v8[6]),
                     "=r"(v8[7])
                   : "r"(tl + col));
      umma::tmem_ld4(tl + col + 8, v4);
#pragma unroll
      for (int u = 0; u < 8; u++) d[b][u] = v8[u];
#pragma unroll
      for (int u = 0; u < 4; u++) d[b][8 + u] = v4[u];
    }
    umma::tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 12; u++) {
      const int q = g + u, j = K + h * HK + q;
      const uint32_t m = C.mod[j], mi = C.minv[j];
      const uint64_t V = (uint64_t)d[0][u] + ((uint64_t)d[1][u] << 8) + ((uint64_t)d[2][u] << 16) +
                         ((uint64_t)d[3][u] << 24);
      const uint32_t qh = redc(V, m, mi);
      uint32_t r = mulr(Tp[q], C.c2[q + h * HK], m, mi) + mulr(qh, C.c3[q + h * HK], m, mi);
      if (r >= 2 * m) r -= 2 * m;
      X[HK + q] = r;
      const uint32_t xp = mulr(r, C.c4[q + h * HK], m, mi);
      sp += (double)xp * C.invp[q + h * HK];
      Tp[q] = xp;  // reuse: xi'
    }
  }
#pragma unroll
  for (int q = 0; q < HK; q += 4) {
    const int chunk = (h * HK + q) / 4;
    *reinterpret_cast<uint4*>(sA + umma::kmajor_off(e, chunk * 16, TILE)) = make_uint4(Tp[q], Tp[q + 1], Tp[q + 2], Tp[q + 3]);
  }
  sS[h * TILE + e] = sp;
  umma::tmem_fence_before();
  __syncthreads();
  {
    const double S = sS[e] + sS[TILE + e];
    const uint32_t beta = (uint32_t)floor(S + 9.5367431640625e-07);  // + 2^-20
    // chunk K/4 holds beta (bytes 0..3) and zeros; chunk K/4 + 1 is zero padding
    if (h == 0)
      *reinterpret_cast<uint4*>(sA + umma::kmajor_off(e, K * 4, TILE)) = make_uint4(beta, 0, 0, 0);
    else
      *reinterpret_cast<uint4*>(sA + umma::kmajor_off(e, K * 4 + 16, TILE)) = make_uint4(0, 0, 0, 0);
  }
  umma::fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    umma::tmem_fence_after();
    const uint32_t a0 = umma::smem_u32(sA), w2 = umma::smem_u32(sm + SM_W2);
    const uint32_t idesc = umma::idesc_i8(TILE, NH);
#pragma unroll 1
    for (int hh = 0; hh < 2; hh++)
#pragma unroll 1
      for (int s = 0; s < K2 / 32; s++)
        umma::mma_i8(tm + hh * NH, umma::desc_kmajor(a0 + s * 2 * TILE * 16, TILE),
                     umma::desc_kmajor(w2 + s * 2 * NOUT * 16 + (hh * NH / 8) * 128, NOUT), idesc, s > 0);
    umma::commit(mbar);
  }
  umma::mbar_wait(mbar, phase);
  phase ^= 1;
  umma::tmem_fence_after();
  // ---- 5. r~ (new B residues) -----------------------------------------------------------------
#pragma unroll
  for (int g = 0; g < HK; g += 12) {
    uint32_t d[4][12];
#pragma unroll
    for (int b = 0; b < 4; b++) {
      uint32_t v8[8], v4[4];
      const uint32_t col = b * K + h * HK + g;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v8[0]), "=r"(v8[1]), "=r"(v8[2]), "=r"(v8[3]), "=r"(v8[4]), "=r"(v8[5]), "=r"(v8[6]),
                     "=r"(v8[7])
                   : "r"(tl + col));
      umma::tmem_ld4(tl + col + 8, v4);
#pragma unroll
      for (int u = 0; u < 8; u++) d[b][u] = v8[u];
#pragma unroll
      for (int u = 0; u < 4; u++) d[b][8 + u] = v4[u];
    }
    umma::tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 12; u++) {
      const int q = g + u, i = h * HK + q;
      const uint64_t V = (uint64_t)d[0][u] + ((uint64_t)d[1][u] << 8) + ((uint64_t)d[2][u] << 16) +
                         ((uint64_t)d[3][u] << 24);
      X[q] = redc(V, C.mod[i], C.minv[i]);
    }
  }
  umma::tmem_fence_before();
}

template <int h>
__device__ __forceinline__ void rns_tiles(const RnsArgs& P, uint8_t* sm, uint32_t tm, uint64_t* mbar, int e, int warp,
                                          uint32_t gt, uint32_t nthr) {
  const RnsConsts& C = P.c;
  const int ntiles = (P.count + TILE - 1) / TILE;
  uint32_t phase = 0;
  // this thread's table: NE entries of K contiguous residues (one base register, immediate offsets)
  uint32_t* const mytab = P.tab + (size_t)gt * (P.ntab + 2) * K;
  auto tab_put = [&](int ent, const uint32_t (&V)[K]) {
    uint4* d = reinterpret_cast<uint4*>(mytab + ent * K);
#pragma unroll
    for (int q = 0; q < K / 4; q++) d[q] = make_uint4(V[4 * q], V[4 * q + 1], V[4 * q + 2], V[4 * q + 3]);
  };
  auto tab_get = [&](int ent, uint32_t (&V)[K]) {
    const uint4* d = reinterpret_cast<const uint4*>(mytab + ent * K);
#pragma unroll
    for (int q = 0; q < K / 4; q++) {
      const uint4 v = d[q];
      V[4 * q] = v.x; V[4 * q + 1] = v.y; V[4 * q + 2] = v.z; V[4 * q + 3] = v.w;
    }
  };
  auto const_get = [&](const uint32_t* c, uint32_t (&V)[K]) {  // c: 2K residues, B then B'
#pragma unroll
    for (int q = 0; q < HK; q++) {
      V[q] = c[h * HK + q];
      V[HK + q] = c[K + h * HK + q];
    }
  };
  // uniform step plan: [pre0] pre1 | x^2 | table (ntab-1) | main (nops-1) | final
  const int npre = P.mode == kRnsPow ? 1 : 2;
  const int s_x2 = npre, s_tab = s_x2 + 1, s_main = s_tab + (P.ntab - 1), s_fin = s_main + (P.nops - 1);
  const int nsteps = s_fin + 1;
  const int park = P.ntab, park_x2 = P.ntab + 1;
  const uint32_t zero = 0;
#pragma unroll 1
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int el = tile * TILE + e;
    const bool live = el < P.count;
    uint32_t X[K], Y[K];
#pragma unroll 1
    for (int s = 0; s < nsteps; s++) {
      // ---- operands ----------------------------------------------------------------------------
      if (s < npre) {
        const bool first = npre == 2 && s == 0;
        const uint32_t* src = &zero;
        int nw = 1;
        const uint32_t* cst = C.r2n;
        if (P.mode == kRnsEnc && first) {         // m n
          if (live) { src = P.m + (size_t)el * P.m_words; nw = P.m_words; }
          cst = C.nM;
        } else if (P.mode == kRnsDec && first) {  // c_hi 2^(32 S) M
          if (live) { src = P.x + (size_t)el * P.x_words + P.S; nw = P.x_words - P.S; }
          cst = C.cr2n;
        } else {                                  // r M / c_lo M / x M
          if (live) { src = P.x + (size_t)el * P.x_words; nw = P.mode == kRnsDec ? P.S : P.x_words; }
        }
        to_rns<h>(X, src, nw, C);
        const_get(cst, Y);
      } else if (s == s_x2) {
#pragma unroll
        for (int q = 0; q < K; q++) Y[q] = X[q];
      } else if (s < s_main) {
        tab_get(park_x2, Y);
      } else if (s < s_fin) {
        const uint8_t op = P.ops[s - s_main + 1];
        if (op == kOpSquare) {
#pragma unroll
          for (int q = 0; q < K; q++) Y[q] = X[q];
        } else {
          tab_get(op, Y);
        }
      } else {
        if (P.mode == kRnsEnc) tab_get(park, Y); else const_get(C.one, Y);
      }
      // ---- the single RNS Montgomery product site -------------------------------------------
      rns_mm<h>(X, Y, P, sm, tm, mbar, phase, e, warp);
      // ---- epilogue ----------------------------------------------------------------------------
      if (s < npre) {
        const bool first = npre == 2 && s == 0;
        if (first) {
          if (P.mode == kRnsEnc) {  // 1 + m n  (plain: the final product cancels one M)
#pragma unroll
            for (int q = 0; q < K; q++) {
              const int pi = q < HK ? h * HK + q : K + h * HK + (q - HK);
              uint32_t v = X[q] + C.one[pi];
              if (v >= 2 * C.mod[pi]) v -= 2 * C.mod[pi];
              X[q] = v;
            }
          }
          tab_put(park, X);
        } else {
          if (P.mode == kRnsDec) {  // c M = c_lo M + c_hi 2^(32 S) M
            tab_get(park, Y);
#pragma unroll
            for (int q = 0; q < K; q++) {
              const int pi = q < HK ? h * HK + q : K + h * HK + (q - HK);
              uint32_t v = X[q] + Y[q];
              if (v >= 2 * C.mod[pi]) v -= 2 * C.mod[pi];
              X[q] = v;
            }
          }
          tab_put(0, X);
        }
      } else if (s == s_x2) {
        tab_put(park_x2, X);
        tab_get(0, X);
      } else if (s < s_main) {
        tab_put(s - s_tab + 1, X);
        if (s == s_main - 1) tab_get(P.ops[0], X);
      } else if (s == s_fin) {
        if (live) {
#pragma unroll
          for (int q = 0; q < HK; q++) P.out[(size_t)el * K + h * HK + q] = X[HK + q];
        }
      }
      if (P.ntab == 1 && s == s_x2) tab_get(P.ops[0], X);
    }
  }
}

__global__ void __launch_bounds__(NTHR, 1) rns_pow_kernel(const __grid_constant__ RnsArgs P) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int e = (warp & 3) * 32 + lane, h = warp >> 2;
  // fixed matrices -> shared memory; zero the A tile (its padding bytes are never written)
  for (uint32_t o = tid * 16; o < (uint32_t)(NOUT * (K1 + K2)); o += NTHR * 16)
    *reinterpret_cast<uint4*>(sm + o) = *reinterpret_cast<const uint4*>(P.wimg + o);
  for (uint32_t o = tid * 16; o < (uint32_t)(TILE * K2); o += NTHR * 16)
    *reinterpret_cast<uint4*>(sm + SM_A + o) = make_uint4(0, 0, 0, 0);
  if (warp == 0) umma::tmem_alloc<512>(&tbase);
  if (tid == 0) umma::mbar_init(&mbar, 1);
  umma::tmem_fence_before();
  __syncthreads();
  umma::tmem_fence_after();
  const uint32_t tm = tbase;
  const uint32_t nthr = gridDim.x * NTHR;
  const uint32_t gt = blockIdx.x * NTHR + tid;
  if (h == 0)
    rns_tiles<0>(P, sm, tm, &mbar, e, warp, gt, nthr);
  else
    rns_tiles<1>(P, sm, tm, &mbar, e, warp, gt, nthr);
  umma::tmem_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<512>(tm);
}

// Exact conversion of the B' residues to the binary residue mod N (one thread per element):
//   xi'_j = REDC(x~'_j C4_j) fully reduced,  r = sum_j xi'_j M'_j - beta M',  y = r mod N.
__global__ void rns_out_kernel(const __grid_constant__ RnsOutArgs P) {
  constexpr int W = kRnsMpWords;
  for (int el = blockIdx.x * blockDim.x + threadIdx.x; el < P.count; el += gridDim.x * blockDim.x) {
    const uint32_t* res = P.res + (size_t)el * K;
    uint32_t r[W + 2];
    for (int w = 0; w < W + 2; w++) r[w] = 0;
    double S = 0.0;
    for (int j = 0; j < K; j++) {
      const uint32_t m = P.mod[j], mi = P.minv[j];
      uint32_t xp = redc((uint64_t)res[j] * P.c4[j], m, mi);
      if (xp >= m) xp -= m;
      S += (double)xp * P.invp[j];
      const uint32_t* Mj = P.mpj + (size_t)j * W;
      uint64_t carry = 0;
      for (int w = 0; w < W; w++) {
        const uint64_t t = (uint64_t)xp * Mj[w] + r[w] + carry;
        r[w] = (uint32_t)t;
        carry = t >> 32;
      }
      for (int w = W; w < W + 2 && carry; w++) {
        const uint64_t t = (uint64_t)r[w] + carry;
        r[w] = (uint32_t)t;
        carry = t >> 32;
      }
    }
    const uint32_t beta = (uint32_t)floor(S + 9.5367431640625e-07);
    {  // r -= beta M'
      int64_t br = 0;
      uint64_t carry = 0;
      for (int w = 0; w < W + 2; w++) {
        const uint64_t pr = (uint64_t)beta * (w < W ? P.mp[w] : 0u) + carry;
        carry = pr >> 32;
        const int64_t d = (int64_t)r[w] - (int64_t)(uint32_t)pr - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    // y = r mod N, r < (2K+2) N: subtract q N with q from the top bits (an underestimate), then
    // at most a few single subtractions
    const int S_ = P.S;
    double rt = 0.0;
    for (int w = W + 1; w >= S_ - 2; w--) rt = rt * 4294967296.0 + (double)r[w];
    const double qd = floor(rt / P.ntop) - 1.0;
    const uint32_t q = qd > 0 ? (uint32_t)qd : 0u;
    if (q) {
      int64_t br = 0;
      uint64_t carry = 0;
      for (int w = 0; w < W + 2; w++) {
        const uint64_t pr = (uint64_t)q * (w < S_ ? P.n[w] : 0u) + carry;
        carry = pr >> 32;
        const int64_t d = (int64_t)r[w] - (int64_t)(uint32_t)pr - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    for (;;) {  // while r >= N: r -= N
      int cmp = 0;
      for (int w = W + 1; w >= 0 && cmp == 0; w--) {
        const uint32_t a = r[w], b = w < S_ ? P.n[w] : 0u;
        cmp = a > b ? 1 : (a < b ? -1 : 0);
      }
      if (cmp < 0) break;
      int64_t br = 0;
      for (int w = 0; w < W + 2; w++) {
        const int64_t d = (int64_t)r[w] - (int64_t)(w < S_ ? P.n[w] : 0u) - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    uint32_t* y = P.y + (size_t)el * S_;
    for (int w = 0; w < S_; w++) y[w] = r[w];
  }
}

pcb_status launch_rns(const RnsModulus& md, int mode, const uint8_t* ops, int nops, int ntab, const uint32_t* x,
                      int x_words, const uint32_t* m, int m_words, size_t count, uint32_t* y, cudaStream_t st,
                      double alg_mac32) {
  if (count == 0) return PCB_OK;
  RnsArgs P;
  P.c = md.c;
  P.wimg = md.d_wimg;
  P.ops = ops;
  P.nops = nops;
  P.ntab = ntab;
  P.x = x;
  P.x_words = x_words;
  P.m = m;
  P.m_words = m_words;
  P.count = (int)count;
  P.mode = mode;
  P.S = md.S;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  // The >48 KB dynamic-smem opt-in is a per-device function attribute: remember it per device
  // (bit dev of an atomic mask), so a second context on another device, or another host
  // thread, never launches without it.  Setting it twice is harmless.
  static std::atomic<uint64_t> attr_dev{0};
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_dev.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(rns_pow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_BYTES) != cudaSuccess)
      return PCB_E_CUDA;
    attr_dev.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int ntiles = (int)((count + TILE - 1) / TILE);
  const int blocks = ntiles < nsm ? ntiles : nsm;
  const size_t nthr = (size_t)blocks * NTHR;
  pcb_status e = scratch_alloc(nthr * (size_t)(ntab + 2) * K * 4, (void**)&P.tab, st);
  uint32_t* res = nullptr;
  if (!e) e = scratch_alloc(count * K * 4, (void**)&res, st);
  P.out = res;
  if (!e) {
    ProfMark pm;
    if (prof_enabled()) pm = prof_start(st);
    rns_pow_kernel<<<blocks, NTHR, SM_BYTES, st>>>(P);
    count_launch();
    if (prof_enabled()) prof_stop(pm, st, alg_mac32 * (double)count);
    e = cuda_check(cudaGetLastError());
  }
  if (!e) {
    RnsOutArgs O = md.out;
    O.res = res;
    O.y = y;
    O.count = (int)count;
    const int grid = (int)((count + 127) / 128 < 4096 ? (count + 127) / 128 : 4096);
    rns_out_kernel<<<grid, 128, 0, st>>>(O);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  scratch_free(P.tab, st);
  scratch_free(res, st);
  return e;
}

// ------------------------------------------------------------------------------------------
// Host: constants for one modulus (computed with the host bignum, uploaded once per context)
// ------------------------------------------------------------------------------------------
namespace {

bool is_prime32(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t p : {2u, 3u, 5u, 7u, 11u, 13u, 17u, 19u, 23u, 29u, 31u, 37u})
    if (n % p == 0) return n == p;
  uint32_t d = n - 1;
  int s = 0;
  while (!(d & 1)) { d >>= 1; s++; }
  auto pw = [&](uint64_t a, uint32_t e) {
    uint64_t r = 1;
    a %= n;
    while (e) {
      if (e & 1) r = r * a % n;
      a = a * a % n;
      e >>= 1;
    }
    return r;
  };
  for (uint32_t a : {2u, 3u, 5u, 7u}) {  // deterministic below 3.2e9
    uint64_t x = pw(a, d);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; r++) {
      x = x * x % n;
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

uint32_t inv_mod(uint64_t a, uint32_t m) {  // a^-1 mod m (m prime, a != 0 mod m)
  int64_t t = 0, nt = 1, r = m, nr = (int64_t)(a % m);
  while (nr) {
    const int64_t q = r / nr;
    int64_t tmp = t - q * nt; t = nt; nt = tmp;
    tmp = r - q * nr; r = nr; nr = tmp;
  }
  return (uint32_t)(t < 0 ? t + m : t);
}

uint32_t big_mod(const HBN& x, uint32_t m) {  // x mod m (limb-wise Horner)
  uint64_t r = 0;
  for (size_t i = x.w.size(); i-- > 0;) r = ((r << 32) | x.w[i]) % m;
  return (uint32_t)r;
}

}  // namespace

bool rns_build(const HBN& N, const HBN& n, int S, RnsModulus* out) {
  if (S > kRnsMaxS || N.bit_length() > (size_t)(32 * S) || !N.is_odd()) return false;
  std::vector<uint32_t> pr;
  for (uint32_t c = (1u << 30) - 1; pr.size() < 2 * (size_t)K; c -= 2)
    if (is_prime32(c)) pr.push_back(c);
  const uint32_t* B = pr.data();
  const uint32_t* Bp = pr.data() + K;
  RnsModulus md;
  md.S = S;
  RnsConsts& C = md.c;
  auto mprod_mod = [&](const uint32_t* base, int skip, uint32_t m) {  // prod_{l != skip} base_l mod m
    uint64_t r = 1;
    for (int l = 0; l < K; l++)
      if (l != skip) r = r * (base[l] % m) % m;
    return (uint32_t)r;
  };
  const uint64_t two32 = 1ull << 32;
  for (int q = 0; q < 2 * K; q++) {
    const uint32_t m = pr[q];
    if (big_mod(N, m) == 0) return false;
    uint32_t inv = 1;  // m^-1 mod 2^32 (Newton)
    for (int it = 0; it < 5; it++) inv *= 2u - m * inv;
    C.mod[q] = m;
    C.minv[q] = (uint32_t)(0u - inv);
    C.one[q] = (uint32_t)(two32 % m);
    C.q64[q] = (uint32_t)((uint64_t)C.one[q] * C.one[q] % m);  // 2^64 mod m
  }
  HBN M(1), Mp(1);
  for (int l = 0; l < K; l++) {
    M = M * HBN(B[l]);
    Mp = Mp * HBN(Bp[l]);
  }
  for (int i = 0; i < K; i++) {
    const uint32_t m = B[i];
    const uint64_t ninv = inv_mod(big_mod(N, m), m), miinv = inv_mod(mprod_mod(B, i, m), m);
    C.c1[i] = (uint32_t)((m - ninv) % m * miinv % m);
  }
  for (int j = 0; j < K; j++) {
    const uint32_t m = Bp[j];
    const uint64_t minvM = inv_mod(big_mod(M, m), m), o = C.one[K + j];
    C.c2[j] = (uint32_t)(minvM * o % m);
    C.c3[j] = (uint32_t)((uint64_t)big_mod(N, m) * minvM % m * C.q64[K + j] % m);
    C.c4[j] = inv_mod(mprod_mod(Bp, j, m), m);
    C.invp[j] = 1.0 / (double)m;
  }
  auto to_res = [&](const HBN& v, uint32_t* dst) {  // lazy-Montgomery residues of v (< M)
    for (int q = 0; q < 2 * K; q++) dst[q] = (uint32_t)((uint64_t)big_mod(v, pr[q]) * C.one[q] % pr[q]);
  };
  const HBN M2 = mod(M * M, N);
  to_res(M2, C.r2n);
  to_res(mod(M2 << (size_t)(32 * S), N), C.cr2n);
  to_res(mod(mod(n, N) * mod(M, N), N), C.nM);
  // W1 (rows (b, j), K bytes 4i+a) and W2 (rows (b, i), K bytes 4j+a, beta slot 4K+a) images
  std::vector<uint8_t> img((size_t)NOUT * (K1 + K2), 0);
  uint8_t* w1 = img.data();
  uint8_t* w2 = img.data() + (size_t)NOUT * K1;
  for (int j = 0; j < K; j++) {
    const uint32_t m = Bp[j];
    for (int i = 0; i < K; i++) {
      const uint64_t base = (uint64_t)mprod_mod(B, i, m) * C.one[K + j] % m;  // M_i 2^32 mod m'_j
      for (int a = 0; a < 4; a++) {
        const uint32_t v = (uint32_t)((base << (8 * a)) % m);
        for (int b = 0; b < 4; b++) w1[umma::kmajor_off(b * K + j, 4 * i + a, NOUT)] = (uint8_t)(v >> (8 * b));
      }
    }
  }
  for (int i = 0; i < K; i++) {
    const uint32_t m = B[i];
    const uint64_t q64 = C.q64[i];
    for (int j = 0; j <= K; j++) {
      uint64_t base;
      if (j < K)
        base = (uint64_t)mprod_mod(Bp, j, m) * q64 % m;  // M'_j 2^64 mod m_i
      else
        base = (m - (uint64_t)big_mod(Mp, m) * q64 % m) % m;  // -M' 2^64 mod m_i
      for (int a = 0; a < 4; a++) {
        const uint32_t v = (uint32_t)((base << (8 * a)) % m);
        for (int b = 0; b < 4; b++) w2[umma::kmajor_off(b * K + i, 4 * j + a, NOUT)] = (uint8_t)(v >> (8 * b));
      }
    }
  }
  // output conversion tables
  std::vector<uint32_t> tabs((size_t)K * kRnsMpWords + kRnsMpWords + S, 0);
  for (int j = 0; j < K; j++) {
    HBN q, r;
    divmod(Mp, HBN(Bp[j]), q, r);
    q.to_limbs(tabs.data() + (size_t)j * kRnsMpWords, kRnsMpWords);
  }
  Mp.to_limbs(tabs.data() + (size_t)K * kRnsMpWords, kRnsMpWords);
  N.to_limbs(tabs.data() + (size_t)K * kRnsMpWords + kRnsMpWords, S);
  if (cudaMalloc(&md.d_wimg, img.size()) != cudaSuccess) return false;
  if (cudaMalloc(&md.d_tabs, tabs.size() * 4) != cudaSuccess) {
    cudaFree(md.d_wimg);
    return false;
  }
  cudaMemcpy(md.d_wimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(md.d_tabs, tabs.data(), tabs.size() * 4, cudaMemcpyHostToDevice);
  RnsOutArgs& O = md.out;
  O.S = S;
  for (int j = 0; j < K; j++) {
    O.mod[j] = C.mod[K + j];
    O.minv[j] = C.minv[K + j];
    O.c4[j] = C.c4[j];
    O.invp[j] = C.invp[j];
  }
  O.mpj = md.d_tabs;
  O.mp = md.d_tabs + (size_t)K * kRnsMpWords;
  O.n = md.d_tabs + (size_t)K * kRnsMpWords + kRnsMpWords;
  double nt = 0.0;
  const std::vector<uint32_t> nl = N.limbs(S);
  for (int w = S - 1; w >= S - 2; w--) nt = nt * 4294967296.0 + (double)nl[w];
  O.ntop = nt;
  md.ok = true;
  *out = md;
  return true;
}

void rns_free(RnsModulus* md) {
  if (md->d_wimg) cudaFree(md->d_wimg);
  if (md->d_tabs) cudaFree(md->d_tabs);
  md->d_wimg = nullptr;
  md->d_tabs = nullptr;
  md->ok = false;
}

}  // namespace pcb
