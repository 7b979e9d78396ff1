// rnsx.cu — streaming RNS Montgomery core for moduli up to 4096 bits (p^2 / q^2 of 2048- and
// 3072-bit keys, n^2 of 2048-bit keys), base extensions on the int8 tensor cores.
//
// Same arithmetic as rns.cu (Bajard-Imbert RNS Montgomery, approximate first / exact second
// base extension; restated and checked in oracle/rns_oracle.py), re-organised so that it scales
// past 2 kbit and keeps both the tensor core and the CUDA cores busy:
//
//  * The two K x K base-extension matrices (byte-split: 4K x 4K bytes each, 2 x 330 KB at
//    K = 144) do not fit in shared memory.  They are streamed from L2 as one periodic sequence of
//    "slices" (NCOL output columns x 32 reduction bytes = one MMA) through an NSTAGE-deep ring
//    filled by cp.async.bulk (mbarrier full/empty handshake).
//  * The GEMM output is produced in chunks of NCOL = 16 PT columns (4 bytes x P primes) into a
//    4-deep TMEM ring.  Every compute thread owns PT primes of EVERY chunk, so while the tensor
//    core computes chunk c+1 all 16 compute warps drain chunk c (tcgen05.ld, then release the
//    buffer) and run its per-prime REDC work.  The MMA of GEMM 2 only waits for the last chunk.
//  * One role warp: lane 0 issues the bulk copies and the MMAs (tcgen05.mma.cta_group::1
//    .kind::i8, M = 128 elements, N = NCOL, K = 32 bytes per instruction).
//  * Per element only the 2K lazy residues live in registers (2 RPT per thread); the multiplier
//    comes from registers (squaring) or global memory (table / constant operands), and
//    t' = x' y' is parked in the x' registers until the GEMM-1 epilogue consumes it.
//
// CTA = 16 compute warps (4 per TMEM lane quadrant; warp w: lanes 32 (w%4).., prime group
// g = w/4) + 1 role warp; one 128-element tile at a time, persistent over tiles.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>
#include <vector>
#include <cstring>
#include <cuda_runtime.h>

#include "host/hbn.hpp"
#include "mont.cuh"
#include "pcb_internal.h"
#include "rnsx.h"
#include "umma.cuh"

#ifndef PCB_RNSX_ROLE_WARPS
#define PCB_RNSX_ROLE_WARPS 4
#endif
#ifndef PCB_RNSX_KCONS
#define PCB_RNSX_KCONS 0  // 1: per-prime constants from the kernel parameters (measured: LDC hoisting spills, slower)
#endif
#ifndef PCB_RNSX_SLOT
#define PCB_RNSX_SLOT 0  // 0: a third of the shared memory left for the ring (Cfg::SLOT)
#endif

namespace pcb {

namespace {

// Chunk layout: the GEMM output (4 bytes x K primes) is produced in chunks of up to 32 primes =
// 128 TMEM columns (one MMA of N = 128 per k-step: the tensor core costs ~64 clocks per
// instruction whatever N <= 128, so wide chunks matter).  Thread group g (warps 4g..4g+3) owns
// PTc = 8 consecutive primes of every full chunk (PTL of the ragged last one); within a thread's
// 4 PTc columns the primes sit in quads of <= 4 primes x 4 bytes ([quad][byte][prime]), so one
// tcgen05.ld x16 returns four complete primes.
// slices per stream stage: bigger bulk copies where the ring has room (8+ stages either way)
__host__ __device__ constexpr int sps_for(int) { return 1; }
// primes in quad j of a chunk with ptc primes per thread group (4, or 2 for a ragged tail)
__host__ __device__ constexpr int rnsx_qt(int ptc, int j) {
  return ptc % 4 == 0 ? 4 : (ptc == 2 ? 2 : (4 * j < ptc - 2 ? 4 : 2));
}
__host__ __device__ constexpr int rnsx_slot(int ptc, int g, int j) {
  return (ptc % 4 == 0 || ptc == 2) ? g * ptc + 4 * j : (4 * j < ptc - 2 ? 16 * j + 4 * g : 16 * (ptc / 4) + 2 * g);
}  // one <= 8 KB slice per stage
// GEMM-output chunks: 64 primes (N = 256 columns) each and a ragged last one -- except K = 72,
// which runs as 32 + 40 primes (N = 128 + 160).  The MMA costs max(N / 2, 32 + N / 4) clk at
// M = 128, K = 32 B (tools/mma_mix.cu, profiles/r02_mma_mix.txt), so {256, 32} takes 171 clk per
// k-step and {128, 160} 144 (the ideal), and 160-column buffers give a 3-deep TMEM ring.  Every
// chunk but the last must be a multiple of 16 primes: a thread's residues are read in quads of 4.
__host__ __device__ constexpr int rnsx_nchunks(int K) { return K == 72 ? 2 : (K + 63) / 64; }
__host__ __device__ constexpr int rnsx_chunk_primes(int K, int c) {
  return K == 72 ? (c == 0 ? 32 : 40) : (c < rnsx_nchunks(K) - 1 ? 64 : K - 64 * (rnsx_nchunks(K) - 1));
}
__host__ __device__ constexpr int rnsx_chunk_first(int K, int c) {
  int f = 0;
  for (int i = 0; i < c; i++) f += rnsx_chunk_primes(K, i);
  return f;
}
__host__ __device__ constexpr int rnsx_max_chunk(int K) {
  int m = 0;
  for (int i = 0; i < rnsx_nchunks(K); i++) m = rnsx_chunk_primes(K, i) > m ? rnsx_chunk_primes(K, i) : m;
  return m;
}

template <int K_, int NT_ = 1, int CG_ = 1>
struct Cfg {
  static constexpr int K = K_, G = 4, NT = NT_;  // NT: tiles in flight per CTA (1 or 2)
  // CG = 2: the CTA pair of a cluster runs every MMA as one cta_group::2 MMA (M = 256, the leader
  // issues); each CTA holds half of every W slice (N / 2 rows), so each SM streams half the bytes
  static constexpr int CG = CG_;
  static constexpr int NC = rnsx_nchunks(K);      // GEMM-output chunks (rnsx_chunk_primes)
  static constexpr int RPT = K / G;                // residues per thread per base
  static constexpr int NQ = (RPT + 3) / 4;         // 4-word vectors per thread per base
  static constexpr int NV = 2 * NQ;                // ... per operand (B quads, then B' quads)
  static constexpr int K1 = 4 * K, K2 = 4 * K + 32, KS1 = K1 / 32, KS2 = K2 / 32;
  static constexpr int NSLICE = NC * (KS1 + KS2);  // MMAs (and streamed slices) per product
  static constexpr int SPS = sps_for(K);           // slices per stream stage (one bulk copy)
  static constexpr int NSTG = (NSLICE + SPS - 1) / SPS;  // stages per product
  // TMEM ring: buffers of the widest chunk (rounded to 32 columns), as many as fit in 512 (<= 3)
  static constexpr int BUFC = (16 * (rnsx_max_chunk(K) / G) + 31) / 32 * 32, TMC = 512;
  static constexpr int NB = TMC / BUFC > 3 ? 3 : TMC / BUFC;
  // + role warps: one MMA issuer and W-stream producers; RW = 8 (two warpgroups at 32 registers)
  // still leaves the compute warps their 112 (16 x 32 x 112 + 8 x 32 x 32 = 64 K registers)
  static constexpr int TILE = 128, NCW = 16, NCT = 32 * NCW, RW = PCB_RNSX_ROLE_WARPS, NTHR = NCT + 32 * RW;
  static constexpr uint32_t ABLK = TILE * (K1 + K2);  // A1 + A2 of one tile
  static constexpr uint32_t OFF_A1 = 0, OFF_A2 = OFF_A1 + TILE * K1, OFF_CONS = NT * ABLK;
  static constexpr uint32_t OFF_S = OFF_CONS + K * 48, OFF_SLT = OFF_S + NT * G * TILE * 8;
  static constexpr uint32_t OFF_BAR = OFF_SLT + NSLICE * 16 + NSTG * 8;
  static constexpr uint32_t OFF_RING = (OFF_BAR + 512 + 1023) & ~1023u;
  // ring slot (CG = 2: halves of one 8 KB slice).  A stage holds spc(c) consecutive slices of one
  // chunk: one issuing warp serialises its bulk copies at ~600 clk each whatever their size
  // (profiles/r02_bulk_bw2.txt), so fewer, bigger stages stream more bytes (20 KB stages: Dec
  // 2048 -10 %, profiles/r02_rnsx_slot_ab.txt).  Default: a third of the ring space, capped at
  // the largest chunk's GEMM-2 slices.
  static constexpr uint32_t SLOT_AUTO_ = ((227u * 1024u - OFF_RING) / 3u) & ~1023u;
  static constexpr uint32_t SLOT_CAP_ = (uint32_t)KS2 * 16u * (uint32_t)(rnsx_max_chunk(K) / 4) * 32u;
  static constexpr int SLOT = CG == 2 ? 8192 / CG
                              : (PCB_RNSX_SLOT > 0 ? PCB_RNSX_SLOT : (int)(SLOT_AUTO_ < SLOT_CAP_ ? SLOT_AUTO_ : SLOT_CAP_));
  static constexpr int NSTAGE_FIT = (int)((227u * 1024u - OFF_RING) / SLOT);
  static constexpr int NSTAGE = NSTAGE_FIT > 12 ? 12 : NSTAGE_FIT;
  static constexpr uint32_t SMEM = OFF_RING + NSTAGE * SLOT;
  __host__ __device__ static constexpr int ptc(int c) { return rnsx_chunk_primes(K, c) / G; }
  __host__ __device__ static constexpr int cp0(int c) { return rnsx_chunk_first(K, c); }      // first prime
  __host__ __device__ static constexpr int cw0(int c) { return rnsx_chunk_first(K, c) / G; }  // first thread residue
  __host__ __device__ static constexpr int ncol(int c) { return 16 * ptc(c); }
  __host__ __device__ static constexpr int spc(int c) { return CG == 2 ? 1 : SLOT / (ncol(c) * 32); }
  // first prime (within chunk c) of quad j of thread group g: group-major when every group's run is
  // 16-byte aligned (ptc a multiple of 4, or 2); otherwise quad-major, groups interleaved per quad
  __host__ __device__ static constexpr int slot(int c, int g, int j) { return rnsx_slot(ptc(c), g, j); }
  static_assert(K % 8 == 0 && rnsx_chunk_primes(K, NC - 1) % 8 == 0 && (NC == 1 || rnsx_chunk_first(K, NC - 1) % 16 == 0),
                "chunks: the last a multiple of 8 primes, all others of 16 (thread residues in quads of 4)");
  static_assert(NB >= 2, "TMEM ring");
  static_assert(NSTAGE >= 3 && SLOT >= 8192 / CG, "stream ring");
  static_assert((3 * NSTAGE + 2 * NB + 2 * NT) * 8 + 4 <= 512, "barriers");
  static_assert(CG == 1 || (CG == 2 && NT == 1), "pair MMA only with one tile per CTA");
  static_assert(NT >= 1 && NT <= 3, "tiles in flight");
};

struct XArgs {
  const uint8_t* wimg;
  const uint8_t* wimg2;  // split-halves stream image (cta_group::2)
  size_t wimg_stride;  // bytes between the replicas of the stream image
  const uint4* cons;
  const uint32_t* cvec;
  const uint32_t* slt;  // per slice of a product {A offset, B offset | LBO, idesc, flags}; per stage {image offset / 16, bytes}
  const uint8_t* ops;
  int nops, ntab;
  uint32_t* tab;  // per-thread tables: word ((entry * NV + v) * NT + gt) * 4 + t
  const uint32_t* x;
  int x_words;
  const uint32_t* m;
  int m_words;
  uint32_t* out;  // count x K: B' residues (lazy Montgomery) of the result
  int count, mode, S;
  int dbg;  // timing experiments: 1 = tensor/stream only, 2 = CUDA cores only
  int cl;   // CTAs per cluster sharing the W stream (1 or 2)
  int nprod;  // W-stream producer warps (PCB_RNSX_NPROD for A/B; default kRxProducers)
  int qbar;   // 1: the GEMM-1 epilogue's beta sum syncs the 4 warps of a lane quadrant, not all 16
  RxProg prog;  // kRxProg
#if PCB_RNSX_KCONS
  // the per-prime constant records in the kernel parameters: every lane of a warp reads the same
  // record (one prime group per warp), so they come from the constant cache as broadcasts and
  // keep the shared-memory pipe to the tensor core, the W stream and the A tiles
  uint4 kcons[144 * 3];
#endif
};

__device__ __forceinline__ uint32_t redc(uint64_t T, uint32_t m, uint32_t minv) {
  const uint32_t u = (uint32_t)T * minv;
  return (uint32_t)((T + (uint64_t)u * m) >> 32);
}
__device__ __forceinline__ uint32_t mulr(uint32_t a, uint32_t b, uint32_t m, uint32_t minv) {
  return redc((uint64_t)a * b, m, minv);
}

// n-word (2 or 4) vector load / store
template <int N>
__device__ __forceinline__ void ldq(uint32_t* y, const uint32_t* p) {
  if constexpr (N == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    y[0] = v.x; y[1] = v.y; y[2] = v.z; y[3] = v.w;
  } else {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    y[0] = v.x; y[1] = v.y;
  }
}
template <int N>
__device__ __forceinline__ void stq(void* p, const uint32_t* y) {
  if constexpr (N == 4)
    *reinterpret_cast<uint4*>(p) = make_uint4(y[0], y[1], y[2], y[3]);
  else
    *reinterpret_cast<uint2*>(p) = make_uint2(y[0], y[1]);
}
template <int N>
__device__ __forceinline__ void tmem_ldq(uint32_t taddr, uint32_t* v) {
  if constexpr (N == 4) {
    uint32_t (&a)[16] = *reinterpret_cast<uint32_t(*)[16]>(v);
    umma::tmem_ld16(taddr, a);
  } else {
    uint32_t (&a)[8] = *reinterpret_cast<uint32_t(*)[8]>(v);
    umma::tmem_ld8(taddr, a);
  }
}

// Per-thread view of the kernel state.
template <class C>
struct Thr {
  uint8_t* sm;
  const uint4* rc;  // this thread group's constant records: [w * 3 + {0,1,2}], w = thread-local residue
  uint32_t tl;      // TMEM address of this warp's lane quadrant
  int e, g, lane, gt, NT;
  uint32_t dbi, dph;
  bool nowait;
  uint32_t rank;  // CTA rank in the pair (cta_group::2): rank 1 signals the leader's barriers
  float cthr;     // sum over this thread's primes of 2^23 (2^8 / m'): the bias of the beta terms
  uint64_t *dfull, *dfree, *a1, *a2;
  uint32_t bar_id, bar_n;  // named barrier of the beta partial sums (quadrant or CTA-wide)
};

// hand-off arrive (A tile ready / TMEM buffer drained): the MMA issuer's barrier is local, or the
// leader CTA's for the peer of a cta_group::2 pair
template <class C>
__device__ __forceinline__ void arrive_issuer(const Thr<C>& T, uint64_t* bar) {
  if (C::CG == 2 && T.rank == 1)
    umma::mbar_arrive_remote(bar, 0);
  else
    umma::mbar_arrive(bar);
}

// x (nw words, LE) -> lazy Montgomery residues of this thread's primes (both bases)
template <class C>
__device__ __forceinline__ void conv_in(uint32_t (&XB)[C::RPT], uint32_t (&XQ)[C::RPT], const uint32_t* w, int nw,
                                        const Thr<C>& T) {
#pragma unroll
  for (int q = 0; q < C::RPT; q++) {
    const uint4 ra = T.rc[q * 3], rq = T.rc[q * 3 + 1], rr = T.rc[q * 3 + 2];
    uint32_t ab = 0, aq = 0;
#pragma unroll 1
    for (int t = nw - 1; t >= 0; t--) {
      const uint32_t wt = w[t];
      uint32_t vb = mulr(ab, ra.w, ra.x, ra.y) + mulr(wt, ra.w, ra.x, ra.y);
      uint32_t vq = mulr(aq, rr.w, rq.x, rq.y) + mulr(wt, rr.w, rq.x, rq.y);
      if (vb >= 2 * ra.x) vb -= 2 * ra.x;
      if (vq >= 2 * rq.x) vq -= 2 * rq.x;
      ab = vb;
      aq = vq;
    }
    XB[q] = ab;
    XQ[q] = aq;
  }
}

// wait for the next TMEM buffer, load this thread's quad j of it, release it when the last quad
// has been read.  Returns the quad in D (4 bytes x QT primes, [byte][prime]).
template <class C, int QT>
__device__ __forceinline__ void d_quad(Thr<C>& T, int ptc, int j, bool first, bool last, uint32_t* D) {
  if (first && !T.nowait) {
    umma::mbar_wait(T.dfull + T.dbi, T.dph);
    umma::tmem_fence_after();
  }
  tmem_ldq<QT>(T.tl + T.dbi * C::BUFC + T.g * 4 * ptc + j * 16, D);
  umma::tmem_wait_ld();
  if (last) {
    umma::tmem_fence_before();
    __syncwarp();
    if (T.lane == 0 && !T.nowait) arrive_issuer<C>(T, T.dfree + T.dbi);
    if (++T.dbi == (uint32_t)C::NB) { T.dbi = 0; T.dph ^= 1; }
  }
}

// One RNS Montgomery product for a tile in three phases (so two tiles can be interleaved):
//   rx_s1: t = x y (both bases), xi = t C1 -> A1, t' parked in XQ; hands A1 to the MMA warp
//   rx_e1: GEMM-1 epilogue: qh', r' (new B'), xi' -> A2, beta; hands A2 to the MMA warp
//   rx_e2: GEMM-2 epilogue: new B residues
// Y = X (sq) or the 4-word vectors at ybase + v * yvs (v < NQ: base-B quad v; v >= NQ: B').
template <class C>
__device__ __forceinline__ void rx_s1(uint32_t (&XB)[C::RPT], uint32_t (&XQ)[C::RPT], bool sq, const uint32_t* ybase,
                                      int yvs, Thr<C>& T, uint8_t* A1, uint64_t* a1) {
  constexpr int NC = C::NC;
  // ---- 1. t = x y: xi = t C1 (B) -> A1; t' parked in XQ ------------------------------------------
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const int ptc = C::ptc(c);
#pragma unroll
    for (int j = 0; j < (ptc + 3) / 4; j++) {
      constexpr int dummy = 0;
      (void)dummy;
      const int QT = rnsx_qt(ptc, j);  // last quad of a ragged chunk: 2 primes
      const int w0 = C::cw0(c) + 4 * j, q = w0 / 4;
      uint32_t yb[4] = {}, yq[4] = {}, xi[4];
      if (!sq) {
        if (QT == 4) {
          ldq<4>(yb, ybase + q * yvs);
          ldq<4>(yq, ybase + (C::NQ + q) * yvs);
        } else {
          ldq<2>(yb, ybase + q * yvs);
          ldq<2>(yq, ybase + (C::NQ + q) * yvs);
        }
      }
#pragma unroll
      for (int t = 0; t < QT; t++) {
        const int w = w0 + t;
        const uint4 ra = T.rc[w * 3], rq = T.rc[w * 3 + 1];
        const uint32_t vb = sq ? XB[w] : yb[t], vq = sq ? XQ[w] : yq[t];
        xi[t] = mulr(mulr(XB[w], vb, ra.x, ra.y), ra.z, ra.x, ra.y);
        XQ[w] = mulr(XQ[w], vq, rq.x, rq.y);
      }
      uint8_t* dst = A1 + umma::kmajor_off(T.e, 4 * (C::cp0(c) + C::slot(c, T.g, j)), C::TILE);
      if (QT == 4) stq<4>(dst, xi); else stq<2>(dst, xi);
    }
  }
  umma::fence_async_smem();
  __syncwarp();
  if (T.lane == 0) arrive_issuer<C>(T, a1);
}

template <class C>
__device__ __forceinline__ void rx_e1(uint32_t (&XQ)[C::RPT], Thr<C>& T, uint8_t* A2, float* sS, uint64_t* a2) {
  constexpr int NC = C::NC;
  // ---- 2. GEMM-1 epilogue per chunk: qh', r' (new B'), xi' -> A2, partial beta ------------------
  // beta = floor(S), S = sum_j xi'_j / m'_j = beta + r'/M' with r'/M' < 2^-24 (M' > 2^24 (2K+2) N).
  // An over-estimate within [S, S + 1 - 2^-24) gives the same floor, so FP32 suffices: each term is
  // f(xi' >> 8) * (2^8 / m') with f(u) = the float 2^23 + u (bit trick, no conversion instruction),
  // the 2^23 parts (T.cthr) subtracted once, and a bias of 2^-8 above the total error bound
  // (~2^-12.5: truncated low bytes, FP32 roundings of 72 terms at magnitude < 2^6).
  float sp = 0.0f;
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const int ptc = C::ptc(c), nq = (ptc + 3) / 4;
#pragma unroll
    for (int j = 0; j < nq; j++) {
      const int QT = rnsx_qt(ptc, j);  // last quad of a ragged chunk: 2 primes
      uint32_t D[16], xp[4];
      if (QT == 4) d_quad<C, 4>(T, ptc, j, j == 0, j == nq - 1, D); else d_quad<C, 2>(T, ptc, j, j == 0, j == nq - 1, D);
#pragma unroll
      for (int t = 0; t < QT; t++) {
        const int w = C::cw0(c) + 4 * j + t;
        const uint4 rq = T.rc[w * 3 + 1], rr = T.rc[w * 3 + 2];
        const uint64_t V = (uint64_t)D[t] + ((uint64_t)D[QT + t] << 8) + ((uint64_t)D[2 * QT + t] << 16) +
                           ((uint64_t)D[3 * QT + t] << 24);
        // GEMM 1 runs on W1' = M_i C3_j mod m'_j, so V = qh C3 2^32 (mod m'_j) and the new B'
        // residue is one REDC of t' C2 + V (< 2m'^2 + 2^49 < 2^62: REDC < 2m', lazy)
        const uint32_t r = redc((uint64_t)XQ[w] * rq.z + V, rq.x, rq.y);
        XQ[w] = r;
        xp[t] = mulr(r, rr.x, rq.x, rq.y);
        sp = __fmaf_rn(__uint_as_float((xp[t] >> 8) | 0x4B000000u), __uint_as_float(rr.y), sp);
      }
      uint8_t* dst = A2 + umma::kmajor_off(T.e, 4 * (C::cp0(c) + C::slot(c, T.g, j)), C::TILE);
      if (QT == 4) stq<4>(dst, xp); else stq<2>(dst, xp);
    }
  }
  sS[T.g * C::TILE + T.e] = __fsub_rn(sp, T.cthr);
  umma::fence_async_smem();
  umma::named_sync(T.bar_id, T.bar_n);
  if (T.g == 0) {
    const float S = sS[T.e] + sS[C::TILE + T.e] + sS[2 * C::TILE + T.e] + sS[3 * C::TILE + T.e];
    const uint32_t beta = (uint32_t)floorf(S + 0.00390625f);  // + 2^-8 (see above)
    *reinterpret_cast<uint4*>(A2 + umma::kmajor_off(T.e, 4 * C::K, C::TILE)) = make_uint4(beta, 0, 0, 0);
    umma::fence_async_smem();
  }
  __syncwarp();
  if (T.lane == 0) arrive_issuer<C>(T, a2);
}

template <class C>
__device__ __forceinline__ void rx_e2(uint32_t (&XB)[C::RPT], Thr<C>& T) {
  constexpr int NC = C::NC;
  // ---- 3. GEMM-2 epilogue per chunk: r (new B residues) -------------------------------------------
#pragma unroll
  for (int c = 0; c < NC; c++) {
    const int ptc = C::ptc(c), nq = (ptc + 3) / 4;
#pragma unroll
    for (int j = 0; j < nq; j++) {
      const int QT = rnsx_qt(ptc, j);  // last quad of a ragged chunk: 2 primes
      uint32_t D[16];
      if (QT == 4) d_quad<C, 4>(T, ptc, j, j == 0, j == nq - 1, D); else d_quad<C, 2>(T, ptc, j, j == 0, j == nq - 1, D);
#pragma unroll
      for (int t = 0; t < QT; t++) {
        const int w = C::cw0(c) + 4 * j + t;
        const uint4 ra = T.rc[w * 3];
        const uint64_t V = (uint64_t)D[t] + ((uint64_t)D[QT + t] << 8) + ((uint64_t)D[2 * QT + t] << 16) +
                           ((uint64_t)D[3 * QT + t] << 24);
        XB[w] = redc(V, ra.x, ra.y);
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void rx_mm(uint32_t (&XB)[C::RPT], uint32_t (&XQ)[C::RPT], bool sq, const uint32_t* ybase,
                                      int yvs, Thr<C>& T) {
  rx_s1<C>(XB, XQ, sq, ybase, yvs, T, T.sm + C::OFF_A1, T.a1);
  rx_e1<C>(XQ, T, T.sm + C::OFF_A2, reinterpret_cast<float*>(T.sm + C::OFF_S), T.a2);
  rx_e2<C>(XB, T);
}

template <class C>
__device__ __forceinline__ void compute_role(const XArgs& P, Thr<C>& T, int mine, int nsteps, int npre, int s_x2,
                                             int s_tab, int s_main, int s_fin) {
  constexpr int NQ = C::NQ, NV = C::NV, RPT = C::RPT;
  const int ntiles = (P.count + C::TILE - 1) / C::TILE;
  const int park = P.ntab, park_x2 = P.ntab + 1;
  const uint32_t zero = 0;
  // per-thread table / constant operand addressing (4-word vectors)
  auto tab_ptr = [&](int ent) { return P.tab + (((size_t)ent * NV) * T.NT + T.gt) * 4; };
  const int tab_vs = T.NT * 4;
  auto cv_ptr = [&](int id) { return P.cvec + (size_t)((id * C::G + T.g) * NV) * 4; };
  auto vec_op = [&](const uint32_t* b, int vs, uint32_t (&XB)[RPT], uint32_t (&XQ)[RPT], int op) {
    // op 0: X = vec, 1: X += vec (lazy), 2: vec = X
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      const int n = RPT - 4 * q < 4 ? RPT - 4 * q : 4;
      uint32_t v[4] = {}, u[4] = {};
      uint32_t* pb = const_cast<uint32_t*>(b) + (size_t)q * vs;
      uint32_t* pq = const_cast<uint32_t*>(b) + (size_t)(NQ + q) * vs;
      if (op == 2) {
#pragma unroll
        for (int t = 0; t < n; t++) {
          v[t] = XB[4 * q + t];
          u[t] = XQ[4 * q + t];
        }
        if (n == 4) { stq<4>(pb, v); stq<4>(pq, u); } else { stq<2>(pb, v); stq<2>(pq, u); }
        continue;
      }
      if (n == 4) { ldq<4>(v, pb); ldq<4>(u, pq); } else { ldq<2>(v, pb); ldq<2>(u, pq); }
#pragma unroll
      for (int t = 0; t < n; t++) {
        const int w = 4 * q + t;
        if (op == 0) {
          XB[w] = v[t];
          XQ[w] = u[t];
        } else {
          const uint32_t mb = T.rc[w * 3].x, mq = T.rc[w * 3 + 1].x;
          uint32_t s1 = XB[w] + v[t], s2 = XQ[w] + u[t];
          if (s1 >= 2 * mb) s1 -= 2 * mb;
          if (s2 >= 2 * mq) s2 -= 2 * mq;
          XB[w] = s1;
          XQ[w] = s2;
        }
      }
    }
  };
  if (P.mode == kRxProg) {
    const RxProg& G = P.prog;
    constexpr int REC = C::G * NV * 4;  // words per RNS record
    // record address of this thread's part of element-record i
    auto rec = [&](const uint32_t* base, size_t i) { return base + i * REC + (size_t)T.g * NV * 4; };
    // operand vector pointer for source (kind, arg) of element el (record layout: vs = 4)
    auto src_ptr = [&](uint8_t kind, uint8_t arg, int el) -> const uint32_t* {
      if (kind == kRsCvec) return cv_ptr(arg);
      if (kind == kRsSelf) return rec(G.mtab, (size_t)el * 64 + arg);
      if (kind == kRsPart) return rec(G.part, (size_t)el * G.nparts + arg);
      // kRsMat: element = (row, chunk)
      const int jl = arg >> 4, w = arg & 15;
      const int row = el / G.nch, col = (el % G.nch) * G.cc + jl;
      const int tcol = (G.brows ? (row / G.brows) * G.cols : 0) + col;
      int d = 0;
      if (col < G.cols) d = (int)((G.expo[(size_t)row * G.cols + col] >> (6 * w)) & 63u);
      if (d == 0) return cv_ptr(kRxOneM);  // digit 0 (and padding columns): the Montgomery one
      return rec(G.mtab, ((size_t)tcol * G.nwin + w) * 64 + d);
    };
#pragma unroll 1
    for (int k = 0; k < mine; k++) {
      const int tile = blockIdx.x + k * gridDim.x;
      const int el0 = tile * C::TILE + T.e;
      const bool live = el0 < P.count;
      const int el = live ? el0 : P.count - 1;  // padding lanes recompute the last element (not stored)
      uint32_t XB[RPT], XQ[RPT];
#pragma unroll 1
      for (int s = 0; s < G.nsteps; s++) {
        const XStep stp = G.st[s];
        if (stp.xs == kRsConv) {
          conv_in<C>(XB, XQ, P.x + (size_t)el * P.x_words, P.x_words, T);
        } else if (stp.xs != kRsKeep) {
          vec_op(src_ptr(stp.xs, stp.xa, el), 4, XB, XQ, 0);
        }
        if (s + 1 < G.nsteps) {  // warm L2 with the next step's gathered multiplier record (no registers)
          const XStep nx = G.st[s + 1];
          if (nx.ys == kRsMat || nx.ys == kRsSelf || nx.ys == kRsPart) {
            const char* pn = reinterpret_cast<const char*>(src_ptr(nx.ys, nx.ya, el));
#pragma unroll
            for (int o = 0; o < NV * 16; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + o));
          }
        }
        if (stp.ys == kRsSq)
          rx_mm<C>(XB, XQ, true, nullptr, 4, T);
        else
          rx_mm<C>(XB, XQ, false, src_ptr(stp.ys, stp.ya, el), 4, T);
        if (!live) continue;
        if (stp.flags & 1) {  // table fill: entry 0 of this element's slot is the Montgomery one
          uint32_t YB[RPT], YQ[RPT];
          vec_op(cv_ptr(kRxOneM), 4, YB, YQ, 0);
          vec_op(rec(G.mtab, (size_t)el * 64), 4, YB, YQ, 2);
        }
        switch (stp.post) {
          case kRpOut: {
            uint32_t* o = P.out + (size_t)el * C::K;
#pragma unroll
            for (int c = 0; c < C::NC; c++) {
              const int ptc = C::ptc(c);
#pragma unroll
              for (int j = 0; j < (ptc + 3) / 4; j++) {
                const int QT = rnsx_qt(ptc, j), w0 = C::cw0(c) + 4 * j;
                uint32_t* d = o + C::cp0(c) + C::slot(c, T.g, j);
                if (QT == 4) stq<4>(d, &XQ[w0]); else stq<2>(d, &XQ[w0]);
              }
            }
            break;
          }
          case kRpChain: vec_op(rec(G.mtab, ((size_t)el * G.nwin + stp.pa) * 64 + 1), 4, XB, XQ, 2); break;
          case kRpSelf: vec_op(rec(G.mtab, (size_t)el * 64 + stp.pa), 4, XB, XQ, 2); break;
          case kRpRec: vec_op(rec(G.pout ? G.pout : G.part, (size_t)el), 4, XB, XQ, 2); break;
          default: break;
        }
      }
    }
    return;
  }
  // ---- exponentiation programs (Enc / Dec / Pow): per-step operand selection and epilogue ------
  // `tt` selects the per-thread window table of tile slot tt (two tiles in flight when C::NT == 2)
  auto tabp = [&](int ent, int tt) { return tab_ptr(ent * C::NT + tt); };
  // PowVar: 4-bit digit w of this element's exponent (dead lanes: 0)
  auto digit = [&](int el, bool live, int w) -> int {
    if (!live) return 0;
    return (int)((P.m[(size_t)el * P.m_words + (w >> 3)] >> (4 * (w & 7))) & 15u);
  };
  // Op bytes of the exponent schedule, 32 steps per warp-wide vector: lane l holds the op of step
  // base + l, the next vector is loaded 32 steps ahead and the current op comes out of a shuffle.
  // (A scalar byte load consumed by the step's branch -- or prefetched one step ahead into a
  // uniform register, which the compiler did right after the load -- put an L2 round trip on
  // every step's critical path; ncu source view, profiles/r02_rnsx72_bench_ncu.json.)
  const bool has_ops = P.mode != kRxPowVar && P.mode != kRxProg && P.ops != nullptr;
  uint32_t op_cur = 0, opv_cur = 0, opv_next = 0;
  auto opv_load = [&](int s0) -> uint32_t {
    const int s = s0 + T.lane;
    return (has_ops && s >= s_main && s < s_fin) ? (uint32_t)P.ops[s - s_main + 1] : 0u;
  };
  auto op_step = [&](int s) {
    if ((s & 31) == 0) {
      opv_cur = s == 0 ? opv_load(0) : opv_next;
      opv_next = opv_load(s + 32);
    }
    op_cur = __shfl_sync(0xffffffffu, opv_cur, s & 31);
  };
  auto prep = [&](int s, uint32_t (&XB)[RPT], uint32_t (&XQ)[RPT], int tt, int el, bool live, bool& sq,
                  const uint32_t*& yb, int& yvs) {
    sq = false;
    yb = nullptr;
    yvs = 4;
    if (P.mode == kRxPowVar && s >= npre) {  // table T_s = T_(s-1) x (s < 16), then 4-bit windows
      if (s < 16) {
        yb = tabp(1, tt);
        yvs = tab_vs;
      } else if (s < s_fin) {
        const int k = s - 16;
        if (k % 5 < 4) {
          sq = true;
        } else {
          yb = tabp(digit(el, live, P.nops - 2 - k / 5), tt);
          yvs = tab_vs;
        }
      } else {
        yb = cv_ptr(kRxOne);
      }
      return;
    }
    if (s < npre) {
      const bool first = npre == 2 && s == 0;
      const uint32_t* src = &zero;
      int nw = 1;
      int cst = kRxR2N;
      if ((P.mode == kRxEnc || P.mode == kRxEncG) && first) {  // m n  (EncG: g, plain, via M mod N)
        if (live) { src = P.m + (size_t)el * P.m_words; nw = P.m_words; }
        cst = P.mode == kRxEnc ? kRxNM : kRxOneM;
      } else if ((P.mode == kRxDec || P.mode == kRxPowVar) && first) {  // c_hi 2^(32 S) M
        // inputs narrower than S words (unbalanced primes: x_words < S) have no high half
        if (live && P.x_words > P.S) { src = P.x + (size_t)el * P.x_words + P.S; nw = P.x_words - P.S; }
        cst = kRxCR2N;
      } else {  // r M / c_lo M / x M
        if (live) {
          src = P.x + (size_t)el * P.x_words;
          nw = (P.mode == kRxDec || P.mode == kRxPowVar) ? min(P.S, P.x_words) : P.x_words;
        }
      }
      conv_in<C>(XB, XQ, src, nw, T);
      yb = cv_ptr(cst);
    } else if (s == s_x2) {
      sq = true;
    } else if (s < s_main) {
      yb = tabp(park_x2, tt);
      yvs = tab_vs;
    } else if (s < s_fin) {
      const uint32_t op = op_cur;
      if (op == kOpSquare) {
        sq = true;
      } else {
        yb = tabp(op, tt);
        yvs = tab_vs;
      }
    } else if (P.mode == kRxEnc || P.mode == kRxEncG) {
      yb = tabp(park, tt);
      yvs = tab_vs;
    } else {
      yb = cv_ptr(kRxOne);
    }
  };
  auto post = [&](int s, uint32_t (&XB)[RPT], uint32_t (&XQ)[RPT], int tt, int el, bool live) {
    if (P.mode == kRxPowVar && s < s_fin) {
      if (s == 0) {
        vec_op(tabp(park, tt), tab_vs, XB, XQ, 2);
      } else if (s == 1) {  // x M = c_lo M + c_hi 2^(32S) M: table entry 1; entry 0 = M mod N (the one)
        vec_op(tabp(park, tt), tab_vs, XB, XQ, 1);
        vec_op(tabp(1, tt), tab_vs, XB, XQ, 2);
        uint32_t OB[RPT], OQ[RPT];
        vec_op(cv_ptr(kRxOneM), 4, OB, OQ, 0);
        vec_op(tabp(0, tt), tab_vs, OB, OQ, 2);
      } else if (s < 16) {
        vec_op(tabp(s, tt), tab_vs, XB, XQ, 2);
        if (s == 15) vec_op(tabp(digit(el, live, P.nops - 1), tt), tab_vs, XB, XQ, 0);  // top window
      }
      return;
    }
    if (s < npre) {
      const bool first = npre == 2 && s == 0;
      if (first) {
        if (P.mode == kRxEnc) vec_op(cv_ptr(kRxOne), 4, XB, XQ, 1);  // 1 + m n (plain)
        vec_op(tabp(park, tt), tab_vs, XB, XQ, 2);
      } else {
        if (P.mode == kRxDec) vec_op(tabp(park, tt), tab_vs, XB, XQ, 1);  // c M = c_lo M + c_hi 2^(32S) M
        vec_op(tabp(0, tt), tab_vs, XB, XQ, 2);
      }
    } else if (s == s_x2) {
      vec_op(tabp(park_x2, tt), tab_vs, XB, XQ, 2);
      vec_op(tabp(0, tt), tab_vs, XB, XQ, 0);
    } else if (s < s_main) {
      vec_op(tabp(s - s_tab + 1, tt), tab_vs, XB, XQ, 2);
      if (s == s_main - 1) vec_op(tabp(P.ops[0], tt), tab_vs, XB, XQ, 0);
    } else if (s == s_fin) {
      if (live) {
        uint32_t* o = P.out + (size_t)el * C::K;
#pragma unroll
        for (int c = 0; c < C::NC; c++) {
          const int ptc = C::ptc(c);
#pragma unroll
          for (int j = 0; j < (ptc + 3) / 4; j++) {
            const int QT = rnsx_qt(ptc, j), w0 = C::cw0(c) + 4 * j;
            uint32_t* d = o + C::cp0(c) + C::slot(c, T.g, j);
            if (QT == 4) stq<4>(d, &XQ[w0]); else stq<2>(d, &XQ[w0]);
          }
        }
      }
    }
    if (P.ntab == 1 && s == s_x2) vec_op(tabp(P.ops[0], tt), tab_vs, XB, XQ, 0);
  };
  if constexpr (C::NT == 2) {
    // Two tiles in flight: compute order A.s1, B.s1, A.e1, B.e1, then (next step) A.e2 + A.s1, ...
    // while the tensor core runs A.G1, B.G1, A.G2, B.G2: each GEMM overlaps the other tile's
    // CUDA-core phase.
    uint8_t* A1a = T.sm + C::OFF_A1;
    uint8_t* A2a = T.sm + C::OFF_A2;
    uint8_t* A1b = A1a + C::ABLK;
    uint8_t* A2b = A2a + C::ABLK;
    float* sSa = reinterpret_cast<float*>(T.sm + C::OFF_S);
    float* sSb = sSa + C::G * C::TILE;
    const int npairs = (ntiles + 1) / 2;
    (void)npairs;
#pragma unroll 1
    for (int k = 0; k < mine; k++) {
      const int pr = blockIdx.x + k * gridDim.x;
      const int ela = (2 * pr) * C::TILE + T.e, elb = (2 * pr + 1) * C::TILE + T.e;
      const bool la = ela < P.count, lb = elb < P.count;
      uint32_t XBa[RPT], XQa[RPT], XBb[RPT], XQb[RPT];
      bool sq;
      const uint32_t* yb;
      int yvs;
#pragma unroll 1
      for (int s = 0; s < nsteps; s++) {
        op_step(s);
        if (s > 0) {
          rx_e2<C>(XBa, T);
          post(s - 1, XBa, XQa, 0, ela, la);
        }
        prep(s, XBa, XQa, 0, ela, la, sq, yb, yvs);
        rx_s1<C>(XBa, XQa, sq, yb, yvs, T, A1a, T.a1);
        if (s > 0) {
          rx_e2<C>(XBb, T);
          post(s - 1, XBb, XQb, 1, elb, lb);
        }
        prep(s, XBb, XQb, 1, elb, lb, sq, yb, yvs);
        rx_s1<C>(XBb, XQb, sq, yb, yvs, T, A1b, T.a1 + 2);
        rx_e1<C>(XQa, T, A2a, sSa, T.a2);
        rx_e1<C>(XQb, T, A2b, sSb, T.a2 + 2);
      }
      rx_e2<C>(XBa, T);
      post(nsteps - 1, XBa, XQa, 0, ela, la);
      rx_e2<C>(XBb, T);
      post(nsteps - 1, XBb, XQb, 1, elb, lb);
    }
    return;
  }
  if constexpr (C::NT == 3) {
    // Three tiles in flight (small K): the same rotation as above over tiles 0, 1, 2.
    constexpr int NT = C::NT;
    float* sS0 = reinterpret_cast<float*>(T.sm + C::OFF_S);
#pragma unroll 1
    for (int k = 0; k < mine; k++) {
      const int pr = blockIdx.x + k * gridDim.x;
      int elt[NT];
      bool lv[NT];
#pragma unroll
      for (int t = 0; t < NT; t++) {
        elt[t] = (NT * pr + t) * C::TILE + T.e;
        lv[t] = elt[t] < P.count;
      }
      uint32_t XB[NT][RPT], XQ[NT][RPT];
      bool sq;
      const uint32_t* yb;
      int yvs;
#pragma unroll 1
      for (int s = 0; s < nsteps; s++) {
        op_step(s);
#pragma unroll
        for (int t = 0; t < NT; t++) {
          if (s > 0) {
            rx_e2<C>(XB[t], T);
            post(s - 1, XB[t], XQ[t], t, elt[t], lv[t]);
          }
          prep(s, XB[t], XQ[t], t, elt[t], lv[t], sq, yb, yvs);
          rx_s1<C>(XB[t], XQ[t], sq, yb, yvs, T, T.sm + C::OFF_A1 + t * C::ABLK, T.a1 + 2 * t);
        }
#pragma unroll
        for (int t = 0; t < NT; t++)
          rx_e1<C>(XQ[t], T, T.sm + C::OFF_A2 + t * C::ABLK, sS0 + t * C::G * C::TILE, T.a2 + 2 * t);
      }
#pragma unroll
      for (int t = 0; t < NT; t++) {
        rx_e2<C>(XB[t], T);
        post(nsteps - 1, XB[t], XQ[t], t, elt[t], lv[t]);
      }
    }
    return;
  }
#pragma unroll 1
  for (int k = 0; k < mine; k++) {
    const int tile = blockIdx.x + k * gridDim.x;
    const int el = tile * C::TILE + T.e;
    const bool live = el < P.count;
    uint32_t XB[RPT], XQ[RPT];
#pragma unroll 1
    for (int s = 0; s < nsteps; s++) {
      op_step(s);
      bool sq;
      const uint32_t* yb;
      int yvs;
      prep(s, XB, XQ, 0, el, live, sq, yb, yvs);
      rx_mm<C>(XB, XQ, sq, yb, yvs, T);
      post(s, XB, XQ, 0, el, live);
    }
  }
}

// Role warp (all 32 lanes run the loop, so every value is warp-uniform; elect.sync issues):
// streams the base-extension slices into the ring (one slice per 4 KB slot) and issues the MMAs.
__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          umma::smem_u32(mbar))
      : "memory");
}

// slice-table flags (host-built per modulus; one entry per MMA of a product)
enum : uint32_t { kFGemm = 1, kFG2 = 2, kFChunk = 4, kFChunkEnd = 8, kFStage = 16, kFStageEnd = 32, kFAcc = 64 };

// Role warp (all 32 lanes run the loop, values warp-uniform; elect.sync issues).  A compact
// interpreter over the per-product slice table {A offset, B offset | LBO, idesc, flags}: the W
// slices stream into the ring (one bulk copy per stage), one MMA per slice.
// Role warpgroup: warp 0 issues the MMAs (a compact interpreter over the per-product slice table
// {A offset, B offset | LBO, idesc, flags}; elect.sync issue), warp 1 streams the W stages into
// the ring (one bulk copy per stage, full/empty mbarrier handshake).  Scalars come by value: a
// noinline callee would otherwise re-read the kernel parameters through generic loads.
__device__ __forceinline__ void commit_elect_mc(uint64_t* mbar, uint16_t mask) {  // arrive in every CTA of mask
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          umma::smem_u32(mbar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mma_elect_cg2(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect_cg2(uint64_t* mbar) {  // arrive in both CTAs of the pair
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          umma::smem_u32(mbar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// cta_group::2 leader (rank 0): one M = 256 MMA per slice for both CTAs' tiles; waits for both
// halves of the slice (own full barrier + the peer's, relayed) and both CTAs' A tiles / drains.
template <class C>
__device__ __noinline__ void mma_pair(uint8_t* sm, uint32_t tm, uint64_t* bars, uint32_t nprod) {
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NSTAGE;
  uint64_t* dfull = bars + 2 * C::NSTAGE;
  uint64_t* dfree = dfull + C::NB;
  uint64_t* abar = dfree + C::NB;
  uint64_t* pfull = abar + 2 * C::NT;
  const uint64_t hi = umma::desc_kmajor(0, 128) & 0xFFFFFFFF00000000ull;
  const uint32_t a1lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A1), C::TILE);
  const uint32_t a2lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A2), C::TILE);
  const uint32_t ring16 = umma::smem_u32(sm + C::OFF_RING) >> 4;
  constexpr uint32_t SLOT16 = C::SLOT / 16;
  uint32_t cslot = 0, cph = 0, dbi = 0, dph = 0, dcnt = 0, bslot = ring16;
#pragma unroll 1
  for (uint32_t pr = 0; pr < nprod; pr++) {
#pragma unroll 1
    for (int gm = 0; gm < 2; gm++) {
      umma::mbar_wait_cluster(abar + gm, pr & 1);
      umma::tmem_fence_after();
      const uint32_t alo = gm ? a2lo : a1lo;
      const int ks = gm ? C::KS2 : C::KS1;
#pragma unroll
      for (int c = 0; c < C::NC; c++) {
        const uint32_t ncol = (uint32_t)C::ncol(c);
        const uint32_t idesc = umma::idesc_i8(2 * C::TILE, (int)ncol);
        if (dcnt >= (uint32_t)C::NB) {
          umma::mbar_wait_cluster(dfree + dbi, dph ^ 1);
          umma::tmem_fence_after();
        }
        const uint32_t dt = tm + dbi * C::BUFC;
#pragma unroll 1
        for (int k = 0; k < ks; k++) {
          umma::mbar_wait(full + cslot, cph);
          umma::mbar_wait_cluster(pfull + cslot, cph);
          mma_elect_cg2(dt, hi | (uint64_t)(alo + (uint32_t)k * (2 * C::TILE * 16 / 16)),
                        hi | (uint64_t)((bslot & 0x3FFFu) | ((ncol / 2) << 16)), idesc, (uint32_t)k);
          commit_elect_cg2(empty + cslot);
          bslot += SLOT16;
          if (++cslot == (uint32_t)C::NSTAGE) { cslot = 0; cph ^= 1; bslot = ring16; }
        }
        commit_elect_cg2(dfull + dbi);
        dcnt++;
        if (++dbi == (uint32_t)C::NB) { dbi = 0; dph ^= 1; }
      }
    }
  }
}

// cta_group::2 peer (rank 1): relay "my half of slice i has landed" to the leader, in order
template <class C>
__device__ __noinline__ void relay_pair(uint64_t* bars, uint32_t nprod, int lane) {
  uint64_t* full = bars;
  uint64_t* pfull = bars + 2 * C::NSTAGE + 2 * C::NB + 2 * C::NT;
  const uint32_t total = nprod * (uint32_t)C::NSLICE;
  uint32_t slot = 0, ph = 0;
#pragma unroll 1
  for (uint32_t i = 0; i < total; i++) {
    umma::mbar_wait(full + slot, ph);
    if (lane == 0) umma::mbar_arrive_remote(pfull + slot, 0);
    __syncwarp();
    if (++slot == (uint32_t)C::NSTAGE) { slot = 0; ph ^= 1; }
  }
}

// The W stream is issued by kRxProducers warps of the role warpgroup in round robin over the ring
// stages: one issuing warp serialises its bulk copies (~600 clk per copy whatever the size or the
// number in flight, tools/bulk_bw2.cu, profiles/r02_bulk_bw2.txt), so one warp caps the stream at
// 8 KB / 600 clk = 13.5 B/clk/SM -- the bound of the whole kernel in the tensor-only timing split
// (profiles/r02_dbg_modes.txt).  Warp pw of npw owns stages i with i % npw == pw.
constexpr int kRxProducers = PCB_RNSX_ROLE_WARPS - 1;

template <class C>
__device__ __noinline__ void producer_role(const uint8_t* wimg0, size_t wstride, uint8_t* sm, uint64_t* bars,
                                           uint32_t nprod, int lane, int cl, uint32_t rank, int pw, int npw,
                                           bool multi_slice) {
  // cl == 2: the CTA pair of a cluster shares the stream; each CTA fetches half of every stage
  // and multicasts it into both CTAs' rings (half the L2 traffic per SM)
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NSTAGE;
  uint8_t* ring = sm + C::OFF_RING;
  const uint2* stg = reinterpret_cast<const uint2*>(sm + C::OFF_SLT + C::NSLICE * 16);
  // every SM streams the same matrices: spread the reads over kRxReplicas copies (L2 slices)
  const uint8_t* wimg = wimg0 + (size_t)(blockIdx.x % kRxReplicas) * wstride;
  // stages: spc consecutive slices of one chunk (contiguous in the image; every slice of a chunk
  // has the same size); the debug interpreter (mma_role, dbg 1/3) and the CTA pair use one slice
  uint32_t issued = 0, pslot = 0, pph = 0;
#pragma unroll 1
  for (uint32_t pr = 0; pr < nprod; pr++) {
#pragma unroll 1
    for (int seg = 0; seg < 2 * C::NT; seg++) {  // G1 per tile, then G2 per tile (MMA issue order)
      const int gm = seg / C::NT;
      const int ks = gm ? C::KS2 : C::KS1;
      int i0 = gm ? C::NC * C::KS1 : 0;
#pragma unroll
      for (int c = 0; c < C::NC; c++) {
        const int sp = multi_slice ? C::spc(c) : 1;
#pragma unroll 1
        for (int k = 0; k < ks; k += sp, issued++) {
          if ((int)(issued % (uint32_t)npw) != pw) {  // another producer warp's stage
            if (++pslot == (uint32_t)C::NSTAGE) { pslot = 0; pph ^= 1; }
            continue;
          }
          if (issued >= (uint32_t)C::NSTAGE) umma::mbar_wait(empty + pslot, pph ^ 1);
          const uint2 d = stg[i0 + k];
          const uint32_t bytes = d.y * (uint32_t)(ks - k < sp ? ks - k : sp);
          if (lane == 0) {
            umma::mbar_arrive_expect_tx(full + pslot, C::CG == 2 ? bytes >> 1 : bytes);
            if (C::CG == 2) {  // wimg is the split-halves image: this CTA's half of the slice
              const uint32_t half = bytes >> 1;
              umma::bulk_g2s(ring + pslot * C::SLOT, wimg + (size_t)d.x * 16 + rank * half, half, full + pslot);
              (void)cl;
            } else if (cl == 2) {
              const uint32_t half = bytes >> 1;
              umma::bulk_g2s_mc(ring + pslot * C::SLOT + rank * half, wimg + (size_t)d.x * 16 + rank * half, half,
                                full + pslot, 0x3);
            } else {
              umma::bulk_g2s(ring + pslot * C::SLOT, wimg + (size_t)d.x * 16, bytes, full + pslot);
            }
          }
          __syncwarp();
          if (++pslot == (uint32_t)C::NSTAGE) { pslot = 0; pph ^= 1; }
        }
        i0 += ks;
      }
    }
  }
}

// DBG: 0 normal, 1 no compute handshakes (tensor + stream only), 3 stream only, 4 MMAs only;
// mma_fast: 5 = production tensor + stream path alone, 6 = it and the compute warps side by side
// without hand-offs (the interference of the two paths, no dependency waits); 7 / 8 = the compute
// warps beside the stream alone / the MMAs alone (single-slice debug loop)
// Production MMA issue loop: the product's structure (GEMM -> chunk -> k-step) is the loop
// structure, so the per-MMA work is one full-barrier wait, the descriptor adds, the MMA and the
// slot release (one 8 KB slice per ring stage).
// WAIT = false (PCB_RNSX_DBG=5): the same loop without the compute hand-offs, to time the tensor +
// stream path on its own
template <class C, bool WAIT = true>
__device__ __noinline__ void mma_fast(uint8_t* sm, uint32_t tm, uint64_t* bars, uint32_t nprod, int cl) {
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NSTAGE;
  uint64_t* dfull = bars + 2 * C::NSTAGE;
  uint64_t* dfree = dfull + C::NB;
  uint64_t* abar = dfree + C::NB;  // per tile: a1, a2
  const uint64_t hi = umma::desc_kmajor(0, 128) & 0xFFFFFFFF00000000ull;
  const uint32_t a1lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A1), C::TILE);
  const uint32_t a2lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A2), C::TILE);
  const uint32_t ring16 = umma::smem_u32(sm + C::OFF_RING) >> 4;
  constexpr uint32_t SLOT16 = C::SLOT / 16, ABLK16 = C::ABLK / 16;
  uint32_t cslot = 0, cph = 0, dbi = 0, dph = 0, dcnt = 0;
  uint32_t bslot = ring16;  // address field of the current ring slot
#pragma unroll 1
  for (uint32_t pr = 0; pr < nprod; pr++) {
#pragma unroll 1
    for (int seg = 0; seg < 2 * C::NT; seg++) {
      const int gm = seg / C::NT, tt = seg % C::NT;
      if (WAIT) {
        umma::mbar_wait(abar + 2 * tt + gm, pr & 1);
        umma::tmem_fence_after();
      }
      const uint32_t alo = (gm ? a2lo : a1lo) + tt * ABLK16;
      const int ks = gm ? C::KS2 : C::KS1;
#pragma unroll
      for (int c = 0; c < C::NC; c++) {
        constexpr int dummy = 0;
        (void)dummy;
        const uint32_t ncol = (uint32_t)C::ncol(c);
        const uint32_t idesc = umma::idesc_i8(C::TILE, (int)ncol);
        const int sp = C::spc(c);  // slices per ring stage (one bulk copy)
        if (WAIT && dcnt >= (uint32_t)C::NB) {
          umma::mbar_wait(dfree + dbi, dph ^ 1);
          umma::tmem_fence_after();
        }
        const uint32_t dt = tm + dbi * C::BUFC;
        uint32_t boff = 0;
        int ks_in = 0;
#pragma unroll 1
        for (int k = 0; k < ks; k++) {
          if (ks_in == 0) {
            umma::mbar_wait(full + cslot, cph);
            boff = 0;
          }
          mma_elect(dt, hi | (uint64_t)(alo + (uint32_t)k * (2 * C::TILE * 16 / 16)),
                    hi | (uint64_t)(((bslot + boff) & 0x3FFFu) | (ncol << 16)), idesc, (uint32_t)k);
          boff += ncol * 2;  // one slice: ncol rows x 32 bytes, in 16-byte units
          if (++ks_in == sp || k == ks - 1) {
            ks_in = 0;
            if (cl == 2) commit_elect_mc(empty + cslot, 0x3); else commit_elect(empty + cslot);
            bslot += SLOT16;
            if (++cslot == (uint32_t)C::NSTAGE) { cslot = 0; cph ^= 1; bslot = ring16; }
          }
        }
        commit_elect(dfull + dbi);
        dcnt++;
        if (++dbi == (uint32_t)C::NB) { dbi = 0; dph ^= 1; }
      }
    }
  }
  if (!WAIT && nprod) umma::mbar_wait(dfull + (dbi + C::NB - 1) % C::NB, (dbi == 0) ? dph ^ 1 : dph);
}

template <class C, int DBG>
__device__ __noinline__ void mma_role(uint8_t* sm, uint32_t tm, uint64_t* bars, uint32_t nprod, int cl) {
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NSTAGE;
  uint64_t* dfull = bars + 2 * C::NSTAGE;
  uint64_t* dfree = dfull + C::NB;
  uint64_t* a1 = dfree + C::NB;
  uint64_t* a2 = a1 + 1;
  const uint4* slt = reinterpret_cast<const uint4*>(sm + C::OFF_SLT);
  constexpr bool kWaitCompute = DBG == 0, kRing = DBG != 4, kMma = DBG != 3;
  uint32_t cslot = 0, cph = 0, dbi = 0, dph = 0, dcnt = 0;
  const uint32_t hi = (uint32_t)(umma::desc_kmajor(0, 128) >> 32);  // SBO / version fields
  const uint32_t a1lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A1), C::TILE);
  const uint32_t a2lo = (uint32_t)umma::desc_kmajor(umma::smem_u32(sm + C::OFF_A2), C::TILE);
  const uint32_t ring16 = umma::smem_u32(sm + C::OFF_RING) >> 4;
  uint4 e = slt[0];
  constexpr int NG1 = C::NC * C::KS1;
  constexpr uint32_t ABLK16 = C::ABLK / 16;
#pragma unroll 1
  for (uint32_t pr = 0; pr < nprod; pr++) {
#pragma unroll 1
    for (int seg = 0; seg < 2 * C::NT; seg++) {  // G1 per tile, then G2 per tile
    const int gm = seg / C::NT, tt = seg % C::NT;
    const int i0 = gm ? NG1 : 0, i1 = gm ? C::NSLICE : NG1;
    e = slt[i0];
#pragma unroll 1
    for (int i = i0; i < i1; i++) {
      const uint4 cur = e;
      e = slt[i + 1 < i1 ? i + 1 : i0];  // prefetch the next entry
      const uint32_t f = cur.w;
      if (f & (kFGemm | kFChunk)) {
        if (kWaitCompute && (f & kFGemm)) {
          umma::mbar_wait((f & kFG2 ? a2 : a1) + 2 * tt, pr & 1);
          umma::tmem_fence_after();
        }
        if (kWaitCompute && (f & kFChunk) && dcnt >= (uint32_t)C::NB) {
          umma::mbar_wait(dfree + dbi, dph ^ 1);
          umma::tmem_fence_after();
        }
      }
      if (kRing && (f & kFStage)) umma::mbar_wait(full + cslot, cph);
      if (kMma) {
        const uint64_t ad = ((uint64_t)hi << 32) | (uint64_t)((f & kFG2 ? a2lo : a1lo) + tt * ABLK16 + cur.x);
        const uint64_t bd =
            ((uint64_t)hi << 32) | (uint64_t)(((ring16 + cslot * (C::SLOT / 16) + (cur.y & 0xFFFFu)) & 0x3FFFu) | (cur.y & 0xFFFF0000u));
        mma_elect(tm + dbi * C::BUFC, ad, bd, cur.z, f & kFAcc);
      }
      if (f & (kFStageEnd | kFChunkEnd)) {
        if (f & kFStageEnd) {
          if (DBG == 3) {
            if ((threadIdx.x & 31) == 0) umma::mbar_arrive(empty + cslot);
            __syncwarp();
          } else if (kRing) {
            if (cl == 2) commit_elect_mc(empty + cslot, 0x3);  // the slot is shared by the CTA pair
            else commit_elect(empty + cslot);
          }
          if (++cslot == (uint32_t)C::NSTAGE) { cslot = 0; cph ^= 1; }
        }
        if (f & kFChunkEnd) {
          commit_elect(dfull + dbi);
          dcnt++;
          if (++dbi == (uint32_t)C::NB) { dbi = 0; dph ^= 1; }
        }
      }
    }
    }
  }
  if (!kWaitCompute && nprod) umma::mbar_wait(dfull + (dbi + C::NB - 1) % C::NB, (dbi == 0) ? dph ^ 1 : dph);
}

template <class C>
__global__ void __launch_bounds__(C::NTHR, 1) rnsx_kernel(const __grid_constant__ XArgs P) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bars + 3 * C::NSTAGE + 2 * C::NB + 2 * C::NT);
  for (uint32_t o = tid * 16; o < (uint32_t)(C::NT * C::ABLK); o += C::NTHR * 16)
    *reinterpret_cast<uint4*>(sm + C::OFF_A1 + o) = make_uint4(0, 0, 0, 0);
  for (int o = tid; o < C::K * 3; o += C::NTHR) reinterpret_cast<uint4*>(sm + C::OFF_CONS)[o] = P.cons[o];
  for (int o = tid; o < 4 * C::NSLICE + 2 * C::NSTG; o += C::NTHR)
    reinterpret_cast<uint32_t*>(sm + C::OFF_SLT)[o] = P.slt[o];
  if (warp == C::NCW) {
    if (C::CG == 2) umma::tmem_alloc_cg2<C::TMC>(tbase);
    else umma::tmem_alloc<C::TMC>(tbase);
  }
  if (tid == 0) {
    const int cn = C::CG == 2 ? 1 : P.cl;  // empty: multicast commits (one per CTA for cluster multicast)
    for (int i = 0; i < C::NSTAGE; i++) umma::mbar_init(bars + i, 1);                  // full
    for (int i = 0; i < C::NSTAGE; i++) umma::mbar_init(bars + C::NSTAGE + i, cn);     // empty
    for (int i = 0; i < C::NB; i++) umma::mbar_init(bars + 2 * C::NSTAGE + i, 1);      // dfull
    // dfree / A-tile hand-offs: every compute warp of the CTA (of both CTAs at the pair leader)
    for (int i = 0; i < C::NB + 2 * C::NT; i++) umma::mbar_init(bars + 2 * C::NSTAGE + C::NB + i, C::NCW * C::CG);
    for (int i = 0; i < C::NSTAGE; i++) umma::mbar_init(bars + 2 * C::NSTAGE + 2 * C::NB + 2 * C::NT + i, 1);  // pfull
  }
  umma::fence_async_smem();
  umma::tmem_fence_before();
  __syncthreads();
  if (P.cl == 2) umma::cluster_sync();  // the peer's barriers exist before any multicast lands
  umma::tmem_fence_after();
  const uint32_t tm = *tbase;
  // uniform step plan: [pre0] pre1 | x^2 | table (ntab-1) | main (nops-1) | final
  const int npre = P.mode == kRxPow ? 1 : 2;
  const int s_x2 = npre, s_tab = s_x2 + 1, s_main = s_tab + (P.ntab - 1);
  int s_fin = s_main + (P.nops - 1);
  if (P.mode == kRxPowVar) s_fin = 16 + 5 * (P.nops - 1);  // 2 pre + 14 table + 5 per window after the top
  const int nsteps = P.mode == kRxProg ? P.prog.nsteps : s_fin + 1;
  const int ntiles = (P.count + C::TILE - 1) / C::TILE;
  // units (tiles, or tile pairs when NT == 2) of this CTA: u = blockIdx.x + k gridDim.x; within a
  // cluster every CTA runs the count of its rank-0 CTA (the other one runs dead tiles at the tail)
  const int units = P.mode == kRxProg ? ntiles : (ntiles + C::NT - 1) / C::NT;
  const int b0 = P.cl == 2 ? (int)(blockIdx.x & ~1u) : (int)blockIdx.x;
  const int mine = b0 < units ? (units - 1 - b0) / (int)gridDim.x + 1 : 0;
  if (warp >= C::NCW) {
    // role warpgroup hands registers to the compute warps (CTA pool: 4 x 64 x 32 = 16 x 16 x 32)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
    const uint32_t np = (uint32_t)(mine * nsteps);
    const uint32_t rank = P.cl == 2 ? umma::cluster_ctarank() : 0;
    if (C::CG == 2) {
      if (warp == C::NCW) {
        if (rank == 0) mma_pair<C>(sm, tm, bars, np);
        else relay_pair<C>(bars, np, lane);
      }
    } else if (warp == C::NCW) {
      if (P.dbg == 0) mma_fast<C>(sm, tm, bars, np, P.cl);
      else if (P.dbg == 5 || P.dbg == 6) mma_fast<C, false>(sm, tm, bars, np, P.cl);
      else if (P.dbg == 1) mma_role<C, 1>(sm, tm, bars, np, P.cl);
      else if (P.dbg == 3 || P.dbg == 7) mma_role<C, 3>(sm, tm, bars, np, P.cl);
      else if (P.dbg == 4 || P.dbg == 8) mma_role<C, 4>(sm, tm, bars, np, P.cl);
    }
    if (warp >= C::NCW + 1 && warp <= C::NCW + kRxProducers && P.dbg != 2 && P.dbg != 4 && P.dbg != 8) {
      const int npw = P.nprod > 0 && P.nprod <= kRxProducers ? P.nprod : kRxProducers;
      if (warp - C::NCW - 1 < npw)
        producer_role<C>(C::CG == 2 ? P.wimg2 : P.wimg, P.wimg_stride, sm, bars, np, lane, P.cl, rank,
                         warp - C::NCW - 1, npw, (P.dbg == 0 || P.dbg == 5 || P.dbg == 6) && C::CG == 1);
    }
    __syncwarp();
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    Thr<C> T;
    T.sm = sm;
    const int qd = warp & 3;
    T.g = warp >> 2;
    T.lane = lane;
    T.e = qd * 32 + lane;
    T.tl = tm + ((uint32_t)(qd * 32) << 16);
#if PCB_RNSX_KCONS
    T.rc = P.kcons + T.g * C::RPT * 3;
#else
    T.rc = reinterpret_cast<const uint4*>(sm + C::OFF_CONS) + T.g * C::RPT * 3;
#endif
    T.cthr = 0.0f;
    for (int w = 0; w < C::RPT; w++) T.cthr = __fmaf_rn(8388608.0f, __uint_as_float(T.rc[w * 3 + 2].y), T.cthr);
    T.NT = gridDim.x * C::NCT;
    T.gt = blockIdx.x * C::NCT + tid;
    T.dbi = 0;
    T.dph = 0;
    T.nowait = P.dbg == 2 || P.dbg >= 6;
    // beta of element e sums the partials of the 4 prime groups, i.e. of the 4 warps that share
    // e's TMEM lane quadrant: a 128-thread named barrier per quadrant (ids 2..5) lets the
    // quadrants run apart instead of all 16 compute warps meeting every product
    T.bar_id = P.qbar ? 2u + (uint32_t)qd : 1u;
    T.bar_n = P.qbar ? 128u : (uint32_t)C::NCT;
    if constexpr (C::CG == 2) T.rank = umma::cluster_ctarank();
    else T.rank = 0;
    T.dfull = bars + 2 * C::NSTAGE;
    T.dfree = T.dfull + C::NB;
    T.a1 = T.dfree + C::NB;
    T.a2 = T.a1 + 1;
    if (P.dbg == 0 || P.dbg == 2 || P.dbg >= 6) compute_role<C>(P, T, mine, nsteps, npre, s_x2, s_tab, s_main, s_fin);
  }
  umma::tmem_fence_before();
  __syncthreads();
  if (P.cl == 2) umma::cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == C::NCW) {
    if (C::CG == 2) umma::tmem_dealloc_cg2<C::TMC>(tm);
    else umma::tmem_dealloc<C::TMC>(tm);
  }
}

// Exact conversion of the B' residues to the binary residue mod N (one thread per element):
//   xi'_j = REDC(x~'_j C4_j) fully reduced,  r = sum_j xi'_j M'_j - beta M',  y = r mod N.
struct XOutArgs {
  const uint32_t* res;
  uint32_t* y;
  const int32_t* skip;  // rows with skip[el] != 0 are left untouched (argument errors)
  const uint32_t* tabs;  // mod[K] minv[K] c4[K] invp[2K] mpj[K][mpw] mp[mpw] n[S]
  int count, K, mpw, S;
  double ntop;
  int ntw;  // word index of the lower of N's two top words (ntop = N / 2^(32 ntw))
};

__global__ void rnsx_out_kernel(const __grid_constant__ XOutArgs P) {
  constexpr int WMAX = 140;
  const int K = P.K, W = P.mpw, S_ = P.S;
  const uint32_t* mod = P.tabs;
  const uint32_t* minv = mod + K;
  const uint32_t* c4 = minv + K;
  const double* invp = reinterpret_cast<const double*>(c4 + K);
  const uint32_t* mpj = c4 + 3 * K;
  const uint32_t* mp = mpj + (size_t)K * W;
  const uint32_t* nn = mp + W;
  for (int el = blockIdx.x * blockDim.x + threadIdx.x; el < P.count; el += gridDim.x * blockDim.x) {
    if (P.skip && P.skip[el] != 0) continue;
    const uint32_t* res = P.res + (size_t)el * K;
    uint32_t r[WMAX + 2];
    for (int w = 0; w < W + 2; w++) r[w] = 0;
    double S = 0.0;
    for (int j = 0; j < K; j++) {
      const uint32_t m = mod[j], mi = minv[j];
      uint32_t xp = redc((uint64_t)res[j] * c4[j], m, mi);
      if (xp >= m) xp -= m;
      S += (double)xp * invp[j];
      const uint32_t* Mj = mpj + (size_t)j * W;
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
    {
      int64_t br = 0;
      uint64_t carry = 0;
      for (int w = 0; w < W + 2; w++) {
        const uint64_t pr = (uint64_t)beta * (w < W ? mp[w] : 0u) + carry;
        carry = pr >> 32;
        const int64_t d = (int64_t)r[w] - (int64_t)(uint32_t)pr - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    double rt = 0.0;
    for (int w = W + 1; w >= P.ntw; w--) rt = rt * 4294967296.0 + (double)r[w];
    const double qd = floor(rt / P.ntop) - 1.0;
    const uint32_t q = qd > 0 ? (uint32_t)qd : 0u;
    if (q) {
      int64_t br = 0;
      uint64_t carry = 0;
      for (int w = 0; w < W + 2; w++) {
        const uint64_t pr = (uint64_t)q * (w < S_ ? nn[w] : 0u) + carry;
        carry = pr >> 32;
        const int64_t d = (int64_t)r[w] - (int64_t)(uint32_t)pr - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    for (int it = 0; it < 8; it++) {  // r < 4 N here for valid residues; bounded for safety
      int cmp = 0;
      for (int w = W + 1; w >= 0 && cmp == 0; w--) {
        const uint32_t a = r[w], b = w < S_ ? nn[w] : 0u;
        cmp = a > b ? 1 : (a < b ? -1 : 0);
      }
      if (cmp < 0) break;
      int64_t br = 0;
      for (int w = 0; w < W + 2; w++) {
        const int64_t d = (int64_t)r[w] - (int64_t)(w < S_ ? nn[w] : 0u) - br;
        r[w] = (uint32_t)d;
        br = d < 0;
      }
    }
    uint32_t* y = P.y + (size_t)el * S_;
    for (int w = 0; w < S_; w++) y[w] = r[w];
  }
}

template <class C>
pcb_status launch_cfg(const RnsXModulus& md, int mode, const uint8_t* ops, int nops, int ntab, const uint32_t* x,
                      int x_words, const uint32_t* m, int m_words, size_t count, uint32_t* y, cudaStream_t st,
                      double alg_mac32, const RxProg* prog = nullptr, const int32_t* skip = nullptr) {
  XArgs P;
  if (prog) P.prog = *prog;
  P.wimg = md.d_wimg;
  P.wimg2 = md.d_wimg2;
  P.wimg_stride = md.wimg_stride;
  P.cons = md.d_cons;
#if PCB_RNSX_KCONS
  if (md.h_cons.size() > sizeof(P.kcons) / 4) return PCB_E_SHAPE;
  memcpy(P.kcons, md.h_cons.data(), md.h_cons.size() * 4);
#endif
  P.cvec = reinterpret_cast<const uint32_t*>(md.d_cvec);
  P.slt = md.d_slt;
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
  {
    const char* d = getenv("PCB_RNSX_DBG");
    P.dbg = d ? atoi(d) : 0;
    const char* np = getenv("PCB_RNSX_NPROD");
    P.nprod = np ? atoi(np) : 0;
    const char* qb = getenv("PCB_RNSX_QBAR");
    P.qbar = qb ? atoi(qb) : 1;
  }
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  // The >48 KB dynamic-smem opt-in is a per-device function attribute: remember it per device
  // (bit dev of an atomic mask), so a second context on another device, or another host
  // thread, never launches without it.  Setting it twice is harmless.
  static std::atomic<uint64_t> attr_dev{0};
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_dev.load(std::memory_order_acquire) & bit)) {
    if (cudaFuncSetAttribute(rnsx_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) != cudaSuccess)
      return PCB_E_CUDA;
    attr_dev.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int ntiles = (int)((count + C::TILE - 1) / C::TILE);
  const int units = mode == kRxProg ? ntiles : (ntiles + C::NT - 1) / C::NT;
  // PCB_RNSX_CL=2: CTA pairs share the W stream (cluster multicast, each CTA fetches half of
  // every stage).  Measured slower on B200 (K = 144 public Enc 277 K/s vs 305 K/s): with clusters
  // of 2 the multicast does not cut the L2 -> SM traffic each SM receives, which is the bound; kept
  // opt-in for the record (profiles/r01_rnsx_cluster_multicast.txt).
  const char* clv = getenv("PCB_RNSX_CL");
  int cl = clv ? atoi(clv) : 1;
  if (cl != 2 || units < 2 || P.dbg != 0) cl = 1;
  if (C::CG == 2) cl = 2;  // a CTA pair always (a single tile runs with a dead peer)
  P.cl = cl;
  int blocks = units < nsm ? units : nsm;
  if (cl == 2) blocks = std::min((units + 1) & ~1, nsm & ~1);
  {
    // PCB_RNSX_NP (A/B): bit 0 = step programs, bit 1 = every other mode, launched one unit per
    // CTA (grid = units) instead of persistent: the block scheduler then hands SMs freed by a
    // concurrent kernel (another stream) to whichever CTAs are pending, instead of a static
    // blockIdx + k gridDim split that waits for the slowest SM.
    const char* npv = getenv("PCB_RNSX_NP");
    const int np = npv ? atoi(npv) : 0;
    if (cl == 1 && (np & (mode == kRxProg ? 1 : 2))) blocks = units;
  }
  const size_t nthr = (size_t)blocks * C::NCT;
  pcb_status e = PCB_OK;
  P.tab = nullptr;
  if (mode != kRxProg) e = scratch_alloc(nthr * (size_t)(ntab + 2) * C::NT * C::NV * 4 * 4, (void**)&P.tab, st);
  uint32_t* res = nullptr;
  if (!e && y) e = scratch_alloc(count * C::K * 4, (void**)&res, st);
  P.out = res;
  if (!e) {
    ProfMark pm;
    if (prof_enabled()) pm = prof_start(st);
    if (cl == 2) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(blocks);
      lc.blockDim = dim3(C::NTHR);
      lc.dynamicSmemBytes = C::SMEM;
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      cudaLaunchKernelEx(&lc, rnsx_kernel<C>, P);
    } else {
      rnsx_kernel<C><<<blocks, C::NTHR, C::SMEM, st>>>(P);
    }
    count_launch();
    if (prof_enabled()) {
      prof_stop(pm, st, alg_mac32 * (double)count);
      double mps = 0;  // int8 MACs per tile-product: every slice is an M = 128 x N = ncol x K = 32 MMA
      for (int c = 0; c < C::NC; c++) mps += (double)C::TILE * C::ncol(c) * 32 * (C::KS1 + C::KS2);
      const int nsteps = mode == kRxProg ? prog->nsteps
                         : mode == kRxPowVar ? 17 + 5 * (nops - 1) : (mode == kRxPow ? 1 : 2) + ntab + nops;
      prof_add_int8(mps * nsteps * (double)(units * C::NT));
    }
    const cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) fprintf(stderr, "rnsx_kernel<K=%d>: %s\n", C::K, cudaGetErrorString(ce));
    e = cuda_check(ce);
  }
  if (!e && P.dbg == 0 && y) {
    XOutArgs O;
    O.res = res;
    O.y = y;
    O.skip = skip;
    O.tabs = md.d_out;
    O.count = (int)count;
    O.K = md.K;
    O.mpw = md.mpw;
    O.S = md.S;
    O.ntop = md.ntop;
    O.ntw = md.ntw;
    const int grid = (int)((count + 127) / 128 < 4096 ? (count + 127) / 128 : 4096);
    rnsx_out_kernel<<<grid, 128, 0, st>>>(O);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  scratch_free(P.tab, st);
  scratch_free(res, st);
  return e;
}

// ------------------------------------------------------------------------------------------
// Host: constants for one modulus
// ------------------------------------------------------------------------------------------
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

uint32_t big_mod(const HBN& x, uint32_t m) {
  uint64_t r = 0;
  for (size_t i = x.w.size(); i-- > 0;) r = ((r << 32) | x.w[i]) % m;
  return (uint32_t)r;
}

// in-place kmajor layout of an R x 32-byte slice
inline size_t slice_off(int r, int k, int R) { return (size_t)(k >> 4) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15); }

}  // namespace

bool rnsx_shape(int bits, int* K) {
  // 30-bit primes; M > (2K+2)^2 N and M' > 2^24 (2K+2) N (checked in rnsx_build)
  if (bits <= 2048) { *K = 72; return true; }
  if (bits <= 3072) { *K = 112; return true; }
  if (bits <= 4096) { *K = 144; return true; }
  return false;
}

bool rnsx_build(const HBN& N, const HBN& n, int S, int K, RnsXModulus* out) {
  if (N.bit_length() > (size_t)(32 * S) || !N.is_odd() || K <= 0 || K > 144) return false;
  const int G = 4, NC = rnsx_nchunks(K);
  for (int c = 0; c < NC; c++)
    if (rnsx_chunk_primes(K, c) % 8) return false;
  auto ptc = [&](int c) { return rnsx_chunk_primes(K, c) / G; };
  const int RPT = K / G, NQ = (RPT + 3) / 4, NV = 2 * NQ;
  // thread-local residue w of thread group g <-> prime index
  auto prime_of = [&](int g, int w) {
    int c = 0;
    while (w >= rnsx_chunk_first(K, c + 1) / G && c + 1 < NC) c++;
    const int t = w - rnsx_chunk_first(K, c) / G;
    return rnsx_chunk_first(K, c) + rnsx_slot(ptc(c), g, t / 4) + t % 4;
  };
  std::vector<uint32_t> pr;
  for (uint32_t c = (1u << 30) - 1; pr.size() < 2 * (size_t)K; c -= 2)
    if (is_prime32(c)) pr.push_back(c);
  const uint32_t* B = pr.data();
  const uint32_t* Bp = pr.data() + K;
  HBN M(1), Mp(1);
  for (int l = 0; l < K; l++) {
    M = M * HBN(B[l]);
    Mp = Mp * HBN(Bp[l]);
  }
  // correctness margins (oracle/rns_oracle.py): M > (2K+2)^2 N, M' > 2^24 (2K+2) N
  const HBN kk((uint64_t)(2 * K + 2));
  if (!(M > kk * kk * N) || !(Mp > (kk * N << 24))) return false;
  std::vector<uint32_t> pm(2 * K), minv(2 * K), one(2 * K), q64(2 * K);
  const uint64_t two32 = 1ull << 32;
  for (int q = 0; q < 2 * K; q++) {
    const uint32_t m = pr[q];
    if (big_mod(N, m) == 0) return false;
    uint32_t inv = 1;
    for (int it = 0; it < 5; it++) inv *= 2u - m * inv;
    pm[q] = m;
    minv[q] = (uint32_t)(0u - inv);
    one[q] = (uint32_t)(two32 % m);
    q64[q] = (uint32_t)((uint64_t)one[q] * one[q] % m);
  }
  auto mprod_mod = [&](const uint32_t* base, int skip, uint32_t m) {
    uint64_t r = 1;
    for (int l = 0; l < K; l++)
      if (l != skip) r = r * (base[l] % m) % m;
    return (uint32_t)r;
  };
  std::vector<uint32_t> c1(K), c2(K), c3(K), c4(K);
  std::vector<double> invp(K);
  for (int i = 0; i < K; i++) {
    const uint32_t m = B[i];
    const uint64_t ninv = inv_mod(big_mod(N, m), m), miinv = inv_mod(mprod_mod(B, i, m), m);
    c1[i] = (uint32_t)((m - ninv) % m * miinv % m);
  }
  for (int j = 0; j < K; j++) {
    const uint32_t m = Bp[j];
    const uint64_t minvM = inv_mod(big_mod(M, m), m), o = one[K + j];
    c2[j] = (uint32_t)(minvM * o % m);
    c3[j] = (uint32_t)((uint64_t)big_mod(N, m) * minvM % m * q64[K + j] % m);
    c4[j] = inv_mod(mprod_mod(Bp, j, m), m);
    invp[j] = 1.0 / (double)m;
  }
  // constant records per (g, w): {m, minv, c1, q64} {m', minv', c2, c3} {c4, f32(2^8 / m'), 0, q64'}
  std::vector<uint32_t> cons((size_t)G * RPT * 12);
  for (int g = 0; g < G; g++)
    for (int w = 0; w < RPT; w++) {
      const int i = prime_of(g, w);
      const float inv8 = (float)(256.0 / (double)Bp[i]);
      uint32_t fb;
      memcpy(&fb, &inv8, 4);
      const uint32_t rec[12] = {B[i], minv[i], c1[i], q64[i], Bp[i], minv[K + i], c2[i], c3[i], c4[i], fb, 0u, q64[K + i]};
      memcpy(&cons[((size_t)g * RPT + w) * 12], rec, sizeof rec);
    }
  // constant operand vectors in thread order: [id][g][v][4]
  auto to_res = [&](const HBN& v, std::vector<uint32_t>& dst) {
    dst.resize(2 * K);
    for (int q = 0; q < 2 * K; q++) dst[q] = (uint32_t)((uint64_t)big_mod(v, pr[q]) * one[q] % pr[q]);
  };
  std::vector<uint32_t> vecs[kRxNumVec];
  vecs[kRxOne] = one;  // 1 in lazy Montgomery form: 2^32 mod m
  const HBN M2 = mod(M * M, N);
  to_res(M2, vecs[kRxR2N]);
  to_res(mod(M2 << (size_t)(32 * S), N), vecs[kRxCR2N]);
  to_res(mod(mod(n, N) * mod(M, N), N), vecs[kRxNM]);
  to_res(mod(M, N), vecs[kRxOneM]);
  std::vector<uint32_t> cvec((size_t)kRxNumVec * G * NV * 4, 0);
  for (int id = 0; id < kRxNumVec; id++)
    for (int g = 0; g < G; g++)
      for (int v = 0; v < NV; v++)
        for (int t = 0; t < 4; t++) {
          const int w = (v < NQ ? v : v - NQ) * 4 + t;
          if (w >= RPT) continue;
          const int i = prime_of(g, w);
          cvec[(((size_t)id * G + g) * NV + v) * 4 + t] = vecs[id][v < NQ ? i : K + i];
        }
  // base-extension stream: GEMM-1 slices (chunk, k-step), then GEMM-2 slices; slice of chunk c is
  // ncol(c) rows x 32 bytes in the K-major core-matrix layout (R = ncol(c))
  const int K1 = 4 * K, K2 = 4 * K + 32, KS1 = K1 / 32, KS2 = K2 / 32;
  std::vector<uint32_t> W1((size_t)K * K), W2((size_t)K * (K + 1));
  // W1'_ji = M_i C3_j mod m'_j: the GEMM-1 epilogue's REDC(qh C3) folded into the matrix (rx_e1)
  for (int j = 0; j < K; j++)
    for (int i = 0; i < K; i++) W1[(size_t)j * K + i] = (uint32_t)((uint64_t)mprod_mod(B, i, Bp[j]) * c3[j] % Bp[j]);
  for (int i = 0; i < K; i++) {
    const uint32_t m = B[i];
    for (int j = 0; j < K; j++) W2[(size_t)i * (K + 1) + j] = (uint32_t)((uint64_t)mprod_mod(Bp, j, m) * q64[i] % m);
    W2[(size_t)i * (K + 1) + K] = (uint32_t)((m - (uint64_t)big_mod(Mp, m) * q64[i] % m) % m);
  }
  std::vector<uint8_t> img, img2;  // img2: every slice as two halves (rows [0, N/2), [N/2, N)), R = N/2 each
  std::vector<uint32_t> slt, soff;  // slice offsets in the image (16-byte units)
  for (int gm = 0; gm < 2; gm++) {
    const int ks = gm ? KS2 : KS1;
    for (int c = 0; c < NC; c++) {
      const int pt = ptc(c), ncol = 16 * pt;
      for (int s = 0; s < ks; s++) {
        const size_t off = img.size();
        img.resize(off + (size_t)ncol * 32, 0);
        img2.resize(off + (size_t)ncol * 32, 0);
        soff.push_back((uint32_t)(off / 16));
        uint8_t* dst = img.data() + off;
        for (int nl = 0; nl < ncol; nl++) {
          // column nl of the chunk: thread group g, quad j, byte b, prime t within the quad
          // (full quads of 4 primes = 16 columns first; a ragged chunk's last quad may hold 2)
          const int g = nl / (4 * pt), r = nl % (4 * pt), j = r / 16, qt = pt - 4 * j < 4 ? pt - 4 * j : 4,
                    b = (r - 16 * j) / qt, t = (r - 16 * j) % qt;
          const int o = rnsx_chunk_first(K, c) + rnsx_slot(pt, g, j) + t;  // output prime (B' for GEMM 1, B for GEMM 2)
          const uint32_t m = gm ? B[o] : Bp[o];
          for (int kk2 = 0; kk2 < 32; kk2++) {
            const int k = 32 * s + kk2, src = k / 4, a = k % 4;
            uint64_t base;
            if (gm == 0)
              base = W1[(size_t)o * K + src];
            else
              base = src <= K ? W2[(size_t)o * (K + 1) + src] : 0;
            const uint32_t v = (uint32_t)((base << (8 * a)) % m);
            dst[slice_off(nl, kk2, ncol)] = (uint8_t)(v >> (8 * b));
            const int hn = ncol / 2, hh = nl / hn;
            img2[off + (size_t)hh * hn * 32 + slice_off(nl - hh * hn, kk2, hn)] = (uint8_t)(v >> (8 * b));
          }
        }
      }
    }
  }
  {  // slice table (role-warp program) and stages of SPS consecutive slices (contiguous in the image)
    const int SPS = sps_for(K), nsl = (int)soff.size(), nst = (nsl + SPS - 1) / SPS;
    int sl = 0;
    for (int gm = 0; gm < 2; gm++) {
      const int ks = gm ? KS2 : KS1;
      for (int c = 0; c < NC; c++) {
        const int ncol = 16 * ptc(c);
        for (int s2 = 0; s2 < ks; s2++, sl++) {
          uint32_t f = 0;
          if (c == 0 && s2 == 0) f |= 1u;                  // kFGemm
          if (gm) f |= 2u;                                 // kFG2
          if (s2 == 0) f |= 4u;                            // kFChunk
          if (s2 == ks - 1) f |= 8u;                       // kFChunkEnd
          if (sl % SPS == 0) f |= 16u;                     // kFStage
          if (sl % SPS == SPS - 1 || sl == nsl - 1) f |= 32u;  // kFStageEnd
          if (s2 > 0) f |= 64u;                            // kFAcc
          const uint32_t rel16 = soff[sl] - soff[sl - sl % SPS];
          slt.push_back((uint32_t)(s2 * (2 * 128 * 16 / 16)));        // A k-step offset (16 B units)
          slt.push_back(rel16 | ((uint32_t)ncol << 16));             // B offset in the slot | LBO field
          slt.push_back((2u << 4) | ((uint32_t)(ncol >> 3) << 17) | ((uint32_t)(128 >> 4) << 24));  // idesc i8
          slt.push_back(f);
        }
      }
    }
    for (int t = 0; t < nst; t++) {
      const int f = t * SPS, l = std::min(nsl, f + SPS);
      const size_t end = l < nsl ? (size_t)soff[l] * 16 : img.size();
      slt.push_back(soff[f]);
      slt.push_back((uint32_t)(end - (size_t)soff[f] * 16));
    }
  }
  // output conversion tables
  RnsXModulus md;
  md.K = K;
  md.S = S;
  md.mpw = (int)((Mp.bit_length() + 31) / 32);
  if (md.mpw > 138) return false;
  std::vector<uint32_t> otab((size_t)5 * K + (size_t)K * md.mpw + md.mpw + S, 0);
  for (int j = 0; j < K; j++) {
    otab[j] = Bp[j];
    otab[K + j] = minv[K + j];
    otab[2 * K + j] = c4[j];
    memcpy(&otab[3 * K + 2 * j], &invp[j], 8);
    HBN q, r;
    divmod(Mp, HBN(Bp[j]), q, r);
    q.to_limbs(otab.data() + 5 * K + (size_t)j * md.mpw, md.mpw);
  }
  Mp.to_limbs(otab.data() + 5 * K + (size_t)K * md.mpw, md.mpw);
  N.to_limbs(otab.data() + 5 * K + (size_t)K * md.mpw + md.mpw, S);
  // the quotient estimate of the output conversion uses N's two TOP words (N may be much narrower
  // than S words, e.g. p^2 of a toy key): ntop = N / 2^(32 ntw)
  double nt = 0.0;
  const std::vector<uint32_t> nl = N.limbs(S);
  const int top = (int)((N.bit_length() + 31) / 32) - 1;
  md.ntw = top > 0 ? top - 1 : 0;
  for (int w = top; w >= md.ntw; w--) nt = nt * 4294967296.0 + (double)nl[w];
  md.ntop = nt;
  md.wimg_stride = (img.size() + 4095) & ~(size_t)4095;
  bool ok = cudaMalloc(&md.d_wimg, md.wimg_stride * kRxReplicas) == cudaSuccess;
  ok = ok && cudaMalloc(&md.d_wimg2, md.wimg_stride * kRxReplicas) == cudaSuccess;
  ok = ok && cudaMalloc(&md.d_cons, cons.size() * 4) == cudaSuccess;
  ok = ok && cudaMalloc(&md.d_cvec, cvec.size() * 4) == cudaSuccess;
  ok = ok && cudaMalloc(&md.d_out, otab.size() * 4) == cudaSuccess;
  ok = ok && cudaMalloc(&md.d_slt, slt.size() * 4) == cudaSuccess;
  for (int r = 0; r < kRxReplicas; r++)
    ok = ok && cudaMemcpy(md.d_wimg + r * md.wimg_stride, img.data(), img.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(md.d_wimg2 + r * md.wimg_stride, img2.data(), img2.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(md.d_cons, cons.data(), cons.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  md.h_cons = cons;
  ok = ok && cudaMemcpy(md.d_cvec, cvec.data(), cvec.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(md.d_out, otab.data(), otab.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(md.d_slt, slt.data(), slt.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    rnsx_free(&md);
    return false;
  }
  md.ok = true;
  *out = md;
  return true;
}

void rnsx_free(RnsXModulus* md) {
  if (md->d_wimg) cudaFree(md->d_wimg);
  if (md->d_wimg2) cudaFree(md->d_wimg2);
  md->d_wimg2 = nullptr;
  if (md->d_cons) cudaFree(md->d_cons);
  if (md->d_cvec) cudaFree(md->d_cvec);
  if (md->d_out) cudaFree(md->d_out);
  if (md->d_slt) cudaFree(md->d_slt);
  md->d_slt = nullptr;
  md->d_wimg = nullptr;
  md->d_cons = nullptr;
  md->d_cvec = nullptr;
  md->d_out = nullptr;
  md->ok = false;
}

int rnsx_rec_words(const RnsXModulus& md) {
  const int RPT = md.K / 4;
  return 4 * 2 * ((RPT + 3) / 4) * 4;
}

pcb_status launch_rnsx_prog(const RnsXModulus& md, const RxProg& prog, const uint32_t* x, int x_words, size_t count,
                            uint32_t* y, cudaStream_t st, double alg_mac32) {
  if (count == 0) return PCB_OK;
  if (!md.ok || prog.nsteps < 1 || prog.nsteps > kRxMaxSteps) return PCB_E_UNSUPPORTED;
  {
    const char* cgv = getenv("PCB_RNSX_CG2");
    if (cgv && atoi(cgv) != 0) {
      if (md.K == 144) return launch_cfg<Cfg<144, 1, 2>>(md, kRxProg, nullptr, 0, 0, x, x_words, nullptr, 0, count, y, st, alg_mac32, &prog);
      if (md.K == 112) return launch_cfg<Cfg<112, 1, 2>>(md, kRxProg, nullptr, 0, 0, x, x_words, nullptr, 0, count, y, st, alg_mac32, &prog);
    }
  }
#define PCB_RX(KK)                                                                                                 \
  if (md.K == KK) return launch_cfg<Cfg<KK>>(md, kRxProg, nullptr, 0, 0, x, x_words, nullptr, 0, count, y, st, alg_mac32, &prog);
  PCB_RX(72)
  PCB_RX(112)
  PCB_RX(144)
#undef PCB_RX
  return PCB_E_UNSUPPORTED;
}

pcb_status launch_rnsx(const RnsXModulus& md, int mode, const uint8_t* ops, int nops, int ntab, const uint32_t* x,
                       int x_words, const uint32_t* m, int m_words, size_t count, uint32_t* y, cudaStream_t st,
                       double alg_mac32, const int32_t* skip) {
  if (count == 0) return PCB_OK;
  if (!md.ok) return PCB_E_UNSUPPORTED;
#define PCB_RX(KK)                                                                                                 \
  if (md.K == KK) return launch_cfg<Cfg<KK>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
  {
    const char* cgv = getenv("PCB_RNSX_CG2");
    if (cgv && atoi(cgv) != 0) {
      if (md.K == 144) return launch_cfg<Cfg<144, 1, 2>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
      if (md.K == 112) return launch_cfg<Cfg<112, 1, 2>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
    }
  }
  if (md.K == 72 || md.K == 40 || md.K == 56) {  // two tiles in flight per CTA (the K <= 72 register budget allows it)
    const char* ppv = getenv("PCB_RNSX_PP");
    const bool pp = !ppv || atoi(ppv) != 0;  // default on; PCB_RNSX_PP=0 runs one tile per CTA
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const char* p3v = getenv("PCB_RNSX_NT3");
    if (pp && md.K == 40 && p3v && atoi(p3v) != 0 && count >= (size_t)nsm * 3 * 128)
      return launch_cfg<Cfg<40, 3>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
    // pairs only pay in latency once every SM has two tiles; background work (a low-priority
    // context) takes them anyway: half the SMs for ~1.3x the time leaves the rest to the critical path
    if (pp && (count >= (size_t)nsm * 2 * 128 || (md.prefer_pairs && count > 128))) {
      if (md.K == 72)
        return launch_cfg<Cfg<72, 2>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
      if (md.K == 56)
        return launch_cfg<Cfg<56, 2>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
      return launch_cfg<Cfg<40, 2>>(md, mode, ops, nops, ntab, x, x_words, m, m_words, count, y, st, alg_mac32, nullptr, skip);
    }
  }
  PCB_RX(40)
  PCB_RX(56)
  PCB_RX(72)
  PCB_RX(112)
  PCB_RX(144)
#undef PCB_RX
  return PCB_E_UNSUPPORTED;
}

}  // namespace pcb
