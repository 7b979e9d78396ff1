// side28.cu — the hot kernel on the carry-free radix-2^r core (mont28.cuh): one CRT half
// (one modulus) of a batch of Paillier exponentiations, same modes as side.cu:
//
//   ENC  y = (1 + m n mod m2) * r^e mod m2        (paillier.cpp:339-342, binomial g)
//   DEC  y = c^e mod m2                            (c^(p-1) form, paillier.cpp:357-358)
//   POW  y = x^e mod m2                            (ModArith::pow, paillier.cpp:26-30)
//
// A warp-uniform step machine around ONE Montgomery product site (keeps code size and register
// allocation under control; see side.cu).  TPI lanes share one residue.  Values stay in [0, 2m)
// (lazy reduction, R = 2^(rN) > 16m); one conditional subtraction at the very end.
#include <cstdint>
#include <cuda_runtime.h>

#include "mont.cuh"
#include "mont28.cuh"
#include "pcb_internal.h"

namespace pcb {

template <int RB, int N, int TPI>
struct Side28Args {
  static constexpr int W = (N * RB + 31) / 32;  // 32-bit words spanned by the limbs
  uint32_t mlimb[N];    // modulus, radix 2^r
  uint32_t mword[W];    // modulus, 32-bit words (final reduction)
  uint32_t r2[N];       // R^2 mod m (radix limbs)
  uint32_t c1[N];       // ENC: n R mod m   DEC: R^3 mod m
  uint32_t minv;        // -m^-1 mod 2^r
  int mwords;           // words of the modulus / outputs
  const uint8_t* ops;
  int nops, ntab;
  uint32_t* tab;        // per-lane table: ((e*K + j) * nlanes + lane)
  const uint32_t* x;    // ENC: r   DEC: c   POW: x   (x_words per element)
  int x_words;
  const uint32_t* m;    // ENC plaintexts (m_words per element)
  int m_words;
  const int32_t* skip;
  uint32_t* y;          // count x y_words
  int y_words;
  int count, mode;
};

#ifndef PCB_R28_MINB
#define PCB_R28_MINB 3
#endif
enum : int { kM28Enc = 0, kM28Dec = 1, kM28Pow = 2 };

template <int RB, int N, int TPI>
__global__ void __launch_bounds__(kThreadsPerBlock, (N / TPI > 40) ? 2 : PCB_R28_MINB) side28_kernel(const __grid_constant__ Side28Args<RB, N, TPI> P) {
  using Cf = r28::Cfg<RB, N, TPI>;
  constexpr int K = Cf::K, G = Cf::G;
  using Slot = r28::DSlot<RB, N, TPI>;
  extern __shared__ __align__(16) uint32_t smem[];
  // block-shared modulus limbs (lane t of a group reads limbs [tK, tK+K))
  for (int j = threadIdx.x; j < N; j += blockDim.x) smem[j] = P.mlimb[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane % TPI, grp = lane / TPI;
  const uint32_t mlane = (uint32_t)__cvta_generic_to_shared(smem) + t * K * 4;
  uint32_t* wbase = smem + ((N + 3) & ~3) + warp * (2 * N * G);
  const Slot Acc{(uint32_t)__cvta_generic_to_shared(wbase + grp)};
  const Slot Op{(uint32_t)__cvta_generic_to_shared(wbase + N * G + grp)};
  const uint32_t nlanes = gridDim.x * blockDim.x;
  const uint32_t gl = blockIdx.x * blockDim.x + threadIdx.x;
  auto tput = [&](int e, const uint32_t (&v)[K]) {
#pragma unroll
    for (int j = 0; j < K; j++) P.tab[(size_t)(e * K + j) * nlanes + gl] = v[j];
  };
  auto tget = [&](int e, uint32_t (&v)[K]) {
#pragma unroll
    for (int j = 0; j < K; j++) v[j] = P.tab[(size_t)(e * K + j) * nlanes + gl];
  };
  auto tslot = [&](int e, const Slot& s) {
#pragma unroll
    for (int j = 0; j < K; j++) s.set(t * K + j, P.tab[(size_t)(e * K + j) * nlanes + gl]);
  };
  auto cslot = [&](const Slot& s, const uint32_t* c) {  // constant radix limbs
#pragma unroll
    for (int j = 0; j < K; j++) s.set(t * K + j, c[t * K + j]);
  };
  const int park = P.ntab;
  const int npre = P.mode == kM28Pow ? 1 : 2;
  const int s_x2 = npre, s_tab = s_x2 + 1, s_main = s_tab + (P.ntab - 1), s_fin = s_main + (P.nops - 1);
  const int nsteps = s_fin + 1;
  const int groups_total = nlanes / TPI;

  for (int i = gl / TPI; i < P.count; i += groups_total) {
    if (P.skip && P.skip[i] != 0) continue;
    const uint32_t* xs = P.x + (size_t)i * P.x_words;
    uint32_t A[K];
#pragma unroll 1
    for (int s = 0; s < nsteps; s++) {
      bool b_is_acc = false;
      if (s < npre) {
        const bool first = s == 0 && npre == 2;
        if (P.mode == kM28Enc && first) {
          r28::words_to_limbs<RB, K>(A, P.m + (size_t)i * P.m_words, P.m_words, t * K);
          cslot(Op, P.c1);
        } else if (P.mode == kM28Dec && first) {  // c_hi = c >> rN
          // words_to_limbs with a bit offset of rN: limb j of c_hi = bits [rN + rj, ...)
          r28::words_to_limbs<RB, K>(A, xs, P.x_words, N + t * K);
          cslot(Op, P.c1);
        } else if (P.mode == kM28Dec) {  // c_lo = c mod 2^(rN)
          r28::words_to_limbs<RB, K>(A, xs, P.x_words, t * K);
          cslot(Op, P.r2);
        } else {
          r28::words_to_limbs<RB, K>(A, xs, P.x_words, t * K);
          cslot(Op, P.r2);
        }
      } else if (s == s_x2) {
        b_is_acc = true;
      } else if (s < s_main) {
        // table build: A = x^(2e-1) (registers), Op = x^2
      } else if (s < s_fin) {
        const uint8_t op = P.ops[s - s_main + 1];
        if (op == kOpSquare)
          b_is_acc = true;
        else
          tslot(op, Op);
      } else {
        if (P.mode == kM28Enc) {
          tslot(park, Op);
        } else {
#pragma unroll
          for (int j = 0; j < K; j++) Op.set(t * K + j, (t == 0 && j == 0) ? 1u : 0u);
        }
      }
      __syncwarp();
      uint32_t R[K];
      r28::mm<RB, N, TPI>(R, A, b_is_acc ? Acc : Op, mlane, P.minv, t);
      __syncwarp();
      if (s < npre) {
        const bool first = s == 0 && npre == 2;
        if (first) {
          if (P.mode == kM28Enc) {  // 1 + m n  (value <= 2m: still a valid lazy operand)
            uint64_t c = (t == 0) ? 1ull : 0ull;
#pragma unroll
            for (int j = 0; j < K; j++) {
              const uint64_t v = (uint64_t)R[j] + c;
              R[j] = (uint32_t)v & Cf::MASK;
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
                  R[j] = (uint32_t)v & Cf::MASK;
                  c = v >> RB;
                }
              }
            }
          }
          tput(park, R);
        } else {
          if (P.mode == kM28Dec) {  // c R = c_lo R + c_hi R^2  (< 4m: R > 16m keeps it lazy-valid)
            uint32_t H[K];
            tget(park, H);
            uint64_t c = 0;
#pragma unroll
            for (int j = 0; j < K; j++) {
              const uint64_t v = (uint64_t)R[j] + H[j] + c;
              R[j] = (uint32_t)v & Cf::MASK;
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
                  R[j] = (uint32_t)v & Cf::MASK;
                  c = v >> RB;
                }
              }
            }
          }
#pragma unroll
          for (int j = 0; j < K; j++) A[j] = R[j];
          Acc.store(R, t);
          tput(0, R);
        }
      } else if (s == s_x2) {
        Op.store(R, t);  // x^2 ; A still holds x
      } else if (s < s_main) {
#pragma unroll
        for (int j = 0; j < K; j++) A[j] = R[j];
        Acc.store(R, t);
        tput(s - s_tab + 1, R);
        if (s == s_main - 1) {  // seed the accumulator
          tget(P.ops[0], A);
          Acc.store(A, t);
        }
      } else if (s < s_fin) {
#pragma unroll
        for (int j = 0; j < K; j++) A[j] = R[j];
        Acc.store(R, t);
      } else {
        // final: value < 2m (<= m for the x 1 form) -> words, conditional subtract, store
        Acc.store(R, t);
        __syncwarp();
        if (t == 0) {
          uint32_t* out = P.y + (size_t)i * P.y_words;
          // compare limbs_value with m (32-bit words, most significant first)
          int cmp = 0;
          for (int k = P.mwords - 1; k >= 0 && cmp == 0; k--) {
            const uint32_t a = r28::limbs_word<RB, N, TPI>(Acc, k), b = P.mword[k];
            cmp = a > b ? 1 : (a < b ? -1 : 0);
          }
          // words beyond the modulus width can only be nonzero for values >= 2^(32 mwords) > m
          for (int k = P.mwords; k < Side28Args<RB, N, TPI>::W && cmp <= 0; k++)
            if (r28::limbs_word<RB, N, TPI>(Acc, k)) cmp = 1;
          int64_t br = 0;
          for (int k = 0; k < P.y_words; k++) {
            const uint32_t a = k < Side28Args<RB, N, TPI>::W ? r28::limbs_word<RB, N, TPI>(Acc, k) : 0u;
            const uint32_t b = (cmp >= 0 && k < P.mwords) ? P.mword[k] : 0u;
            const int64_t d = (int64_t)a - b - br;
            out[k] = (uint32_t)d;
            br = d < 0;
          }
        }
        __syncwarp();
      }
      if (P.ntab == 1 && s == s_x2) {
        tget(P.ops[0], A);
        Acc.store(A, t);
      }
    }
  }
}

template <int RB, int N, int TPI>
pcb_status launch_side28(const uint32_t* mlimb, const uint32_t* mword, int mwords, const uint32_t* r2,
                         const uint32_t* c1, uint32_t minv, const uint8_t* ops, int nops, int ntab, int mode,
                         const uint32_t* x, int x_words, const uint32_t* m, int m_words, const int32_t* skip,
                         size_t count, uint32_t* y, int y_words, cudaStream_t st, double alg_mac32_per_elem) {
  using Args = Side28Args<RB, N, TPI>;
  Args P;
  for (int j = 0; j < N; j++) {
    P.mlimb[j] = mlimb[j];
    P.r2[j] = r2[j];
    P.c1[j] = c1 ? c1[j] : 0u;
  }
  for (int j = 0; j < Args::W; j++) P.mword[j] = j < mwords ? mword[j] : 0u;
  P.minv = minv;
  P.mwords = mwords;
  P.ops = ops;
  P.nops = nops;
  P.ntab = ntab;
  P.x = x;
  P.x_words = x_words;
  P.m = m;
  P.m_words = m_words;
  P.skip = skip;
  P.y = y;
  P.y_words = y_words;
  P.count = (int)count;
  P.mode = mode;
  constexpr int G = 32 / TPI;
  const size_t smem = (size_t)(((N + 3) & ~3) + (kThreadsPerBlock / 32) * 2 * N * G) * 4;
  int blocks = 0;
  if (auto e = item_grid(side28_kernel<RB, N, TPI>, smem, count * TPI, &blocks)) return e;
  const size_t nlanes = (size_t)blocks * kThreadsPerBlock;
  if (auto e = scratch_alloc(nlanes * (ntab + 1) * (N / TPI) * 4, (void**)&P.tab, st)) return e;
  ProfMark pm;
  if (prof_enabled()) pm = prof_start(st);
  side28_kernel<RB, N, TPI><<<blocks, kThreadsPerBlock, smem, st>>>(P);
  count_launch();
  if (prof_enabled()) prof_stop(pm, st, alg_mac32_per_elem * (double)count);
  scratch_free(P.tab, st);
  return cuda_check(cudaGetLastError());
}

#define PCB_SIDE28(RB, N, TPI)                                                                                     \
  template pcb_status launch_side28<RB, N, TPI>(const uint32_t*, const uint32_t*, int, const uint32_t*,            \
                                                const uint32_t*, uint32_t, const uint8_t*, int, int, int,           \
                                                const uint32_t*, int, const uint32_t*, int, const int32_t*, size_t, \
                                                uint32_t*, int, cudaStream_t, double);
PCB_SIDE28(28, 38, 1)   // 1024-bit keys: p^2 <= 1060 bits
PCB_SIDE28(28, 76, 2)   // 2048-bit keys: p^2 <= 2124 bits; n^2 of 1024-bit keys
PCB_SIDE28(28, 112, 2)  // 3072-bit keys: p^2 <= 3132 bits
PCB_SIDE28(27, 152, 4)  // n^2 of 2048-bit keys (public-key encryption)
PCB_SIDE28(27, 240, 8)  // n^2 of 3072-bit keys (6144 bits)
PCB_SIDE28(27, 304, 8)  // n^2 of 4096-bit keys (8192 bits)

}  // namespace pcb
