// wide.cu — operations modulo n^2 (public key suffices) on the radix-2^r core (mont28.cuh),
// driven by a tiny warp-uniform program around ONE Montgomery product site:
//
//   hom_add        out_i = a_i b_i mod n^2            Paillier::hom_add        (paillier.cpp:428-432)
//   hom_scalar_mul out_i = c_i^(k_i) mod n^2, k < 2^64 Paillier::hom_scalar_mul (paillier.cpp:434-439)
//   aggregate      out_c = prod_{i in chunk c} x_i      one level of the product tree (pcb_aggregate)
//
// Each program step computes R = A * B * R^-1 (lazy, < 2m) where A is the register operand and B
// the shared-memory digit operand; the step descriptor says where A and B come from and where R
// goes.  Programs are uniform across the batch (built on the host in abi.cu), per-element data
// only selects WHICH table entry / input feeds a step, so warps never diverge.
#include <cstdint>
#include <cuda_runtime.h>

#include "mont.cuh"
#include "mont28.cuh"
#include "pcb_internal.h"
#include "wide.h"

namespace pcb {

template <int RB, int N, int TPI>
struct WideArgs {
  static constexpr int W = (N * RB + 31) / 32;
  uint32_t mlimb[N];
  uint32_t mword[W];
  uint32_t minv;
  int mwords;             // words per operand / output (= words of n^2)
  WStep prog[kWideMaxSteps];
  int nsteps;
  const uint32_t* consts; // nconst x N radix limbs (device)
  const uint32_t* x;      // primary inputs  (elements of mwords words)
  const uint32_t* b;      // secondary inputs (hom_add)
  const uint64_t* k;      // per-element scalars (hom_scalar_mul)
  int xin_per_out;        // inputs consumed per output (aggregate chunk; 1 otherwise)
  int count;              // number of primary inputs
  int nout;
  uint32_t* tab;          // per-lane scratch table (16 entries)
  uint32_t* y;            // nout x mwords
  // hom_matvec
  uint32_t* mtab;         // power tables: entry (col, w, d) at ((col * nwin + w) * 64 + d) * N words
  const uint64_t* expo;   // rows x cols exponents (row-major)
  int cols, nwin, cc, nch, wcur;
  int brows;              // rows per diagonal block (0: a single block)
};

template <int RB, int N, int TPI>
__global__ void __launch_bounds__(kThreadsPerBlock) wide_kernel(const __grid_constant__ WideArgs<RB, N, TPI> P) {
  using Cf = r28::Cfg<RB, N, TPI>;
  constexpr int K = Cf::K, G = Cf::G, WW = WideArgs<RB, N, TPI>::W;
  using Slot = r28::DSlot<RB, N, TPI>;
  extern __shared__ __align__(16) uint32_t smem[];
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
  const int groups_total = nlanes / TPI;
  const int W = P.mwords;

  auto tab_at = [&](int e, int j) -> uint32_t& { return P.tab[(size_t)(e * K + j) * nlanes + gl]; };

  for (int o = gl / TPI; o < P.nout; o += groups_total) {
    const int first = o * P.xin_per_out;
    const int nin = min(P.xin_per_out, P.count - first);
    const uint64_t kk = P.k ? P.k[o] : 0ull;
    uint32_t A[K];
    // per-element operand fetch (limbs of this lane)
    auto fetch = [&](uint32_t (&v)[K], int src, int arg) {
      if (src == kSrcX) {
        if (arg < nin) {
          r28::words_to_limbs<RB, K>(v, P.x + (size_t)(first + arg) * W, W, t * K);
        } else {  // padding input of a short aggregation chunk: the integer 1 (each step of the
                  // chunk program multiplies by x_j R^-1, so padding must contribute x_j = 1)
#pragma unroll
          for (int j = 0; j < K; j++) v[j] = P.consts[kConstOne * N + t * K + j];
        }
      } else if (src == kSrcB) {
        r28::words_to_limbs<RB, K>(v, P.b + (size_t)o * W, W, t * K);
      } else if (src == kSrcConst) {
#pragma unroll
        for (int j = 0; j < K; j++) v[j] = P.consts[arg * N + t * K + j];
      } else if (src == kSrcTab) {
#pragma unroll
        for (int j = 0; j < K; j++) v[j] = tab_at(arg, j);
      } else if (src == kSrcMatTab) {  // group o = (row, chunk); entry (col, w, digit of E[row][col])
        const int jl = arg >> 4, w = arg & 15;
        const int row = o / P.nch, col = (o % P.nch) * P.cc + jl;
        const int tcol = (P.brows ? (row / P.brows) * P.cols : 0) + col;  // block-diagonal batches
        int d = 0;
        if (col < P.cols) d = (int)((P.expo[(size_t)row * P.cols + col] >> (kMatWin * w)) & ((1u << kMatWin) - 1));
        if (d == 0) {
#pragma unroll
          for (int j = 0; j < K; j++) v[j] = P.consts[kConstOneR * N + t * K + j];
        } else {
          const uint32_t* e = P.mtab + ((size_t)(tcol * P.nwin + w) * 64 + d) * N + t * K;
#pragma unroll
          for (int j = 0; j < K; j++) v[j] = e[j];
        }
      } else if (src == kSrcGEntry) {  // table fill: element o = (column, window) pair
        const uint32_t* e = P.mtab + ((size_t)o * 64 + arg) * N + t * K;
#pragma unroll
        for (int j = 0; j < K; j++) v[j] = e[j];
      } else {  // kSrcTabDigit: entry = 4-bit digit `arg` of this element's scalar
        const int d = (int)((kk >> (4 * arg)) & 15u);
        if (d == 0) {
#pragma unroll
          for (int j = 0; j < K; j++) v[j] = P.consts[kConstOneR * N + t * K + j];
        } else {
#pragma unroll
          for (int j = 0; j < K; j++) v[j] = tab_at(d, j);
        }
      }
    };
#pragma unroll 1
    for (int s = 0; s < P.nsteps; s++) {
      const WStep st = P.prog[s];
      if (st.asrc != kSrcReg) fetch(A, st.asrc, st.aarg);
      const bool b_acc = st.bsrc == kSrcAcc;
      if (!b_acc && st.bsrc != kSrcOpKeep) {
        uint32_t v[K];
        fetch(v, st.bsrc, st.barg);
#pragma unroll
        for (int j = 0; j < K; j++) Op.set(t * K + j, v[j]);
      }
      __syncwarp();
      uint32_t R[K];
      r28::mm<RB, N, TPI>(R, A, b_acc ? Acc : Op, mlane, P.minv, t);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < K; j++) A[j] = R[j];
      if (st.post & kPostAcc) Acc.store(R, t);
      if (st.post & kPostOp) Op.store(R, t);
      if (st.post & kPostGTab) {  // matvec table build (wide.h kPostGTab)
        const size_t ent = P.wcur >= 0 ? (size_t)(o * P.nwin + P.wcur + st.pad0) * 64 + st.tab : (size_t)o * 64 + st.tab;
        uint32_t* e = P.mtab + ent * N + t * K;
#pragma unroll
        for (int j = 0; j < K; j++) e[j] = R[j];
      }
      if (st.post & kPostTab) {
#pragma unroll
        for (int j = 0; j < K; j++) tab_at(st.tab, j) = R[j];
      }
      if (st.post & kPostOut) {
        Acc.store(R, t);
        __syncwarp();
        if (t == 0) {
          uint32_t* out = P.y + (size_t)o * W;
          int cmp = 0;
          for (int kw = WW - 1; kw >= 0 && cmp == 0; kw--) {
            const uint32_t a = r28::limbs_word<RB, N, TPI>(Acc, kw), bw = kw < P.mwords ? P.mword[kw] : 0u;
            cmp = a > bw ? 1 : (a < bw ? -1 : 0);
          }
          int64_t br = 0;
          for (int kw = 0; kw < W; kw++) {
            const uint32_t a = r28::limbs_word<RB, N, TPI>(Acc, kw);
            const uint32_t bw = (cmp >= 0 && kw < P.mwords) ? P.mword[kw] : 0u;
            const int64_t d = (int64_t)a - bw - br;
            out[kw] = (uint32_t)d;
            br = d < 0;
          }
        }
        __syncwarp();
      }
    }
  }
}

template <int RB, int N, int TPI>
pcb_status launch_wide(const WideMod& md, const WStep* prog, int nsteps, const uint32_t* consts_dev,
                       const uint32_t* x, const uint32_t* b, const uint64_t* k, int xin_per_out, size_t count,
                       size_t nout, uint32_t* y, int ntab, cudaStream_t st, const MatvecGeom* mg) {
  using Args = WideArgs<RB, N, TPI>;
  if (nsteps > kWideMaxSteps) return PCB_E_SHAPE;
  Args P;
  for (int j = 0; j < N; j++) P.mlimb[j] = md.mlimb[j];
  for (int j = 0; j < Args::W; j++) P.mword[j] = j < (int)md.mword.size() ? md.mword[j] : 0u;
  P.minv = md.minv;
  P.mwords = md.mwords;
  for (int s = 0; s < nsteps; s++) P.prog[s] = prog[s];
  P.nsteps = nsteps;
  P.consts = consts_dev;
  P.x = x;
  P.b = b;
  P.k = k;
  P.xin_per_out = xin_per_out;
  P.count = (int)count;
  P.nout = (int)nout;
  P.y = y;
  P.mtab = mg ? mg->mtab : nullptr;
  P.expo = mg ? mg->expo : nullptr;
  P.cols = mg ? mg->cols : 0;
  P.nwin = mg ? mg->nwin : 0;
  P.cc = mg ? mg->cc : 1;
  P.nch = mg ? mg->nch : 1;
  P.wcur = mg ? mg->wcur : 0;
  P.brows = mg ? mg->brows : 0;
  constexpr int G = 32 / TPI;
  const size_t smem = (size_t)(((N + 3) & ~3) + (kThreadsPerBlock / 32) * 2 * N * G) * 4;
  int blocks = 0;
  if (auto e = item_grid(wide_kernel<RB, N, TPI>, smem, nout * TPI, &blocks)) return e;
  const size_t nlanes = (size_t)blocks * kThreadsPerBlock;
  if (auto e = scratch_alloc(nlanes * (ntab > 0 ? ntab : 1) * (N / TPI) * 4, (void**)&P.tab, st)) return e;
  wide_kernel<RB, N, TPI><<<blocks, kThreadsPerBlock, smem, st>>>(P);
  count_launch();
  scratch_free(P.tab, st);
  return cuda_check(cudaGetLastError());
}

#define PCB_WIDE(RB, N, TPI)                                                                                      \
  template pcb_status launch_wide<RB, N, TPI>(const WideMod&, const WStep*, int, const uint32_t*, const uint32_t*, \
                                              const uint32_t*, const uint64_t*, int, size_t, size_t, uint32_t*, int, \
                                              cudaStream_t, const MatvecGeom*);
PCB_WIDE(28, 38, 1)   // n^2 <= 1060 bits (toy / 64-bit keys)
PCB_WIDE(28, 76, 2)   // n^2 <= 2124 bits (1024-bit keys)
PCB_WIDE(27, 152, 4)  // n^2 <= 4100 bits (2048-bit keys)
PCB_WIDE(27, 240, 8)  // n^2 <= 6476 bits (3072-bit keys)
PCB_WIDE(27, 304, 8)  // n^2 <= 8204 bits (4096-bit keys)

}  // namespace pcb
