// rnsx.h — streaming RNS Montgomery core (rnsx.cu): any modulus up to 4096 bits (K <= 144 primes
// per base), base-extension matrices streamed from L2 through a shared-memory ring, GEMM output
// chunked through a TMEM ring so the tensor core and the CUDA cores overlap.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "pcb_internal.h"

namespace pcb {

class HBN;

enum : int { kRxEnc = 0, kRxDec = 1, kRxPow = 2, kRxProg = 3, kRxEncG = 4, kRxPowVar = 5 };
// EncG: g r^e with g < N given;  PowVar: x^(e_el) with a per-element exponent (m = exponent words,
// nops = number of 4-bit windows, ntab = 16): the delegated power of the collaborative variant
constexpr int kRxReplicas = 16;  // copies of the stream image (spreads the L2 reads of 148 SMs)
enum : int { kRxOne = 0, kRxR2N = 1, kRxCR2N = 2, kRxNM = 3, kRxOneM = 4, kRxNumVec = 5 };

// ---- step programs (kRxProg): one RNS Montgomery product per step, uniform over the batch -------
// Elements are read / written as RNS records (2K residues, rnsx_rec_words() words each) or as
// binary words.  Operand sources (xs: multiplicand loaded before the product, ys: multiplier):
enum : uint8_t {
  kRsKeep = 0,  // xs: the previous result
  kRsSq = 0,    // ys: square (Y = X)
  kRsConv = 1,  // xs: X = binary input x[el] converted to RNS (lazy residues, plain value)
  kRsCvec = 2,  // constant vector `arg` (kRxOne, kRxR2N, kRxOneM, ...)
  kRsMat = 3,   // matvec table entry (column j = arg >> 4, window w = arg & 15, digit of E[row][col])
  kRsSelf = 4,  // table entry `arg` of this element's own (column, window) slot: mtab[el * 64 + arg]
  kRsPart = 5,  // partial record `arg` of this element: part[el * nparts + arg]
};
enum : uint8_t {
  kRpNone = 0,
  kRpOut = 1,    // result -> binary output y[el] (exact conversion mod N)
  kRpChain = 2,  // result -> mtab[(el * nwin + arg) * 64 + 1]    (window bases, one element per column)
  kRpSelf = 3,   // result -> mtab[el * 64 + arg]                  (table fill, one element per (column, window))
  kRpRec = 4,    // result -> part[el]                             (RNS record out)
};
struct XStep {
  uint8_t xs, xa, ys, ya, post, pa;
  uint8_t flags;  // bit 0: also set mtab[el * 64 + 0] = M mod N (the Montgomery one)
  uint8_t pad;
};
constexpr int kRxMaxSteps = 160;
struct RxProg {
  XStep st[kRxMaxSteps];
  int nsteps = 0;
  uint32_t* mtab = nullptr;       // RNS records
  uint32_t* part = nullptr;       // RNS records
  uint32_t* pout = nullptr;       // kRpRec destination (null: part)
  const uint64_t* expo = nullptr; // rows x cols exponents (matvec)
  int cols = 0, nwin = 0, cc = 1, nch = 1, brows = 0, nparts = 1;
};

struct RnsXModulus {
  int K = 0, S = 0;           // primes per base, words of N
  bool prefer_pairs = false;  // two tiles per CTA whatever the count (background work: least SM time)
  int mpw = 0;                // words of M' (output conversion)
  uint8_t* d_wimg = nullptr;  // base-extension stream: one slice (<= 128 x 32 bytes) per MMA, x kRxReplicas
  uint8_t* d_wimg2 = nullptr; // the same stream with every slice split in two row halves (cta_group::2)
  size_t wimg_stride = 0;
  uint4* d_cons = nullptr;    // per (g, w): {m, minv, c1, q64}, {m', minv', c2, c3}, {c4, invp, q64'}
  std::vector<uint32_t> h_cons;  // host copy (kernel-parameter constants, PCB_RNSX_KCONS)
  uint4* d_cvec = nullptr;    // constant operands in thread order: [id][g][NV][4]
  uint32_t* d_slt = nullptr;  // per slice of a product: {image offset / 16, bytes}
  uint32_t* d_out = nullptr;  // output conversion: mod'[K] minv'[K] c4[K] invp[2K] M'/m'_j[K][mpw] M'[mpw] N[S]
  double ntop = 0.0;          // N / 2^(32 ntw): N's two top words
  int ntw = 0;
  bool ok = false;
};

// Pick K for a modulus of `bits` bits: 2048 -> 72, 3072 -> 104, 4096 -> 144.
bool rnsx_shape(int bits, int* K);
// Build the constants for modulus N (odd, < 2^(32 S)); n is the Paillier modulus (Enc's m n term).
bool rnsx_build(const HBN& N, const HBN& n, int S, int K, RnsXModulus* out);
void rnsx_free(RnsXModulus* md);

// x^e-style uniform programs (Enc: (1 + m n) r^e, Dec: c^e, Pow: x^e), plain residues y mod N out.
int rnsx_rec_words(const RnsXModulus& md);  // words of one RNS record

// Step program over `count` elements (x: binary inputs of x_words words; y: binary outputs of S words).
pcb_status launch_rnsx_prog(const RnsXModulus& md, const RxProg& prog, const uint32_t* x, int x_words, size_t count,
                            uint32_t* y, cudaStream_t st, double alg_mac32);

pcb_status launch_rnsx(const RnsXModulus& md, int mode, const uint8_t* ops, int nops, int ntab, const uint32_t* x,
                       int x_words, const uint32_t* m, int m_words, size_t count, uint32_t* y, cudaStream_t st,
                       double alg_mac32, const int32_t* skip = nullptr);

}  // namespace pcb
