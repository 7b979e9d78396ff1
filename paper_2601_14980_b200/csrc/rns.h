// rns.h — RNS Montgomery core (rns.cu): per-modulus constants and the launcher.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "pcb_internal.h"

namespace pcb {

class HBN;

constexpr int kRnsK = 72;          // primes per base (30-bit): M, M' ~ 2^2160 > (2K+2)^2 N, N <= 2^2048
constexpr int kRnsK2 = 320;        // GEMM 2 reduction bytes: 4 (K + 1) padded to a multiple of 32
constexpr int kRnsMpWords = 68;    // words of M' = prod of the B' primes
constexpr int kRnsMaxS = 64;       // moduli up to 2048 bits (p^2, q^2 of 2048-bit keys)
enum : int { kRnsEnc = 0, kRnsDec = 1, kRnsPow = 2 };

// Kernel-parameter constants.  Index layout: [0, K) base B, [K, 2K) base B'; c1 over B;
// c2/c3/c4/invp over B' (index j - K).  RNS constants are per-prime lazy Montgomery residues.
struct RnsConsts {
  uint32_t mod[2 * kRnsK], minv[2 * kRnsK], q64[2 * kRnsK], one[2 * kRnsK];
  uint32_t c1[kRnsK], c2[kRnsK], c3[kRnsK], c4[kRnsK];
  double invp[kRnsK];
  uint32_t r2n[2 * kRnsK];   // M^2 mod N           (to the Montgomery-M domain)
  uint32_t cr2n[2 * kRnsK];  // 2^(32 S) M^2 mod N  (high half of a 2S-word ciphertext)
  uint32_t nM[2 * kRnsK];    // n M mod N           (m n for Enc)
};

struct RnsOutArgs {
  const uint32_t* res;       // count x K B' residues
  uint32_t* y;               // count x S words
  int count, S;
  uint32_t mod[kRnsK], minv[kRnsK], c4[kRnsK];
  double invp[kRnsK];
  const uint32_t* mpj;       // K x kRnsMpWords: M'/m'_j
  const uint32_t* mp;        // kRnsMpWords: M'
  const uint32_t* n;         // S words: N
  double ntop;               // N / 2^(32 (S-2))
};

struct RnsModulus {
  int S = 0;
  RnsConsts c{};
  RnsOutArgs out{};
  uint8_t* d_wimg = nullptr;  // device: W1 then W2 in the shared-memory image layout
  uint32_t* d_tabs = nullptr; // device: mpj, mp, n
  bool ok = false;
};

// Build the constants for modulus N (odd, coprime to the primes, < 2^(32 S), S <= 64); n is
// the Paillier modulus (for Enc's m n term).  Uploads the matrices; false on failure.
bool rns_build(const HBN& N, const HBN& n, int S, RnsModulus* out);
void rns_free(RnsModulus* md);

pcb_status launch_rns(const RnsModulus& md, int mode, const uint8_t* ops, int nops, int ntab, const uint32_t* x,
                      int x_words, const uint32_t* m, int m_words, size_t count, uint32_t* y, cudaStream_t st,
                      double alg_mac32);

}  // namespace pcb
