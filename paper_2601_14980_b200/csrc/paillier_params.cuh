// paillier_params.cuh — per-key device constants for the Paillier kernels.  Filled once per
// context on the host (abi.cu, from n, p, q) and passed by value as __grid_constant__ kernel
// parameters, so every modulus limb is a constant-bank operand of IMAD.WIDE.
#pragma once
#include <cstdint>

#include "mont.cuh"

namespace pcb {

// Device-resident op stream of one fixed exponent (mont.cuh, mont_pow).
struct Sched {
  const uint8_t* ops;
  int n;
};

// CRT encryption, g = n + 1 (Paillier::crt_encrypt_with_r, paillier.cpp:334-344):
//   c_p = (1 + m n mod p^2) * r^(n mod phi(p^2)) mod p^2, same for q, Garner to mod n^2.
template <int S>
struct CrtEncConsts {
  ModCtx<S> mp, mq;   // p^2, q^2
  uint32_t nRp[S];    // n*R mod p^2  => mont(m, nRp) = m*n mod p^2
  uint32_t nRq[S];    // n*R mod q^2
  uint32_t inv[S];    // (p^2)^-1 mod q^2 (plain)
  uint32_t n[S];      // n (range checks)
};

// CRT decryption (c^(p-1) mod p^2 form; same m as paillier.cpp:354-361 for every unit c).
template <int S>
struct CrtDecConsts {
  ModCtx<S> mp, mq;        // p^2, q^2
  ModCtx<S / 2> sp, sq;    // p, q
  uint32_t r3p[S];         // R^3 mod p^2 (high half of c)
  uint32_t r3q[S];
  uint32_t pinv_lo[S / 2]; // p^-1 mod 2^(16 S)  (exact division L_p)
  uint32_t qinv_lo[S / 2];
  uint32_t hp[S / 2];      // h_p * R_h mod p, h_p = L_p(g^(p-1) mod p^2)^-1 mod p
  uint32_t hq[S / 2];
  uint32_t pinvq[S / 2];   // p^-1 mod q (plain, CRT recombination of m)
  uint32_t p[S / 2];       // p, q (plain)
  uint32_t q[S / 2];
  uint32_t n2[2 * S];      // n^2 (range check c < n^2)
};

// Generic n^2 context for the public-key operations (direct encryption, hom ops).
template <int S>
struct N2Consts {
  ModCtx<S> mn;      // n^2
  uint32_t nR[S];    // n*R mod n^2
  uint32_t n[S];     // n (range checks), zero-padded
};

}  // namespace pcb
