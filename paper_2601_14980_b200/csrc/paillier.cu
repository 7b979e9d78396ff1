// paillier.cu — batched CRT encryption and decryption kernels (the hot path).
//
//   crt_encrypt_kernel : Paillier::crt_encrypt_with_r  (/root/reference/proj/src/paillier.cpp:334-344)
//                        batched as in encrypt_vec (paillier.cpp:495-507)
//   crt_decrypt_kernel : Paillier::crt_decrypt / decrypt (paillier.cpp:346-361), batched as
//                        decrypt_vec (paillier.cpp:509-516)
//
// One element per thread; both CRT halves run in the same thread so the Garner recombination
// stays in registers.  Every exponent is per-key (n mod phi(p^2), p-1, ...), i.e. warp-uniform.
#include <cstdint>
#include <cuda_runtime.h>

#include "bigops.cuh"
#include "mont.cuh"
#include "paillier_params.cuh"
#include "pcb_internal.h"

namespace pcb {


template <int S>
struct CrtEncArgs {
  CrtEncConsts<S> k;
  Sched sp, sq;          // n mod phi(p^2), n mod phi(q^2)
  int ntab;
  uint4* tab;
  const uint32_t* m;     // count x m_limbs
  const uint32_t* r;     // count x L
  uint32_t* c;           // count x 2L
  int32_t* st;           // count (nullable)
  int m_limbs, L, count;
  const double* qv;      // fused quantize prologue (nullable): values -> m
  double zmin, zmax, delta;
  int fine;
  uint64_t* q_out;       // quantized integers (nullable)
  unsigned long long* clamps;  // [2] device counters (nullable)
};

// Quantizers, FP64 with the reference's operation order and no contraction
// (quantize.cpp:31-41; built with --fmad=false).  round() is half-away-from-zero as libm.
__device__ __forceinline__ double clamp_q(double v, double zmin, double zmax, unsigned long long* clamps) {
  if (v < zmin) {
    if (clamps) atomicAdd(&clamps[0], 1ull);
    return zmin;
  }
  if (v > zmax) {
    if (clamps) atomicAdd(&clamps[1], 1ull);
    return zmax;
  }
  return v;
}

// gamma2: (u64) round(delta * ((clamp(v) - zmin) / R))
__device__ __forceinline__ uint64_t gamma2_dev(double v, double zmin, double zmax, double delta,
                                               unsigned long long* clamps) {
  double R = __dsub_rn(zmax, zmin);
  double t = __dmul_rn(delta, __ddiv_rn(__dsub_rn(clamp_q(v, zmin, zmax, clamps), zmin), R));
  return (uint64_t)round(t);
}

// gamma1: (u128) round((delta*delta) * ((clamp(v) - zmin) / (R*R)))  -> lo/hi u64
__device__ __forceinline__ void gamma1_dev(double v, double zmin, double zmax, double delta,
                                           unsigned long long* clamps, uint64_t& lo, uint64_t& hi) {
  double R = __dsub_rn(zmax, zmin);
  double d = __ddiv_rn(__dsub_rn(clamp_q(v, zmin, zmax, clamps), zmin), __dmul_rn(R, R));
  double t = round(__dmul_rn(__dmul_rn(delta, delta), d));
  // exact double -> u128 (t is a non-negative integer-valued double, < 2^128)
  if (t < 18446744073709551616.0) {
    lo = (uint64_t)t;
    hi = 0;
  } else {
    double h = floor(t * 5.421010862427522e-20);  // t / 2^64, exact power-of-two scaling
    hi = (uint64_t)h;
    lo = (uint64_t)(t - h * 18446744073709551616.0);
  }
}

// Slot policy: multiplicand in registers when 3S+4 registers fit next to the kernel state.
template <int S>
struct Areg {
  static constexpr bool value = S <= 64;
};

// Scratch entries appended to the per-thread power table.
enum : int { kParkG = 0, kParkCp = 1, kParkA1 = 2, kParkMp = 0, kNumPark = 3 };

// One CRT half of encryption:  C = (1 + m n mod m2) * r^(n mod phi(m2)) mod m2 (plain), left
// in registers.  (crt_encrypt_with_r per side: g_power_half + half_pow, paillier.cpp:339-342)
template <int S>
__device__ __forceinline__ void enc_half(uint32_t (&C)[S], const Slot<S>& Acc, const Slot<S>& Op,
                                         const GTable<S>& tab, int ntab, const uint32_t* msrc, int m_limbs,
                                         uint64_t qlo, uint64_t qhi, bool quantized, const uint32_t* rsrc, int L,
                                         const SMod<S>& M2, const uint32_t* r2, const uint32_t* nR, const Sched& sc) {
  constexpr bool AR = Areg<S>::value;
  uint32_t R[S];
  // g^m = 1 + m n mod m2  (g_power_half, paillier.cpp:263), parked while r^e runs
  if (quantized) {
    Acc.store_small(0);
    uint4 c0 = make_uint4((uint32_t)qlo, (uint32_t)qhi, 0, 0);  // even limbs m0, m2
    uint4 c1 = make_uint4((uint32_t)(qlo >> 32), (uint32_t)(qhi >> 32), 0, 0);  // odd limbs m1, m3
    Acc.set_chunk(0, c0);
    Acc.set_chunk(S / 8, c1);
  } else {
    Acc.store_global(msrc, m_limbs);
  }
  Op.store_const(nR);
  mont_mul_ss<S, AR>(R, Acc, Op, M2);  // m n mod m2
  mod_inc<S>(R, M2);
  tab.put(ntab + kParkG, R);
  // r^e
  Acc.store_global(rsrc, L);
  Op.store_const(r2);
  mont_mul_ss<S, AR>(R, Acc, Op, M2);  // r R mod m2 (also reduces r)
  Acc.store(R);
  mont_pow<S, AR>(Acc, Op, tab, ntab, sc.ops, sc.n, M2);
  tab.to_slot(ntab + kParkG, Op);
  mont_mul_ss<S, AR>(C, Acc, Op, M2);  // r^e (1 + m n): Montgomery x plain = plain
}

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) crt_encrypt_kernel(const __grid_constant__ CrtEncArgs<S> P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr bool AR = Areg<S>::value;
  const CrtEncConsts<S>& K = P.k;
  // block-shared moduli (broadcast operands), then two per-thread slots
  smod_fill<S>(smem, K.mp.m);
  smod_fill<S>(smem + S, K.mq.m);
  __syncthreads();
  const SMod<S> Mp{smem_addr(smem), K.mp.minv}, Mq{smem_addr(smem + S), K.mq.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + 2 * S;
  const Slot<S> Acc{smem_addr(slots + warp * (64 * S) + lane * 4)};
  const Slot<S> Op{smem_addr(slots + warp * (64 * S) + 32 * S + lane * 4)};
  const uint32_t nthr = gridDim.x * blockDim.x;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  GTable<S> tab{P.tab, nthr, g};

  for (int i = g; i < P.count; i += nthr) {
    uint32_t* out = P.c + (size_t)i * 2 * P.L;
    const uint32_t* rsrc = P.r + (size_t)i * P.L;
    const uint32_t* msrc = P.m ? P.m + (size_t)i * P.m_limbs : nullptr;
    // ---- plaintext (optionally quantized in-kernel) and argument checks -------------------
    uint64_t qlo = 0, qhi = 0;
    int status = PCB_OK;
    if (P.qv) {  // fused quantize prologue (quantize.cpp:31-41)
      const double v = P.qv[i];
      if (!isfinite(v)) {
        status = PCB_E_SHAPE;  // clamp_in throws invalid_argument (quantize.cpp:18-19)
      } else if (P.fine) {
        gamma1_dev(v, P.zmin, P.zmax, P.delta, P.clamps, qlo, qhi);
        if (P.q_out) { P.q_out[2 * (size_t)i] = qlo; P.q_out[2 * (size_t)i + 1] = qhi; }
      } else {
        qlo = gamma2_dev(v, P.zmin, P.zmax, P.delta, P.clamps);
        if (P.q_out) P.q_out[i] = qlo;
      }
      // quantized values are < 2^128 <= n for every supported key; compare anyway
      if (status == PCB_OK) {
        uint32_t mw[4] = {(uint32_t)qlo, (uint32_t)(qlo >> 32), (uint32_t)qhi, (uint32_t)(qhi >> 32)};
        if (!lt_words(mw, 4, K.n, P.L)) status = PCB_E_PLAINTEXT_RANGE;
      }
    } else if (!lt_words(msrc, P.m_limbs, K.n, P.L)) {
      status = PCB_E_PLAINTEXT_RANGE;  // check_plaintext (paillier.cpp:241-243)
    }
    if (status == PCB_OK && (is_zero_words(rsrc, P.L) || !lt_words(rsrc, P.L, K.n, P.L)))
      status = PCB_E_RANDOMNESS_RANGE;  // paillier.cpp:337-338
    if (P.st) P.st[i] = status;
    if (status != PCB_OK) {
      for (int j = 0; j < 2 * P.L; j++) out[j] = 0;
      continue;
    }
    const bool quant = P.qv != nullptr;
    {
      uint32_t C[S];
      enc_half<S>(C, Acc, Op, tab, P.ntab, msrc, P.m_limbs, qlo, qhi, quant, rsrc, P.L, Mp, K.mp.r2, K.nRp, P.sp);
      tab.put(P.ntab + kParkCp, C);
    }
    uint32_t A2[S];
    enc_half<S>(A2, Acc, Op, tab, P.ntab, msrc, P.m_limbs, qlo, qhi, quant, rsrc, P.L, Mq, K.mq.r2, K.nRq, P.sq);
    // ---- Garner (combine_halves, paillier.cpp:307-314): c = cp + p^2 ((cq - cp) (p^2)^-1 mod q^2)
    Acc.store(A2);
    Op.store_const(K.mq.r2);
    mont_mul_ss<S, AR>(A2, Acc, Op, Mq);  // cq R mod q^2
    tab.put(P.ntab + kParkA1, A2);
    tab.to_slot(P.ntab + kParkCp, Acc);
    mont_mul_ss<S, AR>(A2, Acc, Op, Mq);  // cp R mod q^2   (cp < p^2 < R)
    {
      uint32_t A1[S];
      tab.get(P.ntab + kParkA1, A1);
      mod_sub<S>(A1, A2, Mq);  // (cq - cp) R mod q^2
      Acc.store(A1);
    }
    Op.store_const(K.inv);
    mont_mul_ss<S, AR>(A2, Acc, Op, Mq);  // t = (cq - cp) (p^2)^-1 mod q^2, plain
    Op.store(A2);
    {
      uint32_t H[S], Cp[S];
      tab.get(P.ntab + kParkCp, Cp);
      mul_add_smod<S>(H, Cp, Op, Mp);  // c = cp + p^2 t; low S words left in Op
      const int cl = 2 * P.L;
#pragma unroll
      for (int j = 0; j < S; j++)
        if (j < cl) out[j] = Op.digit(j);
#pragma unroll
      for (int j = 0; j < S; j++)
        if (S + j < cl) out[S + j] = H[j];
    }
  }
}

// ------------------------------------------------------------------------------------------
template <int S>
struct CrtDecArgs {
  CrtDecConsts<S> k;
  Sched sp, sq;   // p-1, q-1
  int ntab;
  uint4* tab;
  const uint32_t* c;  // count x 2L
  uint32_t* m;        // count x L
  int32_t* st;
  int L, count;
};

// One CRT half of decryption: returns false for a non-unit (p | c).
//   x = c^(p-1) mod p^2,  u = (x - 1) / p  (exact),  mh = u * h_p mod p.
template <int S>
__device__ __forceinline__ bool dec_half(uint32_t (&Mh)[S / 2], const uint32_t* csrc, int cl, const Slot<S>& Acc,
                                         const Slot<S>& Op, const GTable<S>& tab, int ntab, const Sched& sc,
                                         const SMod<S>& M2, const uint32_t* r2, const uint32_t* r3, const SMod<S / 2>& M1,
                                         const uint32_t* inv_lo, const uint32_t* h, const uint32_t* prime) {
  constexpr int H = S / 2;
  constexpr bool AR = Areg<S>::value;
  uint32_t X[S];
  Acc.store_global(csrc + S, cl - S);  // c_hi
  Op.store_const(r3);
  mont_mul_ss<S, AR>(X, Acc, Op, M2);  // c_hi R^2 = (c_hi 2^(32S)) R
  tab.put(ntab + kParkA1, X);
  Acc.store_global(csrc, cl < S ? cl : S);  // c_lo
  Op.store_const(r2);
  mont_mul_ss<S, AR>(X, Acc, Op, M2);  // c_lo R
  {
    uint32_t Y[S];
    tab.get(ntab + kParkA1, Y);
    mod_add<S>(X, Y, M2);  // c R mod p^2
  }
  Acc.store(X);
  mont_pow<S, AR>(Acc, Op, tab, ntab, sc.ops, sc.n, M2);
  Op.store_small(1);
  mont_mul_ss<S, AR>(X, Acc, Op, M2);  // x = c^(p-1) mod p^2, plain
  // x - 1 (x == 0 -> non-unit)
  bool ok = !is_zero(X);
  uint32_t br;
  asm volatile("sub.cc.u32 %0, %0, 1;" : "+r"(X[0]));
#pragma unroll
  for (int j = 1; j < S; j++) asm volatile("subc.cc.u32 %0, %0, 0;" : "+r"(X[j]));
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(br));
  uint32_t U[H];
  {
    uint32_t lo[H];
#pragma unroll
    for (int j = 0; j < H; j++) lo[j] = X[j];
    mul_lo<H>(U, lo, inv_lo);  // u = (x-1) p^-1 mod 2^(32H)
  }
  ok = mul_eq<H>(U, prime, X) && ok;  // exact division <=> x == 1 mod p
  const Slot<H> Ah{Acc.a}, Oh{Op.a};
  Ah.store(U);
  Oh.store_const(h);
  mont_mul_ss<H, true>(Mh, Ah, Oh, M1);  // u * h_p mod p
  return ok;
}

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) crt_decrypt_kernel(const __grid_constant__ CrtDecArgs<S> P) {
  extern __shared__ __align__(16) uint32_t smem[];
  constexpr int H = S / 2;
  const CrtDecConsts<S>& K = P.k;
  smod_fill<S>(smem, K.mp.m);
  smod_fill<S>(smem + S, K.mq.m);
  smod_fill<H>(smem + 2 * S, K.sp.m);
  smod_fill<H>(smem + 2 * S + H, K.sq.m);
  __syncthreads();
  const SMod<S> Mp_{smem_addr(smem), K.mp.minv}, Mq_{smem_addr(smem + S), K.mq.minv};
  const SMod<H> Sp{smem_addr(smem + 2 * S), K.sp.minv}, Sq{smem_addr(smem + 2 * S + H), K.sq.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + 3 * S;
  const Slot<S> Acc{smem_addr(slots + warp * (64 * S) + lane * 4)};
  const Slot<S> Op{smem_addr(slots + warp * (64 * S) + 32 * S + lane * 4)};
  const uint32_t nthr = gridDim.x * blockDim.x;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  GTable<S> tab{P.tab, nthr, g};

  for (int i = g; i < P.count; i += nthr) {
    const uint32_t* src = P.c + (size_t)i * 2 * P.L;
    uint32_t* out = P.m + (size_t)i * P.L;
    if (!lt_words(src, 2 * P.L, K.n2, 2 * P.L)) {  // c < n^2 (paillier.cpp:356)
      if (P.st) P.st[i] = PCB_E_CIPHER_RANGE;
      for (int j = 0; j < P.L; j++) out[j] = 0;
      continue;
    }
    bool ok;
    {
      uint32_t Mp[H];
      ok = dec_half<S>(Mp, src, 2 * P.L, Acc, Op, tab, P.ntab, P.sp, Mp_, K.mp.r2, K.r3p, Sp, K.pinv_lo, K.hp, K.p);
      uint32_t park[S];
#pragma unroll
      for (int j = 0; j < S; j++) park[j] = j < H ? Mp[j] : 0u;
      tab.put(P.ntab + kParkCp, park);
    }
    uint32_t Mq[H];
    ok = dec_half<S>(Mq, src, 2 * P.L, Acc, Op, tab, P.ntab, P.sq, Mq_, K.mq.r2, K.r3q, Sq, K.qinv_lo, K.hq, K.q) && ok;
    if (!ok) {
      if (P.st) P.st[i] = PCB_E_NOT_UNIT;  // l_function (paillier.cpp:34-41)
      for (int j = 0; j < P.L; j++) out[j] = 0;
      continue;
    }
    // m = m_p + p * ((m_q - m_p) p^-1 mod q)
    const Slot<H> Ah{Acc.a}, Oh{Op.a};
    uint32_t Mp[H], T[H];
    {
      uint32_t park[S];
      tab.get(P.ntab + kParkCp, park);
#pragma unroll
      for (int j = 0; j < H; j++) Mp[j] = park[j];
    }
    Oh.store_const(K.sq.r2);
    Ah.store(Mq);
    mont_mul_ss<H, true>(T, Ah, Oh, Sq);   // m_q R mod q
    Ah.store(Mp);
    mont_mul_ss<H, true>(Mq, Ah, Oh, Sq);  // m_p R mod q (reduces m_p mod q)
    mod_sub<H>(T, Mq, Sq);
    Ah.store(T);
    Oh.store_const(K.pinvq);
    mont_mul_ss<H, true>(T, Ah, Oh, Sq);   // t = (m_q - m_p) p^-1 mod q, plain
    Oh.store(T);
    uint32_t Hi[H];
    mul_add_smod<H>(Hi, Mp, Oh, Sp);
#pragma unroll
    for (int j = 0; j < H; j++)
      if (j < P.L) out[j] = Oh.digit(j);
#pragma unroll
    for (int j = 0; j < H; j++)
      if (H + j < P.L) out[H + j] = Hi[j];
    if (P.st) P.st[i] = PCB_OK;
  }
}

// ------------------------------------------------------------------------------------------
// Launchers (called from abi.cu with the per-context constant blobs).
// ------------------------------------------------------------------------------------------
template <int S>
pcb_status launch_crt_encrypt(const CrtEncConsts<S>& k, Sched sp, Sched sq, int ntab, const uint32_t* m,
                              int m_limbs, const uint32_t* r, int L, size_t count, uint32_t* c, int32_t* st,
                              const double* qv, double zmin, double zmax, double delta, int fine, uint64_t* q_out,
                              unsigned long long* clamps, cudaStream_t stream) {
  CrtEncArgs<S> P;
  P.k = k;
  P.sp = sp;
  P.sq = sq;
  P.ntab = ntab;
  P.m = m;
  P.r = r;
  P.c = c;
  P.st = st;
  P.m_limbs = m_limbs;
  P.L = L;
  P.count = (int)count;
  P.qv = qv;
  P.zmin = zmin;
  P.zmax = zmax;
  P.delta = delta;
  P.fine = fine;
  P.q_out = q_out;
  P.clamps = clamps;
  const size_t smem = (size_t)kThreadsPerBlock * S * 8 + 2 * S * 4;  // moduli + two slots per thread
  int blocks = 0;
  if (auto e = item_grid(crt_encrypt_kernel<S>, smem, count, &blocks)) return e;
  const size_t nthr = (size_t)blocks * kThreadsPerBlock;
  if (auto e = scratch_alloc(nthr * (ntab + kNumPark) * S * 4, (void**)&P.tab, stream)) return e;
  crt_encrypt_kernel<S><<<blocks, kThreadsPerBlock, smem, stream>>>(P);
  count_launch();
  scratch_free(P.tab, stream);
  return cuda_check(cudaGetLastError());
}

template <int S>
pcb_status launch_crt_decrypt(const CrtDecConsts<S>& k, Sched sp, Sched sq, int ntab, const uint32_t* c, int L,
                              size_t count, uint32_t* m, int32_t* st, cudaStream_t stream) {
  CrtDecArgs<S> P;
  P.k = k;
  P.sp = sp;
  P.sq = sq;
  P.ntab = ntab;
  P.c = c;
  P.m = m;
  P.st = st;
  P.L = L;
  P.count = (int)count;
  const size_t smem = (size_t)kThreadsPerBlock * S * 8 + 3 * S * 4;  // moduli + two slots per thread
  int blocks = 0;
  if (auto e = item_grid(crt_decrypt_kernel<S>, smem, count, &blocks)) return e;
  const size_t nthr = (size_t)blocks * kThreadsPerBlock;
  if (auto e = scratch_alloc(nthr * (ntab + kNumPark) * S * 4, (void**)&P.tab, stream)) return e;
  crt_decrypt_kernel<S><<<blocks, kThreadsPerBlock, smem, stream>>>(P);
  count_launch();
  scratch_free(P.tab, stream);
  return cuda_check(cudaGetLastError());
}

#define PCB_INSTANTIATE(S)                                                                                          \
  template pcb_status launch_crt_encrypt<S>(const CrtEncConsts<S>&, Sched, Sched, int, const uint32_t*, int,       \
                                            const uint32_t*, int, size_t, uint32_t*, int32_t*, const double*, double, \
                                            double, double, int, uint64_t*, unsigned long long*, cudaStream_t);      \
  template pcb_status launch_crt_decrypt<S>(const CrtDecConsts<S>&, Sched, Sched, int, const uint32_t*, int, size_t, \
                                            uint32_t*, int32_t*, cudaStream_t);
PCB_INSTANTIATE(32)
PCB_INSTANTIATE(64)

}  // namespace pcb
