// paillier.cu — the light kernels around the hot side kernel (side.cu):
//
//   enc_prep_kernel  argument checks of Paillier::crt_encrypt_with_r / encrypt_with_r
//                    (paillier.cpp:241-243, 322-323, 335-338) and the fused quantize prologue
//                    (gamma1/gamma2, quantize.cpp:17-41) -> plaintext limbs + status
//   garner_kernel    combine_halves (paillier.cpp:307-314): c = c_p + p^2 ((c_q - c_p) (p^2)^-1 mod q^2)
//   dec_prep_kernel  c < n^2 check (paillier.cpp:356)
//   dec_finish_kernel  L_p / h_p / CRT: m = L(c^eps mod n^2) mu mod n computed as
//                    m_p = L_p(c^(p-1) mod p^2) h_p mod p,  m = m_p + p ((m_q - m_p) p^-1 mod q);
//                    non-unit ciphertexts (l_function, paillier.cpp:34-41) -> PCB_E_NOT_UNIT.
//
// These run O(S^2) work per element against O(S^3) in the side kernel, so they favour simple
// code: moduli live in block-shared memory (broadcast loads), one element per thread.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "bigops.cuh"
#include "mont.cuh"
#include "paillier_params.cuh"
#include "pcb_internal.h"

namespace pcb {

// ---- quantizers (FP64, reference operation order, no contraction: built with --fmad=false)
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

// gamma2 (quantize.cpp:31-35): (u64) round(delta * ((clamp(v) - zmin) / R)), R = zmax - zmin
__device__ __forceinline__ uint64_t gamma2_dev(double v, double zmin, double zmax, double delta,
                                               unsigned long long* clamps) {
  const double R = __dsub_rn(zmax, zmin);
  const double t = __dmul_rn(delta, __ddiv_rn(__dsub_rn(clamp_q(v, zmin, zmax, clamps), zmin), R));
  return (uint64_t)round(t);
}

// gamma1 (quantize.cpp:37-41): (u128) round(delta * delta * ((clamp(v) - zmin) / (R * R)))
__device__ __forceinline__ void gamma1_dev(double v, double zmin, double zmax, double delta,
                                           unsigned long long* clamps, uint64_t& lo, uint64_t& hi) {
  const double R = __dsub_rn(zmax, zmin);
  const double d = __ddiv_rn(__dsub_rn(clamp_q(v, zmin, zmax, clamps), zmin), __dmul_rn(R, R));
  const double t = round(__dmul_rn(__dmul_rn(delta, delta), d));
  // exact double -> u128 (t is a non-negative integer-valued double)
  if (t < 18446744073709551616.0) {
    lo = (uint64_t)t;
    hi = 0;
  } else {
    const double h = floor(__dmul_rn(t, 0x1p-64));
    hi = (uint64_t)h;
    lo = (uint64_t)__dsub_rn(t, __dmul_rn(h, 0x1p64));
  }
}

struct EncPrepArgs {
  const uint32_t* m;  // count x m_limbs, or null when quantizing
  int m_limbs;
  const double* v;    // values to quantize (nullable)
  double zmin, zmax, delta;
  int fine;
  uint32_t* m_out;    // count x m_out_limbs (quantized plaintexts), nullable
  int m_out_limbs;
  uint64_t* q_out;    // quantized integers for the caller (nullable)
  unsigned long long* clamps;
  const uint32_t* r;  // count x L
  const uint32_t* n;  // L limbs (device)
  int L;
  int32_t* st;        // count
  int count;
};

__global__ void enc_prep_kernel(const __grid_constant__ EncPrepArgs P) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    int status = PCB_OK;
    if (P.v) {
      const double v = P.v[i];
      uint64_t lo = 0, hi = 0;
      if (!isfinite(v)) {
        status = PCB_E_SHAPE;  // clamp_in: "non-finite value into quantizer" (quantize.cpp:18-19)
      } else if (P.fine) {
        gamma1_dev(v, P.zmin, P.zmax, P.delta, P.clamps, lo, hi);
        if (P.q_out) {
          P.q_out[2 * (size_t)i] = lo;
          P.q_out[2 * (size_t)i + 1] = hi;
        }
      } else {
        lo = gamma2_dev(v, P.zmin, P.zmax, P.delta, P.clamps);
        if (P.q_out) P.q_out[i] = lo;
      }
      uint32_t w[4] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32)};
      if (P.m_out) {
        uint32_t* mo = P.m_out + (size_t)i * P.m_out_limbs;
        for (int j = 0; j < P.m_out_limbs; j++) mo[j] = j < 4 ? w[j] : 0u;
      }
      if (status == PCB_OK && !lt_words(w, 4, P.n, P.L)) status = PCB_E_PLAINTEXT_RANGE;
    } else if (!lt_words(P.m + (size_t)i * P.m_limbs, P.m_limbs, P.n, P.L)) {
      status = PCB_E_PLAINTEXT_RANGE;  // check_plaintext (paillier.cpp:241-243)
    }
    if (status == PCB_OK) {
      const uint32_t* r = P.r + (size_t)i * P.L;
      if (is_zero_words(r, P.L) || !lt_words(r, P.L, P.n, P.L)) status = PCB_E_RANDOMNESS_RANGE;
    }
    P.st[i] = status;
  }
}

template <int S>
struct GarnerArgs {
  ModCtx<S> mp, mq;
  uint32_t inv[S];      // (p^2)^-1 mod q^2, plain
  const uint32_t* cp;   // count x S
  const uint32_t* cq;   // count x S
  const int32_t* st;
  uint32_t* c;          // count x 2L
  int L, count;
};

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) garner_kernel(const __grid_constant__ GarnerArgs<S> P) {
  extern __shared__ __align__(16) uint32_t smem[];
  smod_fill<S>(smem, P.mp.m);
  smod_fill<S>(smem + S, P.mq.m);
  __syncthreads();
  const SMod<S> Mp{smem_addr(smem), P.mp.minv}, Mq{smem_addr(smem + S), P.mq.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + 2 * S;
  const Slot<S> A{smem_addr(slots + warp * (64 * S) + lane * 4)};
  const Slot<S> B{smem_addr(slots + warp * (64 * S) + 32 * S + lane * 4)};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    uint32_t* out = P.c + (size_t)i * 2 * P.L;
    if (P.st[i] != PCB_OK) {
      for (int j = 0; j < 2 * P.L; j++) out[j] = 0;
      continue;
    }
    uint32_t T[S], U[S];
    B.store_const(P.mq.r2);
    A.store_global(P.cq + (size_t)i * S, S);
    mont_mul_ss<S, false, SMod<S>>(T, A, B, Mq);  // c_q R mod q^2
    A.store_global(P.cp + (size_t)i * S, S);
    mont_mul_ss<S, false, SMod<S>>(U, A, B, Mq);  // c_p R mod q^2 (c_p < p^2 < R)
    mod_sub<S, SMod<S>>(T, U, Mq);
    A.store(T);
    B.store_const(P.inv);
    mont_mul_ss<S, false, SMod<S>>(T, A, B, Mq);  // t = (c_q - c_p) (p^2)^-1 mod q^2, plain
    B.store(T);
    const uint32_t* cps = P.cp + (size_t)i * S;
#pragma unroll
    for (int j = 0; j < S; j++) U[j] = cps[j];
    uint32_t H[S];
    mul_add_smod<S>(H, U, B, Mp);  // c = c_p + p^2 t; low words left in B
    const int cl = 2 * P.L;
#pragma unroll
    for (int j = 0; j < S; j++)
      if (j < cl) out[j] = B.digit(j);
#pragma unroll
    for (int j = 0; j < S; j++)
      if (S + j < cl) out[S + j] = H[j];
  }
}

struct DecPrepArgs {
  const uint32_t* c;   // count x 2L
  const uint32_t* n2;  // 2L limbs (device)
  int L;
  int32_t* st;
  int count;
};

__global__ void dec_prep_kernel(const __grid_constant__ DecPrepArgs P) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x)
    P.st[i] = lt_words(P.c + (size_t)i * 2 * P.L, 2 * P.L, P.n2, 2 * P.L) ? PCB_OK : PCB_E_CIPHER_RANGE;
}

template <int S>
struct DecFinishArgs {
  ModCtx<S / 2> sp, sq;     // p, q
  uint32_t pinv_lo[S / 2];  // p^-1 mod 2^(16 S)
  uint32_t qinv_lo[S / 2];
  uint32_t hp[S / 2];       // h_p R_h mod p
  uint32_t hq[S / 2];
  uint32_t pinvq[S / 2];    // p^-1 mod q, plain
  uint32_t p[S / 2], q[S / 2];
  const uint32_t* xp;       // count x S: c^(p-1) mod p^2
  const uint32_t* xq;
  int32_t* st;
  uint32_t* m;              // count x L
  int L, count;
};

// u = (x - 1) / prime exactly (false if prime does not divide x - 1), then mh = u h mod prime.
template <int S>
__device__ __forceinline__ bool l_half(uint32_t (&Mh)[S / 2], const uint32_t* xsrc, const uint32_t* inv_lo,
                                       const uint32_t* prime, const uint32_t* h, const Slot<S / 2>& A,
                                       const Slot<S / 2>& B, const SMod<S / 2>& M1) {
  constexpr int H = S / 2;
  uint32_t X[S];
#pragma unroll
  for (int j = 0; j < S; j++) X[j] = xsrc[j];
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
    mul_lo<H>(U, lo, inv_lo);  // (x - 1) prime^-1 mod 2^(32H)
  }
  ok = mul_eq<H>(U, prime, X) && ok;  // exact division  <=>  x == 1 mod prime
  A.store(U);
  B.store_const(h);
  mont_mul_ss<H, true, SMod<H>>(Mh, A, B, M1);  // u h mod prime
  return ok;
}

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) dec_finish_kernel(const __grid_constant__ DecFinishArgs<S> P) {
  constexpr int H = S / 2;
  extern __shared__ __align__(16) uint32_t smem[];
  smod_fill<H>(smem, P.sp.m);
  smod_fill<H>(smem + H, P.sq.m);
  __syncthreads();
  const SMod<H> Sp{smem_addr(smem), P.sp.minv}, Sq{smem_addr(smem + H), P.sq.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + 2 * H;
  const Slot<H> A{smem_addr(slots + warp * (64 * H) + lane * 4)};
  const Slot<H> B{smem_addr(slots + warp * (64 * H) + 32 * H + lane * 4)};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    uint32_t* out = P.m + (size_t)i * P.L;
    if (P.st[i] != PCB_OK) {
      for (int j = 0; j < P.L; j++) out[j] = 0;
      continue;
    }
    uint32_t Mp[H], Mq[H];
    bool ok = l_half<S>(Mp, P.xp + (size_t)i * S, P.pinv_lo, P.p, P.hp, A, B, Sp);
    ok = l_half<S>(Mq, P.xq + (size_t)i * S, P.qinv_lo, P.q, P.hq, A, B, Sq) && ok;
    if (!ok) {
      P.st[i] = PCB_E_NOT_UNIT;  // l_function (paillier.cpp:34-41)
      for (int j = 0; j < P.L; j++) out[j] = 0;
      continue;
    }
    // m = m_p + p ((m_q - m_p) p^-1 mod q)
    uint32_t T[H], U[H];
    B.store_const(P.sq.r2);
    A.store(Mq);
    mont_mul_ss<H, true, SMod<H>>(T, A, B, Sq);  // m_q R mod q
    A.store(Mp);
    mont_mul_ss<H, true, SMod<H>>(U, A, B, Sq);  // m_p R mod q
    mod_sub<H, SMod<H>>(T, U, Sq);
    A.store(T);
    B.store_const(P.pinvq);
    mont_mul_ss<H, true, SMod<H>>(T, A, B, Sq);  // t, plain
    B.store(T);
    uint32_t Hi[H];
    mul_add_smod<H>(Hi, Mp, B, Sp);
#pragma unroll
    for (int j = 0; j < H; j++)
      if (j < P.L) out[j] = B.digit(j);
#pragma unroll
    for (int j = 0; j < H; j++)
      if (H + j < P.L) out[H + j] = Hi[j];
  }
}

// ------------------------------------------------------------------------------------------
// Master block update (protocol.cpp:494-511): range gate, inverse quantization, soft threshold.
// FP64 in the reference's operation order (built with --fmad=false).
// ------------------------------------------------------------------------------------------
// (double)u128, correctly rounded (__floatuntidf semantics)
__device__ __forceinline__ double u128_to_double_rn(uint64_t lo, uint64_t hi) {
  if (hi == 0) return __ull2double_rn(lo);
  const int sh = 64 - __clzll((long long)hi);            // bits held by hi (1..64)
  uint64_t top = (hi << (64 - sh)) | (sh == 64 ? 0ull : (lo >> sh));
  if (sh == 64) top = hi;
  const uint64_t rest = sh == 64 ? lo : (lo << (64 - sh));
  top |= rest != 0 ? 1ull : 0ull;                          // sticky bit below the rounding point
  return scalbn(__ull2double_rn(top), sh);
}

// BigNat::to_double (bignat.cpp:56-60): limb-wise v = v * 2^64 + (double)limb, top limb first
__device__ __forceinline__ double bignat_to_double(uint64_t lo, uint64_t hi) {
  double v = 0.0;
  if (hi) v = __dadd_rn(__dmul_rn(v, 18446744073709551616.0), __ull2double_rn(hi));
  return __dadd_rn(__dmul_rn(v, 18446744073709551616.0), __ull2double_rn(lo));
}

struct UpdateArgs {
  const uint32_t* m;       // decrypted updates, count x L
  int L;
  const uint64_t* rowsum;  // Gamma2(B) row sums
  const uint64_t* q_z;
  const uint64_t* q_nv;
  const double* sum_zv;    // per block (sequential sums, computed by sumzv_kernel)
  const long long* seg;    // nseg + 1 block offsets (rows of block s: [seg[s], seg[s+1]))
  int nseg;
  double zmin, zmax, delta, kappa;
  double* x;
  double* z;
  double* v;
  int32_t* st;
  int count;
};

// sum_j (2 zmin + step (q_z[j] + q_nv[j])) in the reference's sequential order (quantize.cpp:96-99)
// one thread per block of the batch
__global__ void sumzv_kernel(const uint64_t* q_z, const uint64_t* q_nv, const long long* seg, int nseg, double zmin,
                             double zmax, double delta, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nseg) return;
  const double step = __ddiv_rn(__dsub_rn(zmax, zmin), delta);
  double s = 0.0;
  for (long long j = seg[b]; j < seg[b + 1]; j++)
    s = __dadd_rn(s, __dadd_rn(__dmul_rn(2.0, zmin),
                               __dmul_rn(step, __dadd_rn(__ull2double_rn(q_z[j]), __ull2double_rn(q_nv[j])))));
  out[b] = s;
}

// inverse_quantize_x for one row (quantize.cpp:105-110): the reference's operation order, no FMA
__device__ __forceinline__ double inverse_x_row(uint64_t lo, uint64_t hi, uint64_t rowsum, double cols, double szv,
                                                double zmin, double step, double step2) {
  const double rowsum_b = __dadd_rn(__dmul_rn(cols, zmin), __dmul_rn(step, __ull2double_rn(rowsum)));
  return __dsub_rn(__dadd_rn(__dmul_rn(u128_to_double_rn(lo, hi), step2),
                             __dmul_rn(zmin, __dadd_rn(__dadd_rn(1.0, __dmul_rn(2.0, rowsum_b)), szv))),
                   __dmul_rn(__dmul_rn(__dmul_rn(2.0, zmin), zmin), cols));
}

__global__ void update_kernel(const __grid_constant__ UpdateArgs P) {
  const double range = __dsub_rn(P.zmax, P.zmin);
  const double step = __ddiv_rn(range, P.delta);
  const double step2 = __dmul_rn(step, step);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    if (P.st[i] != PCB_OK) continue;  // decryption already failed
    int lo_s = 0, hi_s = P.nseg - 1;  // block of row i
    while (lo_s < hi_s) {
      const int mid = (lo_s + hi_s + 1) >> 1;
      if (P.seg[mid] <= i) lo_s = mid; else hi_s = mid - 1;
    }
    const double cols = (double)(P.seg[lo_s + 1] - P.seg[lo_s]);
    // check_update_range cap (protocol.cpp:23-24)
    const double cap = __dadd_rn(__ddiv_rn(__dmul_rn(P.delta, P.delta), range),
                                 __dmul_rn(__dmul_rn(__dmul_rn(cols, P.delta), 2.0), P.delta));
    const double lim = __dadd_rn(__dmul_rn(cap, 1.000001), 4.0);
    const double szv = P.sum_zv[lo_s];
    const uint32_t* w = P.m + (size_t)i * P.L;
    bool wide = false;
    for (int j = 4; j < P.L; j++) wide = wide || w[j] != 0;
    const uint64_t lo = (uint64_t)w[0] | ((uint64_t)(P.L > 1 ? w[1] : 0) << 32);
    const uint64_t hi = (uint64_t)(P.L > 2 ? w[2] : 0) | ((uint64_t)(P.L > 3 ? w[3] : 0) << 32);
    if (wide || (hi >> 63) || bignat_to_double(lo, hi) > lim) {  // bit_length > 127 or above the cap
      P.st[i] = PCB_E_RANGE_UPDATE;
      continue;
    }
    const double xi = inverse_x_row(lo, hi, P.rowsum[i], cols, szv, P.zmin, step, step2);
    // protocol.cpp:504-511 + soft_threshold (admm.cpp:18-22)
    const double xv = __dadd_rn(xi, P.v[i]);
    double zz;
    if (xv > P.kappa)
      zz = __dsub_rn(xv, P.kappa);
    else if (xv < -P.kappa)
      zz = __dadd_rn(xv, P.kappa);
    else
      zz = 0.0;
    P.x[i] = xi;
    P.z[i] = zz;
    P.v[i] = __dsub_rn(xv, zz);
  }
}

pcb_status launch_update(const uint32_t* m, int L, const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                         double zmin, double zmax, double delta, double kappa, double* x, double* z, double* v,
                         int32_t* st, size_t count, const long long* seg_dev, int nseg, cudaStream_t stream) {
  double* szv = nullptr;
  if (auto e = scratch_alloc((size_t)nseg * 8, (void**)&szv, stream)) return e;
  sumzv_kernel<<<(nseg + 127) / 128, 128, 0, stream>>>(q_z, q_nv, seg_dev, nseg, zmin, zmax, delta, szv);
  count_launch();
  UpdateArgs P{m, L, rowsum, q_z, q_nv, szv, seg_dev, nseg, zmin, zmax, delta, kappa, x, z, v, st, (int)count};
  const int grid = (int)std::min<size_t>((count + 255) / 256, 4096);
  update_kernel<<<grid > 0 ? grid : 1, 256, 0, stream>>>(P);
  count_launch();
  scratch_free(szv, stream);
  return cuda_check(cudaGetLastError());
}

// ------------------------------------------------------------------------------------------
// Launchers
// ------------------------------------------------------------------------------------------
static int small_grid(size_t count) {
  size_t b = (count + 255) / 256;
  return (int)(b < 4096 ? (b ? b : 1) : 4096);
}

pcb_status launch_enc_prep(const uint32_t* m, int m_limbs, const double* v, double zmin, double zmax, double delta,
                           int fine, uint32_t* m_out, int m_out_limbs, uint64_t* q_out, unsigned long long* clamps,
                           const uint32_t* r, const uint32_t* n_dev, int L, int32_t* st, size_t count,
                           cudaStream_t stream) {
  EncPrepArgs P{m, m_limbs, v, zmin, zmax, delta, fine, m_out, m_out_limbs, q_out, clamps, r, n_dev, L, st, (int)count};
  enc_prep_kernel<<<small_grid(count), 256, 0, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// gamma2_vec / gamma1_vec alone (pcb_quantize_async): no plaintext limbs, no r / n checks; a
// non-finite value records PCB_E_SHAPE in *err (clamp_in, quantize.cpp:18-19)
__global__ void quantize_kernel(const double* v, int count, double zmin, double zmax, double delta, int fine,
                                uint64_t* q, unsigned long long* clamps, int32_t* err) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const double x = v[i];
    uint64_t lo = 0, hi = 0;
    if (!isfinite(x)) {
      if (err) atomicCAS(err, 0, (int32_t)PCB_E_SHAPE);
    } else if (fine) {
      gamma1_dev(x, zmin, zmax, delta, clamps, lo, hi);
    } else {
      lo = gamma2_dev(x, zmin, zmax, delta, clamps);
    }
    if (fine) {
      q[2 * (size_t)i] = lo;
      q[2 * (size_t)i + 1] = hi;
    } else {
      q[i] = lo;
    }
  }
}

pcb_status launch_quantize(const double* v, size_t count, double zmin, double zmax, double delta, int fine,
                           uint64_t* q, unsigned long long* clamps, int32_t* err, cudaStream_t stream) {
  quantize_kernel<<<small_grid(count), 256, 0, stream>>>(v, (int)count, zmin, zmax, delta, fine, q, clamps, err);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// per-element statuses -> the first failure recorded in *err (the asynchronous ABI forms)
__global__ void status_flag_kernel(const int32_t* st, int count, int32_t* err) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    if (st[i] != PCB_OK) atomicCAS(err, 0, st[i]);
}

pcb_status launch_status_flag(const int32_t* st, size_t count, int32_t* err, cudaStream_t stream) {
  if (!err || count == 0) return PCB_OK;
  status_flag_kernel<<<small_grid(count), 256, 0, stream>>>(st, (int)count, err);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// Online half of an offline/online encryption (pcb_encrypt_rn): out = 1 + m n  (2L words, < n^2
// when m < n), with the checks of crt_encrypt_with_r (paillier.cpp:330-336) applied to m and the
// precomputed rn = r^n mod n^2 (0 < rn < n^2).  Failed elements get out = 0.
struct OnePmnArgs {
  const uint32_t* m;   // count x ml
  int ml;
  const uint32_t* rn;  // count x 2L
  const uint32_t* n;   // L limbs (device)
  const uint32_t* n2;  // 2L limbs (device)
  int L;
  uint32_t* out;       // count x 2L
  int32_t* st;
  int count;
};

__global__ void onepmn_kernel(const __grid_constant__ OnePmnArgs P) {
  const int W = 2 * P.L;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    const uint32_t* mi = P.m + (size_t)i * P.ml;
    const uint32_t* ri = P.rn + (size_t)i * W;
    uint32_t* o = P.out + (size_t)i * W;
    int cmp = 0;  // m vs n
    for (int j = max(P.ml, P.L) - 1; j >= 0 && cmp == 0; j--) {
      const uint32_t a = j < P.ml ? mi[j] : 0u, b = j < P.L ? P.n[j] : 0u;
      cmp = a < b ? -1 : (a > b ? 1 : 0);
    }
    int rc = 0;  // rn vs n^2
    bool nz = false;
    for (int j = W - 1; j >= 0; j--) {
      const uint32_t a = ri[j], b = P.n2[j];
      nz = nz || a != 0;
      if (rc == 0) rc = a < b ? -1 : (a > b ? 1 : 0);
    }
    const int32_t s = cmp >= 0 ? PCB_E_PLAINTEXT_RANGE : ((rc >= 0 || !nz) ? PCB_E_RANDOMNESS_RANGE : PCB_OK);
    P.st[i] = s;
    for (int k = 0; k < W; k++) o[k] = 0;
    if (s != PCB_OK) continue;
    int mt = P.ml < P.L ? P.ml : P.L;
    while (mt > 0 && mi[mt - 1] == 0) mt--;
    for (int a = 0; a < mt; a++) {
      uint64_t carry = 0;
      for (int b = 0; b < P.L; b++) {
        const uint64_t t = (uint64_t)mi[a] * P.n[b] + o[a + b] + carry;
        o[a + b] = (uint32_t)t;
        carry = t >> 32;
      }
      o[a + P.L] = (uint32_t)carry;
    }
    uint64_t c = 1;
    for (int k = 0; k < W && c; k++) {
      const uint64_t t = (uint64_t)o[k] + c;
      o[k] = (uint32_t)t;
      c = t >> 32;
    }
  }
}

pcb_status launch_onepmn(const uint32_t* m, int ml, const uint32_t* rn, const uint32_t* n_dev, const uint32_t* n2_dev,
                         int L, uint32_t* out, int32_t* st, size_t count, cudaStream_t stream) {
  OnePmnArgs P{m, ml, rn, n_dev, n2_dev, L, out, st, (int)count};
  const int grid = (int)std::min<size_t>((count + 127) / 128, 4096);
  onepmn_kernel<<<grid > 0 ? grid : 1, 128, 0, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

pcb_status launch_dec_prep(const uint32_t* c, const uint32_t* n2_dev, int L, int32_t* st, size_t count,
                           cudaStream_t stream) {
  DecPrepArgs P{c, n2_dev, L, st, (int)count};
  dec_prep_kernel<<<small_grid(count), 256, 0, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

template <int S>
pcb_status launch_garner(const CrtEncConsts<S>& k, const uint32_t* cp, const uint32_t* cq, const int32_t* st,
                         uint32_t* c, int L, size_t count, cudaStream_t stream) {
  GarnerArgs<S> P;
  P.mp = k.mp;
  P.mq = k.mq;
  for (int j = 0; j < S; j++) P.inv[j] = k.inv[j];
  P.cp = cp;
  P.cq = cq;
  P.st = st;
  P.c = c;
  P.L = L;
  P.count = (int)count;
  const size_t smem = (size_t)kThreadsPerBlock * S * 8 + 2 * S * 4;
  int blocks = 0;
  if (auto e = item_grid(garner_kernel<S>, smem, count, &blocks)) return e;
  garner_kernel<S><<<blocks, kThreadsPerBlock, smem, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

template <int S>
pcb_status launch_dec_finish(const CrtDecConsts<S>& k, const uint32_t* xp, const uint32_t* xq, int32_t* st,
                             uint32_t* m, int L, size_t count, cudaStream_t stream) {
  constexpr int H = S / 2;
  DecFinishArgs<S> P;
  P.sp = k.sp;
  P.sq = k.sq;
  for (int j = 0; j < H; j++) {
    P.pinv_lo[j] = k.pinv_lo[j];
    P.qinv_lo[j] = k.qinv_lo[j];
    P.hp[j] = k.hp[j];
    P.hq[j] = k.hq[j];
    P.pinvq[j] = k.pinvq[j];
    P.p[j] = k.p[j];
    P.q[j] = k.q[j];
  }
  P.xp = xp;
  P.xq = xq;
  P.st = st;
  P.m = m;
  P.L = L;
  P.count = (int)count;
  const size_t smem = (size_t)kThreadsPerBlock * H * 8 + 2 * H * 4;
  int blocks = 0;
  if (auto e = item_grid(dec_finish_kernel<S>, smem, count, &blocks)) return e;
  dec_finish_kernel<S><<<blocks, kThreadsPerBlock, smem, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// half_pow for exponents e = u (p - 1) (paillier.cpp:275-305 with w = 0): with s = b^(p-1) mod p^2,
// b^e mod p^2 = s^u = 1 + p (L_p(s) u mod p) when p does not divide b (s = 1 + p L_p(s)), and 0 when
// it does (then s = 0: p^2 | b^(p-1), and u >= 1).  u comes per element in Montgomery form u R_h mod p.
template <int S>
struct FermatArgs {
  ModCtx<S / 2> sp;        // p
  uint32_t pinv_lo[S / 2]; // p^-1 mod 2^(16 S)
  uint32_t p[S / 2];
  const uint32_t* s;       // count x S: b^(p-1) mod p^2
  const uint32_t* u;       // count x S/2: u R_h mod p
  uint32_t* out;           // count x S: b^(u (p - 1)) mod p^2
  int count;
};

template <int S>
__global__ void __launch_bounds__(kThreadsPerBlock) fermat_finish_kernel(const __grid_constant__ FermatArgs<S> P) {
  constexpr int H = S / 2;
  extern __shared__ __align__(16) uint32_t smem[];
  smod_fill<H>(smem, P.sp.m);
  __syncthreads();
  const SMod<H> Sp{smem_addr(smem), P.sp.minv};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* slots = smem + H;
  const Slot<H> A{smem_addr(slots + warp * (64 * H) + lane * 4)};
  const Slot<H> B{smem_addr(slots + warp * (64 * H) + 32 * H + lane * 4)};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.count; i += gridDim.x * blockDim.x) {
    const uint32_t* si = P.s + (size_t)i * S;
    uint32_t* out = P.out + (size_t)i * S;
    uint32_t K[H];
    if (!l_half<S>(K, si, P.pinv_lo, P.p, P.u + (size_t)i * H, A, B, Sp)) {
      for (int j = 0; j < S; j++) out[j] = 0;  // s = 0: p | b
      continue;
    }
    B.store(K);
    uint32_t one[H], Hi[H];
#pragma unroll
    for (int j = 0; j < H; j++) one[j] = j == 0 ? 1u : 0u;
    mul_add_smod<H>(Hi, one, B, Sp);  // 1 + p K (< p^2)
#pragma unroll
    for (int j = 0; j < H; j++) out[j] = B.digit(j);
#pragma unroll
    for (int j = 0; j < H; j++) out[H + j] = Hi[j];
  }
}

template <int S>
pcb_status launch_fermat_finish(const ModCtx<S / 2>& sp, const uint32_t* pinv_lo, const uint32_t* p,
                                const uint32_t* s, const uint32_t* u, uint32_t* out, size_t count, cudaStream_t stream) {
  constexpr int H = S / 2;
  FermatArgs<S> P;
  P.sp = sp;
  for (int j = 0; j < H; j++) {
    P.pinv_lo[j] = pinv_lo[j];
    P.p[j] = p[j];
  }
  P.s = s;
  P.u = u;
  P.out = out;
  P.count = (int)count;
  const size_t smem = (size_t)kThreadsPerBlock * H * 8 + H * 4;
  int blocks = 0;
  if (auto e = item_grid(fermat_finish_kernel<S>, smem, count, &blocks)) return e;
  fermat_finish_kernel<S><<<blocks, kThreadsPerBlock, smem, stream>>>(P);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// combined_quantized_update (quantize.cpp:66-82) on the device: q_i = qa_i + sum_j qb_ij (qz_j + qnv_j)
// in u128 (wrapping like the reference's u128 arithmetic), one row per thread
__global__ void combined_update_kernel(const uint64_t* qa, const uint64_t* qb, const uint64_t* qz, const uint64_t* qnv,
                                       size_t rows, size_t cols, uint64_t* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows; i += (size_t)gridDim.x * blockDim.x) {
    unsigned __int128 acc = ((unsigned __int128)qa[2 * i + 1] << 64) | qa[2 * i];
    const uint64_t* row = qb + i * cols;
    for (size_t j = 0; j < cols; j++)
      acc += (unsigned __int128)row[j] * ((unsigned __int128)qz[j] + (unsigned __int128)qnv[j]);
    out[2 * i] = (uint64_t)acc;
    out[2 * i + 1] = (uint64_t)(acc >> 64);
  }
}

pcb_status launch_combined_update(const uint64_t* qa, const uint64_t* qb, const uint64_t* qz, const uint64_t* qnv,
                                  size_t rows, size_t cols, uint64_t* out, cudaStream_t stream) {
  combined_update_kernel<<<small_grid(rows), 256, 0, stream>>>(qa, qb, qz, qnv, rows, cols, out);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// inverse_quantize_x (quantize.cpp:84-112) alone: sum_zv in the reference's sequential order
// (sumzv_kernel, one block), then one row per thread
__global__ void inverse_x_kernel(const uint64_t* q, const uint64_t* rowsum, const double* szv, size_t rows,
                                 double cols, double zmin, double zmax, double delta, double* x) {
  const double step = __ddiv_rn(__dsub_rn(zmax, zmin), delta);
  const double step2 = __dmul_rn(step, step);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows; i += (size_t)gridDim.x * blockDim.x)
    x[i] = inverse_x_row(q[2 * i], q[2 * i + 1], rowsum[i], cols, szv[0], zmin, step, step2);
}

pcb_status launch_inverse_x(const uint64_t* q, const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                            size_t rows, size_t cols, double zmin, double zmax, double delta, double* x,
                            cudaStream_t stream) {
  double* szv = nullptr;
  long long* seg = nullptr;
  pcb_status e = scratch_alloc(8, (void**)&szv, stream);
  if (!e) e = scratch_alloc(16, (void**)&seg, stream);
  const long long hseg[2] = {0, (long long)cols};
  if (!e) e = cuda_check(cudaMemcpyAsync(seg, hseg, 16, cudaMemcpyHostToDevice, stream));
  if (!e) {
    sumzv_kernel<<<1, 128, 0, stream>>>(q_z, q_nv, seg, 1, zmin, zmax, delta, szv);
    count_launch();
    inverse_x_kernel<<<small_grid(rows), 256, 0, stream>>>(q, rowsum, szv, rows, (double)cols, zmin, zmax, delta, x);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) e = cuda_check(cudaStreamSynchronize(stream));  // hseg is a host temporary
  scratch_free(szv, stream);
  scratch_free(seg, stream);
  return e;
}

// r = a mod v per element (Knuth algorithm D, remainder only, 32-bit digits): a is count x aw words,
// v (s >= 2 words) arrives normalised (shifted left by `shift` so its top bit is set); out is
// count x s words.  One element per thread, the dividend window in local memory.  Used for the edge's
// exponent reduction obf mod phi(p^2) (delegated_power, protocol.cpp:15-18), which the reference
// does per element before its modexp.
constexpr int kModMaxWords = 260;
__global__ void mod_words_kernel(const uint32_t* a, int aw, int count, const uint32_t* v, int s, int shift,
                                 uint32_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    uint32_t u[kModMaxWords + 2];
    const uint32_t* ai = a + (size_t)i * aw;
    const int n = aw > s ? aw : s;  // dividend digits (zero-extended to at least s)
    // u = a << shift, n + 1 words
    uint32_t carry = 0;
    for (int k = 0; k < n; k++) {
      const uint32_t w = k < aw ? ai[k] : 0u;
      u[k] = shift ? (w << shift) | carry : w;
      carry = shift ? w >> (32 - shift) : 0u;
    }
    u[n] = carry;
    const uint64_t vt = v[s - 1], vt2 = v[s - 2];
    for (int j = n - s; j >= 0; j--) {
      const uint64_t num = ((uint64_t)u[j + s] << 32) | u[j + s - 1];
      uint64_t qh = num / vt, rh = num % vt;
      while (qh >= (1ull << 32) || qh * vt2 > ((rh << 32) | u[j + s - 2])) {
        qh--;
        rh += vt;
        if (rh >= (1ull << 32)) break;
      }
      // u[j .. j+s] -= qh * v
      int64_t borrow = 0;
      uint64_t mc = 0;
      for (int k = 0; k < s; k++) {
        const uint64_t p = qh * v[k] + mc;
        mc = p >> 32;
        const int64_t t = (int64_t)u[j + k] - (int64_t)(uint32_t)p + borrow;
        u[j + k] = (uint32_t)t;
        borrow = t >> 32;
      }
      const int64_t t = (int64_t)u[j + s] - (int64_t)mc + borrow;
      u[j + s] = (uint32_t)t;
      if (t < 0) {  // qh was one too large: add v back
        uint64_t c2 = 0;
        for (int k = 0; k < s; k++) {
          const uint64_t t2 = (uint64_t)u[j + k] + v[k] + c2;
          u[j + k] = (uint32_t)t2;
          c2 = t2 >> 32;
        }
        u[j + s] += (uint32_t)c2;
      }
    }
    uint32_t* o = out + (size_t)i * s;  // remainder = u[0 .. s) >> shift
    for (int k = 0; k < s; k++)
      o[k] = shift ? (u[k] >> shift) | (u[k + 1] << (32 - shift)) : u[k];
  }
}

pcb_status launch_mod_words(const uint32_t* a, int aw, size_t count, const uint32_t* v_norm, int s, int shift,
                            uint32_t* out, cudaStream_t stream) {
  if (s < 2 || aw + 1 > kModMaxWords || s + 1 > kModMaxWords) return PCB_E_UNSUPPORTED;
  mod_words_kernel<<<small_grid(count), 128, 0, stream>>>(a, aw, (int)count, v_norm, s, shift, out);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// out_i = a_i * b + 1 (a_i: aw words per element, b: bw words shared, out: aw + bw words), schoolbook
// per thread -- the binomial collapse of a delegated g power (pcb_delegated_power_binomial)
__global__ void mul_add1_kernel(const uint32_t* a, int aw, const uint32_t* b, int bw, int count, uint32_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint32_t* x = a + (size_t)i * aw;
    uint32_t* o = out + (size_t)i * (aw + bw);
    for (int k = 0; k < aw + bw; k++) o[k] = 0;
    for (int u = 0; u < aw; u++) {
      const uint64_t xu = x[u];
      if (!xu) continue;
      uint64_t carry = 0;
      for (int v = 0; v < bw; v++) {
        const uint64_t t = xu * b[v] + o[u + v] + carry;
        o[u + v] = (uint32_t)t;
        carry = t >> 32;
      }
      o[u + bw] = (uint32_t)carry;
    }
    uint64_t c = 1;
    for (int k = 0; k < aw + bw && c; k++) {
      const uint64_t t = (uint64_t)o[k] + c;
      o[k] = (uint32_t)t;
      c = t >> 32;
    }
  }
}

pcb_status launch_mul_add1(const uint32_t* a, int aw, const uint32_t* b, int bw, size_t count, uint32_t* out,
                           cudaStream_t stream) {
  mul_add1_kernel<<<small_grid(count), 128, 0, stream>>>(a, aw, b, bw, (int)count, out);
  count_launch();
  return cuda_check(cudaGetLastError());
}

// obfuscate_exponent (protocol.cpp:11-13): out = value + mask * n_eps, per element (value: vw words,
// mask: u64, n_eps: nw words shared, out: ow words, ow >= nw + 3)
__global__ void obfuscate_kernel(const uint32_t* value, int vw, const uint64_t* mask, const uint32_t* neps, int nw,
                                 int count, uint32_t* out, int ow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint64_t mk = mask[i];
    const uint32_t m0 = (uint32_t)mk, m1 = (uint32_t)(mk >> 32);
    const uint32_t* v = value + (size_t)i * vw;
    uint32_t* o = out + (size_t)i * ow;
    // o = v + m0 * neps + (m1 * neps << 32): column k takes lo(m0 N[k]) + lo(m1 N[k-1]) and the
    // high halves of the previous column's two products
    uint64_t carry = 0;
    uint32_t hb = 0;  // hi(m1 N[k-2]) for column k
    for (int k = 0; k < ow; k++) {
      const uint64_t a = k < nw ? (uint64_t)m0 * neps[k] : 0ull;
      const uint64_t b = (k >= 1 && k - 1 < nw) ? (uint64_t)m1 * neps[k - 1] : 0ull;
      const uint64_t t = (uint64_t)(k < vw ? v[k] : 0u) + (uint32_t)a + (uint32_t)b + carry + hb;
      o[k] = (uint32_t)t;
      carry = (t >> 32) + (a >> 32);
      hb = (uint32_t)(b >> 32);
    }
  }
}

pcb_status launch_obfuscate(const uint32_t* value, int vw, const uint64_t* mask, const uint32_t* neps, int nw,
                            size_t count, uint32_t* out, int ow, cudaStream_t stream) {
  obfuscate_kernel<<<small_grid(count), 256, 0, stream>>>(value, vw, mask, neps, nw, (int)count, out, ow);
  count_launch();
  return cuda_check(cudaGetLastError());
}

#define PCB_INSTANTIATE(S)                                                                                         \
  template pcb_status launch_garner<S>(const CrtEncConsts<S>&, const uint32_t*, const uint32_t*, const int32_t*,  \
                                       uint32_t*, int, size_t, cudaStream_t);                                      \
  template pcb_status launch_dec_finish<S>(const CrtDecConsts<S>&, const uint32_t*, const uint32_t*, int32_t*,    \
                                           uint32_t*, int, size_t, cudaStream_t);                                  \
  template pcb_status launch_fermat_finish<S>(const ModCtx<S / 2>&, const uint32_t*, const uint32_t*,             \
                                              const uint32_t*, const uint32_t*, uint32_t*, size_t, cudaStream_t);
PCB_INSTANTIATE(32)
PCB_INSTANTIATE(64)
PCB_INSTANTIATE(96)
PCB_INSTANTIATE(128)

}  // namespace pcb
