// prime.cu — Miller-Rabin rounds of key generation on the device.
//
// random_prime (bignat.cpp:497-515) draws a candidate, marches it upward in steps of 2 and runs
// is_probable_prime (bignat.cpp:458-495) on each: trial division, then up to 40 rounds
// x = a^d mod n with bases a drawn from the same splitmix64 stream.  The stream makes the search
// serial, so host/hbn.cpp (random_prime_batched) speculates: the first rounds of the next 16
// marches' survivors form one batch, the remaining rounds of the first candidate that passes
// form a second, and the stream is committed / rewound exactly as the reference consumes it.
// This file evaluates a batch: one thread per (modulus, exponent, base) triple, CIOS Montgomery
// over L u32 limbs with a 4-bit fixed window; R mod n, R^2 mod n and -n^-1 mod 2^32 come from the
// host (they are per-candidate one-off constants).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "host/hbn.hpp"
#include "pcb_internal.h"

namespace pcb {
namespace {

template <int L>
__device__ void mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* n, uint32_t ninv, uint32_t* out) {
  uint32_t t[L + 2];
#pragma unroll
  for (int j = 0; j < L + 2; j++) t[j] = 0;
  for (int i = 0; i < L; i++) {
    uint64_t c = 0;
    const uint32_t bi = b[i];
#pragma unroll
    for (int j = 0; j < L; j++) {
      c += (uint64_t)a[j] * bi + t[j];
      t[j] = (uint32_t)c;
      c >>= 32;
    }
    c += t[L];
    t[L] = (uint32_t)c;
    t[L + 1] = (uint32_t)(c >> 32);
    const uint32_t m = t[0] * ninv;
    c = (uint64_t)m * n[0] + t[0];
    c >>= 32;
#pragma unroll
    for (int j = 1; j < L; j++) {
      c += (uint64_t)m * n[j] + t[j];
      t[j - 1] = (uint32_t)c;
      c >>= 32;
    }
    c += t[L];
    t[L - 1] = (uint32_t)c;
    t[L] = t[L + 1] + (uint32_t)(c >> 32);
  }
  // t < 2n: subtract n once if t >= n
  bool ge = t[L] != 0;
  if (!ge) {
    ge = true;
    for (int j = L - 1; j >= 0; j--)
      if (t[j] != n[j]) {
        ge = t[j] > n[j];
        break;
      }
  }
  if (ge) {
    int64_t br = 0;
#pragma unroll
    for (int j = 0; j < L; j++) {
      const int64_t v = (int64_t)t[j] - n[j] + br;
      out[j] = (uint32_t)v;
      br = v >> 32;
    }
  } else {
#pragma unroll
    for (int j = 0; j < L; j++) out[j] = t[j];
  }
}

// x_i = a_i^d_i mod n_i; all arrays count x L limbs (LE), r1 = R mod n, r2 = R^2 mod n, R = 2^(32L)
template <int L>
__global__ void __launch_bounds__(64) mr_pow_kernel(const uint32_t* __restrict__ n, const uint32_t* __restrict__ ninv,
                                                    const uint32_t* __restrict__ r1, const uint32_t* __restrict__ r2,
                                                    const uint32_t* __restrict__ a, const uint32_t* __restrict__ d,
                                                    uint32_t* __restrict__ x, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint32_t N[L], tab[16][L], acc[L], tmp[L];
  const size_t o = (size_t)i * L;
  for (int j = 0; j < L; j++) N[j] = n[o + j];
  const uint32_t ni = ninv[i];
  for (int j = 0; j < L; j++) {
    tab[0][j] = r1[o + j];  // 1 in Montgomery form
    tmp[j] = a[o + j];
    acc[j] = r2[o + j];
  }
  mont_mul<L>(tmp, acc, N, ni, tab[1]);  // a R mod n
  for (int k = 2; k < 16; k++) mont_mul<L>(tab[k - 1], tab[1], N, ni, tab[k]);
  int top = L - 1;
  while (top > 0 && d[o + top] == 0) top--;
  for (int j = 0; j < L; j++) acc[j] = tab[0][j];
  bool started = false;
  for (int w = top; w >= 0; w--) {
    const uint32_t word = d[o + w];
    for (int nib = 7; nib >= 0; nib--) {
      const uint32_t v = (word >> (4 * nib)) & 15u;
      if (started)
        for (int s = 0; s < 4; s++) {
          mont_mul<L>(acc, acc, N, ni, tmp);
          for (int j = 0; j < L; j++) acc[j] = tmp[j];
        }
      if (v) {
        mont_mul<L>(acc, tab[v], N, ni, tmp);
        for (int j = 0; j < L; j++) acc[j] = tmp[j];
        started = true;
      }
    }
  }
  for (int j = 0; j < L; j++) tmp[j] = j == 0 ? 1u : 0u;
  mont_mul<L>(acc, tmp, N, ni, acc);  // out of Montgomery form
  for (int j = 0; j < L; j++) x[o + j] = acc[j];
}

template <int L>
pcb_status launch_mr(const uint32_t* n, const uint32_t* ninv, const uint32_t* r1, const uint32_t* r2, const uint32_t* a,
                     const uint32_t* d, uint32_t* x, int count, cudaStream_t st) {
  mr_pow_kernel<L><<<(count + 63) / 64, 64, 0, st>>>(n, ninv, r1, r2, a, d, x, count);
  count_launch();
  return cuda_check(cudaGetLastError());
}

struct DevPow {
  int device;
  cudaStream_t st;
  pcb_status err;
};

// the MrPow callback of random_prime_batched, on the device
bool device_pow(const MrBatch& b, std::vector<HBN>& x, void* user) {
  DevPow* u = (DevPow*)user;
  const size_t cnt = b.n.size();
  size_t maxb = 0;
  for (const HBN& n : b.n) maxb = std::max(maxb, n.bit_length());
  const int L = maxb <= 512 ? 16 : maxb <= 1024 ? 32 : maxb <= 1536 ? 48 : 64;
  if (maxb > 2048) {
    u->err = PCB_E_SHAPE;
    return false;
  }
  std::vector<uint32_t> hn(cnt * L), hi(cnt), h1(cnt * L), h2(cnt * L), ha(cnt * L), hd(cnt * L), hx(cnt * L);
  const HBN R = HBN(1) << (32 * L), R2 = HBN(1) << (64 * L);
  for (size_t i = 0; i < cnt; i++) {
    b.n[i].to_limbs(&hn[i * L], L);
    mod(R, b.n[i]).to_limbs(&h1[i * L], L);
    mod(R2, b.n[i]).to_limbs(&h2[i * L], L);
    mod(b.a[i], b.n[i]).to_limbs(&ha[i * L], L);
    b.d[i].to_limbs(&hd[i * L], L);
    uint32_t n0 = hn[i * L], inv = 1;
    for (int k = 0; k < 5; k++) inv *= 2u - n0 * inv;  // n0^-1 mod 2^32 (Newton)
    hi[i] = 0u - inv;
  }
  uint32_t* dv = nullptr;
  const size_t words = cnt * L;
  int prev_dev = 0;
  cudaGetDevice(&prev_dev);  // the caller's current device is restored below
  pcb_status e = cuda_check(cudaSetDevice(u->device));
  if (!e) e = scratch_alloc((5 * words + cnt) * 4, (void**)&dv, u->st);
  uint32_t *dn = dv, *d1 = dv + words, *d2 = dv + 2 * words, *da = dv + 3 * words, *dd = dv + 4 * words,
           *di = dv + 5 * words;
  uint32_t* dxo = nullptr;
  if (!e) e = scratch_alloc(words * 4, (void**)&dxo, u->st);
  auto up = [&](uint32_t* dst, const std::vector<uint32_t>& src) {
    if (!e) e = cuda_check(cudaMemcpyAsync(dst, src.data(), src.size() * 4, cudaMemcpyHostToDevice, u->st));
  };
  up(dn, hn);
  up(d1, h1);
  up(d2, h2);
  up(da, ha);
  up(dd, hd);
  up(di, hi);
  if (!e) {
    if (L == 16) e = launch_mr<16>(dn, di, d1, d2, da, dd, dxo, (int)cnt, u->st);
    if (L == 32) e = launch_mr<32>(dn, di, d1, d2, da, dd, dxo, (int)cnt, u->st);
    if (L == 48) e = launch_mr<48>(dn, di, d1, d2, da, dd, dxo, (int)cnt, u->st);
    if (L == 64) e = launch_mr<64>(dn, di, d1, d2, da, dd, dxo, (int)cnt, u->st);
  }
  if (!e) e = cuda_check(cudaMemcpyAsync(hx.data(), dxo, words * 4, cudaMemcpyDeviceToHost, u->st));
  if (!e) e = cuda_check(cudaStreamSynchronize(u->st));
  scratch_free(dv, u->st);
  scratch_free(dxo, u->st);
  cudaSetDevice(prev_dev);
  if (e) {
    u->err = e;
    return false;
  }
  x.resize(cnt);
  for (size_t i = 0; i < cnt; i++) x[i] = HBN::from_limbs(&hx[i * L], L);
  return true;
}

// the checker's evaluation of the same batches (CPU tests pin the speculation with it)
bool host_pow(const MrBatch& b, std::vector<HBN>& x, void*) {
  x.resize(b.n.size());
  for (size_t i = 0; i < b.n.size(); i++) x[i] = pow_mod(b.a[i], b.d[i], b.n[i]);
  return true;
}

}  // namespace
}  // namespace pcb

extern "C" {

pcb_status pcb_random_prime_speculative(uint64_t* rng_state, uint32_t bits, int device, uint32_t* out) {
  PCB_RANGE("pcb_random_prime_speculative");
  using namespace pcb;
  if (!rng_state || !out || bits < 2) return PCB_E_SHAPE;
  if (bits > 2048) return PCB_E_SHAPE;
  HRng rng(*rng_state);
  HBN p;
  DevPow u{device, nullptr, PCB_OK};
  try {
    if (!random_prime_batched(rng, bits, 40, 16, device >= 0 ? device_pow : host_pow, &u, p))
      return u.err ? u.err : PCB_E_CUDA;
  } catch (...) {
    return PCB_E_SHAPE;
  }
  p.to_limbs(out, (bits + 31) / 32);
  *rng_state = rng.state;
  return PCB_OK;
}

pcb_status pcb_keygen_speculative(uint64_t* rng_state, uint32_t key_bits, int device, uint32_t* n, uint32_t* p,
                                  uint32_t* q) {
  PCB_RANGE("pcb_keygen_speculative");
  using namespace pcb;
  if (!rng_state || !n || !p || !q) return PCB_E_SHAPE;
  HRng rng(*rng_state);
  HBN pp, qq;
  DevPow u{device, nullptr, PCB_OK};
  try {
    if (key_bits != 64 && key_bits != 1024 && key_bits != 2048 && key_bits != 4096) return PCB_E_SHAPE;
    if (!keygen_batched(rng, key_bits, device >= 0 ? device_pow : host_pow, &u, pp, qq))
      return u.err ? u.err : PCB_E_CUDA;
  } catch (...) {
    return PCB_E_SHAPE;
  }
  const size_t L = key_bits / 32;
  (pp * qq).to_limbs(n, L);
  pp.to_limbs(p, L / 2);
  qq.to_limbs(q, L / 2);
  *rng_state = rng.state;
  return PCB_OK;
}

}  // extern "C"
