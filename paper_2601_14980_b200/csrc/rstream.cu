// rstream.cu — count x Paillier::sample_r(rng) on the GPU, bit-identical to the reference's
// serial draw loop (paillier.cpp:233-239 + 497-500, bignat.cpp:388-445).
//
// The reference consumes the splitmix64 stream in fixed blocks of W = ceil(bits(n)/64) words:
// random_below(n) draws random_bits(bits(n)) (W words, little-endian, top word masked) until the
// candidate is < n, and sample_r additionally rejects 0 and gcd(r, n) != 1.  So the stream is a
// sequence of independent W-word candidates and r_i is the i-th accepted one.  splitmix64 is
// counter based (state_j = state_0 + j * gamma), so every candidate is generated independently:
//
//   1. flag_kernel     : candidate k -> accept flag (< n, != 0, p does not divide, q does not)
//   2. cub ExclusiveSum: rank of every accepted candidate
//   3. emit_kernel     : regenerate accepted candidates and scatter them to r_out[rank]
//
// and the final Rng state is state_0 + (index of the count-th accepted candidate + 1) * W * gamma.
// Divisibility uses Montgomery REDC with modulus p (cand < n = p q < p 2^(32H)): REDC(cand) =
// cand 2^(-32H) mod p, which is 0 iff p | cand.  Public-key-only contexts use a binary gcd, one
// warp per candidate (rs_flag_pub_kernel).
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "pcb_internal.h"

namespace pcb {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct RsArgs {
  uint64_t state0;      // Rng::state before the first draw
  uint64_t block0;      // first candidate index of this launch
  int nblocks;          // candidates in this launch
  int W;                // u64 words per candidate
  uint64_t topmask;     // mask of the top word (bits % 64 != 0)
  int L;                // n limbs (u32)
  uint32_t n[128];      // n (LE u32, L limbs; <= 4096-bit keys)
  int has_prv;
  int H;                // p, q limbs
  uint32_t p[64], q[64];
  uint32_t pinv, qinv;  // -p^-1, -q^-1 mod 2^32
  int32_t* flags;       // nblocks
  const int32_t* rank;  // nblocks (emit pass)
  uint32_t* r_out;      // count x L (emit pass)
  int count;
};

// candidate k (absolute index) as L u32 limbs
__device__ __forceinline__ void gen_candidate(const RsArgs& P, uint64_t k, uint32_t* c) {
  const uint64_t j0 = k * (uint64_t)P.W;
  for (int w = 0; w < P.W; w++) {
    uint64_t v = mix64(P.state0 + (j0 + w + 1) * kGamma);
    if (w == P.W - 1) v &= P.topmask;
    if (2 * w < P.L) c[2 * w] = (uint32_t)v;
    if (2 * w + 1 < P.L) c[2 * w + 1] = (uint32_t)(v >> 32);
  }
}

// REDC_p(c): c (L limbs, c < p 2^(32H)) -> c 2^(-32H) mod p; returns true iff the result is 0.
__device__ bool divisible(const uint32_t* c, int L, const uint32_t* p, uint32_t pinv, int H) {
  uint32_t t[2 * 64 + 2];
  for (int i = 0; i < 2 * H + 2; i++) t[i] = i < L ? c[i] : 0u;
  for (int i = 0; i < H; i++) {
    const uint32_t q = t[i] * pinv;
    uint64_t carry = 0;
    for (int j = 0; j < H; j++) {
      const uint64_t s = (uint64_t)q * p[j] + t[i + j] + carry;
      t[i + j] = (uint32_t)s;
      carry = s >> 32;
    }
    for (int j = i + H; carry && j < 2 * H + 2; j++) {
      const uint64_t s = (uint64_t)t[j] + carry;
      t[j] = (uint32_t)s;
      carry = s >> 32;
    }
  }
  // result = t[H .. 2H] < 2p; it is 0 mod p iff it equals 0 or p
  bool zero = true, eqp = true;
  for (int j = 0; j <= H; j++) {
    const uint32_t w = t[H + j];
    zero = zero && w == 0;
    eqp = eqp && w == (j < H ? p[j] : 0u);
  }
  return zero || eqp;
}

// ---- public-key contexts: gcd(r, n) by a warp-cooperative binary gcd ------------------------------
// One warp per candidate; lane i holds bits [128 i, 128 i + 128) of a and b (<= 4096-bit n).  The
// multi-word primitives are warp collectives: zero test and comparison by ballot, the borrow chain of
// a - b by carry-lookahead on the ballot masks (borrow into lane i = bit i of (G + X) ^ X ^ G with
// G = lanes that generate a borrow, X = G | lanes that propagate one), and the shift by the trailing
// zero count through shuffles.  The per-thread version kept 2 x L limbs in local memory and shifted
// one bit at a time (~240 ms for 600 candidates of 2048 bits).
struct W128 {
  uint64_t lo, hi;
};
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool w_is_zero(const W128& a) { return !__any_sync(kFull, (a.lo | a.hi) != 0); }

// sign of a - b
__device__ __forceinline__ int w_cmp(const W128& a, const W128& b) {
  const unsigned m = __ballot_sync(kFull, a.lo != b.lo || a.hi != b.hi);
  if (!m) return 0;
  const int h = 31 - __clz(m);
  const bool gt = a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo);
  return __shfl_sync(kFull, (int)gt, h) ? 1 : -1;
}

// a - b for a >= b
__device__ __forceinline__ W128 w_sub(const W128& a, const W128& b, int lane) {
  const uint64_t lo = a.lo - b.lo;
  uint64_t hi = a.hi - b.hi - (uint64_t)(a.lo < b.lo);
  const bool gen = a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
  const bool prop = a.hi == b.hi && a.lo == b.lo;
  const unsigned G = __ballot_sync(kFull, gen), X = G | __ballot_sync(kFull, prop);
  const uint64_t bin = (((G + X) ^ X ^ G) >> lane) & 1u;
  hi -= (uint64_t)(lo < bin);
  return W128{lo - bin, hi};
}

// a >> (its trailing zero count), a != 0
__device__ __forceinline__ W128 w_strip(const W128& a, int lane) {
  const unsigned m = __ballot_sync(kFull, (a.lo | a.hi) != 0);
  const int f = __ffs(m) - 1;
  const int t0 = a.lo ? __ffsll((long long)a.lo) - 1 : 64 + __ffsll((long long)a.hi) - 1;
  const int tz = 128 * f + __shfl_sync(kFull, t0, f);
  if (tz == 0) return a;
  const int d = tz >> 7;
  int s = tz & 127;
  uint64_t x0 = __shfl_down_sync(kFull, a.lo, d), x1 = __shfl_down_sync(kFull, a.hi, d);
  uint64_t y0 = __shfl_down_sync(kFull, a.lo, (d + 1) & 31), y1 = __shfl_down_sync(kFull, a.hi, (d + 1) & 31);
  if (lane + d > 31) x0 = x1 = 0;
  if (lane + d + 1 > 31) y0 = y1 = 0;
  if (s >= 64) {
    x0 = x1;
    x1 = y0;
    y0 = y1;
    s -= 64;
  }
  if (s == 0) return W128{x0, x1};
  return W128{(x0 >> s) | (x1 << (64 - s)), (x1 >> s) | (y0 << (64 - s))};
}

__global__ void rs_flag_pub_kernel(const __grid_constant__ RsArgs P) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  // n: limbs 4 lane .. 4 lane + 3
  auto limb = [&](int i) -> uint64_t { return i < P.L ? (uint64_t)P.n[i] : 0ull; };
  const W128 n{limb(4 * lane) | limb(4 * lane + 1) << 32, limb(4 * lane + 2) | limb(4 * lane + 3) << 32};
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < P.nblocks; k += warps) {
    // candidate words 2 lane, 2 lane + 1 (gen_candidate)
    const uint64_t j0 = (P.block0 + (uint64_t)k) * (uint64_t)P.W;
    uint64_t w[2];
    for (int h = 0; h < 2; h++) {
      const int wi = 2 * lane + h;
      uint64_t v = wi < P.W ? mix64(P.state0 + (j0 + wi + 1) * kGamma) : 0ull;
      if (wi == P.W - 1) v &= P.topmask;
      w[h] = v;
    }
    W128 a{w[0], w[1]}, b = n;
    bool ok = w_cmp(a, b) < 0 && !w_is_zero(a);  // random_below: < n; sample_r: != 0
    if (ok) {                                    // gcd(r, n) == 1 (paillier.cpp:237); n is odd
      while (!w_is_zero(a)) {
        a = w_strip(a, lane);
        if (w_cmp(a, b) < 0) {
          const W128 t = a;
          a = b;
          b = t;
        }
        a = w_sub(a, b, lane);
      }
      ok = !__any_sync(kFull, lane ? (b.lo | b.hi) != 0 : (b.lo != 1 || b.hi != 0));  // gcd = b == 1
    }
    if (lane == 0) P.flags[k] = ok ? 1 : 0;
  }
}

__global__ void rs_flag_kernel(const __grid_constant__ RsArgs P) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nblocks; k += gridDim.x * blockDim.x) {
    uint32_t c[128];
    gen_candidate(P, P.block0 + k, c);
    // < n ?  (random_below, bignat.cpp:438-445)
    bool lt = false;
    for (int i = P.L - 1; i >= 0; i--)
      if (c[i] != P.n[i]) {
        lt = c[i] < P.n[i];
        break;
      }
    bool nz = false;
    for (int i = 0; i < P.L; i++) nz = nz || c[i] != 0;
    bool ok = lt && nz;  // sample_r: r != 0 (paillier.cpp:236)
    if (ok)  // gcd(r, n) == 1 (paillier.cpp:237): neither p nor q divides r (public keys: rs_flag_pub_kernel)
      ok = !divisible(c, P.L, P.p, P.pinv, P.H) && !divisible(c, P.L, P.q, P.qinv, P.H);
    P.flags[k] = ok ? 1 : 0;
  }
}

__global__ void rs_emit_kernel(const __grid_constant__ RsArgs P, int base_rank) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P.nblocks; k += gridDim.x * blockDim.x) {
    if (!P.flags[k]) continue;
    const int r = base_rank + P.rank[k];
    if (r >= P.count) continue;
    uint32_t c[128];
    gen_candidate(P, P.block0 + k, c);
    uint32_t* dst = P.r_out + (size_t)r * P.L;
    for (int i = 0; i < P.L; i++) dst[i] = c[i];
  }
}

static uint32_t neg_inv(uint32_t m0) {
  uint32_t inv = 1;
  for (int i = 0; i < 5; i++) inv *= 2u - m0 * inv;
  return 0u - inv;
}

// Host driver: fills r_out (device, count x L) and advances *state exactly like the reference.
pcb_status rstream_sample(uint64_t* state, const uint32_t* n, int L, int nbits, const uint32_t* p, const uint32_t* q,
                          int H, size_t count, uint32_t* r_out, cudaStream_t st) {
  if (L > 128 || H > 64) return PCB_E_UNSUPPORTED;
  RsArgs P{};
  P.state0 = *state;
  P.W = (nbits + 63) / 64;
  P.topmask = (nbits % 64) ? (~0ull >> (64 - nbits % 64)) : ~0ull;
  P.L = L;
  for (int i = 0; i < L; i++) P.n[i] = n[i];
  P.has_prv = p && q;
  P.H = H;
  if (P.has_prv) {
    for (int i = 0; i < H; i++) {
      P.p[i] = p[i];
      P.q[i] = q[i];
    }
    P.pinv = neg_inv(p[0]);
    P.qinv = neg_inv(q[0]);
  }
  P.r_out = r_out;
  P.count = (int)count;
  // acceptance >= 1/2 (n has its top bit set within the drawn width); oversample by 2.25x
  size_t chunk = count * 9 / 4 + 256;
  int32_t *flags = nullptr, *rank = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  pcb_status e = scratch_alloc(chunk * 4, (void**)&flags, st);
  if (!e) e = scratch_alloc(chunk * 4, (void**)&rank, st);
  if (!e && cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, rank, (int)chunk, st) != cudaSuccess)
    e = PCB_E_CUDA;
  if (!e) e = scratch_alloc(tmp_bytes, &tmp, st);
  size_t have = 0;
  uint64_t block = 0;
  uint64_t consumed = 0;
  std::vector<int32_t> hflags;
  while (!e && have < count) {
    P.block0 = block;
    P.nblocks = (int)chunk;
    P.flags = flags;
    P.rank = rank;
    const int grid = (int)std::min<size_t>((chunk + 255) / 256, 148 * 16);
    if (P.has_prv) {
      rs_flag_kernel<<<grid, 256, 0, st>>>(P);
    } else {  // a warp per candidate
      const int gridw = (int)std::min<size_t>((chunk * 32 + 255) / 256, 148 * 16);
      rs_flag_pub_kernel<<<gridw, 256, 0, st>>>(P);
    }
    count_launch();
    if (cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags, rank, (int)chunk, st) != cudaSuccess) {
      e = PCB_E_CUDA;
      break;
    }
    rs_emit_kernel<<<grid, 256, 0, st>>>(P, (int)have);
    count_launch();
    // how many accepted in this chunk, and where the count-th one sits
    int32_t last_rank = 0, last_flag = 0;
    cudaMemcpyAsync(&last_rank, rank + chunk - 1, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last_flag, flags + chunk - 1, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      e = PCB_E_CUDA;
      break;
    }
    const size_t acc = (size_t)last_rank + (size_t)last_flag;
    if (have + acc >= count) {
      // find the block holding rank (count - have - 1): scan flags on the host (one pass)
      hflags.resize(chunk);
      cudaMemcpy(hflags.data(), flags, chunk * 4, cudaMemcpyDeviceToHost);
      size_t need = count - have, seen = 0, k = 0;
      for (; k < chunk; k++)
        if (hflags[k] && ++seen == need) break;
      consumed = block + k + 1;
      have = count;
    } else {
      have += acc;
      block += chunk;
    }
  }
  scratch_free(tmp, st);
  scratch_free(flags, st);
  scratch_free(rank, st);
  if (!e) *state = P.state0 + consumed * (uint64_t)P.W * kGamma;
  return e;
}

}  // namespace pcb
