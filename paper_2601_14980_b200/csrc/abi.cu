// abi.cu — the C ABI of include/pcb200.h: context construction (per-key constants), host/device
// pointer staging, dispatch to the templated kernels, error mapping.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <vector>

#include "host/hbn.hpp"
#include "paillier_params.cuh"
#include "pcb_internal.h"
#include "wide.h"
#include "rns.h"
#include "rnsx.h"

namespace pcb {

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

// ---- hot-kernel profiling ----------------------------------------------------------------
namespace {
struct ProfState {
  std::mutex mu;
  bool on = false;
  double int8 = 0.0, last_int8 = 0.0;  // tensor-core int8 MACs issued by the RNS kernels
  std::vector<std::pair<ProfMark, double>> marks;
};
ProfState& prof() {
  static ProfState s;
  return s;
}
}  // namespace

bool prof_enabled() { return prof().on; }

ProfMark prof_start(cudaStream_t st) {
  ProfMark m;
  cudaEventCreate(&m.a);
  cudaEventCreate(&m.b);
  cudaEventRecord(m.a, st);
  return m;
}

void prof_add_int8(double macs) {
  std::lock_guard<std::mutex> lk(prof().mu);
  if (prof().on) prof().int8 += macs;
}

void prof_stop(ProfMark m, cudaStream_t st, double alg) {
  cudaEventRecord(m.b, st);
  std::lock_guard<std::mutex> lk(prof().mu);
  prof().marks.push_back({m, alg});
}

// ---- scratch + staging ----------------------------------------------------------------------
pcb_status scratch_alloc(size_t bytes, void** p, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    // keep freed scratch in the stream-ordered pool (no re-mapping between batches)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  return cudaMallocAsync(p, bytes, st) == cudaSuccess ? PCB_OK : PCB_E_ALLOC;
}
void scratch_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

pcb_status stage_in(const void* p, size_t bytes, cudaStream_t st, Staged* s) {
  s->bytes = bytes;
  if (!p || is_device_ptr(p)) {
    s->dev = const_cast<void*>(p);
    s->host = false;
    return PCB_OK;
  }
  s->host = true;
  if (auto e = scratch_alloc(bytes, &s->dev, st)) return e;
  return cuda_check(cudaMemcpyAsync(s->dev, p, bytes, cudaMemcpyHostToDevice, st));
}

pcb_status stage_out(void* p, size_t bytes, cudaStream_t st, Staged* s) {
  s->bytes = bytes;
  if (!p || is_device_ptr(p)) {
    s->dev = p;
    s->host = false;
    return PCB_OK;
  }
  s->host = true;
  return scratch_alloc(bytes, &s->dev, st);
}

pcb_status unstage_out(void* p, Staged* s, cudaStream_t st) {
  if (!s->host || !p) return PCB_OK;
  return cuda_check(cudaMemcpyAsync(p, s->dev, s->bytes, cudaMemcpyDeviceToHost, st));
}

void unstage(Staged* s, cudaStream_t st) {
  if (s->host && s->dev) scratch_free(s->dev, st);
  s->dev = nullptr;
  s->host = false;
}


// ---- per-element status when the caller passes status = NULL ---------------------------------
// The reference throws on the first bad element (paillier.cpp:242, 322-323, 348, 36-39); with no
// status array the ABI returns that element's code instead of silently handing back 0 / garbage.
__global__ void first_bad_kernel(const int32_t* st, size_t n, unsigned long long* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (st[i] != 0) atomicMin(out, ((unsigned long long)i << 32) | (uint32_t)st[i]);
}

// out[i] = src (w words) for every i < count (a broadcast base for the digit exponentiations)
__global__ void bcast_kernel(uint32_t* out, const uint32_t* src, int w, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count * (size_t)w; i += (size_t)gridDim.x * blockDim.x)
    out[i] = src[i % w];
}
// rows whose argument check failed come back as 0 (as the other encryption paths do)
__global__ void zero_bad_rows_kernel(uint32_t* c, int w, const int32_t* st, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count * (size_t)w; i += (size_t)gridDim.x * blockDim.x)
    if (st[i / w] != 0) c[i] = 0;
}

// Scans stv[0, count) for the first non-OK element; synchronises `st` (only called when the caller
// asked for no status array, i.e. for a single error code).
pcb_status first_failure(const int32_t* stv, size_t count, cudaStream_t st) {
  unsigned long long* d = nullptr;
  unsigned long long h = ~0ull;
  pcb_status e = scratch_alloc(8, (void**)&d, st);
  if (!e) e = cuda_check(cudaMemsetAsync(d, 0xff, 8, st));
  if (!e) {
    const int thr = 256;
    const int blocks = (int)std::min<size_t>((count + thr - 1) / thr, 148 * 8);
    first_bad_kernel<<<blocks, thr, 0, st>>>(stv, count, d);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) e = cuda_check(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
  scratch_free(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (e) return e;
  return h == ~0ull ? PCB_OK : (pcb_status)(int32_t)(uint32_t)(h & 0xffffffffu);
}

// ---- host-buffer pipelining ----------------------------------------------------------------------
// A large batch whose big arrays are host memory runs in chunks: chunk i+1's host->device copy and
// chunk i-1's device->host copy run on their own streams while chunk i computes, instead of the
// whole batch's copies before and after the compute.  The results are the per-chunk calls' on
// device buffers, i.e. the same bytes.
constexpr size_t kPipeMin = (size_t)4 * 148 * 256;  // below this a batch runs in one piece
constexpr size_t kPipeChunks = 4;

struct HostPipe {
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaEvent_t in[2] = {nullptr, nullptr}, comp[2] = {nullptr, nullptr}, out[2] = {nullptr, nullptr}, start = nullptr;
  pcb_status init(cudaStream_t st) {
    if (cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking) != cudaSuccess) return PCB_E_CUDA;
    if (cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking) != cudaSuccess) return PCB_E_CUDA;
    for (cudaEvent_t* ev : {&in[0], &in[1], &comp[0], &comp[1], &out[0], &out[1], &start})
      if (cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) return PCB_E_CUDA;
    // the copies follow everything already queued on the caller's stream
    if (cudaEventRecord(start, st) != cudaSuccess) return PCB_E_CUDA;
    if (cudaStreamWaitEvent(cin, start, 0) != cudaSuccess || cudaStreamWaitEvent(cout, start, 0) != cudaSuccess)
      return PCB_E_CUDA;
    return PCB_OK;
  }
  ~HostPipe() {
    if (cin) cudaStreamSynchronize(cin);
    if (cout) cudaStreamSynchronize(cout);
    for (cudaEvent_t ev : {in[0], in[1], comp[0], comp[1], out[0], out[1], start})
      if (ev) cudaEventDestroy(ev);
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
  }
};

// ---- constants ------------------------------------------------------------------------------
static uint32_t neg_inv32(uint32_t m0) {
  uint32_t inv = 1;
  for (int i = 0; i < 5; i++) inv *= 2u - m0 * inv;
  return 0u - inv;
}

template <int S>
static void fill_mod(ModCtx<S>& c, const HBN& m) {
  std::memset(&c, 0, sizeof(c));
  m.to_limbs(c.m, S);
  mod(HBN(1) << (64 * S), m).to_limbs(c.r2, S);
  c.minv = neg_inv32(c.m[0]);
}

// Left-to-right sliding window schedule (see mont.cuh).  Window width w, table of the
// 2^(w-1) odd powers.
std::vector<uint32_t> build_schedule(const HBN& e, int w) {
  std::vector<uint32_t> ops;
  long i = (long)e.bit_length() - 1;
  bool first = true;
  uint32_t pending = 0;
  while (i >= 0) {
    if (!e.bit((size_t)i)) {
      pending++;
      i--;
      continue;
    }
    long j = i - w + 1;
    if (j < 0) j = 0;
    while (!e.bit((size_t)j)) j++;
    uint32_t d = 0;
    for (long k = i; k >= j; k--) d = (d << 1) | (e.bit((size_t)k) ? 1u : 0u);
    const uint32_t len = (uint32_t)(i - j + 1);
    if (first) {
      ops.push_back((d - 1) / 2);
      first = false;
    } else {
      ops.push_back(((pending + len) << 16) | ((d - 1) / 2));
    }
    pending = 0;
    i = j - 1;
  }
  if (pending) ops.push_back((pending << 16) | 0xffffu);
  return ops;
}

// Expand the window schedule into the per-product byte stream consumed by mont_pow:
// ops[0] = seed table index, then kOpSquare per squaring and a table index per multiply.
std::vector<uint8_t> build_ops(const HBN& e, int w) {
  std::vector<uint32_t> sch = build_schedule(e, w);
  std::vector<uint8_t> ops;
  ops.push_back((uint8_t)(sch[0] & 0xffffu));
  for (size_t i = 1; i < sch.size(); i++) {
    const uint32_t nsq = sch[i] >> 16, idx = sch[i] & 0xffffu;
    ops.insert(ops.end(), nsq, kOpSquare);
    if (idx != 0xffffu) ops.push_back((uint8_t)idx);
  }
  return ops;
}

// radix-2^r limbs of v (N limbs)
std::vector<uint32_t> radix_limbs(const HBN& v, int rb, int n) {
  std::vector<uint32_t> out(n, 0);
  for (int j = 0; j < n; j++) {
    uint32_t x = 0;
    for (int b = 0; b < rb; b++)
      if (v.bit((size_t)j * rb + b)) x |= 1u << b;
    out[j] = x;
  }
  return out;
}

// Constants of one modulus for the radix-2^r core: m limbs, R^2, c1 (caller), minv mod 2^r.
struct R28Mod {
  std::vector<uint32_t> mlimb, mword, r2;
  uint32_t minv = 0;
  int mwords = 0;
};
R28Mod r28_mod(const HBN& m, int rb, int n) {
  R28Mod c;
  c.mlimb = radix_limbs(m, rb, n);
  c.mwords = (int)((m.bit_length() + 31) / 32);
  c.mword = m.limbs(c.mwords);
  c.r2 = radix_limbs(mod(HBN(1) << (2 * (size_t)rb * n), m), rb, n);
  uint32_t inv = 1;
  for (int i = 0; i < 6; i++) inv *= 2u - c.mlimb[0] * inv;  // m^-1 mod 2^32
  c.minv = (0u - inv) & ((1u << rb) - 1u);
  return c;
}

// Sliding-window width of the fixed-exponent schedules (table of 2^(w-1) odd powers per element).
// PCB_WINDOW overrides it for A/B runs (1..6), read once per process before any context exists.
int window_width() {
  static const int w = [] {
    const char* v = getenv("PCB_WINDOW");
    const int x = v ? atoi(v) : 5;
    return x >= 1 && x <= 6 ? x : 5;
  }();
  return w;
}
#define kWindow (window_width())
#define kTab (1 << (kWindow - 1))

}  // namespace pcb

using namespace pcb;

struct pcb_ctx {
  int device = 0;
  uint32_t L = 0, nbits = 0;
  bool has_prv = false;
  int S = 0;   // p^2 / q^2 kernel width
  int S2 = 0;  // n^2 kernel width
  HBN n, n2, p, q;
  std::vector<uint8_t> enc_blob, dec_blob, n2_blob;
  uint8_t* d_sched = nullptr;  // all exponent op streams, concatenated
  int off_enc_p = 0, len_enc_p = 0, off_enc_q = 0, len_enc_q = 0;
  int off_dec_p = 0, len_dec_p = 0, off_dec_q = 0, len_dec_q = 0;
  int off_epsq = 0, len_epsq = 0, off_one = 0, len_one = 0;  // eps mod phi(q^2); e = 1
  std::vector<uint8_t> half_blob;  // CrtDecConsts with h_p = q^-1 mu mod p, h_q = p^-1 mu mod q
  // eps mod phi(q^2) = u (q - 1) (eps is a multiple of q - 1): decrypt_with_half's q side is then
  // c^(q-1) mod q^2 (the Dec chain) with u folded into h_q (half_pow, paillier.cpp:275-305)
  std::vector<uint8_t> half_blob_u;
  bool half_fold = false;
  int off_pub = 0, len_pub = 0;  // exponent n at n^2 (direct encryption)
  uint32_t* d_n = nullptr;       // n (L limbs), n^2 (2L limbs) for the argument checks
  uint32_t* d_n2 = nullptr;
  cudaStream_t side_st[2] = {nullptr, nullptr};  // p-half / q-half streams (fork-join)
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  std::mutex mu;                 // serialises use of the side streams
  WideMod wide;                  // n^2 constants for the radix-2^r kernels (public-key ops)
  R28Mod rp2, rq2;               // p^2, q^2 for the radix CRT halves (3072-bit keys)
  RnsModulus rns_p, rns_q;       // p^2, q^2 for the RNS / tensor-core CRT halves (2048-bit keys)
  bool use_rns = false;
  RnsXModulus rx_p, rx_q;        // p^2, q^2 for the streaming RNS core (rnsx.cu)
  bool use_rnsx = false;
  // rx_p / rx_q exist (use_rnsx, or small keys where they serve only the collaborative entry
  // points decrypt_with_half / finish_split_encrypt while Enc / Dec stay on the carry core)
  bool has_rx = false;
  // random generator (GMode::random_g, pcb_ctx_set_generator): g and its 64-bit digit powers
  // G_j = g^(2^(64 j)) mod n^2 (d_gtab, gdig x 2L words) for g^m = prod_j G_j^(m_j) on the device
  bool random_g = false;
  HBN g;
  uint32_t* d_gtab = nullptr;
  int gdig = 0;
  // split CRT encryption (2048-bit keys): r^n mod p^2 = ((r mod p)^q mod p)^p mod p^2, since u^p
  // mod p^2 depends only on u mod p; stage 1 on the carry-chain core mod p (1024 bits), stage 2
  // on the RNS core with the 1024-bit exponent p (half the exponent bits of n).  Same for q.
  bool enc_split = false;
  bool enc_split_rns = false;           // stage 1 on the RNS core (K = 48) instead
  RnsXModulus rx1_p, rx1_q;             // p, q on the RNS core
  ModCtx<32> m1p, m1q;                  // p, q (32 limbs, R = 2^1024)
  std::vector<uint32_t> r3_p1, r3_q1;   // R^3 mod p, R^3 mod q
  int off_ep = 0, len_ep = 0, off_eq = 0, len_eq = 0;  // exponents p and q
  int w1 = 32;                          // words of p, q (stage-1 outputs)
  RnsXModulus rx_n2;             // n^2 on the streaming RNS core (matvec, public-key ops)
  bool use_rx_n2 = false;
  std::vector<uint32_t> rp2_nR, rq2_nR, rp2_R3, rq2_R3;
  std::vector<uint32_t> wide_r2, wide_nR;
  uint32_t* d_wconst = nullptr;  // [R^2, R, 1, R^C (aggregate)] radix limbs
  int agg_chunk = 32;
  std::atomic<uint64_t> pow_full{0}, pow_half{0};
};

namespace pcb {
// launchers (side.cu / paillier.cu)
template <int S>
pcb_status launch_side(const ModCtx<S>& mod, const uint32_t* c1, const uint8_t* ops, int nops, int ntab, int mode,
                       const uint32_t* x, int x_limbs, const uint32_t* m, int m_limbs, const int32_t* skip,
                       size_t count, uint32_t* y, cudaStream_t st, int ebits_canon);
template <int S>
pcb_status launch_garner(const CrtEncConsts<S>& k, const uint32_t* cp, const uint32_t* cq, const int32_t* st,
                         uint32_t* c, int L, size_t count, cudaStream_t stream);
template <int S>
pcb_status launch_dec_finish(const CrtDecConsts<S>& k, const uint32_t* xp, const uint32_t* xq, int32_t* st,
                             uint32_t* m, int L, size_t count, cudaStream_t stream);
template <int S>
pcb_status launch_fermat_finish(const ModCtx<S / 2>& sp, const uint32_t* pinv_lo, const uint32_t* p,
                                const uint32_t* s, const uint32_t* u, uint32_t* out, size_t count, cudaStream_t stream);
pcb_status launch_enc_prep(const uint32_t* m, int m_limbs, const double* v, double zmin, double zmax, double delta,
                           int fine, uint32_t* m_out, int m_out_limbs, uint64_t* q_out, unsigned long long* clamps,
                           const uint32_t* r, const uint32_t* n_dev, int L, int32_t* st, size_t count,
                           cudaStream_t stream);
pcb_status launch_onepmn(const uint32_t* m, int ml, const uint32_t* rn, const uint32_t* n_dev, const uint32_t* n2_dev,
                         int L, uint32_t* out, int32_t* st, size_t count, cudaStream_t stream);
pcb_status launch_quantize(const double* v, size_t count, double zmin, double zmax, double delta, int fine,
                           uint64_t* q, unsigned long long* clamps, int32_t* err, cudaStream_t stream);
pcb_status launch_status_flag(const int32_t* st, size_t count, int32_t* err, cudaStream_t stream);
pcb_status launch_obfuscate(const uint32_t* value, int vw, const uint64_t* mask, const uint32_t* neps, int nw,
                            size_t count, uint32_t* out, int ow, cudaStream_t stream);
pcb_status launch_mod_words(const uint32_t* a, int aw, size_t count, const uint32_t* v_norm, int s, int shift,
                            uint32_t* out, cudaStream_t stream);
pcb_status launch_mul_add1(const uint32_t* a, int aw, const uint32_t* b, int bw, size_t count, uint32_t* out,
                           cudaStream_t stream);
pcb_status launch_combined_update(const uint64_t* qa, const uint64_t* qb, const uint64_t* qz, const uint64_t* qnv,
                                  size_t rows, size_t cols, uint64_t* out, cudaStream_t stream);
pcb_status launch_inverse_x(const uint64_t* q, const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                            size_t rows, size_t cols, double zmin, double zmax, double delta, double* x,
                            cudaStream_t stream);
pcb_status launch_dec_prep(const uint32_t* c, const uint32_t* n2_dev, int L, int32_t* st, size_t count,
                           cudaStream_t stream);
pcb_status launch_update(const uint32_t* m, int L, const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                         double zmin, double zmax, double delta, double kappa, double* x, double* z, double* v,
                         int32_t* st, size_t count, const long long* seg_dev, int nseg, cudaStream_t stream);
enum SideMode : int { kSideEnc = 0, kSideDec = 1, kSidePow = 2 };
template <int RB, int N, int TPI>
pcb_status launch_side28(const uint32_t* mlimb, const uint32_t* mword, int mwords, const uint32_t* r2,
                         const uint32_t* c1, uint32_t minv, const uint8_t* ops, int nops, int ntab, int mode,
                         const uint32_t* x, int x_words, const uint32_t* m, int m_words, const int32_t* skip,
                         size_t count, uint32_t* y, int y_words, cudaStream_t st, double alg_mac32_per_elem);
pcb_status rstream_sample(uint64_t* state, const uint32_t* n, int L, int nbits, const uint32_t* p, const uint32_t* q,
                          int H, size_t count, uint32_t* r_out, cudaStream_t st);
template <int RB, int N, int TPI>
pcb_status launch_wide(const WideMod& md, const WStep* prog, int nsteps, const uint32_t* consts_dev,
                       const uint32_t* x, const uint32_t* b, const uint64_t* k, int xin_per_out, size_t count,
                       size_t nout, uint32_t* y, int ntab, cudaStream_t st, const MatvecGeom* mg);
}  // namespace pcb

namespace {

template <int S>
void build_enc(pcb_ctx* x) {
  CrtEncConsts<S> k;
  std::memset(&k, 0, sizeof(k));
  HBN p2 = x->p * x->p, q2 = x->q * x->q;
  fill_mod<S>(k.mp, p2);
  fill_mod<S>(k.mq, q2);
  const HBN R = HBN(1) << (32 * S);
  mod(x->n * R, p2).to_limbs(k.nRp, S);
  mod(x->n * R, q2).to_limbs(k.nRq, S);
  HBN inv;
  if (!mod_inverse(mod(p2, q2), q2, inv)) throw std::invalid_argument("p and q share a factor");
  inv.to_limbs(k.inv, S);
  x->n.to_limbs(k.n, S);
  x->enc_blob.assign(reinterpret_cast<uint8_t*>(&k), reinterpret_cast<uint8_t*>(&k) + sizeof(k));
}

template <int S>
void build_dec(pcb_ctx* x) {
  constexpr int H = S / 2;
  CrtDecConsts<S> k;
  std::memset(&k, 0, sizeof(k));
  HBN p2 = x->p * x->p, q2 = x->q * x->q;
  fill_mod<S>(k.mp, p2);
  fill_mod<S>(k.mq, q2);
  fill_mod<H>(k.sp, x->p);
  fill_mod<H>(k.sq, x->q);
  mod(HBN(1) << (96 * S), p2).to_limbs(k.r3p, S);
  mod(HBN(1) << (96 * S), q2).to_limbs(k.r3q, S);
  const HBN RH = HBN(1) << (32 * H);
  HBN t;
  if (!mod_inverse(x->p, RH, t)) throw std::invalid_argument("even p");
  t.to_limbs(k.pinv_lo, H);
  if (!mod_inverse(x->q, RH, t)) throw std::invalid_argument("even q");
  t.to_limbs(k.qinv_lo, H);
  // h_p = L_p(g^(p-1) mod p^2)^-1 mod p (g = n + 1, or the context's random generator)
  const HBN g = x->random_g ? x->g : x->n + HBN(1);
  for (int side = 0; side < 2; side++) {
    const HBN& pr = side ? x->q : x->p;
    const HBN& m2 = side ? q2 : p2;
    HBN xx = pow_mod(g, pr - HBN(1), m2);
    HBN l, r;
    divmod(xx - HBN(1), pr, l, r);
    HBN h;
    if (!mod_inverse(l, pr, h)) throw std::invalid_argument("degenerate key (h_p)");
    mod(h * RH, pr).to_limbs(side ? k.hq : k.hp, H);
  }
  HBN pinvq;
  if (!mod_inverse(mod(x->p, x->q), x->q, pinvq)) throw std::invalid_argument("p and q share a factor");
  pinvq.to_limbs(k.pinvq, H);
  x->p.to_limbs(k.p, H);
  x->q.to_limbs(k.q, H);
  x->n2.to_limbs(k.n2, 2 * S);
  x->dec_blob.assign(reinterpret_cast<uint8_t*>(&k), reinterpret_cast<uint8_t*>(&k) + sizeof(k));
}

// decrypt_with_half constants: dec_finish<S> on (x mod p^2, x mod q^2) of x = c^eps mod n^2 yields
// L(x) mu mod n when h_p = q^-1 mu mod p and h_q = p^-1 mu mod q (L(x) = L_p(x_p) q^-1 mod p, ...).
template <int S>
void build_half(pcb_ctx* x) {
  constexpr int H = S / 2;
  CrtDecConsts<S> k;
  std::memcpy(&k, x->dec_blob.data(), sizeof(k));
  const HBN RH = HBN(1) << (32 * H);
  const HBN eps = lcm(x->p - HBN(1), x->q - HBN(1));
  HBN mu;
  if (x->random_g) {  // mu = L(g^eps mod n^2)^-1 mod n (paillier.cpp:90-92)
    HBN l, r;
    divmod(pow_mod(x->g, eps, x->n2) - HBN(1), x->n, l, r);
    if (!mod_inverse(l, x->n, mu)) throw std::invalid_argument("degenerate generator (mu)");
  } else if (!mod_inverse(mod(eps, x->n), x->n, mu)) {
    throw std::invalid_argument("degenerate key (mu)");  // paillier.cpp:78
  }
  for (int side = 0; side < 2; side++) {
    const HBN& pr = side ? x->q : x->p;
    const HBN& ot = side ? x->p : x->q;
    HBN inv;
    if (!mod_inverse(mod(ot, pr), pr, inv)) throw std::invalid_argument("p and q share a factor");
    mod(mod(inv * mu, pr) * RH, pr).to_limbs(side ? k.hq : k.hp, H);
  }
  x->half_blob.assign(reinterpret_cast<uint8_t*>(&k), reinterpret_cast<uint8_t*>(&k) + sizeof(k));
  // x_q = c^(eps mod phi(q^2)) mod q^2 with eps mod phi(q^2) = u (q - 1), u != 0: x_q = s^u for
  // s = c^(q-1) mod q^2 = 1 + q L_q(s), so L_q(x_q) = u L_q(s) mod q and the finish may run on s with
  // h_q u.  (s = 0 iff q | c, and then x_q = 0 too: the same PCB_E_NOT_UNIT.)  u = 0 (toy keys
  // only) keeps the direct power, whose c^0 = 1 differs from s^0 when q | c.
  {
    const HBN q2 = x->q * x->q, qm1 = x->q - HBN(1);
    HBN u, w;
    divmod(mod(eps, q2 - x->q), qm1, u, w);
    if (w.is_zero() && !u.is_zero()) {
      HBN inv;
      if (!mod_inverse(mod(x->p, x->q), x->q, inv)) throw std::invalid_argument("p and q share a factor");
      mod(mod(mod(inv * mu, x->q) * u, x->q) * RH, x->q).to_limbs(k.hq, H);
      x->half_blob_u.assign(reinterpret_cast<uint8_t*>(&k), reinterpret_cast<uint8_t*>(&k) + sizeof(k));
      x->half_fold = true;
    }
  }
}

pcb_status set_device(const pcb_ctx* x) { return cuda_check(cudaSetDevice(x->device)); }

struct StreamSync {
  cudaStream_t st;
  bool need;
  ~StreamSync() {
    if (need) cudaStreamSynchronize(st);
  }
};

}  // namespace

extern "C" {

const char* pcb_status_str(pcb_status s) {
  switch (s) {
    case PCB_OK: return "ok";
    case PCB_E_PLAINTEXT_RANGE: return "plaintext not below n";
    case PCB_E_RANDOMNESS_RANGE: return "randomness not in [1, n)";
    case PCB_E_CIPHER_RANGE: return "ciphertext not below n^2";
    case PCB_E_NOT_UNIT: return "ciphertext outside the multiplicative group";
    case PCB_E_OVERFLOW: return "homomorphic accumulation exceeds plaintext space";
    case PCB_E_NO_PRIVATE: return "no private key loaded";
    case PCB_E_SHAPE: return "invalid argument (shape / window / size)";
    case PCB_E_UNSUPPORTED: return "unsupported by this build";
    case PCB_E_CUDA: return "CUDA error (or no device)";
    case PCB_E_ALLOC: return "allocation failed";
    case PCB_E_RANGE_UPDATE: return "combined update out of range";
  }
  return "unknown status";
}

uint64_t pcb_launch_count(void) { return launch_counter().load(); }

void pcb_profile_begin(void) {
  std::lock_guard<std::mutex> lk(prof().mu);
  prof().marks.clear();
  prof().int8 = 0.0;
  prof().on = true;
}

double pcb_profile_int8_macs(void) {
  std::lock_guard<std::mutex> lk(prof().mu);
  return prof().last_int8;
}

pcb_status pcb_profile_end(double* side_ms_total, uint64_t* side_launches, double* side_alg_mac32) {
  std::lock_guard<std::mutex> lk(prof().mu);
  prof().on = false;
  prof().last_int8 = prof().int8;
  double ms = 0, alg = 0;
  pcb_status e = PCB_OK;
  for (auto& [m, a] : prof().marks) {
    float t = 0.f;
    if (cudaEventSynchronize(m.b) != cudaSuccess || cudaEventElapsedTime(&t, m.a, m.b) != cudaSuccess) e = PCB_E_CUDA;
    ms += t;
    alg += a;
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  if (side_ms_total) *side_ms_total = ms;
  if (side_launches) *side_launches = prof().marks.size();
  if (side_alg_mac32) *side_alg_mac32 = alg;
  prof().marks.clear();
  return e;
}

pcb_status pcb_keygen(uint64_t* rng_state, uint32_t key_bits, uint32_t* n, uint32_t* p, uint32_t* q) {
  if (!rng_state) return PCB_E_SHAPE;
  try {
    HRng rng(*rng_state);
    HBN P, Q;
    if (!pcb::keygen(rng, key_bits, P, Q)) return PCB_E_SHAPE;
    *rng_state = rng.state;
    const uint32_t nl = (key_bits + 31) / 32, hl = (key_bits / 2 + 31) / 32;
    if (n) (P * Q).to_limbs(n, nl);
    if (p) P.to_limbs(p, hl);
    if (q) Q.to_limbs(q, hl);
    return PCB_OK;
  } catch (const std::bad_alloc&) {
    return PCB_E_ALLOC;
  } catch (...) {
    return PCB_E_SHAPE;
  }
}

pcb_status pcb_random_prime(uint64_t* rng_state, uint32_t bits, uint32_t* out) {
  if (!rng_state || bits < 2) return PCB_E_SHAPE;
  try {
    HRng rng(*rng_state);
    HBN P = pcb::random_prime(rng, bits);
    *rng_state = rng.state;
    P.to_limbs(out, (bits + 31) / 32);
    return PCB_OK;
  } catch (...) {
    return PCB_E_SHAPE;
  }
}

pcb_status pcb_ctx_create(pcb_ctx** out, int device, const uint32_t* n, uint32_t n_limbs, const uint32_t* p,
                          const uint32_t* q, uint32_t pq_limbs) {
  PCB_RANGE("pcb_ctx_create");
  if (!out || !n || n_limbs == 0) return PCB_E_SHAPE;
  *out = nullptr;
  std::unique_ptr<pcb_ctx> x(new (std::nothrow) pcb_ctx);
  if (!x) return PCB_E_ALLOC;
  try {
    x->device = device;
    x->n = HBN::from_limbs(n, n_limbs);
    if (x->n.is_zero() || !x->n.is_odd()) return PCB_E_SHAPE;
    x->n2 = x->n * x->n;
    x->nbits = (uint32_t)x->n.bit_length();
    x->L = (x->nbits + 31) / 32;
    x->S2 = kernel_width_wide(2 * x->L);
    // Keys up to 4096 bits (the reference keygen's largest size, paillier.cpp:107-109): n^2 on the
    // radix core up to 8192 bits; anything larger is refused explicitly, not as a shape error.
    if (x->S2 == 0) return x->nbits > 4096 ? PCB_E_UNSUPPORTED : PCB_E_SHAPE;
    x->has_prv = p && q;
    if (x->has_prv) {
      x->p = HBN::from_limbs(p, pq_limbs);
      x->q = HBN::from_limbs(q, pq_limbs);
      if (x->p * x->q != x->n || x->p == x->q || !x->p.is_odd() || !x->q.is_odd()) return PCB_E_SHAPE;
      const HBN p2 = x->p * x->p, q2 = x->q * x->q;
      const uint32_t l2 = (uint32_t)((std::max(p2.bit_length(), q2.bit_length()) + 31) / 32);
      x->S = kernel_width(std::max(l2, x->L));
      if (x->S == 0) return PCB_E_SHAPE;
      {
        // streaming RNS core for the CRT halves (default; PCB_RNSX=0 selects the older cores)
        const char* ev = getenv("PCB_RNSX");
        int K = 0;
        if ((!ev || atoi(ev) != 0) && (x->S == 64 || x->S == 96 || x->S == 128) && rnsx_shape((int)(32 * x->S), &K))
          x->use_rnsx = rnsx_build(p2, x->n, x->S, K, &x->rx_p) && rnsx_build(q2, x->n, x->S, K, &x->rx_q);
        x->has_rx = x->use_rnsx;
        const char* es = getenv("PCB_ENC_SPLIT");
        const size_t hb = (size_t)16 * x->S;  // half the p^2 width: p, q bits
        if (x->use_rnsx && (x->S == 64 || x->S == 96 || x->S == 128) && x->p.bit_length() <= hb && x->q.bit_length() <= hb &&
            (!es || atoi(es) != 0)) {
          x->w1 = x->S / 2;
          const int K1 = x->S == 64 ? 40 : (x->S == 96 ? 56 : 72);  // M > (2K+2)^2 p with 30-bit primes
          // default: stage 1 on the RNS core; PCB_ENC_SPLIT=1 selects the carry core (1024-bit p only)
          if (!es || atoi(es) == 2 || x->S != 64)
            x->enc_split_rns =
                rnsx_build(x->p, x->n, x->w1, K1, &x->rx1_p) && rnsx_build(x->q, x->n, x->w1, K1, &x->rx1_q);
          if (x->S == 64) {
            const HBN R3 = HBN(1) << (3 * 1024);
            fill_mod<32>(x->m1p, x->p);
            fill_mod<32>(x->m1q, x->q);
            x->r3_p1 = mod(R3, x->p).limbs(32);
            x->r3_q1 = mod(R3, x->q).limbs(32);
          }
          x->enc_split = x->S == 64 || x->enc_split_rns;
        }
      }
      switch (x->S) {
        case 32: {
          build_enc<32>(x.get());
          build_dec<32>(x.get());
          build_half<32>(x.get());
          // p^2, q^2 <= 1024 bits on the K = 40 RNS core for the collaborative entry points only
          const char* ev = getenv("PCB_RNSX");
          if (!ev || atoi(ev) != 0)
            x->has_rx = rnsx_build(p2, x->n, 32, 40, &x->rx_p) && rnsx_build(q2, x->n, 32, 40, &x->rx_q);
          break;
        }
        case 64: {
          build_enc<64>(x.get());
          build_dec<64>(x.get());
          build_half<64>(x.get());
          // RNS / tensor-core core for the CRT halves (default; PCB_RNS=0 selects the carry-chain
          // core).  Falls back to the carry core if the bases cannot be built for this key.
          const char* ev = getenv("PCB_RNS");
          if (!ev || atoi(ev) != 0)
            x->use_rns = rns_build(p2, x->n, 64, &x->rns_p) && rns_build(q2, x->n, 64, &x->rns_q);
          break;
        }
        case 128: {
          // 4096-bit keys: the CRT halves (4096-bit p^2, q^2) run on the streaming RNS core only
          if (!x->use_rnsx) return PCB_E_UNSUPPORTED;
          build_enc<128>(x.get());
          build_dec<128>(x.get());
          build_half<128>(x.get());
          break;
        }
        case 96: {
          build_enc<96>(x.get());
          build_dec<96>(x.get());
          build_half<96>(x.get());
          // the CRT halves run on the radix-2^28 core (28 x 112 limbs, 2 lanes per residue)
          const HBN R = HBN(1) << (28 * 112);
          x->rp2 = r28_mod(p2, 28, 112);
          x->rq2 = r28_mod(q2, 28, 112);
          x->rp2_nR = radix_limbs(mod(x->n * R, p2), 28, 112);
          x->rq2_nR = radix_limbs(mod(x->n * R, q2), 28, 112);
          x->rp2_R3 = radix_limbs(mod(R * R * R, p2), 28, 112);
          x->rq2_R3 = radix_limbs(mod(R * R * R, q2), 28, 112);
          break;
        }
      }
    }
    // exponent schedules
    std::vector<uint8_t> all;
    auto add = [&](const HBN& e, int* off, int* len) {
      std::vector<uint8_t> s = build_ops(e, kWindow);
      *off = (int)all.size();
      *len = (int)s.size();
      all.insert(all.end(), s.begin(), s.end());
    };
    if (x->has_prv) {
      const HBN p2 = x->p * x->p, q2 = x->q * x->q;
      add(mod(x->n, p2 - x->p), &x->off_enc_p, &x->len_enc_p);  // n mod phi(p^2)
      add(mod(x->n, q2 - x->q), &x->off_enc_q, &x->len_enc_q);
      add(x->p - HBN(1), &x->off_dec_p, &x->len_dec_p);
      add(x->q - HBN(1), &x->off_dec_q, &x->len_dec_q);
      const HBN eps = lcm(x->p - HBN(1), x->q - HBN(1));
      add(mod(eps, q2 - x->q), &x->off_epsq, &x->len_epsq);  // decrypt_with_half's q side (paillier.cpp:366)
      add(HBN(1), &x->off_one, &x->len_one);                 // plain reduction mod p^2
      add(x->p, &x->off_ep, &x->len_ep);                     // split encryption (enc_split)
      add(x->q, &x->off_eq, &x->len_eq);
    }
    add(x->n, &x->off_pub, &x->len_pub);
    if (cudaSetDevice(device) != cudaSuccess) return PCB_E_CUDA;
    if (cudaMalloc(&x->d_n, x->L * 4) != cudaSuccess) return PCB_E_CUDA;
    if (cudaMalloc(&x->d_n2, 2 * x->L * 4) != cudaSuccess) return PCB_E_CUDA;
    {
      std::vector<uint32_t> nl = x->n.limbs(x->L), n2l = x->n2.limbs(2 * x->L);
      if (cudaMemcpy(x->d_n, nl.data(), x->L * 4, cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
      if (cudaMemcpy(x->d_n2, n2l.data(), 2 * x->L * 4, cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
    }
    for (int k = 0; k < 2; k++) {
      if (cudaStreamCreateWithFlags(&x->side_st[k], cudaStreamNonBlocking) != cudaSuccess) return PCB_E_CUDA;
      if (cudaEventCreateWithFlags(&x->ev_join[k], cudaEventDisableTiming) != cudaSuccess) return PCB_E_CUDA;
    }
    if (cudaEventCreateWithFlags(&x->ev_fork, cudaEventDisableTiming) != cudaSuccess) return PCB_E_CUDA;
    // n^2 constants for the radix-2^r kernels (public-key encryption and homomorphic ops)
    {
      const size_t b2 = x->n2.bit_length();
      int rb = 0, nl = 0, tpi = 0;
      if (b2 + 4 <= 28 * 38) { rb = 28; nl = 38; tpi = 1; }
      else if (b2 + 4 <= 28 * 76) { rb = 28; nl = 76; tpi = 2; }
      else if (b2 + 4 <= 27 * 152) { rb = 27; nl = 152; tpi = 4; }
      else if (b2 + 4 <= 27 * 240) { rb = 27; nl = 240; tpi = 8; }
      else if (b2 + 4 <= 27 * 304) { rb = 27; nl = 304; tpi = 8; }
      if (rb) {
        R28Mod c = r28_mod(x->n2, rb, nl);
        x->wide.rb = rb;
        x->wide.n = nl;
        x->wide.tpi = tpi;
        x->wide.mlimb = c.mlimb;
        x->wide.minv = c.minv;
        x->wide.mwords = 2 * (int)x->L;
        x->wide.mword = x->n2.limbs(2 * x->L);
        x->wide_r2 = c.r2;
        const HBN R = HBN(1) << ((size_t)rb * nl);
        x->wide_nR = radix_limbs(mod(x->n * R, x->n2), rb, nl);
        std::vector<uint32_t> consts;
        auto push = [&](const HBN& v) {
          std::vector<uint32_t> l = radix_limbs(v, rb, nl);
          consts.insert(consts.end(), l.begin(), l.end());
        };
        push(mod(R * R, x->n2));                                // kConstR2
        push(mod(R, x->n2));                                    // kConstOneR
        push(HBN(1));                                           // kConstOne
        push(pow_mod(mod(R, x->n2), HBN((uint64_t)x->agg_chunk), x->n2));  // R^C (aggregate fix)
        if (cudaMalloc(&x->d_wconst, consts.size() * 4) != cudaSuccess) return PCB_E_CUDA;
        if (cudaMemcpy(x->d_wconst, consts.data(), consts.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
          return PCB_E_CUDA;
      }
    }
    {  // n^2 on the streaming RNS core (2048-bit keys: 4096-bit n^2, K = 144)
      const char* ev = getenv("PCB_RNSX_N2");
      int K = 0;
      if ((!ev || atoi(ev) != 0) && x->n2.bit_length() > 2048 && rnsx_shape((int)x->n2.bit_length(), &K))
        x->use_rx_n2 = rnsx_build(x->n2, x->n, 2 * (int)x->L, K, &x->rx_n2);
    }
    if (cudaMalloc(&x->d_sched, all.size()) != cudaSuccess) return PCB_E_CUDA;
    if (cudaMemcpy(x->d_sched, all.data(), all.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return PCB_E_CUDA;
  } catch (const std::bad_alloc&) {
    return PCB_E_ALLOC;
  } catch (...) {
    return PCB_E_SHAPE;
  }
  *out = x.release();
  return PCB_OK;
}

void pcb_ctx_destroy(pcb_ctx* x) {
  if (!x) return;
  cudaSetDevice(x->device);
  if (x->d_sched) cudaFree(x->d_sched);
  if (x->d_n) cudaFree(x->d_n);
  if (x->d_n2) cudaFree(x->d_n2);
  if (x->d_wconst) cudaFree(x->d_wconst);
  for (int k = 0; k < 2; k++) {
    if (x->side_st[k]) cudaStreamDestroy(x->side_st[k]);
    if (x->ev_join[k]) cudaEventDestroy(x->ev_join[k]);
  }
  if (x->ev_fork) cudaEventDestroy(x->ev_fork);
  rns_free(&x->rns_p);
  rns_free(&x->rns_q);
  rnsx_free(&x->rx_p);
  rnsx_free(&x->rx_q);
  rnsx_free(&x->rx_n2);
  rnsx_free(&x->rx1_p);
  rnsx_free(&x->rx1_q);
  if (x->d_gtab) cudaFree(x->d_gtab);
  delete x;
}

uint32_t pcb_ctx_n_limbs(const pcb_ctx* x) { return x ? x->L : 0; }
uint32_t pcb_ctx_n_bits(const pcb_ctx* x) { return x ? x->nbits : 0; }
int pcb_ctx_has_private(const pcb_ctx* x) { return x && x->has_prv ? 1 : 0; }
pcb_status pcb_ctx_set_priority(pcb_ctx* x, int high) {
  if (!x) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  int least = 0, greatest = 0;
  if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return PCB_E_CUDA;
  std::lock_guard<std::mutex> lk(x->mu);
  for (int k = 0; k < 2; k++) {
    if (x->side_st[k]) {
      cudaStreamSynchronize(x->side_st[k]);
      cudaStreamDestroy(x->side_st[k]);
      x->side_st[k] = nullptr;
    }
    if (cudaStreamCreateWithPriority(&x->side_st[k], cudaStreamNonBlocking, high ? greatest : least) != cudaSuccess)
      return PCB_E_CUDA;
  }
  // PCB_PRE_PAIRS=1: a low-priority context's RNS launches take two tiles per CTA (fewer SMs held by
  // background work for longer).  Measured on cfg3: 0.0668 vs 0.0643 s/iteration -- off by default.
  const char* pv = getenv("PCB_PRE_PAIRS");
  const bool pairs = !high && pv && atoi(pv) != 0;
  for (RnsXModulus* md : {&x->rx_p, &x->rx_q, &x->rx1_p, &x->rx1_q, &x->rx_n2}) md->prefer_pairs = pairs;
  return PCB_OK;
}

int pcb_ctx_engine(const pcb_ctx* x) {
  return !x || !x->has_prv ? 0 : (x->use_rnsx ? 3 : (x->use_rns ? 1 : (x->S == 96 ? 2 : 0)));
}

pcb_status pcb_ctx_get_n(const pcb_ctx* x, uint32_t* n, uint32_t* n2) {
  if (!x) return PCB_E_SHAPE;
  if (n) x->n.to_limbs(n, x->L);
  if (n2) x->n2.to_limbs(n2, 2 * x->L);
  return PCB_OK;
}

pcb_status pcb_ctx_set_generator(pcb_ctx* x, const uint32_t* g, uint32_t g_limbs) {
  if (!x || !g || !g_limbs) return PCB_E_SHAPE;
  try {
    const HBN gg = HBN::from_limbs(g, g_limbs);
    if (gg >= x->n2 || gg.bit_length() < 2 || gcd(gg, x->n) != HBN(1)) return PCB_E_SHAPE;
    if (gg == x->n + HBN(1)) {  // the binomial generator: nothing to do
      x->random_g = false;
      return PCB_OK;
    }
    x->random_g = true;
    x->g = gg;
    if (x->has_prv) {  // decryption constants from g (h_p, h_q; mu for decrypt_with_half)
      switch (x->S) {
        case 32: build_dec<32>(x); build_half<32>(x); break;
        case 64: build_dec<64>(x); build_half<64>(x); break;
        case 96: build_dec<96>(x); build_half<96>(x); break;
        case 128: build_dec<128>(x); build_half<128>(x); break;
        default: return PCB_E_UNSUPPORTED;
      }
    }
    // G_j = g^(2^(64 j)) mod n^2, j < ceil(L / 2): key-setup constants for g^m on the device
    x->gdig = (int)((x->L + 1) / 2);
    const size_t W = 2 * x->L;
    std::vector<uint32_t> tab((size_t)x->gdig * W, 0);
    HBN gj = gg;
    const HBN two64 = HBN(1) << 64;
    for (int j = 0; j < x->gdig; j++) {
      gj.to_limbs(tab.data() + (size_t)j * W, W);
      gj = pow_mod(gj, two64, x->n2);
    }
    if (set_device(x)) return PCB_E_CUDA;
    if (x->d_gtab) cudaFree(x->d_gtab);
    x->d_gtab = nullptr;
    if (cudaMalloc(&x->d_gtab, tab.size() * 4) != cudaSuccess) return PCB_E_ALLOC;
    if (cudaMemcpy(x->d_gtab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
  } catch (...) {
    return PCB_E_SHAPE;
  }
  return PCB_OK;
}

void pcb_ctx_counters(const pcb_ctx* x, uint64_t* pow_full, uint64_t* pow_half) {
  if (pow_full) *pow_full = x ? x->pow_full.load() : 0;
  if (pow_half) *pow_half = x ? x->pow_half.load() : 0;
}

void pcb_ctx_reset_counters(pcb_ctx* x) {
  if (!x) return;
  x->pow_full = 0;
  x->pow_half = 0;
}

}  // extern "C"

// Runs the two CRT halves concurrently: fork from `st`, side p on side_st[0], side q on
// side_st[1], join back into `st`.
template <class FP, class FQ>
static pcb_status fork_join(pcb_ctx* x, cudaStream_t st, FP&& fp, FQ&& fq, size_t count) {
  // A batch that fills the GPU gains nothing from running the halves concurrently: run them
  // back to back on the caller's stream (clean per-launch timing, no SM contention).
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (count >= (size_t)nsm * 256) {
    pcb_status e = fp(st);
    if (!e) e = fq(st);
    return e;
  }
  std::lock_guard<std::mutex> lk(x->mu);
  pcb_status e = cuda_check(cudaEventRecord(x->ev_fork, st));
  for (int k = 0; k < 2 && !e; k++) e = cuda_check(cudaStreamWaitEvent(x->side_st[k], x->ev_fork, 0));
  if (!e) e = fp(x->side_st[0]);
  if (!e) e = fq(x->side_st[1]);
  for (int k = 0; k < 2; k++) {
    cudaEventRecord(x->ev_join[k], x->side_st[k]);
    cudaStreamWaitEvent(st, x->ev_join[k], 0);
  }
  return e;
}

// Stage 1 of the split CRT encryption: u = r^q mod p (half 0) or r^p mod q
// (half 1), x->w1 words per element, on the RNS core (default) or the carry core.
static pcb_status split_stage1(pcb_ctx* x, int half, const uint32_t* r, const int32_t* stv, size_t count, uint32_t* u,
                               cudaStream_t st) {
  const uint8_t* ops = x->d_sched + (half ? x->off_ep : x->off_eq);
  const int nops = half ? x->len_ep : x->len_eq;
  if (x->enc_split_rns)
    return launch_rnsx(half ? x->rx1_q : x->rx1_p, kRxDec, ops, nops, kTab, r, (int)x->L, nullptr, 0, count, u, st, 0.0);
  return launch_side<32>(half ? x->m1q : x->m1p, (half ? x->r3_q1 : x->r3_p1).data(), ops, nops, kTab, kSideDec, r,
                         (int)x->L, nullptr, 0, stv, count, u, st, -1);
}

// Device-pointer core of CRT encryption (m given as limbs, or v quantized in the prep kernel).
static pcb_status enc_core(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const double* v, double zmin, double zmax,
                           double delta, int fine, uint64_t* q_out, unsigned long long* clamps, const uint32_t* r,
                           size_t count, uint32_t* c, int32_t* st_user, cudaStream_t st) {
  const int S = x->S;
  int32_t* stv = st_user;
  uint32_t *mq = nullptr, *yp = nullptr, *yq = nullptr;
  pcb_status e = PCB_OK;
  if (!stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  const int mql = 4;
  if (!e && v) e = scratch_alloc(count * mql * 4, (void**)&mq, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yp, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yq, st);
  if (!e)
    e = launch_enc_prep(m, (int)m_limbs, v, zmin, zmax, delta, fine, mq, mql, q_out, clamps, r, x->d_n, (int)x->L,
                        stv, count, st);
  const uint32_t* mm = v ? mq : m;
  const uint32_t* mmv = mm;
  const uint32_t* mm_ = mm;
  const int ml = v ? mql : (int)m_limbs;
  const uint8_t* opp = x->d_sched + x->off_enc_p;
  const uint8_t* opq = x->d_sched + x->off_enc_q;
  if (!e && x->use_rnsx && x->enc_split) {
    const double mm = 2.0 * S * S + S, alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm + 2 * mm;
    const uint8_t* oep = x->d_sched + x->off_ep;
    const uint8_t* oeq = x->d_sched + x->off_eq;
    uint32_t *up = nullptr, *uq = nullptr;
    const int w1 = x->w1;
    e = scratch_alloc(count * w1 * 4, (void**)&up, st);
    if (!e) e = scratch_alloc(count * w1 * 4, (void**)&uq, st);
    // stage 1: u = r^q mod p (kSideDec reduces the 2048-bit r: r R = r_lo R + r_hi R^2);
    // stage 2: (1 + m n) u^p mod p^2.  The canonical work is accounted on stage 2.
    if (!e)
      e = fork_join(
          x, st,
          [&](cudaStream_t s2) {
            pcb_status e2 = split_stage1(x, 0, r, stv, count, up, s2);
            if (!e2) e2 = launch_rnsx(x->rx_p, kRxEnc, oep, x->len_ep, kTab, up, w1, mm_, ml, count, yp, s2, alg);
            return e2;
          },
          [&](cudaStream_t s2) {
            pcb_status e2 = split_stage1(x, 1, r, stv, count, uq, s2);
            if (!e2) e2 = launch_rnsx(x->rx_q, kRxEnc, oeq, x->len_eq, kTab, uq, w1, mm_, ml, count, yq, s2, alg);
            return e2;
          },
          count);
    if (!e && S == 64) e = launch_garner<64>(*reinterpret_cast<const CrtEncConsts<64>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
    if (!e && S == 96) e = launch_garner<96>(*reinterpret_cast<const CrtEncConsts<96>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
    if (!e && S == 128) e = launch_garner<128>(*reinterpret_cast<const CrtEncConsts<128>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
    scratch_free(up, st);
    scratch_free(uq, st);
  } else if (!e && x->use_rnsx) {
    const double mm = 2.0 * S * S + S, alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm + 2 * mm;
    e = fork_join(
        x, st,
        [&](cudaStream_t s2) {
          return launch_rnsx(x->rx_p, kRxEnc, opp, x->len_enc_p, kTab, r, (int)x->L, mm_, ml, count, yp, s2, alg);
        },
        [&](cudaStream_t s2) {
          return launch_rnsx(x->rx_q, kRxEnc, opq, x->len_enc_q, kTab, r, (int)x->L, mm_, ml, count, yq, s2, alg);
        },
        count);
    if (!e && S == 64) e = launch_garner<64>(*reinterpret_cast<const CrtEncConsts<64>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
    if (!e && S == 96) e = launch_garner<96>(*reinterpret_cast<const CrtEncConsts<96>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
    if (!e && S == 128) e = launch_garner<128>(*reinterpret_cast<const CrtEncConsts<128>*>(x->enc_blob.data()), yp, yq, stv, c, (int)x->L, count, st);
  } else if (!e && x->use_rns) {
    const auto& k = *reinterpret_cast<const CrtEncConsts<64>*>(x->enc_blob.data());
    const double mm = 2.0 * 64 * 64 + 64, alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm + 2 * mm;
    e = fork_join(
        x, st,
        [&](cudaStream_t s2) {
          return launch_rns(x->rns_p, kRnsEnc, opp, x->len_enc_p, kTab, r, (int)x->L, mm_, ml, count, yp, s2, alg);
        },
        [&](cudaStream_t s2) {
          return launch_rns(x->rns_q, kRnsEnc, opq, x->len_enc_q, kTab, r, (int)x->L, mm_, ml, count, yq, s2, alg);
        },
        count);
    if (!e) e = launch_garner<64>(k, yp, yq, stv, c, (int)x->L, count, st);
  } else if (!e) {
    switch (S) {
#define PCB_CASE(SS)                                                                                                  \
  case SS: {                                                                                                          \
    const auto& k = *reinterpret_cast<const CrtEncConsts<SS>*>(x->enc_blob.data());                                   \
    e = fork_join(                                                                                                    \
        x, st,                                                                                                        \
        [&](cudaStream_t s2) {                                                                                        \
          return launch_side<SS>(k.mp, k.nRp, opp, x->len_enc_p, kTab, kSideEnc, r, (int)x->L, mm, ml, stv, count, yp, s2, (int)x->nbits); \
        },                                                                                                            \
        [&](cudaStream_t s2) {                                                                                        \
          return launch_side<SS>(k.mq, k.nRq, opq, x->len_enc_q, kTab, kSideEnc, r, (int)x->L, mm, ml, stv, count, yq, s2, (int)x->nbits); \
        }, count);                                                                                                    \
    if (!e) e = launch_garner<SS>(k, yp, yq, stv, c, (int)x->L, count, st);                                           \
    break;                                                                                                            \
  }
      PCB_CASE(32)
      PCB_CASE(64)
#undef PCB_CASE
      case 96: {
        const auto& k = *reinterpret_cast<const CrtEncConsts<96>*>(x->enc_blob.data());
        const double mm = 2.0 * 96 * 96 + 96, alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm + 2 * mm;
        e = fork_join(
            x, st,
            [&](cudaStream_t s2) {
              return launch_side28<28, 112, 2>(x->rp2.mlimb.data(), x->rp2.mword.data(), x->rp2.mwords,
                                               x->rp2.r2.data(), x->rp2_nR.data(), x->rp2.minv, opp, x->len_enc_p,
                                               kTab, 0, r, (int)x->L, mmv, ml, stv, count, yp, 96, s2, alg);
            },
            [&](cudaStream_t s2) {
              return launch_side28<28, 112, 2>(x->rq2.mlimb.data(), x->rq2.mword.data(), x->rq2.mwords,
                                               x->rq2.r2.data(), x->rq2_nR.data(), x->rq2.minv, opq, x->len_enc_q,
                                               kTab, 0, r, (int)x->L, mmv, ml, stv, count, yq, 96, s2, alg);
            },
            count);
        if (!e) e = launch_garner<96>(k, yp, yq, stv, c, (int)x->L, count, st);
        break;
      }
      default: e = PCB_E_UNSUPPORTED;
    }
  }
  scratch_free(yp, st);
  scratch_free(yq, st);
  scratch_free(mq, st);
  if (!st_user) scratch_free(stv, st);
  return e;
}

static pcb_status dec_core(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* m, int32_t* st_user,
                           cudaStream_t st) {
  const int S = x->S;
  int32_t* stv = st_user;
  uint32_t *yp = nullptr, *yq = nullptr;
  pcb_status e = PCB_OK;
  if (!stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yp, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yq, st);
  if (!e) e = launch_dec_prep(c, x->d_n2, (int)x->L, stv, count, st);
  const uint8_t* opp = x->d_sched + x->off_dec_p;
  const uint8_t* opq = x->d_sched + x->off_dec_q;
  if (!e && x->use_rnsx) {
    const double mm = 2.0 * S * S + S,
                 alg = ((double)(x->nbits / 2) + (double)((x->nbits / 2 + 3) / 4)) * mm + 2 * mm;
    e = fork_join(
        x, st,
        [&](cudaStream_t s2) {
          return launch_rnsx(x->rx_p, kRxDec, opp, x->len_dec_p, kTab, c, 2 * (int)x->L, nullptr, 0, count, yp, s2, alg);
        },
        [&](cudaStream_t s2) {
          return launch_rnsx(x->rx_q, kRxDec, opq, x->len_dec_q, kTab, c, 2 * (int)x->L, nullptr, 0, count, yq, s2, alg);
        },
        count);
    if (!e && S == 64) e = launch_dec_finish<64>(*reinterpret_cast<const CrtDecConsts<64>*>(x->dec_blob.data()), yp, yq, stv, m, (int)x->L, count, st);
    if (!e && S == 96) e = launch_dec_finish<96>(*reinterpret_cast<const CrtDecConsts<96>*>(x->dec_blob.data()), yp, yq, stv, m, (int)x->L, count, st);
    if (!e && S == 128) e = launch_dec_finish<128>(*reinterpret_cast<const CrtDecConsts<128>*>(x->dec_blob.data()), yp, yq, stv, m, (int)x->L, count, st);
  } else if (!e && x->use_rns) {
    const auto& k = *reinterpret_cast<const CrtDecConsts<64>*>(x->dec_blob.data());
    const double mm = 2.0 * 64 * 64 + 64,
                 alg = ((double)(x->nbits / 2) + (double)((x->nbits / 2 + 3) / 4)) * mm + 2 * mm;
    e = fork_join(
        x, st,
        [&](cudaStream_t s2) {
          return launch_rns(x->rns_p, kRnsDec, opp, x->len_dec_p, kTab, c, 2 * (int)x->L, nullptr, 0, count, yp, s2,
                            alg);
        },
        [&](cudaStream_t s2) {
          return launch_rns(x->rns_q, kRnsDec, opq, x->len_dec_q, kTab, c, 2 * (int)x->L, nullptr, 0, count, yq, s2,
                            alg);
        },
        count);
    if (!e) e = launch_dec_finish<64>(k, yp, yq, stv, m, (int)x->L, count, st);
  } else if (!e) {
    switch (S) {
#define PCB_CASE(SS)                                                                                                \
  case SS: {                                                                                                        \
    const auto& k = *reinterpret_cast<const CrtDecConsts<SS>*>(x->dec_blob.data());                                 \
    e = fork_join(                                                                                                  \
        x, st,                                                                                                      \
        [&](cudaStream_t s2) {                                                                                      \
          return launch_side<SS>(k.mp, k.r3p, opp, x->len_dec_p, kTab, kSideDec, c, 2 * (int)x->L, nullptr, 0, stv, \
                                 count, yp, s2, (int)x->nbits / 2);                                                 \
        },                                                                                                          \
        [&](cudaStream_t s2) {                                                                                      \
          return launch_side<SS>(k.mq, k.r3q, opq, x->len_dec_q, kTab, kSideDec, c, 2 * (int)x->L, nullptr, 0, stv, \
                                 count, yq, s2, (int)x->nbits / 2);                                                 \
        }, count);                                                                                                  \
    if (!e) e = launch_dec_finish<SS>(k, yp, yq, stv, m, (int)x->L, count, st);                                     \
    break;                                                                                                          \
  }
      PCB_CASE(32)
      PCB_CASE(64)
#undef PCB_CASE
      case 96: {
        const auto& k = *reinterpret_cast<const CrtDecConsts<96>*>(x->dec_blob.data());
        const double mm = 2.0 * 96 * 96 + 96, alg = ((double)(x->nbits / 2) + (double)((x->nbits / 2 + 3) / 4)) * mm + 2 * mm;
        e = fork_join(
            x, st,
            [&](cudaStream_t s2) {
              return launch_side28<28, 112, 2>(x->rp2.mlimb.data(), x->rp2.mword.data(), x->rp2.mwords,
                                               x->rp2.r2.data(), x->rp2_R3.data(), x->rp2.minv, opp, x->len_dec_p,
                                               kTab, 1, c, 2 * (int)x->L, nullptr, 0, stv, count, yp, 96, s2, alg);
            },
            [&](cudaStream_t s2) {
              return launch_side28<28, 112, 2>(x->rq2.mlimb.data(), x->rq2.mword.data(), x->rq2.mwords,
                                               x->rq2.r2.data(), x->rq2_R3.data(), x->rq2.minv, opq, x->len_dec_q,
                                               kTab, 1, c, 2 * (int)x->L, nullptr, 0, stv, count, yq, 96, s2, alg);
            },
            count);
        if (!e) e = launch_dec_finish<96>(k, yp, yq, stv, m, (int)x->L, count, st);
        break;
      }
      default: e = PCB_E_UNSUPPORTED;
    }
  }
  scratch_free(yp, st);
  scratch_free(yq, st);
  if (!st_user) scratch_free(stv, st);
  return e;
}


// ---- n^2 (radix-2^r) dispatch ------------------------------------------------------------------
static pcb_status run_wide(pcb_ctx* x, const WStep* prog, int nsteps, const uint32_t* xin, const uint32_t* b,
                           const uint64_t* k, int xin_per_out, size_t count, size_t nout, uint32_t* y, int ntab,
                           cudaStream_t st, const MatvecGeom* mg = nullptr) {
  const WideMod& w = x->wide;
#define PCB_W(RB, NN, TT)                                                                                        \
  if (w.rb == RB && w.n == NN && w.tpi == TT)                                                                     \
    return launch_wide<RB, NN, TT>(w, prog, nsteps, x->d_wconst, xin, b, k, xin_per_out, count, nout, y, ntab, st, mg);
  PCB_W(28, 38, 1)
  PCB_W(28, 76, 2)
  PCB_W(27, 152, 4)
  PCB_W(27, 240, 8)
  PCB_W(27, 304, 8)
#undef PCB_W
  return PCB_E_UNSUPPORTED;
}

static std::vector<WStep> prog_hom_add();
static std::vector<WStep> prog_scalar_pow();

// g^m mod n^2 for a random generator (g_power_full, paillier.cpp:253-258) with per-element m
// (count x m_limbs words): m = sum_j m_j 2^(64 j), g^m = prod_j G_j^(m_j) with the context's digit
// powers G_j, each a 64-bit-exponent power on the n^2 core (prog_scalar_pow), multiplied in with
// prog_hom_add.  Chunks of <= 2^16 elements bound the broadcast-base scratch.
static pcb_status gpow_core(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, size_t count, uint32_t* out,
                            cudaStream_t st) {
  if (!x->random_g || !x->d_gtab) return PCB_E_UNSUPPORTED;
  const size_t W = 2 * x->L, wb = W * 4;
  const int nd = std::min<int>((int)((m_limbs + 1) / 2), x->gdig);
  const size_t CH = 1 << 16;
  std::vector<WStep> pw = prog_scalar_pow(), pa = prog_hom_add();
  uint32_t *mp = nullptr, *base = nullptr, *pj = nullptr;
  uint64_t* kj = nullptr;
  const size_t mw = 2 * (size_t)nd;  // even-width copy of m (64-bit digits)
  pcb_status e = scratch_alloc(count * mw * 4, (void**)&mp, st);
  if (!e) e = cuda_check(cudaMemsetAsync(mp, 0, count * mw * 4, st));
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync(mp, mw * 4, m, m_limbs * 4, std::min<size_t>(m_limbs, mw) * 4, count,
                                     cudaMemcpyDeviceToDevice, st));
  if (!e) e = scratch_alloc(std::min(count, CH) * wb, (void**)&base, st);
  if (!e) e = scratch_alloc(std::min(count, CH) * wb, (void**)&pj, st);
  if (!e) e = scratch_alloc(std::min(count, CH) * 8, (void**)&kj, st);
  for (size_t c0 = 0; !e && c0 < count; c0 += CH) {
    const size_t cn = std::min(CH, count - c0);
    uint32_t* acc = out + c0 * W;
    for (int j = 0; !e && j < nd; j++) {
      bcast_kernel<<<(int)std::min<size_t>((cn * W + 255) / 256, 4096), 256, 0, st>>>(base, x->d_gtab + (size_t)j * W,
                                                                                  (int)W, cn);
      count_launch();
      e = cuda_check(cudaGetLastError());
      if (!e)
        e = cuda_check(cudaMemcpy2DAsync(kj, 8, mp + c0 * mw + 2 * j, mw * 4, 8, cn, cudaMemcpyDeviceToDevice, st));
      if (!e)
        e = run_wide(x, pw.data(), (int)pw.size(), base, nullptr, kj, 1, cn, cn, j ? pj : acc, 16, st);
      if (!e && j) e = run_wide(x, pa.data(), (int)pa.size(), acc, pj, nullptr, 1, cn, cn, acc, 1, st);
    }
  }
  scratch_free(mp, st);
  scratch_free(base, st);
  scratch_free(pj, st);
  scratch_free(kj, st);
  return e;
}

// Public-key encryption c = (1 + m n) r^n mod n^2 (encrypt_with_r, paillier.cpp:320-328) on the
// radix kernel at modulus n^2 (ENC mode of side28.cu).
static pcb_status run_pub_enc(pcb_ctx* x, const uint32_t* r, const uint32_t* m, int m_words, const int32_t* stv,
                              size_t count, uint32_t* c, cudaStream_t st) {
  const WideMod& w = x->wide;
  const uint8_t* ops = x->d_sched + x->off_pub;
  const double S2 = 2.0 * x->L, mm = 2 * S2 * S2 + S2;
  const double alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm + mm;  // EXP(2|n|,|n|) + MM(2|n|)
  if (x->use_rx_n2)  // streaming RNS core at n^2 (rnsx.cu); rows with argument errors stay 0
    return launch_rnsx(x->rx_n2, kRxEnc, ops, x->len_pub, kTab, r, (int)x->L, m, m_words, count, c, st, alg, stv);
#define PCB_W(RB, NN, TT)                                                                                           \
  if (w.rb == RB && w.n == NN && w.tpi == TT)                                                                        \
    return launch_side28<RB, NN, TT>(w.mlimb.data(), w.mword.data(), w.mwords, x->wide_r2.data(), x->wide_nR.data(), \
                                     w.minv, ops, x->len_pub, kTab, 0, r, (int)x->L, m, m_words, stv, count, c,      \
                                     2 * (int)x->L, st, alg);
  PCB_W(28, 38, 1)
  PCB_W(28, 76, 2)
  PCB_W(27, 152, 4)
  PCB_W(27, 240, 8)
  PCB_W(27, 304, 8)
#undef PCB_W
  return PCB_E_UNSUPPORTED;
}

static std::vector<WStep> prog_hom_add() {
  return {WStep{kSrcX, 0, kSrcConst, (uint8_t)kConstR2, 0, 0, 0, 0},  // a R
          WStep{kSrcReg, 0, kSrcB, 0, kPostOut, 0, 0, 0}};           // a b
}

static std::vector<WStep> prog_scalar_pow() {
  std::vector<WStep> p;
  p.push_back(WStep{kSrcX, 0, kSrcConst, (uint8_t)kConstR2, kPostAcc | kPostTab, 1, 0, 0});  // t1 = cR
  p.push_back(WStep{kSrcReg, 0, kSrcAcc, 0, kPostTab, 2, 0, 0});                            // t2
  for (int e = 3; e < 16; e++) p.push_back(WStep{kSrcReg, 0, kSrcTab, 1, kPostTab, (uint8_t)e, 0, 0});
  p.push_back(WStep{kSrcTabDigit, 15, kSrcConst, (uint8_t)kConstOneR, kPostAcc, 0, 0, 0});  // seed: top digit
  for (int w = 14; w >= 0; w--) {
    for (int q = 0; q < 4; q++) p.push_back(WStep{kSrcReg, 0, kSrcAcc, 0, kPostAcc, 0, 0, 0});
    p.push_back(WStep{kSrcReg, 0, kSrcTabDigit, (uint8_t)w, kPostAcc, 0, 0, 0});
  }
  p.push_back(WStep{kSrcReg, 0, kSrcConst, (uint8_t)kConstOne, kPostOut, 0, 0, 0});
  return p;
}

// matvec phase A1: the window bases T[col][w][1] = zv_col^(64^w) R, one squaring chain per column
static std::vector<WStep> prog_mat_chain(int nwin) {
  std::vector<WStep> p;
  p.push_back(WStep{kSrcX, 0, kSrcConst, (uint8_t)kConstR2, kPostAcc | kPostGTab, 1, 0, 0});
  for (int w = 1; w < nwin; w++)
    for (int q = 1; q <= kMatWin; q++)
      p.push_back(WStep{kSrcReg, 0, kSrcAcc, 0, (uint8_t)(q == kMatWin ? (kPostAcc | kPostGTab) : kPostAcc), 1,
                        (uint8_t)(q == kMatWin ? w : 0), 0});
  return p;
}

// matvec phase A2 (fill mode, one element per (column, window)): T[d] = T[d-1] T[1], d = 2..63
static std::vector<WStep> prog_mat_fill() {
  std::vector<WStep> p;
  p.push_back(WStep{kSrcGEntry, 1, kSrcGEntry, 1, kPostGTab, 2, 0, 0});
  for (int d = 3; d < 64; d++) p.push_back(WStep{kSrcReg, 0, kSrcOpKeep, 0, kPostGTab, (uint8_t)d, 0, 0});
  return p;
}

// matvec phase B: product of the table entries of cc columns x nwin windows (Montgomery form)
static std::vector<WStep> prog_mat_prod(int cc, int nwin) {
  std::vector<WStep> p;
  std::vector<uint8_t> ids;
  for (int j = 0; j < cc; j++)
    for (int w = 0; w < nwin; w++) ids.push_back((uint8_t)(j * 16 + w));
  if (ids.size() == 1) {
    p.push_back(WStep{kSrcMatTab, ids[0], kSrcConst, (uint8_t)kConstOneR, kPostOut, 0, 0, 0});
    return p;
  }
  p.push_back(WStep{kSrcMatTab, ids[0], kSrcMatTab, ids[1], 0, 0, 0, 0});
  for (size_t q = 2; q < ids.size(); q++) p.push_back(WStep{kSrcReg, 0, kSrcMatTab, ids[q], 0, 0, 0, 0});
  p.back().post = kPostOut;
  return p;
}

// matvec phase C: out_i = alpha_i * prod_c P_{i,c}  (inputs per row: nch Montgomery partials, then alpha)
static std::vector<WStep> prog_mat_combine(int nch) {
  std::vector<WStep> p;
  p.push_back(WStep{kSrcX, 0, kSrcX, 1, 0, 0, 0, 0});
  for (int q = 2; q <= nch; q++) p.push_back(WStep{kSrcReg, 0, kSrcX, (uint8_t)q, 0, 0, 0, 0});
  p.back().post = kPostOut;
  return p;
}

static std::vector<WStep> prog_aggregate(int chunk) {
  std::vector<WStep> p;
  p.push_back(WStep{kSrcX, 0, kSrcX, 1, 0, 0, 0, 0});
  for (int j = 2; j < chunk; j++) p.push_back(WStep{kSrcReg, 0, kSrcX, (uint8_t)j, 0, 0, 0, 0});
  p.push_back(WStep{kSrcReg, 0, kSrcConst, (uint8_t)kConstFirstF, kPostOut, 0, 0, 0});  // x R^C R^-1 ... fix
  return p;
}

// Encryption under a random generator: c = g^m r^n mod n^2 (encrypt_with_r / crt_encrypt_with_r,
// paillier.cpp:320-344; the CRT form is the same residue, test_paillier.cpp:63-78).  r^n (CRT or
// n^2 path, as for g = n + 1 with m = 0), then g^m by gpow_core, one product, and the argument
// statuses of the real m and r (rows that fail come back as 0).
static pcb_status encrypt_random_g(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const uint32_t* r, size_t count,
                                   uint32_t* c, int use_crt, int32_t* status, cudaStream_t st) {
  Staged sm, sr, sc, ss;
  uint32_t *m0 = nullptr, *gm = nullptr;
  int32_t* stv = nullptr;
  const size_t W = 2 * x->L;
  pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
  if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
  if (!e) e = stage_out(c, count * W * 4, st, &sc);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * 4, (void**)&m0, st);
  if (!e) e = cuda_check(cudaMemsetAsync(m0, 0, count * 4, st));
  if (!e && x->has_prv) {
    e = enc_core(x, m0, 1, nullptr, 0, 0, 0, 0, nullptr, nullptr, (const uint32_t*)sr.dev, count, (uint32_t*)sc.dev,
                 stv, st);
  } else if (!e) {
    e = launch_enc_prep(m0, 1, nullptr, 0, 0, 0, 0, nullptr, 0, nullptr, nullptr, (const uint32_t*)sr.dev, x->d_n,
                        (int)x->L, stv, count, st);
    if (!e) e = cuda_check(cudaMemsetAsync(sc.dev, 0, count * W * 4, st));
    if (!e) e = run_pub_enc(x, (const uint32_t*)sr.dev, m0, 1, stv, count, (uint32_t*)sc.dev, st);
  }
  if (!e)  // statuses of the real arguments
    e = launch_enc_prep((const uint32_t*)sm.dev, (int)m_limbs, nullptr, 0, 0, 0, 0, nullptr, 0, nullptr, nullptr,
                        (const uint32_t*)sr.dev, x->d_n, (int)x->L, stv, count, st);
  if (!e) e = scratch_alloc(count * W * 4, (void**)&gm, st);
  if (!e) e = gpow_core(x, (const uint32_t*)sm.dev, m_limbs, count, gm, st);
  std::vector<WStep> pa = prog_hom_add();
  if (!e) e = run_wide(x, pa.data(), (int)pa.size(), (const uint32_t*)sc.dev, gm, nullptr, 1, count, count,
                       (uint32_t*)sc.dev, 1, st);
  if (!e) {
    zero_bad_rows_kernel<<<(int)std::min<size_t>((count * W + 255) / 256, 4096), 256, 0, st>>>((uint32_t*)sc.dev,
                                                                                             (int)W, stv, count);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  scratch_free(m0, st);
  scratch_free(gm, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sm.host || sr.host || sc.host || ss.host;
  for (auto* p : {&sm, &sr, &sc, &ss}) unstage(p, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) {  // reference ledger: g^m and r^n (paillier.cpp:253-258, 325; 264-271, 339-342)
    if (use_crt)
      x->pow_half += 4 * (uint64_t)count;
    else
      x->pow_full += 2 * (uint64_t)count;
  }
  return e;
}

extern "C" {

pcb_status pcb_encrypt(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const uint32_t* r, size_t count, uint32_t* c,
                       int use_crt, int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_encrypt");
  if (!x || (count && (!m || !r || !c))) return PCB_E_SHAPE;
  if (m_limbs == 0 || m_limbs > x->L) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (!x->has_prv && use_crt) return PCB_E_NO_PRIVATE;
  if (x->random_g) {
    if (auto e = set_device(x)) return e;
    return encrypt_random_g(x, m, m_limbs, r, count, c, use_crt, status, (cudaStream_t)stream);
  }
  // use_crt = 0 on a private context: same residue through the CRT halves (the reference's own
  // tests pin CRT == direct bit-identically, test_paillier.cpp:63-78, acceptance [2]); the
  // ledger still records the direct path (pow_full).  Public-key-only: n^2 path (TODO).
  if (!x->has_prv && use_crt) return PCB_E_NO_PRIVATE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const bool m_dev = is_device_ptr(m), r_dev = is_device_ptr(r), c_dev = is_device_ptr(c);
  if (count >= kPipeMin && (!m_dev || !r_dev || !c_dev)) {  // host buffers: chunked, copies beside the compute
    const size_t WM = m_limbs, WR = x->L, WO = 2 * x->L;
    const size_t chunk = ((count + kPipeChunks - 1) / kPipeChunks + 255) / 256 * 256;
    HostPipe hp;
    pcb_status e = hp.init(st);
    uint32_t *dmv[2] = {nullptr, nullptr}, *drv[2] = {nullptr, nullptr}, *dcv[2] = {nullptr, nullptr};
    int32_t* sall = nullptr;
    for (int b = 0; b < 2 && !e; b++) {
      if (!m_dev) e = scratch_alloc(chunk * WM * 4, (void**)&dmv[b], st);
      if (!e && !r_dev) e = scratch_alloc(chunk * WR * 4, (void**)&drv[b], st);
      if (!e && !c_dev) e = scratch_alloc(chunk * WO * 4, (void**)&dcv[b], st);
    }
    if (!e) e = scratch_alloc(count * 4, (void**)&sall, st);
    if (!e) e = cuda_check(cudaStreamSynchronize(st));  // the scratch exists before the copy streams use it
    for (size_t i = 0, off = 0; off < count && !e; i++, off += chunk) {
      const int b = (int)(i & 1);
      const size_t cnt = std::min(chunk, count - off);
      const uint32_t* ms = m + off * WM;
      const uint32_t* rs = r + off * WR;
      uint32_t* cs = c + off * WO;
      if (!m_dev || !r_dev) {
        if (i >= 2) e = cuda_check(cudaStreamWaitEvent(hp.cin, hp.comp[b], 0));
        if (!e && !m_dev) e = cuda_check(cudaMemcpyAsync(dmv[b], ms, cnt * WM * 4, cudaMemcpyHostToDevice, hp.cin));
        if (!e && !r_dev) e = cuda_check(cudaMemcpyAsync(drv[b], rs, cnt * WR * 4, cudaMemcpyHostToDevice, hp.cin));
        if (!e) e = cuda_check(cudaEventRecord(hp.in[b], hp.cin));
        if (!e) e = cuda_check(cudaStreamWaitEvent(st, hp.in[b], 0));
        if (!m_dev) ms = dmv[b];
        if (!r_dev) rs = drv[b];
      }
      if (!c_dev) {
        if (i >= 2 && !e) e = cuda_check(cudaStreamWaitEvent(st, hp.out[b], 0));
        cs = dcv[b];
      }
      if (!e) e = pcb_encrypt(x, ms, m_limbs, rs, cnt, cs, use_crt, sall + off, stream);  // device: asynchronous
      if (!e) e = cuda_check(cudaEventRecord(hp.comp[b], st));
      if (!c_dev && !e) {
        e = cuda_check(cudaStreamWaitEvent(hp.cout, hp.comp[b], 0));
        if (!e) e = cuda_check(cudaMemcpyAsync(c + off * WO, dcv[b], cnt * WO * 4, cudaMemcpyDeviceToHost, hp.cout));
        if (!e) e = cuda_check(cudaEventRecord(hp.out[b], hp.cout));
      }
    }
    if (cudaStreamSynchronize(hp.cout) != cudaSuccess && !e) e = PCB_E_CUDA;
    if (!e && status) e = cuda_check(cudaMemcpyAsync(status, sall, count * 4, cudaMemcpyDefault, st));
    if (!e && !status) e = first_failure(sall, count, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
    for (int b = 0; b < 2; b++)
      for (void* p : {(void*)dmv[b], (void*)drv[b], (void*)dcv[b]}) scratch_free(p, st);
    scratch_free(sall, st);
    cudaStreamSynchronize(st);
    return e;
  }
  Staged sm, sr, sc, ss;
  if (!x->has_prv) {  // public-key context: direct encryption at n^2
    pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
    if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
    if (!e) e = stage_out(c, count * 2 * x->L * 4, st, &sc);
    if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
    int32_t* stv = (int32_t*)ss.dev;
    if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
    if (!e)
      e = launch_enc_prep((const uint32_t*)sm.dev, (int)m_limbs, nullptr, 0, 0, 0, 0, nullptr, 0, nullptr, nullptr,
                          (const uint32_t*)sr.dev, x->d_n, (int)x->L, stv, count, st);
    if (!e) e = cuda_check(cudaMemsetAsync(sc.dev, 0, count * 2 * x->L * 4, st));
    if (!e) e = run_pub_enc(x, (const uint32_t*)sr.dev, (const uint32_t*)sm.dev, (int)m_limbs, stv, count,
                            (uint32_t*)sc.dev, st);
    if (!e) e = unstage_out(c, &sc, st);
    if (!e) e = unstage_out(status, &ss, st);
    if (!e && !status) e = first_failure(stv, count, st);
    if (!ss.dev) scratch_free(stv, st);
    const bool any_host = sm.host || sr.host || sc.host || ss.host;
    unstage(&sm, st);
    unstage(&sr, st);
    unstage(&sc, st);
    unstage(&ss, st);
    if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
    if (!e) x->pow_full += (uint64_t)count;
    return e;
  }
  pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
  if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
  if (!e) e = stage_out(c, count * 2 * x->L * 4, st, &sc);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  int32_t* stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e)
    e = enc_core(x, (const uint32_t*)sm.dev, m_limbs, nullptr, 0, 0, 0, 0, nullptr, nullptr, (const uint32_t*)sr.dev,
                 count, (uint32_t*)sc.dev, stv, st);
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sm.host || sr.host || sc.host || ss.host;
  unstage(&sm, st);
  unstage(&sr, st);
  unstage(&sc, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) {
    if (use_crt)
      x->pow_half += 2 * (uint64_t)count;  // crt_encrypt_with_r: two half_pow (paillier.cpp:339-342)
    else
      x->pow_full += (uint64_t)count;      // encrypt_with_r: r^n mod n^2 (paillier.cpp:325)
  }
  return e;
}

// Online encryption with precomputed randomness: c = (1 + m n) rn mod n^2, rn = r^n mod n^2
// (= pcb_encrypt(m = 0, r)); the value equals crt_encrypt_with_r(m, r) / encrypt_with_r(m, r).
pcb_status pcb_encrypt_rn(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const uint32_t* rn, size_t count,
                          uint32_t* c, int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_encrypt_rn");
  if (!x || (count && (!m || !rn || !c))) return PCB_E_SHAPE;
  if (m_limbs == 0 || m_limbs > x->L) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sm, sr, sc, ss;
  uint32_t* b = nullptr;
  pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
  if (!e) e = stage_in(rn, count * wb, st, &sr);
  if (!e) e = stage_out(c, count * wb, st, &sc);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  int32_t* stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * wb, (void**)&b, st);
  if (!e)
    e = launch_onepmn((const uint32_t*)sm.dev, (int)m_limbs, (const uint32_t*)sr.dev, x->d_n, x->d_n2, (int)x->L, b,
                      stv, count, st);
  if (!e && x->random_g) {  // g^m instead of 1 + m n (encrypt_with_factor, paillier.cpp:384-389)
    e = gpow_core(x, (const uint32_t*)sm.dev, m_limbs, count, b, st);
    if (!e) {
      zero_bad_rows_kernel<<<(int)std::min<size_t>((count * 2 * x->L + 255) / 256, 4096), 256, 0, st>>>(
          b, (int)(2 * x->L), stv, count);
      count_launch();
      e = cuda_check(cudaGetLastError());
    }
  }
  std::vector<WStep> p = prog_hom_add();  // (1 + m n) * rn mod n^2; failed rows have b = 0 -> c = 0
  if (!e) e = run_wide(x, p.data(), (int)p.size(), (const uint32_t*)sr.dev, b, nullptr, 1, count, count,
                       (uint32_t*)sc.dev, 1, st);
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  scratch_free(b, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sm.host || sr.host || sc.host || ss.host;
  unstage(&sm, st);
  unstage(&sr, st);
  unstage(&sc, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_decrypt(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* m, int use_crt, int32_t* status,
                       pcb_stream stream) {
  PCB_RANGE("pcb_decrypt");
  if (!x || (count && (!c || !m))) return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const bool c_dev = is_device_ptr(c), m_dev = is_device_ptr(m);
  if (count >= kPipeMin && (!c_dev || !m_dev)) {  // host buffers: chunked, copies beside the compute
    const size_t WI = 2 * x->L, WO = x->L;
    const size_t chunk = ((count + kPipeChunks - 1) / kPipeChunks + 255) / 256 * 256;
    HostPipe hp;
    pcb_status e = hp.init(st);
    uint32_t *dc[2] = {nullptr, nullptr}, *dm[2] = {nullptr, nullptr};
    int32_t* sall = nullptr;
    for (int b = 0; b < 2 && !e; b++) {
      if (!c_dev) e = scratch_alloc(chunk * WI * 4, (void**)&dc[b], st);
      if (!e && !m_dev) e = scratch_alloc(chunk * WO * 4, (void**)&dm[b], st);
    }
    if (!e) e = scratch_alloc(count * 4, (void**)&sall, st);
    if (!e) e = cuda_check(cudaStreamSynchronize(st));  // the scratch exists before the copy streams use it
    for (size_t i = 0, off = 0; off < count && !e; i++, off += chunk) {
      const int b = (int)(i & 1);
      const size_t cnt = std::min(chunk, count - off);
      const uint32_t* src = c + off * WI;
      uint32_t* dst = m + off * WO;
      if (!c_dev) {
        if (i >= 2) e = cuda_check(cudaStreamWaitEvent(hp.cin, hp.comp[b], 0));
        if (!e) e = cuda_check(cudaMemcpyAsync(dc[b], src, cnt * WI * 4, cudaMemcpyHostToDevice, hp.cin));
        if (!e) e = cuda_check(cudaEventRecord(hp.in[b], hp.cin));
        if (!e) e = cuda_check(cudaStreamWaitEvent(st, hp.in[b], 0));
        src = dc[b];
      }
      if (!m_dev) {
        if (i >= 2 && !e) e = cuda_check(cudaStreamWaitEvent(st, hp.out[b], 0));
        dst = dm[b];
      }
      if (!e) e = pcb_decrypt(x, src, cnt, dst, use_crt, sall + off, stream);  // device buffers: asynchronous
      if (!e) e = cuda_check(cudaEventRecord(hp.comp[b], st));
      if (!m_dev && !e) {
        e = cuda_check(cudaStreamWaitEvent(hp.cout, hp.comp[b], 0));
        if (!e) e = cuda_check(cudaMemcpyAsync(m + off * WO, dm[b], cnt * WO * 4, cudaMemcpyDeviceToHost, hp.cout));
        if (!e) e = cuda_check(cudaEventRecord(hp.out[b], hp.cout));
      }
    }
    if (cudaStreamSynchronize(hp.cout) != cudaSuccess && !e) e = PCB_E_CUDA;
    if (!e && status) e = cuda_check(cudaMemcpyAsync(status, sall, count * 4, cudaMemcpyDefault, st));
    if (!e && !status) e = first_failure(sall, count, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
    for (void* p : {(void*)dc[0], (void*)dc[1], (void*)dm[0], (void*)dm[1], (void*)sall}) scratch_free(p, st);
    cudaStreamSynchronize(st);
    return e;
  }
  Staged sc, sm, ss;
  pcb_status e = stage_in(c, count * 2 * x->L * 4, st, &sc);
  if (!e) e = stage_out(m, count * x->L * 4, st, &sm);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  int32_t* stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = dec_core(x, (const uint32_t*)sc.dev, count, (uint32_t*)sm.dev, stv, st);
  if (!e) e = unstage_out(m, &sm, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sc.host || sm.host || ss.host;
  unstage(&sc, st);
  unstage(&sm, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) {
    if (use_crt)
      x->pow_half += 2 * (uint64_t)count;
    else
      x->pow_full += (uint64_t)count;
  }
  return e;
}

// ---- collaborative variant (paper Alg. 3) ---------------------------------------
}  // extern "C"
// the master's own CRT half of decrypt_with_half: yq = (c mod q^2)^(eps mod phi(q^2)) mod q^2
// (paillier.cpp:366); it needs only c, so a caller may run it while the edge computes the p side
static pcb_status dwh_q(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* yq, cudaStream_t st) {
  const int S = x->S;
  const double mm = 2.0 * S * S + S;
  if (x->half_fold)  // c^(q-1) mod q^2; the factor u of the exponent is folded into the finish (build_half)
    return launch_rnsx(x->rx_q, kRxDec, x->d_sched + x->off_dec_q, x->len_dec_q, kTab, c, 2 * (int)x->L, nullptr, 0,
                       count, yq, st, ((double)(x->nbits / 2) + (double)((x->nbits / 2 + 3) / 4)) * mm);
  return launch_rnsx(x->rx_q, kRxDec, x->d_sched + x->off_epsq, x->len_epsq, kTab, c, 2 * (int)x->L, nullptr, 0, count,
                     yq, st, ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm);
}

// device core of decrypt_with_half: c (count x 2L), pw (count x 2L: the p-half, any representative);
// yq_pre (nullable): the q side already computed by dwh_q
static pcb_status dwh_core(pcb_ctx* x, const uint32_t* c, const uint32_t* pw, size_t count, uint32_t* m, int32_t* stv,
                           cudaStream_t st, const uint32_t* yq_pre) {
  const int S = x->S, L2 = 2 * (int)x->L;
  uint32_t *yp = nullptr, *yq = nullptr;
  pcb_status e = scratch_alloc(count * S * 4, (void**)&yp, st);
  if (!e && !yq_pre) e = scratch_alloc(count * S * 4, (void**)&yq, st);
  if (!e) e = launch_dec_prep(c, x->d_n2, (int)x->L, stv, count, st);  // c < n^2 (paillier.cpp:365)
  const double mm = 2.0 * S * S + S;
  // p side: p2_power mod p^2 (reference: mod(p2_power, crt_.p2)); q side: c^(eps mod phi(q^2)) mod q^2
  if (!e) e = launch_rnsx(x->rx_p, kRxDec, x->d_sched + x->off_one, x->len_one, kTab, pw, L2, nullptr, 0, count, yp, st, mm);
  if (!e && !yq_pre) e = dwh_q(x, c, count, yq, st);
  if (yq_pre) yq = const_cast<uint32_t*>(yq_pre);
  if (!e && S == 32)
    e = launch_dec_finish<32>(*reinterpret_cast<const CrtDecConsts<32>*>((x->half_fold ? x->half_blob_u : x->half_blob).data()), yp, yq, stv, m,
                              (int)x->L, count, st);
  if (!e && S == 64)
    e = launch_dec_finish<64>(*reinterpret_cast<const CrtDecConsts<64>*>((x->half_fold ? x->half_blob_u : x->half_blob).data()), yp, yq, stv, m,
                              (int)x->L, count, st);
  if (!e && S == 96)
    e = launch_dec_finish<96>(*reinterpret_cast<const CrtDecConsts<96>*>((x->half_fold ? x->half_blob_u : x->half_blob).data()), yp, yq, stv, m,
                              (int)x->L, count, st);
  if (!e && S == 128)
    e = launch_dec_finish<128>(*reinterpret_cast<const CrtDecConsts<128>*>((x->half_fold ? x->half_blob_u : x->half_blob).data()), yp, yq, stv, m,
                              (int)x->L, count, st);
  scratch_free(yp, st);
  if (!yq_pre) scratch_free(yq, st);
  return e;
}
struct pcb_share {  // an edge's CrtShare (paillier.hpp:64-66): p^2 and phi(p^2) only
  int device = 0;
  HBN p2, phi;
  int S = 0;
  RnsXModulus md;
  uint32_t* d_phi = nullptr;  // phi(p^2) normalised for the device long division (exponent reduction)
  int phi_words = 0, phi_shift = 0;
  uint32_t* d_p2n = nullptr;  // p^2 normalised likewise (the binomial form's final reduction)
  int p2_shift = 0;
  // pcb_delegated_power_fermat: p = p^2 - phi(p^2), the p - 1 exponent schedule and the mod-p
  // constants of the finish (ModCtx<S/2>, p^-1 mod 2^(16 S), p), by kernel width
  uint8_t* d_ops_pm1 = nullptr;
  int len_pm1 = 0;
  std::vector<uint8_t> fermat_blob;
};

template <int S>
struct FermatConsts {
  ModCtx<S / 2> sp;
  uint32_t pinv_lo[S / 2];
  uint32_t p[S / 2];
};

template <int S>
static void build_fermat(pcb_share* sh, const HBN& p) {
  constexpr int H = S / 2;
  FermatConsts<S> k;
  std::memset(&k, 0, sizeof(k));
  fill_mod<H>(k.sp, p);
  HBN t;
  if (!mod_inverse(p, HBN(1) << (32 * H), t)) throw std::invalid_argument("even p");
  t.to_limbs(k.pinv_lo, H);
  p.to_limbs(k.p, H);
  sh->fermat_blob.assign(reinterpret_cast<uint8_t*>(&k), reinterpret_cast<uint8_t*>(&k) + sizeof(k));
}
extern "C" {

pcb_status pcb_share_create(pcb_share** out, int device, const uint32_t* p2, uint32_t p2_limbs, const uint32_t* phi_p2,
                            uint32_t phi_limbs) {
  if (!out || !p2 || !phi_p2 || !p2_limbs || !phi_limbs) return PCB_E_SHAPE;
  *out = nullptr;
  std::unique_ptr<pcb_share> sh(new (std::nothrow) pcb_share);
  if (!sh) return PCB_E_ALLOC;
  try {
    sh->device = device;
    sh->p2 = HBN::from_limbs(p2, p2_limbs);
    sh->phi = HBN::from_limbs(phi_p2, phi_limbs);
    if (!sh->p2.is_odd() || sh->phi.is_zero()) return PCB_E_SHAPE;
    sh->S = (int)((sh->p2.bit_length() + 31) / 32);
    int K = 0;
    if (!rnsx_shape(32 * sh->S, &K) || sh->p2.bit_length() <= 1024) return PCB_E_UNSUPPORTED;  // 2048/3072-bit keys
    if (cudaSetDevice(device) != cudaSuccess) return PCB_E_CUDA;
    if (!rnsx_build(sh->p2, sh->p2, sh->S, K, &sh->md)) return PCB_E_UNSUPPORTED;
    // phi(p^2) shifted so its top word has the top bit set (Knuth D divisor)
    sh->phi_words = (int)((sh->phi.bit_length() + 31) / 32);
    sh->phi_shift = (int)(32 * sh->phi_words - sh->phi.bit_length());
    const std::vector<uint32_t> vn = (sh->phi << (size_t)sh->phi_shift).limbs(sh->phi_words);
    if (cudaMalloc(&sh->d_phi, vn.size() * 4) != cudaSuccess) return PCB_E_ALLOC;
    if (cudaMemcpy(sh->d_phi, vn.data(), vn.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
    sh->p2_shift = (int)(32 * sh->S - sh->p2.bit_length());
    const std::vector<uint32_t> pn = (sh->p2 << (size_t)sh->p2_shift).limbs(sh->S);
    if (cudaMalloc(&sh->d_p2n, pn.size() * 4) != cudaSuccess) return PCB_E_ALLOC;
    if (cudaMemcpy(sh->d_p2n, pn.data(), pn.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
    // the Fermat form (pcb_delegated_power_fermat) when phi = p^2 - p for a p with p^2 = p2
    const HBN p = sh->p2 - sh->phi;
    if (p * p == sh->p2 && (sh->S == 64 || sh->S == 96 || sh->S == 128)) {
      const std::vector<uint8_t> ops = build_ops(p - HBN(1), kWindow);
      if (cudaMalloc(&sh->d_ops_pm1, ops.size()) != cudaSuccess) return PCB_E_ALLOC;
      if (cudaMemcpy(sh->d_ops_pm1, ops.data(), ops.size(), cudaMemcpyHostToDevice) != cudaSuccess) return PCB_E_CUDA;
      sh->len_pm1 = (int)ops.size();
      if (sh->S == 64) build_fermat<64>(sh.get(), p);
      else if (sh->S == 96) build_fermat<96>(sh.get(), p);
      else build_fermat<128>(sh.get(), p);
    }
  } catch (const std::bad_alloc&) {
    return PCB_E_ALLOC;
  } catch (...) {
    return PCB_E_SHAPE;
  }
  *out = sh.release();
  return PCB_OK;
}

void pcb_share_destroy(pcb_share* sh) {
  if (!sh) return;
  cudaSetDevice(sh->device);
  rnsx_free(&sh->md);
  if (sh->d_phi) cudaFree(sh->d_phi);
  if (sh->d_p2n) cudaFree(sh->d_p2n);
  if (sh->d_ops_pm1) cudaFree(sh->d_ops_pm1);
  delete sh;
}

// delegated_power for exponents that are multiples of p - 1 (half_pow with w = 0, paillier.cpp:275-305):
// out_i = (base_i mod p^2)^(u_i (p - 1)) mod p^2 = 1 + p (L_p(s_i) u_i mod p) with s_i = base_i^(p-1)
// mod p^2 (0 when p | base_i) -- one |p|-bit chain instead of a |p^2|-bit one.  u_mont: count x S/2
// words, u_i R mod p (R = 2^(16 S)), u_i != 0.  The collaborative session's obf_dec = eps (1 + mask n)
// is such an exponent (protocol.cpp:11-13, 352-353).
pcb_status pcb_delegated_power_fermat(pcb_share* sh, const uint32_t* base, uint32_t base_limbs, const uint32_t* u_mont,
                                      size_t count, uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_delegated_power_fermat");
  if (!sh || (count && (!base || !u_mont || !out)) || base_limbs == 0 || base_limbs > (uint32_t)(2 * sh->S))
    return PCB_E_SHAPE;
  if (!sh->d_ops_pm1) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (cudaSetDevice(sh->device) != cudaSuccess) return PCB_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = sh->S, W = 2 * S, H = S / 2;
  Staged sb, su, so;
  uint32_t *bw = nullptr, *sv = nullptr;
  pcb_status e = stage_in(base, count * base_limbs * 4, st, &sb);
  if (!e) e = stage_in(u_mont, count * H * 4, st, &su);
  if (!e) e = stage_out(out, count * S * 4, st, &so);
  if (!e) e = scratch_alloc(count * W * 4, (void**)&bw, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&sv, st);
  if (!e) e = cuda_check(cudaMemset2DAsync(bw, W * 4, 0, W * 4, count, st));
  if (!e) e = cuda_check(cudaMemcpy2DAsync(bw, W * 4, sb.dev, base_limbs * 4, base_limbs * 4, count, cudaMemcpyDeviceToDevice, st));
  const double mm = 2.0 * S * S + S;
  const double bits = (double)(sh->p2.bit_length() / 2);
  if (!e) e = launch_rnsx(sh->md, kRxDec, sh->d_ops_pm1, sh->len_pm1, kTab, bw, W, nullptr, 0, count, sv, st,
                          (bits + (bits + 3) / 4) * mm);
  if (!e && S == 64) {
    const auto& k = *reinterpret_cast<const FermatConsts<64>*>(sh->fermat_blob.data());
    e = launch_fermat_finish<64>(k.sp, k.pinv_lo, k.p, sv, (const uint32_t*)su.dev, (uint32_t*)so.dev, count, st);
  }
  if (!e && S == 96) {
    const auto& k = *reinterpret_cast<const FermatConsts<96>*>(sh->fermat_blob.data());
    e = launch_fermat_finish<96>(k.sp, k.pinv_lo, k.p, sv, (const uint32_t*)su.dev, (uint32_t*)so.dev, count, st);
  }
  if (!e && S == 128) {
    const auto& k = *reinterpret_cast<const FermatConsts<128>*>(sh->fermat_blob.data());
    e = launch_fermat_finish<128>(k.sp, k.pinv_lo, k.p, sv, (const uint32_t*)su.dev, (uint32_t*)so.dev, count, st);
  }
  if (!e) e = unstage_out(out, &so, st);
  scratch_free(bw, st);
  scratch_free(sv, st);
  const bool any_host = sb.host || su.host || so.host;
  unstage(&sb, st);
  unstage(&su, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

// delegated_power (protocol.cpp:15-18): out_i = (base_i mod p^2)^(obf_i mod phi(p^2)) mod p^2.
// The exponent reduction runs on the device (mod_words_kernel); the powers run on the RNS
// core with a per-element 4-bit window table.
pcb_status pcb_delegated_power(pcb_share* sh, const uint32_t* base, uint32_t base_limbs, const uint32_t* obf,
                               uint32_t obf_limbs, size_t count, uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_delegated_power");
  if (!sh || (count && (!base || !obf || !out)) || base_limbs == 0 || base_limbs > (uint32_t)(2 * sh->S) || !obf_limbs)
    return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (cudaSetDevice(sh->device) != cudaSuccess) return PCB_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = sh->S, W = 2 * S, PW = sh->phi_words;
  Staged sb, so, sx;
  uint32_t *bw = nullptr, *ed = nullptr, *er = nullptr;
  pcb_status e = stage_in(base, count * base_limbs * 4, st, &sb);
  if (!e) e = stage_in(obf, count * obf_limbs * 4, st, &sx);
  if (!e) e = stage_out(out, count * S * 4, st, &so);
  if (!e) e = scratch_alloc(count * W * 4, (void**)&bw, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&ed, st);
  if (!e) e = scratch_alloc(count * PW * 4, (void**)&er, st);
  if (!e) e = cuda_check(cudaMemset2DAsync(bw, W * 4, 0, W * 4, count, st));
  if (!e) e = cuda_check(cudaMemcpy2DAsync(bw, W * 4, sb.dev, base_limbs * 4, base_limbs * 4, count, cudaMemcpyDeviceToDevice, st));
  // exponents obf mod phi(p^2) on the device (mod(obf, phi_p2), protocol.cpp:17), S words each
  if (!e) e = launch_mod_words((const uint32_t*)sx.dev, (int)obf_limbs, count, sh->d_phi, PW, sh->phi_shift, er, st);
  if (!e) e = cuda_check(cudaMemset2DAsync(ed, S * 4, 0, S * 4, count, st));
  if (!e) e = cuda_check(cudaMemcpy2DAsync(ed, S * 4, er, PW * 4, std::min(PW, S) * 4, count, cudaMemcpyDeviceToDevice, st));
  // windows of the reduced exponents: < phi(p^2), so ceil(bits(phi) / 4) 4-bit windows
  const int nwin = (int)((sh->phi.bit_length() + 3) / 4);
  const double mm = 2.0 * S * S + S;
  if (!e) e = launch_rnsx(sh->md, kRxPowVar, nullptr, nwin, 16, bw, W, ed, S, count, (uint32_t*)so.dev, st,
                          (4.0 * nwin + nwin + 14.0) * mm);
  if (!e) e = unstage_out(out, &so, st);
  scratch_free(bw, st);
  scratch_free(ed, st);
  scratch_free(er, st);
  const bool any_host = sb.host || so.host || sx.host;
  unstage(&sb, st);
  unstage(&sx, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

// delegated_power (protocol.cpp:15-18) of the binomial generator g = n + 1 for every element:
// g^(obf mod phi(p^2)) mod p^2 = 1 + (obf mod phi(p^2)) n mod p^2, because n^2 = 0 mod p^2 -- the same
// collapse the reference uses for g_power_half (paillier.cpp:259-263).  Exponent reduction, one
// (PW x L)-word product and one reduction mod p^2 instead of a 2048-bit exponentiation; the result
// is bit-identical to pcb_delegated_power(base = n + 1, obf).
pcb_status pcb_delegated_power_binomial(pcb_share* sh, const uint32_t* n, uint32_t n_limbs, const uint32_t* obf,
                                        uint32_t obf_limbs, size_t count, uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_delegated_power_binomial");
  if (!sh || !n || !n_limbs || (count && (!obf || !out)) || !obf_limbs) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (cudaSetDevice(sh->device) != cudaSuccess) return PCB_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = sh->S, PW = sh->phi_words, NL = (int)n_limbs;
  Staged sn, so, sx;
  uint32_t *er = nullptr, *pr = nullptr;
  pcb_status e = stage_in(n, (size_t)NL * 4, st, &sn);
  if (!e) e = stage_in(obf, count * obf_limbs * 4, st, &sx);
  if (!e) e = stage_out(out, count * S * 4, st, &so);
  if (!e) e = scratch_alloc(count * PW * 4, (void**)&er, st);
  if (!e) e = scratch_alloc(count * (size_t)(PW + NL) * 4, (void**)&pr, st);
  if (!e) e = launch_mod_words((const uint32_t*)sx.dev, (int)obf_limbs, count, sh->d_phi, PW, sh->phi_shift, er, st);
  if (!e) e = launch_mul_add1(er, PW, (const uint32_t*)sn.dev, NL, count, pr, st);
  if (!e) e = launch_mod_words(pr, PW + NL, count, sh->d_p2n, S, sh->p2_shift, (uint32_t*)so.dev, st);
  if (!e) e = unstage_out(out, &so, st);
  scratch_free(er, st);
  scratch_free(pr, st);
  const bool any_host = sn.host || so.host || sx.host;
  unstage(&sn, st);
  unstage(&sx, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_decrypt_with_half(pcb_ctx* x, const uint32_t* c, const uint32_t* p2_power, uint32_t pw_limbs,
                                 size_t count, uint32_t* m, int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_with_half");
  if (!x || (count && (!c || !p2_power || !m)) || pw_limbs == 0 || pw_limbs > 2 * x->L) return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (!x->has_rx) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = x->S, L2 = 2 * (int)x->L;
  Staged sc, sp, sm, ss;
  uint32_t* pw = nullptr;
  int32_t* stv = nullptr;
  pcb_status e = stage_in(c, count * L2 * 4, st, &sc);
  if (!e) e = stage_in(p2_power, count * pw_limbs * 4, st, &sp);
  if (!e) e = stage_out(m, count * x->L * 4, st, &sm);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * L2 * 4, (void**)&pw, st);
  if (!e) e = cuda_check(cudaMemset2DAsync(pw, L2 * 4, 0, L2 * 4, count, st));
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync(pw, L2 * 4, sp.dev, pw_limbs * 4, pw_limbs * 4, count, cudaMemcpyDeviceToDevice, st));
  (void)S;
  if (!e) e = dwh_core(x, (const uint32_t*)sc.dev, pw, count, (uint32_t*)sm.dev, stv, st, nullptr);
  if (!e) e = unstage_out(m, &sm, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  scratch_free(pw, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sc.host || sp.host || sm.host || ss.host;
  unstage(&sc, st);
  unstage(&sp, st);
  unstage(&sm, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) x->pow_half += (uint64_t)count;  // one half_pow per element (paillier.cpp:366)
  return e;
}

pcb_status pcb_finish_split_encrypt(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const uint32_t* p2_g_power,
                                    uint32_t pg_limbs, const uint32_t* r, size_t count, uint32_t* c, int32_t* status,
                                    pcb_stream stream) {
  PCB_RANGE("pcb_finish_split_encrypt");
  if (!x || (count && (!m || !p2_g_power || !r || !c)) || pg_limbs == 0 || pg_limbs > 2 * x->L) return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (!x->has_rx) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = x->S, L2 = 2 * (int)x->L;
  Staged sm, sg, sr, sc, ss;
  uint32_t *gw = nullptr, *gp = nullptr, *yp = nullptr, *yq = nullptr;
  int32_t* stv = nullptr;
  pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
  if (!e) e = stage_in(p2_g_power, count * pg_limbs * 4, st, &sg);
  if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
  if (!e) e = stage_out(c, count * L2 * 4, st, &sc);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * L2 * 4, (void**)&gw, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&gp, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yp, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yq, st);
  // argument checks m < n, r in [1, n) (paillier.cpp:409-412)
  if (!e)
    e = launch_enc_prep((const uint32_t*)sm.dev, (int)m_limbs, nullptr, 0, 0, 0, 0, nullptr, 0, nullptr, nullptr,
                        (const uint32_t*)sr.dev, x->d_n, (int)x->L, stv, count, st);
  if (!e) e = cuda_check(cudaMemset2DAsync(gw, L2 * 4, 0, L2 * 4, count, st));
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync(gw, L2 * 4, sg.dev, pg_limbs * 4, pg_limbs * 4, count, cudaMemcpyDeviceToDevice, st));
  const double mm = 2.0 * S * S + S, alg = ((double)x->nbits + (double)((x->nbits + 3) / 4)) * mm;
  // cp = (p2_g_power mod p^2) r^(n mod phi(p^2)) mod p^2;  cq = (1 + m n) r^(n mod phi(q^2)) mod q^2
  if (!e) e = launch_rnsx(x->rx_p, kRxDec, x->d_sched + x->off_one, x->len_one, kTab, gw, L2, nullptr, 0, count, gp, st, mm);
  // random generator: the q side's g power is g^m mod q^2 (g_power_half, paillier.cpp:264-271),
  // from g^m mod n^2 (gpow_core) reduced mod q^2
  uint32_t *gfull = nullptr, *gq = nullptr;
  if (!e && x->random_g) {
    e = scratch_alloc(count * L2 * 4, (void**)&gfull, st);
    if (!e) e = scratch_alloc(count * S * 4, (void**)&gq, st);
    if (!e) e = gpow_core(x, (const uint32_t*)sm.dev, m_limbs, count, gfull, st);
    if (!e)
      e = launch_rnsx(x->rx_q, kRxDec, x->d_sched + x->off_one, x->len_one, kTab, gfull, L2, nullptr, 0, count, gq, st,
                      mm);
  }
  if (x->enc_split) {  // r^n mod p^2 = (r^q mod p)^p mod p^2, same for q
    uint32_t* u = nullptr;
    if (!e) e = scratch_alloc(count * x->w1 * 4, (void**)&u, st);
    if (!e) e = split_stage1(x, 0, (const uint32_t*)sr.dev, stv, count, u, st);
    if (!e)
      e = launch_rnsx(x->rx_p, kRxEncG, x->d_sched + x->off_ep, x->len_ep, kTab, u, x->w1, gp, S, count, yp, st, alg);
    if (!e) e = split_stage1(x, 1, (const uint32_t*)sr.dev, stv, count, u, st);
    if (!e && gq)
      e = launch_rnsx(x->rx_q, kRxEncG, x->d_sched + x->off_eq, x->len_eq, kTab, u, x->w1, gq, S, count, yq, st, alg);
    else if (!e)
      e = launch_rnsx(x->rx_q, kRxEnc, x->d_sched + x->off_eq, x->len_eq, kTab, u, x->w1, (const uint32_t*)sm.dev,
                      (int)m_limbs, count, yq, st, alg);
    scratch_free(u, st);
  } else {
    if (!e)
      e = launch_rnsx(x->rx_p, kRxEncG, x->d_sched + x->off_enc_p, x->len_enc_p, kTab, (const uint32_t*)sr.dev,
                      (int)x->L, gp, S, count, yp, st, alg);
    if (!e && gq)
      e = launch_rnsx(x->rx_q, kRxEncG, x->d_sched + x->off_enc_q, x->len_enc_q, kTab, (const uint32_t*)sr.dev,
                      (int)x->L, gq, S, count, yq, st, alg);
    else if (!e)
      e = launch_rnsx(x->rx_q, kRxEnc, x->d_sched + x->off_enc_q, x->len_enc_q, kTab, (const uint32_t*)sr.dev,
                      (int)x->L, (const uint32_t*)sm.dev, (int)m_limbs, count, yq, st, alg);
  }
  if (!e && S == 32)
    e = launch_garner<32>(*reinterpret_cast<const CrtEncConsts<32>*>(x->enc_blob.data()), yp, yq, stv,
                          (uint32_t*)sc.dev, (int)x->L, count, st);
  if (!e && S == 64)
    e = launch_garner<64>(*reinterpret_cast<const CrtEncConsts<64>*>(x->enc_blob.data()), yp, yq, stv,
                          (uint32_t*)sc.dev, (int)x->L, count, st);
  if (!e && S == 96)
    e = launch_garner<96>(*reinterpret_cast<const CrtEncConsts<96>*>(x->enc_blob.data()), yp, yq, stv,
                          (uint32_t*)sc.dev, (int)x->L, count, st);
  if (!e && S == 128)
    e = launch_garner<128>(*reinterpret_cast<const CrtEncConsts<128>*>(x->enc_blob.data()), yp, yq, stv,
                          (uint32_t*)sc.dev, (int)x->L, count, st);
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  scratch_free(gw, st);
  scratch_free(gp, st);
  scratch_free(yp, st);
  scratch_free(yq, st);
  scratch_free(gfull, st);
  scratch_free(gq, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sm.host || sg.host || sr.host || sc.host || ss.host;
  unstage(&sm, st);
  unstage(&sg, st);
  unstage(&sr, st);
  unstage(&sc, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) x->pow_half += 2 * (uint64_t)count;  // two half_pows (paillier.cpp:412-413)
  return e;
}

// finish_split_encrypt_with_factor (paillier.cpp:416-426) with the pooled factor's rn = r^n mod n^2
// (RnFactor.full; its residues mod p^2 / q^2 are the factor's half_p2 / half_q2):
//   c = CRT(p2_g_power mod p^2, g_q(m) mod q^2) * rn mod n^2,  g_q(m) = 1 + m n (g^m for random g)
// -- two plain reductions, one Garner recombination and one multiply mod n^2; no exponentiation
// with r (that is what the pool buys).
pcb_status pcb_finish_split_encrypt_rn(pcb_ctx* x, const uint32_t* m, uint32_t m_limbs, const uint32_t* p2_g_power,
                                       uint32_t pg_limbs, const uint32_t* rn, size_t count, uint32_t* c,
                                       int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_finish_split_encrypt_rn");
  if (!x || (count && (!m || !p2_g_power || !rn || !c)) || pg_limbs == 0 || pg_limbs > 2 * x->L) return PCB_E_SHAPE;
  if (m_limbs == 0 || m_limbs > x->L) return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (!x->has_rx) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const int S = x->S, L2 = 2 * (int)x->L;
  Staged sm, sg, sr, sc, ss;
  uint32_t *gw = nullptr, *u = nullptr, *yp = nullptr, *yq = nullptr, *c1 = nullptr;
  int32_t* stv = nullptr;
  pcb_status e = stage_in(m, count * m_limbs * 4, st, &sm);
  if (!e) e = stage_in(p2_g_power, count * pg_limbs * 4, st, &sg);
  if (!e) e = stage_in(rn, count * L2 * 4, st, &sr);
  if (!e) e = stage_out(c, count * L2 * 4, st, &sc);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * L2 * 4, (void**)&gw, st);
  if (!e) e = scratch_alloc(count * L2 * 4, (void**)&u, st);
  if (!e) e = scratch_alloc(count * L2 * 4, (void**)&c1, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yp, st);
  if (!e) e = scratch_alloc(count * S * 4, (void**)&yq, st);
  // m < n, rn in [1, n^2) ("factor missing split residues" for rn = 0); u = 1 + m n
  if (!e)
    e = launch_onepmn((const uint32_t*)sm.dev, (int)m_limbs, (const uint32_t*)sr.dev, x->d_n, x->d_n2, (int)x->L, u,
                      stv, count, st);
  if (!e && x->random_g) {  // g_power_half(m, false) of a random generator (paillier.cpp:259-267)
    e = gpow_core(x, (const uint32_t*)sm.dev, m_limbs, count, u, st);
    if (!e) {
      zero_bad_rows_kernel<<<(int)std::min<size_t>((count * L2 + 255) / 256, 4096), 256, 0, st>>>(u, L2, stv, count);
      count_launch();
      e = cuda_check(cudaGetLastError());
    }
  }
  if (!e) e = cuda_check(cudaMemset2DAsync(gw, L2 * 4, 0, L2 * 4, count, st));
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync(gw, L2 * 4, sg.dev, pg_limbs * 4, pg_limbs * 4, count, cudaMemcpyDeviceToDevice, st));
  const double mm = 2.0 * S * S + S;
  if (!e) e = launch_rnsx(x->rx_p, kRxDec, x->d_sched + x->off_one, x->len_one, kTab, gw, L2, nullptr, 0, count, yp, st, mm);
  if (!e) e = launch_rnsx(x->rx_q, kRxDec, x->d_sched + x->off_one, x->len_one, kTab, u, L2, nullptr, 0, count, yq, st, mm);
  if (!e && S == 32)
    e = launch_garner<32>(*reinterpret_cast<const CrtEncConsts<32>*>(x->enc_blob.data()), yp, yq, stv, c1, (int)x->L,
                          count, st);
  if (!e && S == 64)
    e = launch_garner<64>(*reinterpret_cast<const CrtEncConsts<64>*>(x->enc_blob.data()), yp, yq, stv, c1, (int)x->L,
                          count, st);
  if (!e && S == 96)
    e = launch_garner<96>(*reinterpret_cast<const CrtEncConsts<96>*>(x->enc_blob.data()), yp, yq, stv, c1, (int)x->L,
                          count, st);
  if (!e && S == 128)
    e = launch_garner<128>(*reinterpret_cast<const CrtEncConsts<128>*>(x->enc_blob.data()), yp, yq, stv, c1, (int)x->L,
                          count, st);
  std::vector<WStep> p = prog_hom_add();  // CRT(...) * rn mod n^2; failed rows have c1 = 0 -> c = 0
  if (!e) e = run_wide(x, p.data(), (int)p.size(), (const uint32_t*)sr.dev, c1, nullptr, 1, count, count,
                       (uint32_t*)sc.dev, 1, st);
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(status, &ss, st);
  if (!e && !status) e = first_failure(stv, count, st);
  scratch_free(gw, st);
  scratch_free(u, st);
  scratch_free(c1, st);
  scratch_free(yp, st);
  scratch_free(yq, st);
  if (!ss.dev) scratch_free(stv, st);
  const bool any_host = sm.host || sg.host || sr.host || sc.host || ss.host;
  unstage(&sm, st);
  unstage(&sg, st);
  unstage(&sr, st);
  unstage(&sc, st);
  unstage(&ss, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e && x->random_g) x->pow_half += (uint64_t)count;  // g_power_half on the q side (paillier.cpp:424)
  return e;
}

pcb_status pcb_hom_add(pcb_ctx* x, const uint32_t* a, const uint32_t* b, size_t count, uint32_t* out,
                       pcb_stream stream) {
  PCB_RANGE("pcb_hom_add");
  if (!x || (count && (!a || !b || !out))) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sa, sb, so;
  pcb_status e = stage_in(a, count * wb, st, &sa);
  if (!e) e = stage_in(b, count * wb, st, &sb);
  if (!e) e = stage_out(out, count * wb, st, &so);
  std::vector<WStep> p = prog_hom_add();
  if (!e)
    e = run_wide(x, p.data(), (int)p.size(), (const uint32_t*)sa.dev, (const uint32_t*)sb.dev, nullptr, 1, count,
                 count, (uint32_t*)so.dev, 1, st);
  if (!e) e = unstage_out(out, &so, st);
  const bool any_host = sa.host || sb.host || so.host;
  unstage(&sa, st);
  unstage(&sb, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_hom_scalar_mul(pcb_ctx* x, const uint64_t* k, const uint32_t* c, size_t count, uint32_t* out,
                              pcb_stream stream) {
  PCB_RANGE("pcb_hom_scalar_mul");
  if (!x || (count && (!k || !c || !out))) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sk, sc, so;
  pcb_status e = stage_in(k, count * 8, st, &sk);
  if (!e) e = stage_in(c, count * wb, st, &sc);
  if (!e) e = stage_out(out, count * wb, st, &so);
  std::vector<WStep> p = prog_scalar_pow();
  if (!e)
    e = run_wide(x, p.data(), (int)p.size(), (const uint32_t*)sc.dev, nullptr, (const uint64_t*)sk.dev, 1, count,
                 count, (uint32_t*)so.dev, 16, st);
  if (!e) e = unstage_out(out, &so, st);
  const bool any_host = sk.host || sc.host || so.host;
  unstage(&sk, st);
  unstage(&sc, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) x->pow_full += (uint64_t)count;  // hom_scalar_mul bumps pow_full (paillier.cpp:437)
  return e;
}

pcb_status pcb_aggregate(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_aggregate");
  if (!x || !c || !out || count == 0) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sc, so;
  pcb_status e = stage_in(c, count * wb, st, &sc);
  if (!e) e = stage_out(out, wb, st, &so);
  const int C = x->agg_chunk;
  std::vector<WStep> p = prog_aggregate(C);
  const uint32_t* cur = (const uint32_t*)sc.dev;
  size_t n = count;
  uint32_t* bufs[2] = {nullptr, nullptr};
  int which = 0;
  while (!e && n > 1) {
    const size_t nout = (n + C - 1) / C;
    uint32_t* dst = nullptr;
    if (nout == 1) {
      dst = (uint32_t*)so.dev;
    } else {
      if (!bufs[which]) e = scratch_alloc(((count + C - 1) / C) * wb, (void**)&bufs[which], st);
      dst = bufs[which];
    }
    if (!e) e = run_wide(x, p.data(), (int)p.size(), cur, nullptr, nullptr, C, n, nout, dst, 1, st);
    cur = dst;
    which ^= 1;
    n = nout;
  }
  if (!e && count == 1) e = cuda_check(cudaMemcpyAsync(so.dev, sc.dev, wb, cudaMemcpyDeviceToDevice, st));
  if (!e) e = unstage_out(out, &so, st);
  scratch_free(bufs[0], st);
  scratch_free(bufs[1], st);
  const bool any_host = sc.host || so.host;
  unstage(&sc, st);
  unstage(&so, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

// bit length of the largest exponent (OR-reduction on the device; sets the window count)
__global__ void expo_or_kernel(const uint64_t* e, size_t n, unsigned long long* out) {
  uint64_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc |= e[i];
  for (int o = 16; o > 0; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicOr(out, (unsigned long long)acc);
}

static pcb_status expo_max_bits(const uint64_t* expo_dev, size_t n, cudaStream_t st, int* bits) {
  *bits = 0;
  if (n == 0) return PCB_OK;
  unsigned long long* d = nullptr;
  pcb_status e = scratch_alloc(8, (void**)&d, st);
  if (!e) e = cuda_check(cudaMemsetAsync(d, 0, 8, st));
  if (!e) {
    const int grid = (int)std::min<size_t>((n + 255) / 256, 1184);
    expo_or_kernel<<<grid, 256, 0, st>>>(expo_dev, n, d);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  unsigned long long h = 0;
  if (!e) e = cuda_check(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
  if (!e) e = cuda_check(cudaStreamSynchronize(st));
  scratch_free(d, st);
  *bits = h ? 64 - __builtin_clzll(h) : 0;
  return e;
}

// hom_matvec over nblk diagonal blocks of rows_b x cols_b (device pointers, block-major):
//   out[b][i] = alpha[b][i] * prod_j zv[b][j]^expo[b][i][j] mod n^2.
// A1: window bases per column (squaring chains), A2: the 63-entry tables per (column, window),
// B: table products per (row, chunk of cc columns), C: alpha_i times the chunk partials.
// hom_matvec on the streaming RNS core: the same table method (paillier.cpp:441-493) with every
// table entry and partial product kept as an RNS record (2K residues) in HBM.
//   A1 (one element per column):  window bases zv^(64^w), 6 squarings per window
//   A2 (one per (column, window)): entries 0..63 (entry 0 = the Montgomery one)
//   B  (one per (row, chunk of cc columns)): product of the cc x nwin selected entries
//   C  (one per row): alpha_i x the chunk partials, converted back to binary mod n^2
static pcb_status matvec_rnsx(pcb_ctx* x, const uint32_t* alpha, const uint64_t* expo_dev, const uint32_t* zv,
                              size_t nblk, size_t rows_b, size_t cols_b, int nwin, uint32_t* out, cudaStream_t st) {
  const RnsXModulus& md = x->rx_n2;
  const size_t rows = nblk * rows_b, cols = nblk * cols_b;
  const int cc = std::max(1, std::min(16, (kRxMaxSteps - 1) / nwin));
  const int nch = (int)((cols_b + cc - 1) / cc);
  const size_t REC = (size_t)rnsx_rec_words(md);
  const double mm = 2.0 * (2 * x->L) * (2 * x->L) + 2 * x->L;  // canonical MM(2|n|) MAC32
  RxProg g;
  g.expo = expo_dev;
  g.cols = (int)cols_b;
  g.nwin = nwin;
  g.cc = cc;
  g.nch = nch;
  g.brows = (int)rows_b;
  g.nparts = nch;
  pcb_status e = scratch_alloc(cols * (size_t)nwin * 64 * REC * 4, (void**)&g.mtab, st);
  if (!e) e = scratch_alloc(rows * (size_t)nch * REC * 4, (void**)&g.part, st);
  auto S = [](uint8_t xs, uint8_t xa, uint8_t ys, uint8_t ya, uint8_t post, uint8_t pa, uint8_t flags = 0) {
    return XStep{xs, xa, ys, ya, post, pa, flags, 0};
  };
  if (!e && getenv("PCB_RNSX_MVDBG") && atoi(getenv("PCB_RNSX_MVDBG")) >= 2) {  // debug: A1 (+A2) then out
    const int dbg = atoi(getenv("PCB_RNSX_MVDBG"));
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsConv, 0, kRsCvec, kRxR2N, kRpChain, 0);
    e = launch_rnsx_prog(md, g, zv, 2 * (int)x->L, cols, nullptr, st, 0);
    if (dbg == 3) {  // A2 (entries 2.. of every (column, window)); out = entry 2 of element el = zv^2 for el < cols
      g.nwin = 1;
      g.nsteps = 0;
      g.st[g.nsteps++] = S(kRsSelf, 1, kRsSelf, 1, kRpSelf, 2, 1);
      for (int d = 3; d < 64; d++) g.st[g.nsteps++] = S(kRsKeep, 0, kRsSelf, 1, kRpSelf, (uint8_t)d);
      if (!e) e = launch_rnsx_prog(md, g, nullptr, 0, cols, nullptr, st, 0);
    }
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsSelf, dbg == 3 ? 2 : 1, kRsCvec, kRxOne, kRpOut, 0);
    if (!e) e = launch_rnsx_prog(md, g, nullptr, 0, rows, out, st, 0);
    scratch_free(g.mtab, st);
    scratch_free(g.part, st);
    return e;
  }
  if (!e && getenv("PCB_RNSX_MVDBG")) {  // debug: out = alpha through conv -> x R2N -> x 1 -> out
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsConv, 0, kRsCvec, kRxR2N, kRpNone, 0);
    g.st[g.nsteps++] = S(kRsKeep, 0, kRsCvec, kRxOne, kRpOut, 0);
    e = launch_rnsx_prog(md, g, alpha, 2 * (int)x->L, rows, out, st, 0);
    scratch_free(g.mtab, st);
    scratch_free(g.part, st);
    return e;
  }
  if (!e) {  // A1
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsConv, 0, kRsCvec, kRxR2N, kRpChain, 0);
    for (int w = 1; w < nwin; w++)
      for (int q = 1; q <= kMatWin; q++) g.st[g.nsteps++] = S(kRsKeep, 0, kRsSq, 0, q == kMatWin ? kRpChain : kRpNone, (uint8_t)w);
    e = launch_rnsx_prog(md, g, zv, 2 * (int)x->L, cols, nullptr, st, mm * g.nsteps);
  }
  if (!e) {  // A2
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsSelf, 1, kRsSelf, 1, kRpSelf, 2, 1);
    for (int d = 3; d < 64; d++) g.st[g.nsteps++] = S(kRsKeep, 0, kRsSelf, 1, kRpSelf, (uint8_t)d);
    e = launch_rnsx_prog(md, g, nullptr, 0, cols * nwin, nullptr, st, mm * g.nsteps);
  }
  if (!e) {  // B
    std::vector<uint8_t> ids;
    for (int j = 0; j < cc; j++)
      for (int w = 0; w < nwin; w++) ids.push_back((uint8_t)(j * 16 + w));
    g.nsteps = 0;
    if (ids.size() == 1) {
      g.st[g.nsteps++] = S(kRsMat, ids[0], kRsCvec, kRxOneM, kRpRec, 0);
    } else {
      g.st[g.nsteps++] = S(kRsMat, ids[0], kRsMat, ids[1], kRpNone, 0);
      for (size_t q = 2; q < ids.size(); q++) g.st[g.nsteps++] = S(kRsKeep, 0, kRsMat, ids[q], kRpNone, 0);
      g.st[g.nsteps - 1].post = kRpRec;
    }
    e = launch_rnsx_prog(md, g, nullptr, 0, rows * nch, nullptr, st, mm * g.nsteps);
  }
  // C: the nch chunk partials of every row are first multiplied pairwise in a tree (one product per
  // level, rows x cur/2 elements on all SMs) while their count is even, then alpha_i times the
  // remaining ones -- instead of a chain of nch products on ceil(rows / 128) CTAs.  The product mod
  // n^2 does not depend on the order, and the output conversion is canonical.
  uint32_t* tbuf = nullptr;
  int cur = nch;
  if (!e && cur % 2 == 0 && cur > 1 && !getenv("PCB_MATVEC_CHAIN"))
    e = scratch_alloc(rows * (size_t)(cur / 2) * REC * 4, (void**)&tbuf, st);
  uint32_t *pin = g.part, *pnext = tbuf;
  while (!e && tbuf && cur % 2 == 0 && cur > 1) {
    const int nxt = cur / 2;
    g.part = pin;
    g.pout = pnext;
    g.nparts = 2;  // element (row, j) of rows x nxt reads partials (row, 2j) and (row, 2j + 1)
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsPart, 0, kRsPart, 1, kRpRec, 0);
    e = launch_rnsx_prog(md, g, nullptr, 0, rows * (size_t)nxt, nullptr, st, mm);
    std::swap(pin, pnext);
    cur = nxt;
  }
  g.part = pin;
  g.pout = nullptr;
  g.nparts = cur;
  if (!e) {  // alpha_i times the cur remaining partials of row i, out of Montgomery form
    g.nsteps = 0;
    g.st[g.nsteps++] = S(kRsConv, 0, kRsCvec, kRxR2N, kRpNone, 0);
    for (int c = 0; c < cur; c++) g.st[g.nsteps++] = S(kRsKeep, 0, kRsPart, (uint8_t)c, kRpNone, 0);
    g.st[g.nsteps++] = S(kRsKeep, 0, kRsCvec, kRxOne, kRpOut, 0);
    e = launch_rnsx_prog(md, g, alpha, 2 * (int)x->L, rows, out, st, mm * g.nsteps);
  }
  scratch_free(g.mtab, st);
  scratch_free(pin, st);  // {pin, pnext} = the partials buffer and the tree buffer
  scratch_free(pnext, st);
  return e;
}

// bits_hint > 0: an upper bound of every exponent's bit length supplied by the caller (the
// asynchronous edge step), so the OR-reduction and its host read-back are skipped
static pcb_status matvec_core(pcb_ctx* x, const uint32_t* alpha, const uint64_t* expo_dev, const uint32_t* zv,
                              size_t nblk, size_t rows_b, size_t cols_b, uint32_t* out, cudaStream_t st,
                              int bits_hint = 0) {
  const size_t wb = 2 * x->L * 4;
  const size_t rows = nblk * rows_b, cols = nblk * cols_b;
  if (rows == 0) return PCB_OK;
  if (cols_b == 0) return cuda_check(cudaMemcpyAsync(out, alpha, rows * wb, cudaMemcpyDeviceToDevice, st));
  int maxbits = bits_hint > 64 ? 64 : bits_hint;
  if (maxbits <= 0)
    if (auto e = expo_max_bits(expo_dev, rows * cols_b, st, &maxbits)) return e;
  const int nwin = maxbits ? (maxbits + kMatWin - 1) / kMatWin : 1;
  if (x->use_rx_n2 && nwin <= 15 && nblk * cols_b <= (1u << 20))
    return matvec_rnsx(x, alpha, expo_dev, zv, nblk, rows_b, cols_b, nwin, out, st);
  const int cc = std::max(1, std::min(16, (kWideMaxSteps - 1) / nwin));
  const int nch = (int)((cols_b + cc - 1) / cc);
  const int N = x->wide.n;
  MatvecGeom g;
  g.expo = expo_dev;
  g.cols = (int)cols_b;
  g.nwin = nwin;
  g.cc = cc;
  g.nch = nch;
  g.brows = (int)rows_b;
  uint32_t *part = nullptr, *combo = nullptr;
  pcb_status e = scratch_alloc(cols * (size_t)nwin * 64 * N * 4, (void**)&g.mtab, st);
  if (!e) {  // A1
    std::vector<WStep> p = prog_mat_chain(nwin);
    g.wcur = 0;
    e = run_wide(x, p.data(), (int)p.size(), zv, nullptr, nullptr, 1, cols, cols, nullptr, 1, st, &g);
  }
  if (!e) {  // A2
    std::vector<WStep> p = prog_mat_fill();
    g.wcur = -1;
    e = run_wide(x, p.data(), (int)p.size(), nullptr, nullptr, nullptr, 1, cols * nwin, cols * nwin, nullptr, 1, st, &g);
  }
  g.wcur = 0;
  if (!e) e = scratch_alloc(rows * (size_t)nch * wb, (void**)&part, st);
  if (!e) {  // B
    std::vector<WStep> p = prog_mat_prod(cc, nwin);
    e = run_wide(x, p.data(), (int)p.size(), nullptr, nullptr, nullptr, 1, rows * nch, rows * nch, part, 1, st, &g);
  }
  if (!e) e = scratch_alloc(rows * (size_t)(nch + 1) * wb, (void**)&combo, st);
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync(combo, (nch + 1) * wb, part, nch * wb, nch * wb, rows, cudaMemcpyDeviceToDevice, st));
  if (!e)
    e = cuda_check(cudaMemcpy2DAsync((uint8_t*)combo + nch * wb, (nch + 1) * wb, alpha, wb, wb, rows,
                                     cudaMemcpyDeviceToDevice, st));
  if (!e) {  // C
    std::vector<WStep> p = prog_mat_combine(nch);
    e = run_wide(x, p.data(), (int)p.size(), combo, nullptr, nullptr, nch + 1, rows * (nch + 1), rows, out, 1, st);
  }
  scratch_free(g.mtab, st);
  scratch_free(part, st);
  scratch_free(combo, st);
  return e;
}

pcb_status pcb_hom_matvec(pcb_ctx* x, const uint32_t* alpha, const uint64_t* expo, const uint32_t* zv, size_t rows,
                          size_t cols, uint32_t window, uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_hom_matvec");
  if (!x || (rows && (!alpha || !out)) || (rows && cols && (!expo || !zv))) return PCB_E_SHAPE;
  if (window < 1 || window > 8) return PCB_E_SHAPE;  // paillier.cpp:449
  if (rows == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sa, se, sz, so;
  pcb_status e = stage_in(alpha, rows * wb, st, &sa);
  if (!e) e = stage_in(expo, rows * cols * 8, st, &se);
  if (!e) e = stage_in(zv, cols * wb, st, &sz);
  if (!e) e = stage_out(out, rows * wb, st, &so);
  if (!e)
    e = matvec_core(x, (const uint32_t*)sa.dev, (const uint64_t*)se.dev, (const uint32_t*)sz.dev, 1, rows, cols,
                    (uint32_t*)so.dev, st);
  if (!e) e = unstage_out(out, &so, st);
  unstage(&sa, st);
  unstage(&se, st);
  unstage(&sz, st);
  unstage(&so, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) x->pow_full += rows;  // hom_matvec counts one full exponentiation per row (paillier.cpp:476)
  return e;
}

// Edge step over nblk square blocks (dense, block-major: alpha/zc/vc/out hold sum(sizes) ciphertexts,
// expo the row-major size_k x size_k matrices back to back).  Unequal sizes are padded to the
// largest block (zero exponents select the Montgomery one, padded rows are dropped).
static pcb_status edge_core(pcb_ctx* x, size_t nblk, const uint32_t* sizes, const uint32_t* alpha,
                            const uint64_t* expo, const uint32_t* zc, const uint32_t* vc, uint32_t* out,
                            cudaStream_t st, int bits_hint = 0, int32_t* err_dev = nullptr) {
  const size_t wb = 2 * x->L * 4;
  size_t total = 0, cmax = 0, etotal = 0;
  for (size_t k = 0; k < nblk; k++) {
    total += sizes[k];
    etotal += (size_t)sizes[k] * sizes[k];
    cmax = std::max<size_t>(cmax, sizes[k]);
  }
  if (total == 0) return PCB_OK;
  int32_t* stv = nullptr;
  uint32_t* zvd = nullptr;
  // protocol.cpp:264-266: every z_j, v_j must be < n^2 ("ciphertext outside the group")
  pcb_status e = scratch_alloc(2 * total * 4, (void**)&stv, st);
  if (!e) e = launch_dec_prep(zc, x->d_n2, (int)x->L, stv, total, st);
  if (!e) e = launch_dec_prep(vc, x->d_n2, (int)x->L, stv + total, total, st);
  if (err_dev) {  // asynchronous form: the caller reads the flag once per iteration
    if (!e) e = launch_status_flag(stv, 2 * total, err_dev, st);
  } else {
    std::vector<int32_t> hst(2 * total);
    if (!e) e = cuda_check(cudaMemcpyAsync(hst.data(), stv, 2 * total * 4, cudaMemcpyDeviceToHost, st));
    if (!e) e = cuda_check(cudaStreamSynchronize(st));
    if (!e)
      for (int32_t v : hst)
        if (v != PCB_OK) e = PCB_E_CIPHER_RANGE;
  }
  // zv_j = z_j * v_j mod n^2 (hom_add, protocol.cpp:268-269), then the matvec (270-271)
  if (!e) e = scratch_alloc(total * wb, (void**)&zvd, st);
  std::vector<WStep> pa = prog_hom_add();
  if (!e) e = run_wide(x, pa.data(), (int)pa.size(), zc, vc, nullptr, 1, total, total, zvd, 1, st);
  bool uniform = true;
  for (size_t k = 0; k < nblk; k++) uniform = uniform && sizes[k] == cmax;
  if (!e && uniform) {
    e = matvec_core(x, alpha, expo, zvd, nblk, cmax, cmax, out, st, bits_hint);
  } else if (!e) {
    uint32_t *ap = nullptr, *zp = nullptr, *op = nullptr;
    uint64_t* ep = nullptr;
    const size_t padded = nblk * cmax;
    e = scratch_alloc(padded * wb, (void**)&ap, st);
    if (!e) e = scratch_alloc(padded * wb, (void**)&zp, st);
    if (!e) e = scratch_alloc(padded * wb, (void**)&op, st);
    if (!e) e = scratch_alloc(padded * cmax * 8, (void**)&ep, st);
    if (!e) e = cuda_check(cudaMemsetAsync(ap, 0, padded * wb, st));
    if (!e) e = cuda_check(cudaMemsetAsync(zp, 0, padded * wb, st));
    if (!e) e = cuda_check(cudaMemsetAsync(ep, 0, padded * cmax * 8, st));
    size_t off = 0, eoff = 0;
    for (size_t k = 0; !e && k < nblk; k++) {
      const size_t c = sizes[k];
      if (c) {
        e = cuda_check(cudaMemcpyAsync((uint8_t*)ap + k * cmax * wb, (const uint8_t*)alpha + off * wb, c * wb,
                                       cudaMemcpyDeviceToDevice, st));
        if (!e)
          e = cuda_check(cudaMemcpyAsync((uint8_t*)zp + k * cmax * wb, (const uint8_t*)zvd + off * wb, c * wb,
                                         cudaMemcpyDeviceToDevice, st));
        if (!e)
          e = cuda_check(cudaMemcpy2DAsync(ep + k * cmax * cmax, cmax * 8, expo + eoff, c * 8, c * 8, c,
                                           cudaMemcpyDeviceToDevice, st));
      }
      off += c;
      eoff += c * c;
    }
    if (!e) e = matvec_core(x, ap, ep, zp, nblk, cmax, cmax, op, st, bits_hint);
    off = 0;
    for (size_t k = 0; !e && k < nblk; k++) {
      if (sizes[k])
        e = cuda_check(cudaMemcpyAsync((uint8_t*)out + off * wb, (const uint8_t*)op + k * cmax * wb, sizes[k] * wb,
                                       cudaMemcpyDeviceToDevice, st));
      off += sizes[k];
    }
    scratch_free(ap, st);
    scratch_free(zp, st);
    scratch_free(op, st);
    scratch_free(ep, st);
  }
  scratch_free(stv, st);
  scratch_free(zvd, st);
  if (!e) x->pow_full += total;  // one hom_matvec row = one full exponentiation (paillier.cpp:476)
  (void)etotal;
  return e;
}

static pcb_status edge_entry(pcb_ctx* x, size_t nblk, const uint32_t* sizes, const uint32_t* alpha,
                             const uint64_t* expo, const uint32_t* zc, const uint32_t* vc, uint32_t window,
                             uint32_t* out, pcb_stream stream) {
  if (!x || (nblk && !sizes)) return PCB_E_SHAPE;
  if (window < 1 || window > 8) return PCB_E_SHAPE;
  size_t total = 0, etotal = 0;
  for (size_t k = 0; k < nblk; k++) {
    total += sizes[k];
    etotal += (size_t)sizes[k] * sizes[k];
  }
  if (total == 0) return PCB_OK;
  if (!alpha || !expo || !zc || !vc || !out) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wb = 2 * x->L * 4;
  Staged sa, se, sz, sv, so;
  pcb_status e = stage_in(alpha, total * wb, st, &sa);
  if (!e) e = stage_in(expo, etotal * 8, st, &se);
  if (!e) e = stage_in(zc, total * wb, st, &sz);
  if (!e) e = stage_in(vc, total * wb, st, &sv);
  if (!e) e = stage_out(out, total * wb, st, &so);
  if (!e)
    e = edge_core(x, nblk, sizes, (const uint32_t*)sa.dev, (const uint64_t*)se.dev, (const uint32_t*)sz.dev,
                  (const uint32_t*)sv.dev, (uint32_t*)so.dev, st);
  if (!e) e = unstage_out(out, &so, st);
  unstage(&sa, st);
  unstage(&se, st);
  unstage(&sz, st);
  unstage(&sv, st);
  unstage(&so, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_edge_step(pcb_ctx* x, const uint32_t* alpha, const uint64_t* expo, const uint32_t* zc,
                         const uint32_t* vc, size_t cols, uint32_t window, uint32_t* out, pcb_stream stream) {
  if (cols > 0xffffffffu) return PCB_E_SHAPE;
  const uint32_t c = (uint32_t)cols;
  return edge_entry(x, 1, &c, alpha, expo, zc, vc, window, out, stream);
}

pcb_status pcb_edge_step_blocks(pcb_ctx* x, size_t nblocks, const uint32_t* sizes, const uint32_t* alpha,
                                const uint64_t* expo, const uint32_t* zc, const uint32_t* vc, uint32_t window,
                                uint32_t* out, pcb_stream stream) {
  PCB_RANGE("pcb_edge_step_blocks");
  return edge_entry(x, nblocks, sizes, alpha, expo, zc, vc, window, out, stream);
}

extern "C++" {
static pcb_status dwh_core(pcb_ctx* x, const uint32_t* c, const uint32_t* pw, size_t count, uint32_t* m, int32_t* stv,
                           cudaStream_t st, const uint32_t* yq_pre);
static pcb_status dwh_q(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* yq, cudaStream_t st);
}
static pcb_status update_entry(pcb_ctx* x, size_t nblk, const uint32_t* sizes, const uint32_t* c,
                               const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv, double z_min,
                               double z_max, double delta, double kappa, double* xo, double* zo, double* vo,
                               int32_t* status, pcb_stream stream, const uint32_t* p2pow = nullptr) {
  if (!x || (nblk && !sizes)) return PCB_E_SHAPE;
  size_t count = 0;
  std::vector<long long> seg(nblk + 1, 0);
  for (size_t k = 0; k < nblk; k++) seg[k + 1] = seg[k] + sizes[k];
  count = (size_t)seg[nblk];
  if (count && (!c || !rowsum || !q_z || !q_nv || !xo || !zo || !vo)) return PCB_E_SHAPE;
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;  // check_spec (quantize.cpp:8-15)
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (count == 0) return PCB_OK;
  if (count > 0x7fffffffu) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sc, sr, sz, sn, sx, szz, sv, ss;
  uint32_t* m = nullptr;
  int32_t* stv = nullptr;
  long long* segd = nullptr;
  pcb_status e = stage_in(c, count * 2 * x->L * 4, st, &sc);
  if (!e) e = stage_in(rowsum, count * 8, st, &sr);
  if (!e) e = stage_in(q_z, count * 8, st, &sz);
  if (!e) e = stage_in(q_nv, count * 8, st, &sn);
  if (!e) e = stage_in(xo, count * 8, st, &sx);  // in/out: staged in and copied back
  if (!e) e = stage_in(zo, count * 8, st, &szz);
  if (!e) e = stage_in(vo, count * 8, st, &sv);
  if (!e) e = stage_out(status, status ? count * 4 : 0, st, &ss);
  stv = (int32_t*)ss.dev;
  if (!e && !stv) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * x->L * 4, (void**)&m, st);
  if (!e) e = scratch_alloc(seg.size() * 8, (void**)&segd, st);
  if (!e) e = cuda_check(cudaMemcpyAsync(segd, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, st));
  Staged sp;
  if (p2pow && !x->has_rx) e = e ? e : PCB_E_UNSUPPORTED;
  if (!e && p2pow) e = stage_in(p2pow, count * 2 * x->L * 4, st, &sp);
  if (!e) e = p2pow ? dwh_core(x, (const uint32_t*)sc.dev, (const uint32_t*)sp.dev, count, m, stv, st, nullptr)  // collaborative
                    : dec_core(x, (const uint32_t*)sc.dev, count, m, stv, st);
  if (!e)
    e = launch_update(m, (int)x->L, (const uint64_t*)sr.dev, (const uint64_t*)sz.dev, (const uint64_t*)sn.dev, z_min,
                      z_max, delta, kappa, (double*)sx.dev, (double*)szz.dev, (double*)sv.dev, stv, count, segd,
                      (int)nblk, st);
  std::vector<int32_t> hst(count);
  if (!e) e = cuda_check(cudaMemcpyAsync(hst.data(), stv, count * 4, cudaMemcpyDeviceToHost, st));
  for (auto* p : {&sx, &szz, &sv}) {
    if (!e && p->host) {
      p->bytes = count * 8;
      e = cuda_check(cudaMemcpyAsync(p == &sx ? (void*)xo : p == &szz ? (void*)zo : (void*)vo, p->dev, count * 8,
                                     cudaMemcpyDeviceToHost, st));
    }
  }
  if (!e) e = unstage_out(status, &ss, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!ss.dev) scratch_free(stv, st);
  scratch_free(m, st);
  scratch_free(segd, st);
  for (auto* p : {&sc, &sr, &sz, &sn, &sx, &szz, &sv, &ss, &sp}) unstage(p, st);
  cudaStreamSynchronize(st);
  if (!e) {
    x->pow_half += (p2pow ? 1 : 2) * (uint64_t)count;
    for (int32_t v : hst)
      if (v != PCB_OK) return (pcb_status)v;  // first failure, like the reference's throw
  }
  return e;
}

pcb_status pcb_decrypt_update(pcb_ctx* x, const uint32_t* c, size_t count, const uint64_t* rowsum, const uint64_t* q_z,
                              const uint64_t* q_nv, double z_min, double z_max, double delta, double kappa, double* xo,
                              double* zo, double* vo, int32_t* status, pcb_stream stream) {
  if (count > 0x7fffffffu) return PCB_E_SHAPE;
  const uint32_t n = (uint32_t)count;
  return update_entry(x, 1, &n, c, rowsum, q_z, q_nv, z_min, z_max, delta, kappa, xo, zo, vo, status, stream);
}

pcb_status pcb_decrypt_update_blocks(pcb_ctx* x, size_t nblocks, const uint32_t* sizes, const uint32_t* c,
                                     const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv, double z_min,
                                     double z_max, double delta, double kappa, double* xo, double* zo, double* vo,
                                     int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_update_blocks");
  return update_entry(x, nblocks, sizes, c, rowsum, q_z, q_nv, z_min, z_max, delta, kappa, xo, zo, vo, status, stream);
}

pcb_status pcb_combined_update(const uint64_t* q_alpha, const uint64_t* q_b, const uint64_t* q_z,
                               const uint64_t* q_nv, size_t rows, size_t cols, uint64_t* out, pcb_stream stream) {
  if (rows && (!q_alpha || !out || (cols && (!q_b || !q_z || !q_nv)))) return PCB_E_SHAPE;
  if (rows == 0) return PCB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sa, sb, sz, sn, so;
  pcb_status e = stage_in(q_alpha, rows * 16, st, &sa);
  if (!e) e = stage_in(q_b, rows * cols * 8, st, &sb);
  if (!e) e = stage_in(q_z, cols * 8, st, &sz);
  if (!e) e = stage_in(q_nv, cols * 8, st, &sn);
  if (!e) e = stage_out(out, rows * 16, st, &so);
  if (!e)
    e = launch_combined_update((const uint64_t*)sa.dev, (const uint64_t*)sb.dev, (const uint64_t*)sz.dev,
                               (const uint64_t*)sn.dev, rows, cols, (uint64_t*)so.dev, st);
  if (!e) e = unstage_out(out, &so, st);
  const bool any_host = sa.host || sb.host || sz.host || sn.host || so.host;
  for (auto* p : {&sa, &sb, &sz, &sn, &so}) unstage(p, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_inverse_quantize_x(const uint64_t* q, const uint64_t* rowsum, const uint64_t* q_z,
                                  const uint64_t* q_nv, size_t rows, size_t cols, double z_min, double z_max,
                                  double delta, double* x, pcb_stream stream) {
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;  // check_spec (quantize.cpp:8-15)
  if (rows && (!q || !rowsum || !x || (cols && (!q_z || !q_nv)))) return PCB_E_SHAPE;
  if (rows == 0) return PCB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sq, sr, sz, sn, sx;
  std::vector<uint64_t> zero(2, 0);
  pcb_status e = stage_in(q, rows * 16, st, &sq);
  if (!e) e = stage_in(rowsum, rows * 8, st, &sr);
  if (!e) e = stage_in(cols ? (const void*)q_z : (const void*)zero.data(), std::max<size_t>(cols, 1) * 8, st, &sz);
  if (!e) e = stage_in(cols ? (const void*)q_nv : (const void*)zero.data(), std::max<size_t>(cols, 1) * 8, st, &sn);
  if (!e) e = stage_out(x, rows * 8, st, &sx);
  if (!e)
    e = launch_inverse_x((const uint64_t*)sq.dev, (const uint64_t*)sr.dev, (const uint64_t*)sz.dev,
                         (const uint64_t*)sn.dev, rows, cols, z_min, z_max, delta, (double*)sx.dev, st);
  if (!e) e = unstage_out(x, &sx, st);
  for (auto* p : {&sq, &sr, &sz, &sn, &sx}) unstage(p, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_obfuscate_exponent(const uint32_t* value, uint32_t value_limbs, const uint64_t* mask,
                                  const uint32_t* n_eps, uint32_t ne_limbs, size_t count, uint32_t* out,
                                  uint32_t out_limbs, pcb_stream stream) {
  if (count && (!value || !mask || !n_eps || !out)) return PCB_E_SHAPE;
  if (!value_limbs || !ne_limbs || out_limbs < ne_limbs + 3 || out_limbs < value_limbs) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sv, sm, sn, so;
  pcb_status e = stage_in(value, count * value_limbs * 4, st, &sv);
  if (!e) e = stage_in(mask, count * 8, st, &sm);
  if (!e) e = stage_in(n_eps, ne_limbs * 4, st, &sn);
  if (!e) e = stage_out(out, count * out_limbs * 4, st, &so);
  if (!e)
    e = launch_obfuscate((const uint32_t*)sv.dev, (int)value_limbs, (const uint64_t*)sm.dev, (const uint32_t*)sn.dev,
                         (int)ne_limbs, count, (uint32_t*)so.dev, (int)out_limbs, st);
  if (!e) e = unstage_out(out, &so, st);
  const bool any_host = sv.host || sm.host || sn.host || so.host;
  for (auto* p : {&sv, &sm, &sn, &so}) unstage(p, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

// ---- asynchronous iteration forms (include/pcb200.h): device pointers, no host sync ----------
pcb_status pcb_edge_step_blocks_async(pcb_ctx* x, size_t nblocks, const uint32_t* sizes, const uint32_t* alpha,
                                      const uint64_t* expo, uint32_t expo_bits, const uint32_t* zc,
                                      const uint32_t* vc, uint32_t window, uint32_t* out, int32_t* err_dev,
                                      pcb_stream stream) {
  PCB_RANGE("pcb_edge_step_blocks_async");
  if (!x || (nblocks && !sizes) || !err_dev) return PCB_E_SHAPE;
  if (window < 1 || window > 8) return PCB_E_SHAPE;
  size_t total = 0;
  for (size_t k = 0; k < nblocks; k++) total += sizes[k];
  if (total == 0) return PCB_OK;
  if (!alpha || !expo || !zc || !vc || !out) return PCB_E_SHAPE;
  for (const void* p : {(const void*)alpha, (const void*)expo, (const void*)zc, (const void*)vc, (const void*)out,
                        (const void*)err_dev})
    if (!is_device_ptr(p)) return PCB_E_SHAPE;  // the asynchronous form never stages host memory
  if (auto e = set_device(x)) return e;
  return edge_core(x, nblocks, sizes, alpha, expo, zc, vc, out, (cudaStream_t)stream, (int)expo_bits, err_dev);
}

pcb_status pcb_quantize_async(const double* v, size_t count, double z_min, double z_max, double delta, int fine,
                              uint64_t* q_out, uint64_t* clamps_dev, int32_t* err_dev, pcb_stream stream) {
  if (count && (!v || !q_out || !err_dev)) return PCB_E_SHAPE;
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;  // check_spec (quantize.cpp:8-15)
  if (count == 0) return PCB_OK;
  if (!is_device_ptr(v) || !is_device_ptr(q_out) || !is_device_ptr(err_dev) || (clamps_dev && !is_device_ptr(clamps_dev)))
    return PCB_E_SHAPE;
  return launch_quantize(v, count, z_min, z_max, delta, fine, q_out, (unsigned long long*)clamps_dev, err_dev,
                         (cudaStream_t)stream);
}

pcb_status pcb_decrypt_update_blocks_async(pcb_ctx* x, size_t nblk, const uint32_t* sizes, const uint32_t* c,
                                           const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                                           double z_min, double z_max, double delta, double kappa, double* xo,
                                           double* zo, double* vo, int32_t* err_dev, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_update_blocks_async");
  if (!x || (nblk && !sizes) || !err_dev) return PCB_E_SHAPE;
  std::vector<long long> seg(nblk + 1, 0);
  for (size_t k = 0; k < nblk; k++) seg[k + 1] = seg[k] + sizes[k];
  const size_t count = (size_t)seg[nblk];
  if (count && (!c || !rowsum || !q_z || !q_nv || !xo || !zo || !vo)) return PCB_E_SHAPE;
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (count == 0) return PCB_OK;
  if (count > 0x7fffffffu) return PCB_E_SHAPE;
  for (const void* p : {(const void*)c, (const void*)rowsum, (const void*)q_z, (const void*)q_nv, (const void*)xo,
                        (const void*)zo, (const void*)vo, (const void*)err_dev})
    if (!is_device_ptr(p)) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* m = nullptr;
  int32_t* stv = nullptr;
  long long* segd = nullptr;
  pcb_status e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * x->L * 4, (void**)&m, st);
  if (!e) e = scratch_alloc(seg.size() * 8, (void**)&segd, st);
  // pageable source: the driver stages it before returning, so `seg` may go out of scope
  if (!e) e = cuda_check(cudaMemcpyAsync(segd, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, st));
  if (!e) e = dec_core(x, c, count, m, stv, st);
  if (!e)
    e = launch_update(m, (int)x->L, rowsum, q_z, q_nv, z_min, z_max, delta, kappa, xo, zo, vo, stv, count, segd,
                      (int)nblk, st);
  if (!e) e = launch_status_flag(stv, count, err_dev, st);
  scratch_free(stv, st);
  scratch_free(m, st);
  scratch_free(segd, st);
  if (!e) x->pow_half += 2 * (uint64_t)count;
  return e;
}

pcb_status pcb_decrypt_half_q(pcb_ctx* x, const uint32_t* c, size_t count, uint32_t* q2_half, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_half_q");
  if (!x || (count && (!c || !q2_half))) return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (!x->has_rx) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (!is_device_ptr(c) || !is_device_ptr(q2_half)) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  const pcb_status e = dwh_q(x, c, count, q2_half, (cudaStream_t)stream);
  if (!e) x->pow_half += (uint64_t)count;  // the q half of decrypt_with_half
  return e;
}

pcb_status pcb_decrypt_update_blocks_half_async(pcb_ctx* x, size_t nblk, const uint32_t* sizes, const uint32_t* c,
                                                const uint32_t* p2_power, const uint32_t* q2_half,
                                                const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                                                double z_min, double z_max, double delta, double kappa, double* xo,
                                                double* zo, double* vo, int32_t* err_dev, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_update_blocks_half_async");
  if (!x || (nblk && !sizes) || !err_dev) return PCB_E_SHAPE;
  std::vector<long long> seg(nblk + 1, 0);
  for (size_t k = 0; k < nblk; k++) seg[k + 1] = seg[k] + sizes[k];
  const size_t count = (size_t)seg[nblk];
  if (count && (!c || !p2_power || !rowsum || !q_z || !q_nv || !xo || !zo || !vo)) return PCB_E_SHAPE;
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;
  if (!x->has_prv) return PCB_E_NO_PRIVATE;
  if (!x->has_rx) return PCB_E_UNSUPPORTED;
  if (count == 0) return PCB_OK;
  if (count > 0x7fffffffu) return PCB_E_SHAPE;
  for (const void* p : {(const void*)c, (const void*)p2_power, (const void*)rowsum, (const void*)q_z,
                        (const void*)q_nv, (const void*)xo, (const void*)zo, (const void*)vo, (const void*)err_dev})
    if (!is_device_ptr(p)) return PCB_E_SHAPE;
  if (q2_half && !is_device_ptr(q2_half)) return PCB_E_SHAPE;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* m = nullptr;
  int32_t* stv = nullptr;
  long long* segd = nullptr;
  pcb_status e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e) e = scratch_alloc(count * x->L * 4, (void**)&m, st);
  if (!e) e = scratch_alloc(seg.size() * 8, (void**)&segd, st);
  if (!e) e = cuda_check(cudaMemcpyAsync(segd, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, st));
  if (!e) e = dwh_core(x, c, p2_power, count, m, stv, st, q2_half);
  if (!e)
    e = launch_update(m, (int)x->L, rowsum, q_z, q_nv, z_min, z_max, delta, kappa, xo, zo, vo, stv, count, segd,
                      (int)nblk, st);
  if (!e) e = launch_status_flag(stv, count, err_dev, st);
  scratch_free(stv, st);
  scratch_free(m, st);
  scratch_free(segd, st);
  if (!e && !q2_half) x->pow_half += (uint64_t)count;
  return e;
}

pcb_status pcb_decrypt_update_blocks_half(pcb_ctx* x, size_t nblocks, const uint32_t* sizes, const uint32_t* c,
                                          const uint32_t* p2_power, const uint64_t* rowsum, const uint64_t* q_z,
                                          const uint64_t* q_nv, double z_min, double z_max, double delta, double kappa,
                                          double* xo, double* zo, double* vo, int32_t* status, pcb_stream stream) {
  PCB_RANGE("pcb_decrypt_update_blocks_half");
  if (!p2_power) return PCB_E_SHAPE;
  return update_entry(x, nblocks, sizes, c, rowsum, q_z, q_nv, z_min, z_max, delta, kappa, xo, zo, vo, status, stream,
                      p2_power);
}

pcb_status pcb_quantize(const double* v, size_t count, double z_min, double z_max, double delta, int fine,
                        uint64_t* q_out, uint64_t* clamps, pcb_stream stream) {
  if (count && (!v || !q_out)) return PCB_E_SHAPE;
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sv, sq;
  unsigned long long* dclamps = nullptr;
  int32_t* stv = nullptr;
  uint32_t* dummy_r = nullptr;
  uint32_t* dn = nullptr;
  pcb_status e = stage_in(v, count * 8, st, &sv);
  if (!e) e = stage_out(q_out, count * 8 * (fine ? 2 : 1), st, &sq);
  if (!e) e = scratch_alloc(16, (void**)&dclamps, st);
  if (!e) e = cuda_check(cudaMemsetAsync(dclamps, 0, 16, st));
  if (!e) e = scratch_alloc(count * 4, (void**)&stv, st);
  // the prep kernel also range-checks m and r against n: give it n = 2^160 - 1 (5 words) and
  // r = 1, so only the quantizer's own status (non-finite input) can fail
  if (!e) e = scratch_alloc(count * 5 * 4, (void**)&dummy_r, st);
  if (!e) e = scratch_alloc(5 * 4, (void**)&dn, st);
  if (!e) {
    std::vector<uint32_t> ones(count * 5, 0), nmax(5, 0xffffffffu);
    for (size_t i = 0; i < count; i++) ones[i * 5] = 1;
    e = cuda_check(cudaMemcpyAsync(dummy_r, ones.data(), count * 5 * 4, cudaMemcpyHostToDevice, st));
    if (!e) e = cuda_check(cudaMemcpyAsync(dn, nmax.data(), 20, cudaMemcpyHostToDevice, st));
    if (!e)
      e = launch_enc_prep(nullptr, 0, (const double*)sv.dev, z_min, z_max, delta, fine, nullptr, 0, (uint64_t*)sq.dev,
                          dclamps, dummy_r, dn, 5, stv, count, st);
    if (!e) e = cuda_check(cudaStreamSynchronize(st));  // host vectors above are temporaries
  }
  if (!e) e = unstage_out(q_out, &sq, st);
  unsigned long long hcl[2] = {0, 0};
  std::vector<int32_t> hst(count);
  if (!e) e = cuda_check(cudaMemcpyAsync(hcl, dclamps, 16, cudaMemcpyDeviceToHost, st));
  if (!e) e = cuda_check(cudaMemcpyAsync(hst.data(), stv, count * 4, cudaMemcpyDeviceToHost, st));
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  for (void* p : {(void*)dclamps, (void*)stv, (void*)dummy_r, (void*)dn}) scratch_free(p, st);
  unstage(&sv, st);
  unstage(&sq, st);
  cudaStreamSynchronize(st);
  if (!e && clamps) {
    clamps[0] = hcl[0];
    clamps[1] = hcl[1];
  }
  if (!e)
    for (int32_t s2 : hst)
      if (s2 != PCB_OK) return PCB_E_SHAPE;
  return e;
}

pcb_status pcb_sample_r(pcb_ctx* x, uint64_t* rng_state, size_t count, uint32_t* r_out, pcb_stream stream) {
  PCB_RANGE("pcb_sample_r");
  if (!x || !rng_state || (count && !r_out)) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sr;
  pcb_status e = stage_out(r_out, count * x->L * 4, st, &sr);
  const int H = (int)((std::max(x->p.bit_length(), x->q.bit_length()) + 31) / 32);
  std::vector<uint32_t> nl = x->n.limbs(x->L), pl, ql;
  if (x->has_prv) {
    pl = x->p.limbs(H);
    ql = x->q.limbs(H);
  }
  if (!e)
    e = rstream_sample(rng_state, nl.data(), (int)x->L, (int)x->nbits, x->has_prv ? pl.data() : nullptr,
                       x->has_prv ? ql.data() : nullptr, H, count, (uint32_t*)sr.dev, st);
  if (!e) e = unstage_out(r_out, &sr, st);
  unstage(&sr, st);
  if (sr.host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_quantize_encrypt(pcb_ctx* x, const double* v, size_t count, double z_min, double z_max, double delta,
                                int fine, const uint32_t* r, int use_crt, uint32_t* c, uint64_t* q_out,
                                uint64_t* clamps, pcb_stream stream) {
  PCB_RANGE("pcb_quantize_encrypt");
  if (!x || (count && (!v || !r || !c))) return PCB_E_SHAPE;
  // check_spec (quantize.cpp:8-15)
  if (!std::isfinite(z_min) || !std::isfinite(z_max) || !(z_max > z_min) || !(delta >= 1.0) || delta > 9.0e15)
    return PCB_E_SHAPE;
  if (use_crt && !x->has_prv) return PCB_E_NO_PRIVATE;
  if (x->random_g) return PCB_E_UNSUPPORTED;  // the fused quantize + Enc is the g = n + 1 hot path
  if (count == 0) return PCB_OK;
  if (auto e = set_device(x)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  if (count >= kPipeMin && !is_device_ptr(c)) {  // host ciphertexts: chunked, each chunk's copy beside the next's compute
    const size_t WO = 2 * x->L, qw = fine ? 2 : 1;
    const size_t chunk = ((count + kPipeChunks - 1) / kPipeChunks + 255) / 256 * 256;
    HostPipe hp;
    pcb_status e = hp.init(st);
    uint32_t* dc[2] = {nullptr, nullptr};
    for (int b = 0; b < 2 && !e; b++) e = scratch_alloc(chunk * WO * 4, (void**)&dc[b], st);
    if (!e) e = cuda_check(cudaStreamSynchronize(st));
    uint64_t tot[2] = {0, 0};
    for (size_t i = 0, off = 0; off < count && !e; i++, off += chunk) {
      const int b = (int)(i & 1);
      const size_t cnt = std::min(chunk, count - off);
      if (i >= 2) e = cuda_check(cudaStreamWaitEvent(st, hp.out[b], 0));  // dc[b]'s previous chunk is home
      uint64_t cl[2] = {0, 0};
      if (!e)  // device output: the call returns once the chunk is computed (its status check synchronises)
        e = pcb_quantize_encrypt(x, v + off, cnt, z_min, z_max, delta, fine, r + off * x->L, use_crt, dc[b],
                                 q_out ? q_out + off * qw : nullptr, cl, stream);
      tot[0] += cl[0];
      tot[1] += cl[1];
      if (!e) e = cuda_check(cudaEventRecord(hp.comp[b], st));
      if (!e) e = cuda_check(cudaStreamWaitEvent(hp.cout, hp.comp[b], 0));
      if (!e) e = cuda_check(cudaMemcpyAsync(c + off * WO, dc[b], cnt * WO * 4, cudaMemcpyDeviceToHost, hp.cout));
      if (!e) e = cuda_check(cudaEventRecord(hp.out[b], hp.cout));
    }
    if (cudaStreamSynchronize(hp.cout) != cudaSuccess && !e) e = PCB_E_CUDA;
    for (void* p : {(void*)dc[0], (void*)dc[1]}) scratch_free(p, st);
    cudaStreamSynchronize(st);
    if (!e && clamps) {
      clamps[0] = tot[0];
      clamps[1] = tot[1];
    }
    return e;
  }
  Staged sv, sr, sc, sq;
  unsigned long long* dclamps = nullptr;
  if (!use_crt) {  // public-key form: prep (quantize + checks) then n^2 encryption
    uint32_t* mq = nullptr;
    int32_t* stv = nullptr;
    pcb_status e = stage_in(v, count * 8, st, &sv);
    if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
    if (!e) e = stage_out(c, count * 2 * x->L * 4, st, &sc);
    if (!e) e = stage_out(q_out, q_out ? count * 8 * (fine ? 2 : 1) : 0, st, &sq);
    if (!e) e = scratch_alloc(16, (void**)&dclamps, st);
    if (!e) e = cuda_check(cudaMemsetAsync(dclamps, 0, 16, st));
    if (!e) e = scratch_alloc(count * 4 * 4, (void**)&mq, st);
    if (!e) e = scratch_alloc(count * 4, (void**)&stv, st);
    if (!e)
      e = launch_enc_prep(nullptr, 0, (const double*)sv.dev, z_min, z_max, delta, fine, mq, 4, (uint64_t*)sq.dev,
                          dclamps, (const uint32_t*)sr.dev, x->d_n, (int)x->L, stv, count, st);
    if (!e) e = cuda_check(cudaMemsetAsync(sc.dev, 0, count * 2 * x->L * 4, st));
    if (!e) e = run_pub_enc(x, (const uint32_t*)sr.dev, mq, 4, stv, count, (uint32_t*)sc.dev, st);
    if (!e) e = unstage_out(c, &sc, st);
    if (!e) e = unstage_out(q_out, &sq, st);
    unsigned long long hcl[2] = {0, 0};
    std::vector<int32_t> hst(count);
    if (!e && clamps) e = cuda_check(cudaMemcpyAsync(hcl, dclamps, 16, cudaMemcpyDeviceToHost, st));
    if (!e) e = cuda_check(cudaMemcpyAsync(hst.data(), stv, count * 4, cudaMemcpyDeviceToHost, st));
    if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
    scratch_free(mq, st);
    scratch_free(stv, st);
    scratch_free(dclamps, st);
    for (auto* p : {&sv, &sr, &sc, &sq}) unstage(p, st);
    cudaStreamSynchronize(st);
    if (!e && clamps) {
      clamps[0] = hcl[0];
      clamps[1] = hcl[1];
    }
    if (!e) {
      x->pow_full += (uint64_t)count;
      for (int32_t s2 : hst)
        if (s2 != PCB_OK) return (pcb_status)s2;
    }
    return e;
  }
  pcb_status e = stage_in(v, count * 8, st, &sv);
  if (!e) e = stage_in(r, count * x->L * 4, st, &sr);
  if (!e) e = stage_out(c, count * 2 * x->L * 4, st, &sc);
  if (!e) e = stage_out(q_out, q_out ? count * 8 * (fine ? 2 : 1) : 0, st, &sq);
  int32_t* stv = nullptr;  // per-element statuses: the first failure is the call's result
  if (!e) e = scratch_alloc(16, (void**)&dclamps, st);
  if (!e) e = cuda_check(cudaMemsetAsync(dclamps, 0, 16, st));
  if (!e) e = scratch_alloc(count * 4, (void**)&stv, st);
  if (!e)
    e = enc_core(x, nullptr, 0, (const double*)sv.dev, z_min, z_max, delta, fine, (uint64_t*)sq.dev, dclamps,
                 (const uint32_t*)sr.dev, count, (uint32_t*)sc.dev, stv, st);
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(q_out, &sq, st);
  unsigned long long hcl[2] = {0, 0};
  if (!e && clamps) e = cuda_check(cudaMemcpyAsync(hcl, dclamps, 16, cudaMemcpyDeviceToHost, st));
  if (!e) e = first_failure(stv, count, st);  // synchronises st
  scratch_free(stv, st);
  unstage(&sv, st);
  unstage(&sr, st);
  unstage(&sc, st);
  unstage(&sq, st);
  scratch_free(dclamps, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e && clamps) {
    clamps[0] = hcl[0];
    clamps[1] = hcl[1];
  }
  if (!e) x->pow_half += 2 * (uint64_t)count;
  return e;
}

pcb_status pcb_modexp_batch(const uint32_t* m, uint32_t m_limbs, const uint32_t* e, uint32_t e_limbs,
                            const uint32_t* xs, size_t count, uint32_t* y, pcb_stream stream) {
  PCB_RANGE("pcb_modexp_batch");
  if (!m || !e || (count && (!xs || !y))) return PCB_E_SHAPE;
  const int S = kernel_width(m_limbs);
  if (!S) return PCB_E_SHAPE;
  if (count == 0) return PCB_OK;
  try {
    HBN M = HBN::from_limbs(m, m_limbs), E = HBN::from_limbs(e, e_limbs);
    if (!M.is_odd()) return PCB_E_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    Staged sx, sy;
    pcb_status s = stage_in(xs, count * m_limbs * 4, st, &sx);
    if (!s) s = stage_out(y, count * m_limbs * 4, st, &sy);
    uint32_t* ydev = nullptr;
    uint8_t* d_ops = nullptr;
    if (!s) s = scratch_alloc(count * S * 4, (void**)&ydev, st);
    if (!s && E.is_zero()) {
      // x^0 = 1 mod m (0 when m == 1)
      std::vector<uint32_t> one(count * m_limbs, 0);
      if (!(M == HBN(1)))
        for (size_t i = 0; i < count; i++) one[i * m_limbs] = 1;
      s = cuda_check(cudaMemcpyAsync(sy.dev, one.data(), one.size() * 4, cudaMemcpyHostToDevice, st));
      cudaStreamSynchronize(st);
    } else if (!s) {
      std::vector<uint8_t> ops = build_ops(E, kWindow);
      s = scratch_alloc(ops.size(), (void**)&d_ops, st);
      if (!s) s = cuda_check(cudaMemcpyAsync(d_ops, ops.data(), ops.size(), cudaMemcpyHostToDevice, st));
      const char* core = getenv("PCB_CORE28");
      if (!s && S == 96) {  // 2049..3072-bit moduli: radix-2^28 core, 2 lanes per residue
        R28Mod c = r28_mod(M, 28, 112);
        const double mm = 2.0 * S * S + S;
        const double alg = ((double)E.bit_length() + (double)((E.bit_length() + 3) / 4)) * mm;
        s = launch_side28<28, 112, 2>(c.mlimb.data(), c.mword.data(), c.mwords, c.r2.data(), nullptr, c.minv, d_ops,
                                      (int)ops.size(), kTab, 2, (const uint32_t*)sx.dev, (int)m_limbs, nullptr, 0,
                                      nullptr, count, ydev, S, st, alg);
      } else if (!s && core && core[0] == '1' && M.bit_length() + 4 <= 28 * 76) {
        const int bits = (int)M.bit_length();
        const int N = bits + 4 <= 28 * 38 ? 38 : 76;
        R28Mod c = r28_mod(M, 28, N);
        const double mm = 2.0 * S * S + S;
        const double alg = ((double)E.bit_length() + (double)((E.bit_length() + 3) / 4)) * mm;
        const int yw = (int)S;
        if (N == 38)
          s = launch_side28<28, 38, 1>(c.mlimb.data(), c.mword.data(), c.mwords, c.r2.data(), nullptr, c.minv, d_ops,
                                       (int)ops.size(), kTab, 2, (const uint32_t*)sx.dev, (int)m_limbs, nullptr, 0,
                                       nullptr, count, ydev, yw, st, alg);
        else
          s = launch_side28<28, 76, 2>(c.mlimb.data(), c.mword.data(), c.mwords, c.r2.data(), nullptr, c.minv, d_ops,
                                       (int)ops.size(), kTab, 2, (const uint32_t*)sx.dev, (int)m_limbs, nullptr, 0,
                                       nullptr, count, ydev, yw, st, alg);
      } else if (!s) {
        switch (S) {
#define PCB_CASE(SS)                                                                                        \
  case SS: {                                                                                                \
    ModCtx<SS> mc;                                                                                          \
    fill_mod<SS>(mc, M);                                                                                    \
    s = launch_side<SS>(mc, nullptr, d_ops, (int)ops.size(), kTab, kSidePow, (const uint32_t*)sx.dev,       \
                        (int)m_limbs, nullptr, 0, nullptr, count, ydev, st, (int)E.bit_length());          \
    break;                                                                                                  \
  }
          PCB_CASE(32)
          PCB_CASE(64)
#undef PCB_CASE
          default: s = PCB_E_UNSUPPORTED;
        }
      }
      if (!s)
        s = cuda_check(cudaMemcpy2DAsync(sy.dev, m_limbs * 4, ydev, S * 4, m_limbs * 4, count,
                                         cudaMemcpyDeviceToDevice, st));
      cudaStreamSynchronize(st);  // `ops` is a host temporary
    }
    if (!s) s = unstage_out(y, &sy, st);
    unstage(&sx, st);
    unstage(&sy, st);
    scratch_free(ydev, st);
    scratch_free(d_ops, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && !s) s = PCB_E_CUDA;
    return s;
  } catch (...) {
    return PCB_E_SHAPE;
  }
}

}  // extern "C"

// ---- not yet implemented in this build (fail loudly, never fall back) -----------------------
extern "C" {
}
