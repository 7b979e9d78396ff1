// factor.cu — the edges' node factors on the device, all blocks of a session in one batch:
//   node_factor (admm.cpp:63-75): normal = A_k^T A_k + rho I,  B_k = rho normal^-1,
//   alpha_k = normal^-1 A_k^T y_s  (y_s = y / K under YScaling::over_k).
// The reference factors `normal` once with Eigen's LDLT and solves against I and A^T y.  Here the
// same SPD system goes through a blocked Cholesky, a blocked triangular inverse and the product
// normal^-1 = L^-T L^-1, every FLOP on FP64 tensor cores (DMMA 8x8x4, mma.sync f64 -- tcgen05 has
// no f64 kind) in one generic 64 x 64 tile kernel driven by task lists:
//
//   Gram       N_k[i,j] = sum_r A[r, i] A[r, j]  (+ rho on the diagonal)   lower tiles, K = rows
//   potrf      diagonal 64 x 64 block: unblocked Cholesky + its triangular inverse in shared memory
//   panel      L_ij = N_ij Linv_jj^T                                          (trsm by the inverse)
//   syrk       N_ik -= L_ij L_kj^T                                            trailing lower tiles
//   trtri      M = L^-1 by block rows: T_ik = L_i,[k,i) M_[k,i),k ; M_ik = -Linv_ii T_ik
//   lauum      B_k = rho M^T M                                                lower tiles, mirrored
//   alpha      u = A_k^T y_s ; v = M u ; alpha = M^T v
//
// Numerics: FP64 throughout; results agree with the reference's LDLT solve to rounding (the
// factorisation and the summation order differ), tests/test_gpu_factor.py states the tolerance.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "pcb_internal.h"

namespace pcb {
namespace {

constexpr int TB = 64;  // tile edge
constexpr int KC = 16;  // k chunk staged in shared memory
constexpr int SA = KC + 4;  // row strides chosen so the DMMA fragment loads are conflict-free
constexpr int SB = TB + 4;

struct TileTask {
  const double* A;
  const double* B;
  double* C;
  int lda, ldb, ldc;
  int m, n, k;       // C is m x n (<= 64), the reduction depth is k
  int ta, tb, mode;  // opA = A (ta 0: A[i lda + kk]) or A^T (ta 1: A[kk lda + i]); opB likewise
  double scale;      // mode 0: C = scale opA opB (+ diag on the tile's diagonal); 1: C -= opA opB; 2: C = -opA opB
  double diag;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One 64 x 64 output tile per CTA, 4 warps of 32 x 32 (4 x 4 DMMA tiles each).  The k loop stages
// 64 x 16 of opA and 16 x 64 of opB per step; the next chunk's loads are issued into registers
// before the current chunk's MMAs.  The output tile is written after every chunk was read, so a
// task may overwrite its own A tile (the in-place panel solve).
__global__ void __launch_bounds__(128) tile_kernel(const TileTask* __restrict__ tasks) {
  __shared__ double As[TB][SA];
  __shared__ double Bs[KC][SB];
  const TileTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      int i, kk;
      if (t.ta == 0) {
        kk = tid & 15;
        i = (tid >> 4) + 8 * r;
      } else {
        i = tid & 63;
        kk = (tid >> 6) + 2 * r;
      }
      const int gk = k0 + kk;
      ra[r] = (i < t.m && gk < t.k) ? (t.ta == 0 ? t.A[(size_t)i * t.lda + gk] : t.A[(size_t)gk * t.lda + i]) : 0.0;
      int j;
      if (t.tb == 0) {
        j = tid & 63;
        kk = (tid >> 6) + 2 * r;
      } else {
        kk = tid & 15;
        j = (tid >> 4) + 8 * r;
      }
      const int gk2 = k0 + kk;
      rb[r] = (j < t.n && gk2 < t.k) ? (t.tb == 0 ? t.B[(size_t)gk2 * t.ldb + j] : t.B[(size_t)j * t.ldb + gk2]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      if (t.ta == 0)
        As[(tid >> 4) + 8 * r][tid & 15] = ra[r];
      else
        As[tid & 63][(tid >> 6) + 2 * r] = ra[r];
      if (t.tb == 0)
        Bs[(tid >> 6) + 2 * r][tid & 63] = rb[r];
      else
        Bs[tid & 15][(tid >> 4) + 8 * r] = rb[r];
    }
  };

  load(0);
  for (int k0 = 0; k0 < t.k; k0 += KC) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + KC < t.k) load(k0 + KC);
#pragma unroll
    for (int k4 = 0; k4 < KC; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; a++) af[a] = As[wm * 32 + a * 8 + (lane >> 2)][k4 + (lane & 3)];
#pragma unroll
      for (int b = 0; b < 4; b++) bf[b] = Bs[k4 + (lane & 3)][wn * 32 + b * 8 + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b], af[a], bf[b]);
    }
  }
  // epilogue: lane holds C[row = lane / 4][col = 2 (lane % 4) + {0, 1}] of each 8 x 8 tile
  __syncthreads();  // every chunk read before the (possibly aliasing) tile is written
#pragma unroll
  for (int a = 0; a < 4; a++) {
    const int i = wm * 32 + a * 8 + (lane >> 2);
    if (i >= t.m) continue;
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = wn * 32 + b * 8 + 2 * (lane & 3) + h;
        if (j >= t.n) continue;
        double* c = t.C + (size_t)i * t.ldc + j;
        const double v = acc[a][b][h];
        if (t.mode == 0)
          *c = i == j ? t.scale * v + t.diag : t.scale * v;
        else if (t.mode == 1)
          *c = *c - v;
        else
          *c = -v;
      }
  }
}

struct PotrfTask {
  double* D;     // diagonal block (in place: lower = L_jj, upper zeroed)
  double* Dinv;  // its inverse (lower triangular, upper zeroed)
  int ld, m;
};

// Unblocked right-looking Cholesky of one m x m (m <= 64) diagonal block in shared memory, then
// its inverse by column-parallel forward substitution.  A non-positive or non-finite pivot
// (normal is SPD for rho > 0; only NaN/Inf input gets here) sets *err.
__global__ void __launch_bounds__(256) potrf_kernel(const PotrfTask* __restrict__ tasks, int* err) {
  extern __shared__ double sm[];
  double (*S)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(sm);
  double (*X)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(sm + TB * (TB + 1));
  const PotrfTask t = tasks[blockIdx.x];
  const int tid = threadIdx.x, m = t.m;
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    S[i][j] = j <= i ? t.D[(size_t)i * t.ld + j] : 0.0;
  }
  __syncthreads();
  for (int p = 0; p < m; p++) {
    if (tid == 0) {
      const double d = S[p][p];
      if (!(d > 0.0) || !isfinite(d)) atomicCAS(err, 0, 1);
      S[p][p] = sqrt(d);
    }
    __syncthreads();
    const double piv = S[p][p];
    for (int i = p + 1 + tid; i < m; i += blockDim.x) S[i][p] = S[i][p] / piv;
    __syncthreads();
    const int r = m - p - 1;  // trailing (r x r) lower triangle
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int i = p + 1 + e / r, j = p + 1 + e % r;
      if (j <= i) S[i][j] = S[i][j] - S[i][p] * S[j][p];
    }
    __syncthreads();
  }
  if (tid < m) {  // column c of L^-1
    const int c = tid;
    X[c][c] = 1.0 / S[c][c];
    for (int i = c + 1; i < m; i++) {
      double s = 0.0;
      for (int k = c; k < i; k++) s += S[i][k] * X[k][c];
      X[i][c] = -s / S[i][i];
    }
  }
  __syncthreads();
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    t.D[(size_t)i * t.ld + j] = j <= i ? S[i][j] : 0.0;
    t.Dinv[(size_t)i * t.ld + j] = j <= i ? X[i][j] : 0.0;
  }
}

// B_k upper triangle from its lower triangle (the product M^T M is symmetric)
__global__ void mirror_kernel(double* b, const uint64_t* mat_off, const uint32_t* sizes, int nblocks) {
  const int k = blockIdx.y;
  if (k >= nblocks) return;
  const size_t c = sizes[k];
  double* m = b + mat_off[k];
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < c * c; e += (size_t)gridDim.x * blockDim.x) {
    const size_t i = e / c, j = e % c;
    if (j > i) m[e] = m[j * c + i];
  }
}

__global__ void scale_kernel(const double* y, size_t n, double k_total, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = y[i] / k_total;
}

}  // namespace

pcb_status node_factors_core(const double* a, size_t rows, size_t cols, size_t lda, const double* y, size_t nblocks,
                             const uint32_t* sizes, double rho, uint32_t k_total, int over_k, double* b_bar,
                             double* alpha, cudaStream_t st) {
  std::vector<uint64_t> col_off(nblocks), mat_off(nblocks);
  uint64_t cs = 0, ms = 0;
  int nbmax = 0;
  for (size_t k = 0; k < nblocks; k++) {
    col_off[k] = cs;
    mat_off[k] = ms;
    cs += sizes[k];
    ms += (uint64_t)sizes[k] * sizes[k];
    nbmax = std::max(nbmax, (int)((sizes[k] + TB - 1) / TB));
  }
  // task lists of every launch, uploaded once
  std::vector<TileTask> tt;
  std::vector<PotrfTask> pt;
  struct Launch {
    int kind;  // 0 tile, 1 potrf
    size_t first, count;
  };
  std::vector<Launch> plan;
  double *nm = nullptr, *mm = nullptr, *tsc = nullptr, *ys = nullptr, *u = nullptr, *v = nullptr;
  pcb_status e = scratch_alloc(ms * 8, (void**)&nm, st);
  if (!e) e = scratch_alloc(ms * 8, (void**)&mm, st);
  if (!e) e = scratch_alloc(nblocks * (size_t)std::max(nbmax, 1) * TB * TB * 8, (void**)&tsc, st);
  if (!e) e = scratch_alloc(rows * 8, (void**)&ys, st);
  if (!e) e = scratch_alloc(cols * 8, (void**)&u, st);
  if (!e) e = scratch_alloc(cols * 8, (void**)&v, st);
  auto tile = [&](const double* A, int lda_, int ta, const double* B, int ldb_, int tb, double* C, int ldc, int m, int n,
                  int k, int mode, double scale = 1.0, double diag = 0.0) {
    tt.push_back(TileTask{A, B, C, lda_, ldb_, ldc, m, n, k, ta, tb, mode, scale, diag});
  };
  auto close = [&](int kind, size_t first) {
    const size_t cnt = (kind == 0 ? tt.size() : pt.size()) - first;
    if (cnt) plan.push_back({kind, first, cnt});
  };
  if (!e) {
    const double* yv = over_k ? ys : y;
    // Gram + rho I (lower tiles)
    size_t f = tt.size();
    for (size_t k = 0; k < nblocks; k++) {
      const int c = (int)sizes[k];
      double* N = nm + mat_off[k];
      for (int i0 = 0; i0 < c; i0 += TB)
        for (int j0 = 0; j0 <= i0; j0 += TB)
          tile(a + col_off[k] + i0, (int)lda, 1, a + col_off[k] + j0, (int)lda, 0, N + (size_t)i0 * c + j0, c,
               std::min(TB, c - i0), std::min(TB, c - j0), (int)rows, 0, 1.0, i0 == j0 ? rho : 0.0);
    }
    close(0, f);
    // blocked Cholesky
    for (int jb = 0; jb < nbmax; jb++) {
      const int j0 = jb * TB;
      size_t fp = pt.size();
      for (size_t k = 0; k < nblocks; k++) {
        const int c = (int)sizes[k];
        if (j0 >= c) continue;
        pt.push_back(PotrfTask{nm + mat_off[k] + (size_t)j0 * c + j0, mm + mat_off[k] + (size_t)j0 * c + j0, c,
                               std::min(TB, c - j0)});
      }
      close(1, fp);
      f = tt.size();
      for (size_t k = 0; k < nblocks; k++) {
        const int c = (int)sizes[k];
        double *N = nm + mat_off[k], *M = mm + mat_off[k];
        const int w = std::min(TB, c - j0);
        for (int i0 = j0 + TB; i0 < c; i0 += TB)
          tile(N + (size_t)i0 * c + j0, c, 0, M + (size_t)j0 * c + j0, c, 1, N + (size_t)i0 * c + j0, c,
               std::min(TB, c - i0), w, w, 0);
      }
      close(0, f);
      f = tt.size();
      for (size_t k = 0; k < nblocks; k++) {
        const int c = (int)sizes[k];
        double* N = nm + mat_off[k];
        const int w = std::min(TB, c - j0);
        for (int i0 = j0 + TB; i0 < c; i0 += TB)
          for (int k0 = j0 + TB; k0 <= i0; k0 += TB)
            tile(N + (size_t)i0 * c + j0, c, 0, N + (size_t)k0 * c + j0, c, 1, N + (size_t)i0 * c + k0, c,
                 std::min(TB, c - i0), std::min(TB, c - k0), w, 1);
      }
      close(0, f);
    }
    // M = L^-1 by block rows (diagonal blocks came from potrf)
    for (int ib = 1; ib < nbmax; ib++) {
      const int i0 = ib * TB;
      f = tt.size();
      for (size_t k = 0; k < nblocks; k++) {
        const int c = (int)sizes[k];
        if (i0 >= c) continue;
        double *N = nm + mat_off[k], *M = mm + mat_off[k], *T = tsc + k * (size_t)nbmax * TB * TB;
        for (int k0 = 0; k0 < i0; k0 += TB)
          tile(N + (size_t)i0 * c + k0, c, 0, M + (size_t)k0 * c + k0, c, 0, T + (size_t)(k0 / TB) * TB * TB, TB,
               std::min(TB, c - i0), TB, i0 - k0, 0);
      }
      close(0, f);
      f = tt.size();
      for (size_t k = 0; k < nblocks; k++) {
        const int c = (int)sizes[k];
        if (i0 >= c) continue;
        double *M = mm + mat_off[k], *T = tsc + k * (size_t)nbmax * TB * TB;
        const int w = std::min(TB, c - i0);
        for (int k0 = 0; k0 < i0; k0 += TB)
          tile(M + (size_t)i0 * c + i0, c, 0, T + (size_t)(k0 / TB) * TB * TB, TB, 0, M + (size_t)i0 * c + k0, c, w, TB,
               w, 2);
      }
      close(0, f);
    }
    // B = rho M^T M (lower tiles) and u = A^T y_s (independent: one launch)
    f = tt.size();
    for (size_t k = 0; k < nblocks; k++) {
      const int c = (int)sizes[k];
      double* M = mm + mat_off[k];
      for (int a0 = 0; a0 < c; a0 += TB)
        for (int b0 = 0; b0 <= a0; b0 += TB)
          tile(M + (size_t)a0 * c + a0, c, 1, M + (size_t)a0 * c + b0, c, 0, b_bar + mat_off[k] + (size_t)a0 * c + b0, c,
               std::min(TB, c - a0), std::min(TB, c - b0), c - a0, 0, rho);
      for (int i0 = 0; i0 < c; i0 += TB)
        tile(a + col_off[k] + i0, (int)lda, 1, yv, 1, 0, u + col_off[k] + i0, 1, std::min(TB, c - i0), 1, (int)rows, 0);
    }
    close(0, f);
    // v = M u, then alpha = M^T v
    f = tt.size();
    for (size_t k = 0; k < nblocks; k++) {
      const int c = (int)sizes[k];
      double* M = mm + mat_off[k];
      for (int i0 = 0; i0 < c; i0 += TB) {
        const int w = std::min(TB, c - i0);
        tile(M + (size_t)i0 * c, c, 0, u + col_off[k], 1, 0, v + col_off[k] + i0, 1, w, 1, i0 + w, 0);
      }
    }
    close(0, f);
    f = tt.size();
    for (size_t k = 0; k < nblocks; k++) {
      const int c = (int)sizes[k];
      double* M = mm + mat_off[k];
      for (int a0 = 0; a0 < c; a0 += TB)
        tile(M + (size_t)a0 * c + a0, c, 1, v + col_off[k] + a0, 1, 0, alpha + col_off[k] + a0, 1,
             std::min(TB, c - a0), 1, c - a0, 0);
    }
    close(0, f);
  }
  TileTask* dtt = nullptr;
  PotrfTask* dpt = nullptr;
  uint64_t* dmo = nullptr;
  uint32_t* dsz = nullptr;
  int* derr = nullptr;
  if (!e) e = scratch_alloc(std::max<size_t>(tt.size(), 1) * sizeof(TileTask), (void**)&dtt, st);
  if (!e) e = scratch_alloc(std::max<size_t>(pt.size(), 1) * sizeof(PotrfTask), (void**)&dpt, st);
  if (!e) e = scratch_alloc(nblocks * 8, (void**)&dmo, st);
  if (!e) e = scratch_alloc(nblocks * 4, (void**)&dsz, st);
  if (!e) e = scratch_alloc(4, (void**)&derr, st);
  if (!e) e = cuda_check(cudaMemcpyAsync(dtt, tt.data(), tt.size() * sizeof(TileTask), cudaMemcpyHostToDevice, st));
  if (!e && !pt.empty())
    e = cuda_check(cudaMemcpyAsync(dpt, pt.data(), pt.size() * sizeof(PotrfTask), cudaMemcpyHostToDevice, st));
  if (!e) e = cuda_check(cudaMemcpyAsync(dmo, mat_off.data(), nblocks * 8, cudaMemcpyHostToDevice, st));
  if (!e) e = cuda_check(cudaMemcpyAsync(dsz, sizes, nblocks * 4, cudaMemcpyHostToDevice, st));
  if (!e) e = cuda_check(cudaMemsetAsync(derr, 0, 4, st));
  if (!e) e = cuda_check(cudaMemsetAsync(mm, 0, ms * 8, st));  // M's strictly upper blocks stay zero
  if (!e && over_k) {
    scale_kernel<<<(int)std::min<size_t>((rows + 255) / 256, 1184), 256, 0, st>>>(y, rows, (double)k_total, ys);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  const int potrf_smem = 2 * TB * (TB + 1) * 8;
  if (!e) e = cuda_check(cudaFuncSetAttribute(potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, potrf_smem));
  for (const Launch& l : plan) {
    if (e) break;
    if (l.kind == 0)
      tile_kernel<<<(unsigned)l.count, 128, 0, st>>>(dtt + l.first);
    else
      potrf_kernel<<<(unsigned)l.count, 256, potrf_smem, st>>>(dpt + l.first, derr);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) {
    dim3 g(64, (unsigned)nblocks);
    mirror_kernel<<<g, 256, 0, st>>>(b_bar, dmo, dsz, (int)nblocks);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  int herr = 0;
  if (!e) e = cuda_check(cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, st));
  if (!e) e = cuda_check(cudaStreamSynchronize(st));
  if (!e && herr) e = PCB_E_SHAPE;  // normal not positive definite (non-finite input)
  for (void* p : {(void*)nm, (void*)mm, (void*)tsc, (void*)ys, (void*)u, (void*)v, (void*)dtt, (void*)dpt, (void*)dmo,
                  (void*)dsz, (void*)derr})
    scratch_free(p, st);
  return e;
}

}  // namespace pcb

extern "C" pcb_status pcb_node_factors(const double* a, size_t rows, size_t cols, size_t lda, const double* y,
                                       size_t nblocks, const uint32_t* sizes, double rho, uint32_t k_total,
                                       int over_k, double* b_bar, double* alpha, pcb_stream stream) {
  PCB_RANGE("pcb_node_factors");
  using namespace pcb;
  // check_inputs (admm.cpp:8-16), node_factor's k_total check (admm.cpp:66), split shape
  if (!a || !y || !sizes || !b_bar || !alpha || rows == 0 || cols == 0 || lda < cols || nblocks == 0)
    return PCB_E_SHAPE;
  if (!(rho > 0.0) || k_total < 1 || rows > (size_t)INT32_MAX || lda > (size_t)INT32_MAX) return PCB_E_SHAPE;
  size_t total = 0, msz = 0;
  for (size_t k = 0; k < nblocks; k++) {
    if (sizes[k] == 0) return PCB_E_SHAPE;
    total += sizes[k];
    msz += (size_t)sizes[k] * sizes[k];
  }
  if (total != cols) return PCB_E_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sa, sy, sb, sl;
  pcb_status e = stage_in(a, ((rows - 1) * lda + cols) * 8, st, &sa);
  if (!e) e = stage_in(y, rows * 8, st, &sy);
  if (!e) e = stage_out(b_bar, msz * 8, st, &sb);
  if (!e) e = stage_out(alpha, cols * 8, st, &sl);
  if (!e)
    e = node_factors_core((const double*)sa.dev, rows, cols, lda, (const double*)sy.dev, nblocks, sizes, rho, k_total,
                          over_k, (double*)sb.dev, (double*)sl.dev, st);
  if (!e) e = unstage_out(b_bar, &sb, st);
  if (!e) e = unstage_out(alpha, &sl, st);
  const bool any_host = sa.host || sy.host || sb.host || sl.host;
  unstage(&sa, st);
  unstage(&sy, st);
  unstage(&sb, st);
  unstage(&sl, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}
