// pcb_internal.h — shared host/device plumbing of the CUDA library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstddef>
#include <cstdint>

#include "../../include/pcb200.h"

namespace pcb {

constexpr int kThreadsPerBlock = 128;

// Process-wide launch ledger (bench.py reports it as gpu_launches).
std::atomic<uint64_t>& launch_counter();
inline void count_launch(uint64_t k = 1) { launch_counter().fetch_add(k, std::memory_order_relaxed); }

inline pcb_status cuda_check(cudaError_t e) { return e == cudaSuccess ? PCB_OK : PCB_E_CUDA; }

// Grid = (#SMs) x (max resident CTAs per SM for this kernel / smem): a persistent grid.
template <class K>
pcb_status occupancy_grid(K kernel, size_t smem, int* blocks) {
  int dev = 0, nsm = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PCB_E_CUDA;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return PCB_E_CUDA;
  if (smem > 48 * 1024)
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return PCB_E_CUDA;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreadsPerBlock, smem) != cudaSuccess)
    return PCB_E_CUDA;
  if (per_sm < 1) return PCB_E_CUDA;
  *blocks = nsm * per_sm;
  return PCB_OK;
}

// Grid for `count` one-thread-per-element items: the persistent grid, shrunk when the batch
// is smaller (so a small batch still spreads over all SMs one warp at a time).
template <class K>
pcb_status item_grid(K kernel, size_t smem, size_t count, int* blocks) {
  int full = 0;
  if (auto e = occupancy_grid(kernel, smem, &full)) return e;
  size_t need = (count + kThreadsPerBlock - 1) / kThreadsPerBlock;
  *blocks = (int)(need < (size_t)full ? (need ? need : 1) : (size_t)full);
  return PCB_OK;
}

// Hot-kernel profiling (pcb_profile_begin/end): record an event pair around a launch.
struct ProfMark {
  cudaEvent_t a = nullptr, b = nullptr;
};
bool prof_enabled();
ProfMark prof_start(cudaStream_t st);
void prof_stop(ProfMark m, cudaStream_t st, double alg_mac32);
void prof_add_int8(double macs);  // int8 tensor-core MACs issued (RNS base extensions)

// Stream-ordered device scratch (cudaMallocAsync on the caller's stream; freed on the same
// stream once the kernels using it are enqueued).
pcb_status scratch_alloc(size_t bytes, void** p, cudaStream_t st);
void scratch_free(void* p, cudaStream_t st);

// Host/device pointer staging for the ABI: if `p` is a host pointer, copy `bytes` to a device
// scratch buffer (in) or allocate one (out).  `host` tells the caller to copy back.
struct Staged {
  void* dev = nullptr;
  bool host = false;
  size_t bytes = 0;
};
bool is_device_ptr(const void* p);
pcb_status stage_in(const void* p, size_t bytes, cudaStream_t st, Staged* s);
pcb_status stage_out(void* p, size_t bytes, cudaStream_t st, Staged* s);
pcb_status unstage_out(void* p, Staged* s, cudaStream_t st);  // copies back if host
void unstage(Staged* s, cudaStream_t st);

// NVTX range around an ABI call (header-only NVTX v3: a no-op unless a profiler injects itself),
// so nsys / ncu --nvtx timelines show the library's calls by name.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PCB_RANGE(name) ::pcb::NvtxRange pcb_nvtx_range_(name)

// Kernel width (limbs) used for a modulus of `limbs` limbs.
inline int kernel_width(uint32_t limbs) {
  if (limbs <= 32) return 32;
  if (limbs <= 64) return 64;
  if (limbs <= 96) return 96;
  if (limbs <= 128) return 128;  // 4096-bit keys: p^2, q^2 (RNS core only)
  return 0;
}
inline int kernel_width_wide(uint32_t limbs) {
  if (limbs <= 64) return 64;
  if (limbs <= 128) return 128;
  if (limbs <= 192) return 192;
  if (limbs <= 256) return 256;  // 4096-bit keys: n^2 = 8192 bits
  return 0;
}


}  // namespace pcb
