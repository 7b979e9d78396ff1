// wire.cu — the reference's ciphertext wire format, packed and parsed on the device, so GPU
// ciphertexts interoperate byte-for-byte with a reference SimCarrier / TcpCarrier session:
//   put_cipher_vec / get_cipher_vec (wire.cpp:125-146): u32 BE count, then per element
//     u32 BE byte length, the minimal big-endian magnitude (bignat.cpp:414-418 wire_put), u32 BE
//     plain_bits;
//   encode_envelope (wire.cpp:148-159): u32 BE (7 + payload), type, u16 BE session, u32 BE
//     iteration, payload.
// One warp per element moves the magnitude bytes; the variable-length layout is placed by an
// exclusive scan of the per-element sizes (CUB).
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <cstring>
#include <vector>

#include "pcb_internal.h"

namespace pcb {
namespace {

__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24);
  p[1] = (uint8_t)(v >> 16);
  p[2] = (uint8_t)(v >> 8);
  p[3] = (uint8_t)v;
}
__device__ __forceinline__ uint32_t get_be32(const uint8_t* p) {
  return ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | (uint32_t)p[3];
}

// minimal magnitude length in bytes of every element (0 for zero), record size = 8 + len
__global__ void wire_len_kernel(const uint32_t* c, int W, size_t count, uint32_t* len, uint64_t* rec) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t* x = c + i * W;
    int top = W - 1;
    while (top >= 0 && x[top] == 0) top--;
    uint32_t bytes = 0;
    if (top >= 0) bytes = 4 * (uint32_t)top + (32 - __clz(x[top]) + 7) / 8;
    len[i] = bytes;
    rec[i] = 8ull + bytes;
  }
}

// one warp per element: length, big-endian magnitude, plain_bits at 4 + offs[i]
__global__ void wire_put_kernel(const uint32_t* c, int W, const uint32_t* plain_bits, size_t count,
                                const uint32_t* len, const uint64_t* offs, uint8_t* out) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) put_be32(out, (uint32_t)count);
  for (size_t i = warp; i < count; i += nwarps) {
    uint8_t* o = out + 4 + offs[i];
    const uint32_t nb = len[i];
    const uint32_t* x = c + i * W;
    if (lane == 0) {
      put_be32(o, nb);
      put_be32(o + 4 + nb, plain_bits ? plain_bits[i] : 0u);
    }
    for (uint32_t b = lane; b < nb; b += 32) {  // byte b of the BE magnitude = LE byte nb - 1 - b
      const uint32_t le = nb - 1 - b;
      o[4 + b] = (uint8_t)(x[le / 4] >> (8 * (le % 4)));
    }
  }
}

// sequential walk of the length fields (device-resident frames): offs[i] = start of element i
__global__ void wire_walk_kernel(const uint8_t* in, size_t in_len, size_t off0, size_t count, int W, uint64_t* offs,
                                 int* err, uint64_t* end) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  size_t off = off0;
  for (size_t i = 0; i < count; i++) {
    if (off + 4 > in_len) { *err = PCB_E_SHAPE; return; }
    const uint32_t nb = get_be32(in + off);
    if (nb > 4u * (uint32_t)W || off + 8 + nb > in_len) { *err = PCB_E_SHAPE; return; }
    offs[i] = off;
    off += 8 + nb;
  }
  *end = off;
}

// one warp per element: magnitude bytes -> W LE u32 limbs (zero-extended), plain_bits
__global__ void wire_get_kernel(const uint8_t* in, const uint64_t* offs, size_t count, int W, uint32_t* c,
                                uint32_t* plain_bits) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t i = warp; i < count; i += nwarps) {
    const uint8_t* p = in + offs[i];
    const uint32_t nb = get_be32(p);
    uint32_t* x = c + i * W;
    for (int w = lane; w < W; w += 32) {
      uint32_t v = 0;
      for (int k = 3; k >= 0; k--) {  // LE byte 4w + k sits at BE index nb - 1 - (4w + k)
        const uint32_t le = 4u * (uint32_t)w + (uint32_t)k;
        v = (v << 8) | (le < nb ? p[4 + nb - 1 - le] : 0u);
      }
      x[w] = v;
    }
    if (lane == 0 && plain_bits) plain_bits[i] = get_be32(p + 4 + nb);
  }
}

int warp_grid(size_t count) {
  const size_t b = (count * 32 + 255) / 256;
  return (int)(b < 4096 ? (b ? b : 1) : 4096);
}

}  // namespace
}  // namespace pcb

using namespace pcb;

extern "C" {

pcb_status pcb_wire_put_cipher_vec(const uint32_t* c, uint32_t W, const uint32_t* plain_bits, size_t count,
                                   uint8_t* out, size_t out_cap, size_t* out_len, pcb_stream stream) {
  PCB_RANGE("pcb_wire_put_cipher_vec");
  if (!out_len || W == 0 || (count && !c) || count > 0xffffffffu) return PCB_E_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  Staged sc, sp, so;
  uint32_t* len = nullptr;
  uint64_t *rec = nullptr, *offs = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  pcb_status e = stage_in(c, count * W * 4, st, &sc);
  if (!e) e = stage_in(plain_bits, plain_bits ? count * 4 : 0, st, &sp);
  if (!e) e = scratch_alloc(count * 4, (void**)&len, st);
  if (!e) e = scratch_alloc((count + 1) * 8, (void**)&rec, st);
  if (!e) e = scratch_alloc((count + 1) * 8, (void**)&offs, st);
  if (!e && count) {
    wire_len_kernel<<<(int)std::min<size_t>((count + 255) / 256, 4096), 256, 0, st>>>((const uint32_t*)sc.dev, (int)W,
                                                                                       count, len, rec);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) e = cuda_check(cudaMemsetAsync(rec + count, 0, 8, st));
  if (!e) e = cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rec, offs, count + 1, st));
  if (!e) e = scratch_alloc(tmp_bytes, &tmp, st);
  if (!e) e = cuda_check(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rec, offs, count + 1, st));
  uint64_t body = 0;
  if (!e) e = cuda_check(cudaMemcpyAsync(&body, offs + count, 8, cudaMemcpyDeviceToHost, st));
  if (!e) e = cuda_check(cudaStreamSynchronize(st));  // the caller needs the frame length
  const size_t total = 4 + (size_t)body;
  *out_len = total;
  if (!e && out) {
    if (out_cap < total) e = PCB_E_SHAPE;
    if (!e) e = stage_out(out, total, st, &so);
    if (!e) {
      wire_put_kernel<<<warp_grid(count), 256, 0, st>>>((const uint32_t*)sc.dev, (int)W, (const uint32_t*)sp.dev, count,
                                                        len, offs, (uint8_t*)so.dev);
      count_launch();
      e = cuda_check(cudaGetLastError());
    }
    if (!e) e = unstage_out(out, &so, st);
  }
  scratch_free(len, st);
  scratch_free(rec, st);
  scratch_free(offs, st);
  scratch_free(tmp, st);
  const bool any_host = sc.host || sp.host || so.host;
  for (auto* p : {&sc, &sp, &so}) unstage(p, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  return e;
}

pcb_status pcb_wire_get_cipher_vec(const uint8_t* in, size_t in_len, size_t* off, uint32_t W, size_t max_count,
                                   size_t* count_out, uint32_t* c, uint32_t* plain_bits, pcb_stream stream) {
  PCB_RANGE("pcb_wire_get_cipher_vec");
  if (!in || !off || !count_out || W == 0) return PCB_E_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev_in = is_device_ptr(in);
  // the element count and the length fields: read in place from host frames, walked by one
  // device thread for device-resident frames
  uint8_t hdr[4];
  if (*off + 4 > in_len) return PCB_E_SHAPE;
  if (dev_in) {
    if (cudaMemcpyAsync(hdr, in + *off, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return PCB_E_CUDA;
  } else {
    std::memcpy(hdr, in + *off, 4);
  }
  const size_t count = ((size_t)hdr[0] << 24) | ((size_t)hdr[1] << 16) | ((size_t)hdr[2] << 8) | hdr[3];
  *count_out = count;
  if (count > max_count) return PCB_E_SHAPE;
  if (count && !c) return PCB_E_SHAPE;
  Staged si, sc, sp;
  uint64_t* offs = nullptr;
  size_t end = *off + 4;
  pcb_status e = scratch_alloc((count + 1) * 8, (void**)&offs, st);
  if (!e && !dev_in) {
    std::vector<uint64_t> h(count);
    size_t o = *off + 4;
    for (size_t i = 0; i < count && !e; i++) {
      if (o + 4 > in_len) { e = PCB_E_SHAPE; break; }
      const uint32_t nb = ((uint32_t)in[o] << 24) | ((uint32_t)in[o + 1] << 16) | ((uint32_t)in[o + 2] << 8) | in[o + 3];
      if (nb > 4u * W || o + 8 + nb > in_len) { e = PCB_E_SHAPE; break; }
      h[i] = o;
      o += 8 + nb;
    }
    end = o;
    // pageable source: staged by the driver before the call returns
    if (!e && count) e = cuda_check(cudaMemcpyAsync(offs, h.data(), count * 8, cudaMemcpyHostToDevice, st));
    if (!e) e = stage_in(in, end, st, &si);
  } else if (!e) {
    si.dev = const_cast<uint8_t*>(in);
    int* derr = nullptr;
    uint64_t* dend = nullptr;
    e = scratch_alloc(4, (void**)&derr, st);
    if (!e) e = scratch_alloc(8, (void**)&dend, st);
    if (!e) e = cuda_check(cudaMemsetAsync(derr, 0, 4, st));
    if (!e) {
      wire_walk_kernel<<<1, 32, 0, st>>>(in, in_len, *off + 4, count, (int)W, offs, derr, dend);
      count_launch();
      e = cuda_check(cudaGetLastError());
    }
    int herr = 0;
    uint64_t hend = 0;
    if (!e) e = cuda_check(cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, st));
    if (!e) e = cuda_check(cudaMemcpyAsync(&hend, dend, 8, cudaMemcpyDeviceToHost, st));
    if (!e) e = cuda_check(cudaStreamSynchronize(st));
    if (!e && herr) e = (pcb_status)herr;
    end = (size_t)hend;
    scratch_free(derr, st);
    scratch_free(dend, st);
  }
  if (!e) e = stage_out(c, count * W * 4, st, &sc);
  if (!e) e = stage_out(plain_bits, plain_bits ? count * 4 : 0, st, &sp);
  if (!e && count) {
    wire_get_kernel<<<warp_grid(count), 256, 0, st>>>((const uint8_t*)si.dev, offs, count, (int)W, (uint32_t*)sc.dev,
                                                      (uint32_t*)sp.dev);
    count_launch();
    e = cuda_check(cudaGetLastError());
  }
  if (!e) e = unstage_out(c, &sc, st);
  if (!e) e = unstage_out(plain_bits, &sp, st);
  scratch_free(offs, st);
  const bool any_host = si.host || sc.host || sp.host;
  for (auto* p : {&si, &sc, &sp}) unstage(p, st);
  if (any_host && cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;
  if (!e) *off = end;
  return e;
}

pcb_status pcb_encode_envelope(uint8_t type, uint16_t session, uint32_t iteration, const uint8_t* payload,
                               size_t payload_len, uint8_t* out, size_t out_cap, size_t* out_len, pcb_stream stream) {
  if (!out_len || (payload_len && !payload) || type < 1 || type > 7) return PCB_E_SHAPE;
  const size_t body = 7 + payload_len;
  if (body > ((size_t)256 << 20)) return PCB_E_SHAPE;  // kFrameCap (wire.hpp:14): length_error
  *out_len = 4 + body;
  if (!out) return PCB_OK;
  if (out_cap < 4 + body) return PCB_E_SHAPE;
  const uint8_t hdr[11] = {(uint8_t)(body >> 24), (uint8_t)(body >> 16), (uint8_t)(body >> 8), (uint8_t)body, type,
                           (uint8_t)(session >> 8), (uint8_t)session,  (uint8_t)(iteration >> 24),
                           (uint8_t)(iteration >> 16), (uint8_t)(iteration >> 8), (uint8_t)iteration};
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev_out = is_device_ptr(out), dev_pl = payload_len && is_device_ptr(payload);
  if (!dev_out && !dev_pl) {  // host to host: plain copies
    std::memcpy(out, hdr, 11);
    if (payload_len) std::memcpy(out + 11, payload, payload_len);
    return PCB_OK;
  }
  pcb_status e = cuda_check(cudaMemcpyAsync(out, hdr, 11, cudaMemcpyDefault, st));
  if (!e && payload_len) e = cuda_check(cudaMemcpyAsync(out + 11, payload, payload_len, cudaMemcpyDefault, st));
  if (cudaStreamSynchronize(st) != cudaSuccess && !e) e = PCB_E_CUDA;  // hdr is a host temporary
  return e;
}

}  // extern "C"
