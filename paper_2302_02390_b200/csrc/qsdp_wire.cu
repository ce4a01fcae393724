// GPU wire codec: byte-exact encode / decode of one
// quantized segment between the device layout (packed codes + float[nb][3]
// meta) and the reference's message format (wire.py:1-20, 108-184):
//
//   header  <BBIII  version=1, bit_width, bucket_size (= blocks[0].length),
//                   block_count, total_length                        14 bytes
//   block j <fff    shift, scale_lo, scale_hi                        12 bytes
//           payload ceil(len_j * bits / 8) bytes, LSB-first, zero-padded
//
// Both directions run one warp per block; the payload copy writes aligned 4-byte
// destination words assembled from aligned source words with funnel shifts (the
// message puts payloads at offsets = 2 mod 4), so the codec is a single
// HBM-bound pass (read c, write c bytes per element).
// Decode also validates every complete block: nonzero padding bits
// (DecodeError, wire.py:90-91) and scale_lo <= scale_hi (QuantizedBlock,
// quantize.py:109-110), reporting the first failing block per kind.
#include <cuda_runtime.h>

#include <cstdint>

#include "qsdp_device.cuh"

namespace qsdp {


// Warp-cooperative copy of n bytes between arbitrarily aligned buffers: single
// bytes up to an 8-aligned destination, then whole 8-byte destination words
// assembled from two aligned source words (64-bit funnel shift; 4 words in
// flight per lane), then the tail bytes.
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t n,
                                          int lane) {
  int64_t h = (8 - ((uintptr_t)dst & 7)) & 7;
  if (h > n) h = n;
  if (lane < h) dst[lane] = src[lane];
  const int64_t nw = (n - h) >> 3;  // whole destination words
  const uint8_t* s0 = src + h;
  const int sh = (int)((uintptr_t)s0 & 7);
  const unsigned long long* sa = reinterpret_cast<const unsigned long long*>(s0 - sh);
  unsigned long long* dw = reinterpret_cast<unsigned long long*>(dst + h);
  // with sh != 0 the last word read, sa[nw], is the word holding the last body
  // byte (s0 + 8*nw - 1), so no read leaves the source span's words
  constexpr int U = 4;
  for (int64_t i0 = lane; i0 < nw; i0 += 32 * U) {
    unsigned long long lo[U], hi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + 32 * u;
      lo[u] = i < nw ? sa[i] : 0ull;
      hi[u] = (sh && i < nw) ? sa[i + 1] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + 32 * u;
      if (i < nw) dw[i] = sh ? (lo[u] >> (8 * sh)) | (hi[u] << (64 - 8 * sh)) : lo[u];
    }
  }
  for (int64_t k = h + 8 * nw + lane; k < n; k += 32) dst[k] = src[k];
}

// One warp per block: the block's 12 meta bytes and payload go to their message
// offsets (14 + j*blk); block 0's warp also writes the 14 header bytes.
__global__ void __launch_bounds__(256) wire_encode_kernel(const uint8_t* __restrict__ codes,
                                                          const float* __restrict__ meta,
                                                          const __grid_constant__ WireGeom g, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint8_t* mb = reinterpret_cast<const uint8_t*>(meta);
  if (warp == 0 && lane < 14) out[lane] = g.header[lane];
  for (int64_t j = warp; j < g.nb; j += nwarps) {
    uint8_t* d = out + 14 + j * g.blk;
    if (lane < 12) d[lane] = mb[12 * j + lane];
    warp_copy(d + 12, codes + j * g.pbs, j == g.nb - 1 ? g.last_pb : g.pbs, lane);
  }
}

// Decode the first `nblk` (complete) blocks, one warp per block: payload to the
// packed layout, meta to float[nb][3]; err[0] = first block with nonzero padding
// bits, err[1] = first block with !(lo <= hi) (atomicMin; init UINT64_MAX).
__global__ void __launch_bounds__(256) wire_decode_kernel(const uint8_t* __restrict__ msg, const __grid_constant__ WireGeom g,
                                                          int64_t nblk, uint8_t* __restrict__ codes,
                                                          float* __restrict__ meta, unsigned long long* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < nblk; j += nwarps) {
    const uint8_t* h = msg + 14 + j * g.blk;
    const int64_t n = j == g.nb - 1 ? g.last_n : (int64_t)g.bucket;
    const int64_t pb = j == g.nb - 1 ? g.last_pb : g.pbs;
    warp_copy(codes + j * g.pbs, h + 12, pb, lane);
    if (lane == 0) {
      float m[3];
      uint8_t* mbytes = reinterpret_cast<uint8_t*>(m);
      for (int k = 0; k < 12; ++k) mbytes[k] = h[k];
      meta[3 * j] = m[0];
      meta[3 * j + 1] = m[1];
      meta[3 * j + 2] = m[2];
      const int used = (int)((n * g.bits) & 7);
      if (used != 0 && (h[12 + pb - 1] >> used) != 0) atomicMin(&err[0], (unsigned long long)j);
      if (!(m[1] <= m[2])) atomicMin(&err[1], (unsigned long long)j);
    }
  }
}

// uint32 codes (one per element) <-> the packed device layout (per bucket,
// LSB-first, each bucket zero-padded to a byte: wire.py:82-95).  Widths 1..32.
__global__ void __launch_bounds__(256) pack_codes_kernel(const uint32_t* __restrict__ codes, int64_t length,
                                                         int bucket, int bits, uint8_t* __restrict__ out,
                                                         int64_t out_bytes) {
  const int64_t pbs = payload_bytes(bucket, bits);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < out_bytes; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = c / pbs, w = c - j * pbs;
    const int64_t base = j * bucket;
    const int64_t nbits = (int64_t)min((int64_t)bucket, length - base) * bits;
    uint32_t v = 0;
    for (int b = 0; b < 8; ++b) {
      const int64_t bp = 8 * w + b;
      if (bp < nbits) v |= ((codes[base + bp / bits] >> (bp % bits)) & 1u) << b;
    }
    out[c] = (uint8_t)v;
  }
}

__global__ void __launch_bounds__(256) unpack_codes_kernel(const uint8_t* __restrict__ packed, int64_t length,
                                                           int bucket, int bits, uint32_t* __restrict__ codes) {
  const int64_t pbs = payload_bytes(bucket, bits);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < length; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / bucket, i = e - j * bucket;
    const int64_t n = min((int64_t)bucket, length - j * bucket);
    const int64_t lim = payload_bytes(n, bits);
    const int64_t bp = i * bits, by = bp >> 3;
    const uint8_t* p = packed + j * pbs;
    uint64_t w = 0;  // up to 7 + 32 bits
    for (int k = 0; k < 5; ++k)
      if (by + k < lim) w |= (uint64_t)p[by + k] << (8 * k);
    codes[e] = (uint32_t)((w >> (bp & 7)) & ((1ull << bits) - 1ull));
  }
}

static int grid_for_bytes(int64_t bytes, int sms) {
  const int64_t chunks = (bytes + 15) / 16;
  int64_t blocks = (chunks + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

static int grid_for_blocks(int64_t nb, int sms) {
  int64_t blocks = (nb + 7) / 8;  // 8 warps per CTA, one warp per block
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_wire_encode(const uint8_t* codes, const float* meta, const WireGeom& g, uint8_t* out, int sms,
                               cudaStream_t s) {
  wire_encode_kernel<<<grid_for_blocks(g.nb, sms), 256, 0, s>>>(codes, meta, g, out);
  return cudaGetLastError();
}

cudaError_t launch_wire_decode(const uint8_t* msg, const WireGeom& g, int64_t nblk, uint8_t* codes, float* meta,
                               unsigned long long* err, int sms, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  wire_decode_kernel<<<grid_for_blocks(nblk, sms), 256, 0, s>>>(msg, g, nblk, codes, meta, err);
  return cudaGetLastError();
}

cudaError_t launch_pack_codes(const uint32_t* codes, int64_t length, int bucket, int bits, uint8_t* out,
                              int64_t out_bytes, int sms, cudaStream_t s) {
  if (out_bytes <= 0) return cudaSuccess;
  pack_codes_kernel<<<grid_for_bytes(16 * out_bytes, sms), 256, 0, s>>>(codes, length, bucket, bits, out, out_bytes);
  return cudaGetLastError();
}

cudaError_t launch_unpack_codes(const uint8_t* packed, int64_t length, int bucket, int bits, uint32_t* codes, int sms,
                                cudaStream_t s) {
  if (length <= 0) return cudaSuccess;
  unpack_codes_kernel<<<grid_for_bytes(16 * length, sms), 256, 0, s>>>(packed, length, bucket, bits, codes);
  return cudaGetLastError();
}

}  // namespace qsdp
