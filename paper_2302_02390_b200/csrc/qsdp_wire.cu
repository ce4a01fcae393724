// GPU wire codec: byte-exact encode / decode of one
// quantized segment between the device layout (packed codes + float[nb][3]
// meta) and the reference's message format (wire.py:1-20, 108-184):
//
//   header  <BBIII  version=1, bit_width, bucket_size (= blocks[0].length),
//                   block_count, total_length                        14 bytes
//   block j <fff    shift, scale_lo, scale_hi                        12 bytes
//           payload ceil(len_j * bits / 8) bytes, LSB-first, zero-padded
//
// Both directions are gathers: one thread produces 16 consecutive output bytes
// (vector store when aligned), locating its block once and walking forward, so
// the codec is a single HBM-bound pass (read c, write c bytes per element).
// Decode also validates every complete block: nonzero padding bits
// (DecodeError, wire.py:90-91) and scale_lo <= scale_hi (QuantizedBlock,
// quantize.py:109-110), reporting the first failing block per kind.
#include <cuda_runtime.h>

#include <cstdint>

#include "qsdp_device.cuh"

namespace qsdp {


// byte o (>= 14) of the message: block j, offset w inside the block's wire bytes
__device__ __forceinline__ uint8_t wire_byte_at(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ meta,
                                                const WireGeom& g, int64_t j, int64_t w) {
  if (w < 12) return meta[12 * j + w];
  return codes[j * g.pbs + (w - 12)];
}

__global__ void __launch_bounds__(256) wire_encode_kernel(const uint8_t* __restrict__ codes,
                                                          const float* __restrict__ meta,
                                                          const __grid_constant__ WireGeom g, uint8_t* __restrict__ out) {
  const uint8_t* mb = reinterpret_cast<const uint8_t*>(meta);
  const int64_t nchunk = (g.msg_bytes + 15) / 16;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunk; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o0 = 16 * c;
    uint8_t buf[16];
    // locate the block of the first body byte of the chunk once, then walk
    int64_t j = 0, w = 0;
    if (o0 >= 14) {
      j = (o0 - 14) / g.blk;
      w = (o0 - 14) - j * g.blk;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t o = o0 + k;
      uint8_t v = 0;
      if (o < 14) {
        v = g.header[o];
      } else if (o < g.msg_bytes) {
        v = wire_byte_at(codes, mb, g, j, w);
        if (++w == g.blk) {
          w = 0;
          ++j;
        }
      }
      buf[k] = v;
    }
    uint8_t* dst = out + o0;
    if (o0 + 16 <= g.msg_bytes && ((uintptr_t)dst & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(buf);
    } else {
      for (int k = 0; k < 16 && o0 + k < g.msg_bytes; ++k) dst[k] = buf[k];
    }
  }
}

// Decode the first `nblk` (complete) blocks: codes chunks are gathered from the
// payloads, meta from the block headers; err[0] = first block with nonzero
// padding bits, err[1] = first block with !(lo <= hi) (atomicMin; init INT64_MAX).
__global__ void __launch_bounds__(256) wire_decode_kernel(const uint8_t* __restrict__ msg, const __grid_constant__ WireGeom g,
                                                          int64_t nblk, uint8_t* __restrict__ codes,
                                                          float* __restrict__ meta, unsigned long long* err) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t cbytes = nblk == g.nb ? g.codes_bytes : nblk * g.pbs;
  const int64_t nchunk = (cbytes + 15) / 16;
  for (int64_t c = tid; c < nchunk; c += nth) {
    const int64_t c0 = 16 * c;
    int64_t j = c0 / g.pbs, w = c0 - j * g.pbs;
    uint8_t buf[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint8_t v = 0;
      if (c0 + k < cbytes) {
        v = msg[14 + j * g.blk + 12 + w];
        if (++w == g.pbs) {
          w = 0;
          ++j;
        }
      }
      buf[k] = v;
    }
    uint8_t* dst = codes + c0;
    if (c0 + 16 <= cbytes && ((uintptr_t)dst & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(buf);
    } else {
      for (int k = 0; k < 16 && c0 + k < cbytes; ++k) dst[k] = buf[k];
    }
  }
  // per block: meta + validation
  for (int64_t j = tid; j < nblk; j += nth) {
    const uint8_t* h = msg + 14 + j * g.blk;
    float m[3];
    uint8_t* mb = reinterpret_cast<uint8_t*>(m);
    for (int k = 0; k < 12; ++k) mb[k] = h[k];
    meta[3 * j] = m[0];
    meta[3 * j + 1] = m[1];
    meta[3 * j + 2] = m[2];
    const int64_t n = j == g.nb - 1 ? g.last_n : (int64_t)g.bucket;
    const int64_t pb = j == g.nb - 1 ? g.last_pb : g.pbs;
    const int used = (int)((n * g.bits) & 7);
    if (used != 0 && (h[12 + pb - 1] >> used) != 0) atomicMin(&err[0], (unsigned long long)j);
    if (!(m[1] <= m[2])) atomicMin(&err[1], (unsigned long long)j);
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

cudaError_t launch_wire_encode(const uint8_t* codes, const float* meta, const WireGeom& g, uint8_t* out, int sms,
                               cudaStream_t s) {
  wire_encode_kernel<<<grid_for_bytes(g.msg_bytes, sms), 256, 0, s>>>(codes, meta, g, out);
  return cudaGetLastError();
}

cudaError_t launch_wire_decode(const uint8_t* msg, const WireGeom& g, int64_t nblk, uint8_t* codes, float* meta,
                               unsigned long long* err, int sms, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  wire_decode_kernel<<<grid_for_bytes(nblk * g.blk, sms), 256, 0, s>>>(msg, g, nblk, codes, meta, err);
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
