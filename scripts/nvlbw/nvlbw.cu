// NVLink write-bandwidth probe (measurement tool, not product code): one GPU pushes a buffer
// into P-1 peers' memory with (0) per-lane 16-byte stores, (1) TMA bulk stores from shared
// memory in 4 KB chunks, several in flight per warp.  Built by scripts/nvlbw/Makefile.
#include <cuda_runtime.h>
#include <cstdint>

extern "C" int nvlbw_enable_peers(int n) {
  for (int i = 0; i < n; ++i) {
    cudaSetDevice(i);
    for (int j = 0; j < n; ++j)
      if (i != j) {
        cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return (int)e;
      }
  }
  cudaGetLastError();
  return 0;
}

struct Dsts { uint8_t* d[8]; int n; };

__global__ void st16_kernel(const uint4* __restrict__ src, Dsts dst, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    for (int k = 0; k < dst.n; ++k) reinterpret_cast<uint4*>(dst.d[k])[i] = v;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one warp per 4 KB chunk stream; lane 0 issues; NBUF buffers per warp
template <int NBUF>
__global__ void tma_kernel(const uint8_t* __restrict__ src, Dsts dst, int64_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int CH = 4096;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  uint8_t* buf = sm + (size_t)warp * NBUF * CH;
  __shared__ __align__(8) uint64_t bars[32 * NBUF];
  uint64_t* bar = bars + warp * NBUF;
  if (lane == 0)
    for (int b = 0; b < NBUF; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar + b)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t nch = bytes / CH;
  const int64_t gw = (int64_t)blockIdx.x * wpc + warp, nw = (int64_t)gridDim.x * wpc;
  uint32_t phase[NBUF] = {};
  int it = 0;
  for (int64_t c = gw; c < nch; c += nw, ++it) {
    const int b = it % NBUF;
    if (lane == 0) {
      if (it >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar + b)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(buf + b * CH)),
                   "l"(src + c * CH), "r"(CH), "r"(smem_u32(bar + b))
                   : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(bar + b)), "r"(phase[b]) : "memory");
      phase[b] ^= 1u;
      for (int k = 0; k < dst.n; ++k)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst.d[k] + c * CH),
                     "r"(smem_u32(buf + b * CH)), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int nvlbw_run(int mode, const void* src, void** dsts, int ndst, long long bytes, int grid, int block,
                         void* stream) {
  Dsts d{};
  for (int k = 0; k < ndst; ++k) d.d[k] = static_cast<uint8_t*>(dsts[k]);
  d.n = ndst;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mode == 0) {
    st16_kernel<<<grid, block, 0, s>>>(static_cast<const uint4*>(src), d, bytes / 16);
  } else {
    const int nbuf = mode;  // 1..4 buffers
    const size_t smem = (size_t)(block / 32) * nbuf * 4096;
    if (nbuf == 2) {
      cudaFuncSetAttribute(tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      tma_kernel<2><<<grid, block, smem, s>>>(static_cast<const uint8_t*>(src), d, bytes);
    } else {
      cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      tma_kernel<4><<<grid, block, smem, s>>>(static_cast<const uint8_t*>(src), d, bytes);
    }
  }
  return (int)cudaGetLastError();
}
