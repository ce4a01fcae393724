// Fused single-launch C1 (quantized all-gather) and C2 (quantized
// reduce-scatter) instantiations: fp32 weights/gradients, direct widths,
// buckets of 128..2048 elements (one warp per bucket).
#include "qsdp_kernels.cuh"

namespace qsdp {

template <int INNER, int BITS, bool ACC, int OUT>
static cudaError_t launch_fused_t(const QJobTable& qt, const DJobTable& dt, const FuseSync& fs, int sms,
                                  cudaStream_t s) {
  constexpr int NST = 2;
  const size_t stage = (size_t)qt.bucket * sizeof(float);
  const int wpc = 8;
  size_t smem = (size_t)wpc * NST * stage + (size_t)wpc * NST * sizeof(uint64_t) + (size_t)wpc * 32 * sizeof(SeedOut);
  const size_t acc_rows = (size_t)wpc * 8 * 3 * sizeof(double);
  if (smem < acc_rows) smem = acc_rows;
  auto kern = fused_collective_kernel<float, INNER, BITS, NST, ACC, OUT>;
  static thread_local size_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  // every CTA must be co-resident (in-kernel grid barrier): grid = one full wave at most
  static thread_local int per_sm = 0;
  static thread_local size_t per_sm_smem = 0;
  if (per_sm == 0 || per_sm_smem != smem) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, wpc * 32, smem) != cudaSuccess || v < 1) v = 1;
    per_sm = v;
    per_sm_smem = smem;
  }
  const int64_t work = qt.total_buckets > dt.total_buckets ? qt.total_buckets : dt.total_buckets;
  int64_t grid = (work + wpc - 1) / wpc;
  const int64_t cap = (int64_t)sms * per_sm;
  grid = grid < 1 ? 1 : (grid > cap ? cap : grid);
  kern<<<(int)grid, wpc * 32, smem, s>>>(qt, dt, fs);
  return cudaGetLastError();
}

template <int INNER, bool ACC, int OUT>
static cudaError_t launch_fused_bits(const QJobTable& qt, const DJobTable& dt, const FuseSync& fs, int sms,
                                     cudaStream_t s) {
  switch (qt.bits) {
    case 8: return launch_fused_t<INNER, 8, ACC, OUT>(qt, dt, fs, sms, s);
    case 4: return launch_fused_t<INNER, 4, ACC, OUT>(qt, dt, fs, sms, s);
    case 2: return launch_fused_t<INNER, 2, ACC, OUT>(qt, dt, fs, sms, s);
    default: return launch_fused_t<INNER, 16, ACC, OUT>(qt, dt, fs, sms, s);
  }
}

// all_gather: INNER 0 (shift), K3 pull;  reduce_scatter: INNER 1 (stochastic), K4 pull.
cudaError_t launch_fused(const QJobTable& qt, const DJobTable& dt, const FuseSync& fs, int sms, cudaStream_t s) {
  if (qt.inner == 0) {
    return dt.out_dtype == 2 ? launch_fused_bits<0, false, 2>(qt, dt, fs, sms, s)
                             : launch_fused_bits<0, false, 0>(qt, dt, fs, sms, s);
  }
  return launch_fused_bits<1, true, 0>(qt, dt, fs, sms, s);
}

cudaError_t upload_jump_fused(const JumpEntry* host) {
  return cudaMemcpyToSymbol(g_jump, host, sizeof(JumpEntry) * kJumpTable);
}

}  // namespace qsdp
