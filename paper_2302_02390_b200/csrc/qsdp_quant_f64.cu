// fp64-input instantiations of K1/K2 (the reference protocol's float64 shards).
#include "qsdp_kernels.cuh"

namespace qsdp {
cudaError_t launch_quantize_f64(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  return tab.inner ? launch_q_t<double, 1>(tab, vec, sms, s) : launch_q_t<double, 0>(tab, vec, sms, s);
}
cudaError_t upload_jump_f64(const JumpEntry* host) {
  return cudaMemcpyToSymbol(g_jump, host, sizeof(JumpEntry) * kJumpTable);
}
}  // namespace qsdp
