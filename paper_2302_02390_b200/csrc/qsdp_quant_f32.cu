// fp32-input instantiations of K1/K2 (the GPT / FSDP hot path).
#include "qsdp_kernels.cuh"

namespace qsdp {
cudaError_t launch_quantize_f32(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  return tab.inner ? launch_q_t<float, 1>(tab, vec, sms, s) : launch_q_t<float, 0>(tab, vec, sms, s);
}
cudaError_t upload_jump_f32(const JumpEntry* host) {
  return cudaMemcpyToSymbol(g_jump, host, sizeof(JumpEntry) * kJumpTable);
}
}  // namespace qsdp
