// Counter-based (numpy Philox4x64-10) instantiations of K1/K2, both input types:
// the team kernels with the Philox Coder and the generic kernel (own TU: parallel build).
#include "qsdp_kernels.cuh"

namespace qsdp {
cudaError_t launch_quantize_philox(const QJobTable& tab, bool f64, bool vec, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  if (f64) return tab.inner ? launch_q_philox<double, 1>(tab, vec, sms, s) : launch_q_philox<double, 0>(tab, vec, sms, s);
  return tab.inner ? launch_q_philox<float, 1>(tab, vec, sms, s) : launch_q_philox<float, 0>(tab, vec, sms, s);
}
}  // namespace qsdp
