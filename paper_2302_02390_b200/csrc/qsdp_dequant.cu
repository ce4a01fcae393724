// K3 (dequantize) / K4 (ordered dequantize-accumulate) instantiations.
#include "qsdp_kernels.cuh"

namespace qsdp {
template <int BITS, int TL, int OUT, bool ACC>
static cudaError_t launch_d_tl(const DJobTable& tab, bool vec, int sms, cudaStream_t s) {
  auto go = [&](auto kern) {
    kern<<<persistent_grid(kern, 256, 0, tab.total_buckets, 32 / TL, sms), 256, 0, s>>>(tab);
  };
  if constexpr (ACC) {
    if (tab.lat_on) {  // K4 with the fused lattice-projected step
      if constexpr (TL == 32 && (BITS == 8 || BITS == 4)) {
        int ns = 0;
        for (int j = 0; j < tab.njobs; ++j) ns = ns > tab.jobs[j].nsrc ? ns : tab.jobs[j].nsrc;
        if (vec && tab.codes_vec && (tab.bucket & 127) == 0 && tab.bucket <= 1024) {
          auto pick = [&](auto xt) {
            using XT = decltype(xt);
            if (ns <= 2) go(dequant_lat_fast_kernel<BITS, OUT, 2, XT>);
            else if (ns <= 4) go(dequant_lat_fast_kernel<BITS, OUT, 4, XT>);
            else go(dequant_lat_fast_kernel<BITS, OUT, 8, XT>);
          };
          if (tab.lat_xdtype == 1) pick(0.0);
          else pick(0.0f);
          return cudaGetLastError();
        }
      }
      if (vec) go(dequant_kernel<BITS, TL, OUT, true, ACC, true>);
      else go(dequant_kernel<BITS, TL, OUT, false, ACC, true>);
      return cudaGetLastError();
    }
  }
  if (vec) go(dequant_kernel<BITS, TL, OUT, true, ACC>);
  else go(dequant_kernel<BITS, TL, OUT, false, ACC>);
  return cudaGetLastError();
}

template <int BITS, int OUT, bool ACC>
static cudaError_t launch_d_bits(const DJobTable& tab, bool vec, int sms, cudaStream_t s) {
  int tl = team_lanes(tab.bucket);
  // small buckets (S <= 64): narrower teams -- more buckets per warp iteration share the
  // per-bucket work (job lookup, scales) and each lane keeps several groups' loads in flight
  if (tl == 16) tl = ACC ? 8 : 4;
  if constexpr (ACC) {  // per-source scale rows are filled by lanes 0..nsrc-1: teams of >= 8 lanes
    if (tl <= 8) return launch_d_tl<BITS, 8, OUT, ACC>(tab, vec, sms, s);
    if (tl == 16) return launch_d_tl<BITS, 16, OUT, ACC>(tab, vec, sms, s);
    return launch_d_tl<BITS, 32, OUT, ACC>(tab, vec, sms, s);
  } else {
    switch (tl) {
      case 1: return launch_d_tl<BITS, 1, OUT, ACC>(tab, vec, sms, s);
      case 2: return launch_d_tl<BITS, 2, OUT, ACC>(tab, vec, sms, s);
      case 4: return launch_d_tl<BITS, 4, OUT, ACC>(tab, vec, sms, s);
      case 8: return launch_d_tl<BITS, 8, OUT, ACC>(tab, vec, sms, s);
      case 16: return launch_d_tl<BITS, 16, OUT, ACC>(tab, vec, sms, s);
      default: return launch_d_tl<BITS, 32, OUT, ACC>(tab, vec, sms, s);
    }
  }
}

template <int OUT, bool ACC>
static cudaError_t launch_d_out(const DJobTable& tab, bool vec, int sms, cudaStream_t s) {
  switch (tab.bits) {
    case 8: return launch_d_bits<8, OUT, ACC>(tab, vec, sms, s);
    case 4: return launch_d_bits<4, OUT, ACC>(tab, vec, sms, s);
    default: return launch_d_bits<0, OUT, ACC>(tab, vec, sms, s);
  }
}

template <bool ACC>
static cudaError_t launch_d_acc(const DJobTable& tab, bool vec, int sms, cudaStream_t s) {
  switch (tab.out_dtype) {
    case 0: return launch_d_out<0, ACC>(tab, vec, sms, s);
    case 1: return launch_d_out<1, ACC>(tab, vec, sms, s);
    default: return launch_d_out<2, ACC>(tab, vec, sms, s);
  }
}

cudaError_t launch_dequant(const DJobTable& tab, bool vec, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  return tab.accumulate ? launch_d_acc<true>(tab, vec, sms, s) : launch_d_acc<false>(tab, vec, sms, s);
}
}  // namespace qsdp
