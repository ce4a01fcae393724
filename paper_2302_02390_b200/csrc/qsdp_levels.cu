// Learned quantization levels on B200: the reference's
// inner="levels" mode and Alg. 2 level learning.
//
//   quantize_bucket(v, b, "levels", rng, levels)  quantize.py:235-286 with
//     quantize_with_levels(u, table, stochastic=False)  quantize.py:400-422:
//     u = clip((v-lo)/(hi-lo), 0, 1); mids = (q[:-1]+q[1:])/2;
//     code = searchsorted(mids, u, side="left")  (= #{mids < u}); shift = 0
//   dequantize(block, "levels", table)            quantize.py:225-231:
//     lo + q[code] * (hi - lo)
//   learn_levels(values, table, lr)               quantize.py:366-397:
//     for x in values: i = argmin|q - x|; q[i] -= lr*(q[i] - x)   (sequential)
//
// u is evaluated with the certified fast path (u' = (v-lo)*fl(1/span), |u' - u|
// < 4e-16); an element whose u' lies within that bound of a mid is recomputed
// with the exact division.  One warp per bucket; the mids of tables up to
// 2^12 levels live in shared memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "qsdp_kernels.cuh"

namespace qsdp {

constexpr int kSmemLevelBits = 12;  // mids of tables up to 2^12 levels are staged in smem

// mids[i] = (q[i] + q[i+1]) / 2, from smem when staged, else computed from the
// global table (2^13..2^16 levels).
struct Mids {
  const double* sm;
  const double* q;
  __device__ __forceinline__ double operator[](int i) const {
    return sm != nullptr ? sm[i] : __dmul_rn(__dadd_rn(__ldg(q + i), __ldg(q + i + 1)), 0.5);
  }
};

template <typename T>
__global__ void __launch_bounds__(256) quantize_levels_kernel(const __grid_constant__ QJobTable tab,
                                                              const double* __restrict__ levels, int nl) {
  extern __shared__ double smids[];
  const bool staged = nl <= (1 << kSmemLevelBits);
  if (staged)
    for (int i = threadIdx.x; i < nl - 1; i += blockDim.x)
      smids[i] = __dmul_rn(__dadd_rn(levels[i], levels[i + 1]), 0.5);  // (q[:-1] + q[1:]) / 2
  __syncthreads();
  const Mids mids{staged ? smids : nullptr, levels};
  const double q0 = levels[0], qL = levels[nl - 1];
  const int64_t poff = q_parity_off(tab);
  using Tr = InTraits<T>;
  using K = typename Tr::Key;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket;
  const int bits = tab.bits;
  const int64_t pbs = payload_bytes(S, bits);
  // code = #{mids < u}  (searchsorted side="left")
  auto search = [&](double u) -> uint32_t {
    int lo_i = 0, hi_i = nl - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (mids[mid] < u) lo_i = mid + 1;
      else hi_i = mid;
    }
    return (uint32_t)lo_i;
  };
  // clip(u, 0, 1) (quantize_bucket) then clip(u, q[0], q[-1]) (quantize_with_levels)
  auto clip2 = [&](double u) { return fmin(fmax(fmin(fmax(u, 0.0), 1.0), q0), qL); };
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const BucketRef br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const T* x = reinterpret_cast<const T*>(J.x) + br.off;
    K mnk = Tr::kMax, mxk = Tr::kMin;
    for (int i = lane; i < n; i += 32) {
      const K kk = Tr::key(x[i]);
      mnk = min(mnk, kk);
      mxk = max(mxk, kk);
    }
    mnk = team_min_k<32>(mnk);
    mxk = team_max_k<32>(mxk);
    const bool nonfinite = n > 0 && !(Tr::kNegInf < mnk && mxk < Tr::kPosInf);
    const float lof = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mnk));
    const float hif = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mxk));
    const bool degenerate = nonfinite || !(lof < hif);
    if (nonfinite && lane == 0 && tab.bad_index != nullptr) {
      const int i = first_nonfinite<T>(x, n);
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + i));
    }
    const double lo = (double)lof;
    const double span = __dsub_rn((double)hif, lo);
    const double inv = __drcp_rn(span);
    uint8_t* cbase = J.codes + poff + br.lb * pbs;
    // each lane packs 8-element groups (8 codes = `bits` whole bytes)
    for (int g = lane; 8 * g < n; g += 32) {
      unsigned __int128 w = 0;
      for (int i = 0; i < 8; ++i) {
        const int e = 8 * g + i;
        uint32_t c = 0;
        if (!degenerate && nl > 1 && e < n) {
          const double a = __dsub_rn(Tr::to_d(x[e]), lo);
          const double u1 = clip2(__dmul_rn(a, inv));
          c = search(u1);
          // |u' - u| < 4e-16 (both clipped): certified unless u' is that close to
          // mids[c-1] or mids[c]; then redo with the exact quotient
          const bool near_lo = c > 0 && fabs(u1 - mids[c - 1]) <= 4e-16;
          const bool near_hi = c < (uint32_t)(nl - 1) && fabs(mids[c] - u1) <= 4e-16;
          if (near_lo || near_hi) c = search(clip2(__ddiv_rn(a, span)));
        }
        w |= (unsigned __int128)c << (i * bits);
      }
      const int64_t o = (int64_t)g * bits;
      const int64_t lim = payload_bytes(n, bits);
      for (int k = 0; k < bits && o + k < lim; ++k) cbase[o + k] = (uint8_t)(w >> (8 * k));
    }
    if (lane == 0) {
      float* m = meta_at(J.meta, poff) + 3 * br.lb;
      m[0] = 0.0f;  // levels blocks carry no shift
      m[1] = lof;
      m[2] = hif;
    }
  }
}

__global__ void __launch_bounds__(256) dequant_levels_kernel(const __grid_constant__ DJobTable tab,
                                                             const double* __restrict__ levels) {
  extern __shared__ double sq[];
  const int nl = 1 << tab.bits;
  const bool staged = tab.bits <= kSmemLevelBits;
  if (staged)
    for (int i = threadIdx.x; i < nl; i += blockDim.x) sq[i] = levels[i];
  __syncthreads();
  const double* q = staged ? sq : levels;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket, bits = tab.bits;
  const uint32_t mask = (1u << bits) - 1u;
  const int64_t pbs = payload_bytes(S, bits);
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    const float* m = J.meta[0] + 3 * lb;
    const double lo = (double)m[1];
    const double span = __dsub_rn((double)m[2], lo);  // scale_hi - scale_lo
    const uint8_t* cp = J.codes[0] + lb * pbs;
    const int64_t lim = payload_bytes(n, bits);
    for (int e = lane; e < n; e += 32) {
      const int64_t bit = (int64_t)e * bits, by = bit >> 3;
      uint32_t w = 0;
      for (int k = 0; k < 3; ++k)
        if (by + k < lim) w |= (uint32_t)cp[by + k] << (8 * k);
      const uint32_t c = (w >> (bit & 7)) & mask;
      const double v = __dadd_rn(lo, __dmul_rn(q[c], span));  // lo + levels[codes] * span
      if (tab.out_dtype == 0) reinterpret_cast<float*>(J.out)[off + e] = __double2float_rn(v);
      else if (tab.out_dtype == 1) reinterpret_cast<double*>(J.out)[off + e] = v;
      else reinterpret_cast<__nv_bfloat16*>(J.out)[off + e] = __float2bfloat16_rn(__double2float_rn(v));
    }
  }
}

// learn_levels: one warp walks the values in order (the update is sequential);
// the nearest level is found with a warp argmin (first index on ties, np.argmin).
__global__ void learn_levels_kernel(const double* __restrict__ values, int64_t n, double* q, int nl, double lr) {
  extern __shared__ double sq[];
  const int lane = threadIdx.x;
  for (int i = lane; i < nl; i += 32) sq[i] = q[i];
  __syncwarp();
  for (int64_t t = 0; t < n; ++t) {
    const double x = values[t];
    double best = INFINITY;
    int bi = 0x7fffffff;
    for (int i = lane; i < nl; i += 32) {
      const double d = fabs(__dsub_rn(sq[i], x));
      if (d < best) { best = d; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) sq[bi] = __dsub_rn(sq[bi], __dmul_rn(lr, __dsub_rn(sq[bi], x)));  // q[i] -= lr*(q[i]-x)
    __syncwarp();
  }
  // np.any(diff <= 0) -> sort, then nudge exact collisions by max(ptp, 1)*1e-12
  // (indices of the collisions taken before any nudge, as the reference does)
  if (lane == 0) {
    bool broken = false;
    for (int i = 0; i + 1 < nl; ++i) broken |= !(__dsub_rn(sq[i + 1], sq[i]) > 0.0);
    if (broken) {
      for (int i = 1; i < nl; ++i) {  // insertion sort: rare path, <= 2^12 levels
        const double v = sq[i];
        int j = i - 1;
        while (j >= 0 && sq[j] > v) { sq[j + 1] = sq[j]; --j; }
        sq[j + 1] = v;
      }
      const double ptp = __dsub_rn(sq[nl - 1], sq[0]);
      const double eps = __dmul_rn(ptp > 1.0 ? ptp : 1.0, 1e-12);
      // dup = flatnonzero(diff(q) <= 0) is taken on the sorted table before any
      // nudge; q[j+1] = q[j] + eps then runs in order.  Keep the un-nudged value
      // of q[i] to evaluate the original diff at i.
      double orig_i = sq[0];
      for (int i = 0; i + 1 < nl; ++i) {
        const double orig_next = sq[i + 1];
        if (!(__dsub_rn(orig_next, orig_i) > 0.0)) sq[i + 1] = __dadd_rn(sq[i], eps);
        orig_i = orig_next;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < nl; i += 32) q[i] = sq[i];
}

cudaError_t launch_quantize_levels(const QJobTable& tab, int in_f64, const double* levels, int nl, int sms,
                                   cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  const int grid = grid_for(tab.total_buckets, 1, sms);
  const size_t sm = nl <= (1 << kSmemLevelBits) ? sizeof(double) * nl : 0;
  if (in_f64) quantize_levels_kernel<double><<<grid, 256, sm, s>>>(tab, levels, nl);
  else quantize_levels_kernel<float><<<grid, 256, sm, s>>>(tab, levels, nl);
  return cudaGetLastError();
}

cudaError_t launch_dequant_levels(const DJobTable& tab, const double* levels, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  const size_t sm = tab.bits <= kSmemLevelBits ? sizeof(double) << tab.bits : 0;
  dequant_levels_kernel<<<grid_for(tab.total_buckets, 1, sms), 256, sm, s>>>(tab, levels);
  return cudaGetLastError();
}

cudaError_t launch_learn_levels(const double* values, int64_t n, double* q, int nl, double lr, cudaStream_t s) {
  // nl <= 2^16 levels: 512 KB does not fit; tables beyond 2^13 levels are
  // rejected by the host (learning tables that wide is not a use the paper has)
  learn_levels_kernel<<<1, 32, sizeof(double) * nl, s>>>(values, n, q, nl, lr);
  return cudaGetLastError();
}

}  // namespace qsdp
