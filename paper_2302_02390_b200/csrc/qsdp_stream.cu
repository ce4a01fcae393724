// qsdp_stream.cu -- bucketed quantization with ONE shared generator consumed in bucket order:
// the reference's bucketed_quantize(v, bucket, bits, inner, rng) (quantize.py:289-313) as used by
// the theory side (UniformStochasticGradientQuantizer, optimizer.py:177-191).
//
// The shared numpy PCG64 stream is consumed sequentially: a non-degenerate bucket draws one
// uniform (shift, quantize.py:130-132) or n doubles (stochastic, quantize.py:316-321); a
// degenerate bucket draws nothing (quantize.py:256-264).  The host restates that prefix sum
// and hands the device every bucket's starting generator state (state, inc); here a warp
// takes a bucket, lane L starts at state_{L+1} (its first element's draw) and jumps 32 draws
// per element, the codes come from the exact __ddiv_rn chain (this is the theory-side path,
// not the FSDP hot path) into a uint32 scratch, packed LSB-first by the wire kernel.
#include <cuda_runtime.h>

#include "qsdp_kernels.cuh"

namespace qsdp {

cudaError_t launch_pack_codes(const uint32_t* codes, int64_t length, int bucket, int bits, uint8_t* out,
                              int64_t out_bytes, int sms, cudaStream_t s);

// (A_k, G_k) with state_k = A_k * state_0 + G_k * inc  (PCG advance by doubling).
__device__ __forceinline__ void pcg_advance_coeffs(uint64_t k, U128& A, U128& G) {
  U128 am{1, 0}, ap{0, 0}, cm = pcg_mult(), cp{1, 0};
  const U128 one{1, 0};
  while (k) {
    if (k & 1ull) {
      am = mul128(am, cm);
      ap = add128(mul128(ap, cm), cp);
    }
    cp = mul128(add128(cm, one), cp);
    cm = mul128(cm, cm);
    k >>= 1;
  }
  A = am;
  G = ap;
}

template <typename T, int INNER>
__global__ void __launch_bounds__(256) quantize_stream_kernel(const T* __restrict__ x, int64_t length, int S, int bits,
                                                              const ulonglong4* __restrict__ states,
                                                              uint32_t* __restrict__ codes32, float* __restrict__ meta) {
  using Tr = InTraits<T>;
  using K = typename Tr::Key;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nb = (length + S - 1) / S;
  const double top = (double)((1u << bits) - 1u);
  const double pitch = __ddiv_rn(1.0, top);
  U128 A32, G32;
  pcg_advance_coeffs(32, A32, G32);
  for (int64_t b = warp; b < nb; b += nwarps) {
    const int64_t off = b * S;
    const int n = (int)min((int64_t)S, length - off);
    const T* v = x + off;
    K mnk = Tr::kMax, mxk = Tr::kMin;
    for (int e = lane; e < n; e += 32) {
      const K k = Tr::key(v[e]);
      mnk = min(mnk, k);
      mxk = max(mxk, k);
    }
    mnk = team_min_k<32>(mnk);
    mxk = team_max_k<32>(mxk);
    const float lof = (float)Tr::to_d(Tr::from_key(mnk)), hif = (float)Tr::to_d(Tr::from_key(mxk));
    const bool degenerate = !(lof < hif);  // the host has raised on non-finite input
    float shift_f = 0.0f;
    if (degenerate) {
      for (int e = lane; e < n; e += 32) codes32[off + e] = 0u;
    } else {
      const ulonglong4 w = states[b];
      const U128 s0{w.x, w.y}, inc{w.z, w.w};
      const double lo = (double)lof, span = __dsub_rn((double)hif, lo);
      if (INNER == 0) {  // sample_shift: one draw, rng.uniform(-p/2, p/2) unfused
        const double d = u64_to_unit_double(pcg_output(pcg_step(s0, inc)));
        const double r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
        shift_f = __double2float_rn(__dmul_rn(r, span));
        for (int e = lane; e < n; e += 32)
          codes32[off + e] = exact_shift_code(__dsub_rn(Tr::to_d(v[e]), lo), span, r, pitch, top);
      } else {  // element e draws the (e+1)-th output of the bucket's stream
        U128 A, G;
        pcg_advance_coeffs((uint64_t)lane + 1u, A, G);
        U128 st = add128(mul128(A, s0), mul128(G, inc));
        const U128 c32 = mul128(G32, inc);
        for (int e = lane; e < n; e += 32) {
          codes32[off + e] = exact_stoch_code(__dsub_rn(Tr::to_d(v[e]), lo), span, top, st);
          st = add128(mul128(A32, st), c32);
        }
      }
    }
    if (lane == 0) {
      meta[3 * b + 0] = degenerate ? 0.0f : shift_f;
      meta[3 * b + 1] = lof;
      meta[3 * b + 2] = hif;
    }
  }
}

// quantize_with_levels(v, table, stochastic=True, rng) (quantize.py:400-422): v clipped to
// [q0, q_last]; low = clip(searchsorted(q, v, "right") - 1, 0, L-2); code = low + (d_i < frac)
// with frac = (v - q[low]) / (q[low+1] - q[low]) and d_i the i-th double of the shared numpy
// PCG64 stream (state0 = before the first draw).  A thread takes CH consecutive elements: one
// jump to its first draw, then one LCG step per element.
template <int CH>
__global__ void __launch_bounds__(256) levels_stochastic_kernel(const double* __restrict__ v, int64_t n,
                                                                const double* __restrict__ q, int nl, ulonglong4 s,
                                                                uint32_t* __restrict__ codes) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = t * CH;
  if (i0 >= n) return;
  const U128 s0{s.x, s.y}, inc{s.z, s.w};
  U128 A, G;
  pcg_advance_coeffs((uint64_t)i0, A, G);
  U128 st = add128(mul128(A, s0), mul128(G, inc));  // state before draw i0
  const double lo_q = q[0], hi_q = q[nl - 1];
  for (int64_t i = i0; i < n && i < i0 + CH; ++i) {
    st = pcg_step(st, inc);
    const double d = u64_to_unit_double(pcg_output(st));
    const double x = fmin(fmax(v[i], lo_q), hi_q);  // np.clip
    int a = 0, b = nl;  // searchsorted(q, x, "right"): first index with q[idx] > x
    while (a < b) {
      const int m = (a + b) >> 1;
      if (q[m] <= x) a = m + 1;
      else b = m;
    }
    int low = a - 1;
    low = low < 0 ? 0 : (low > nl - 2 ? nl - 2 : low);
    const double frac = __ddiv_rn(__dsub_rn(x, q[low]), __dsub_rn(q[low + 1], q[low]));
    codes[i] = (uint32_t)low + (d < frac ? 1u : 0u);
  }
}

cudaError_t launch_levels_stochastic(const double* v, int64_t n, const double* q, int nl, const uint64_t* state,
                                     uint32_t* codes, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  constexpr int CH = 16;
  const int64_t threads = (n + CH - 1) / CH;
  const ulonglong4 st = make_ulonglong4(state[0], state[1], state[2], state[3]);
  levels_stochastic_kernel<CH><<<(int)((threads + 255) / 256), 256, 0, s>>>(v, n, q, nl, st, codes);
  return cudaGetLastError();
}

cudaError_t launch_quantize_stream(const void* x, bool f64, int64_t length, int S, int bits, int inner,
                                   const uint64_t* states, uint32_t* scratch, uint8_t* codes, int64_t codes_bytes,
                                   float* meta, int sms, cudaStream_t s) {
  if (length <= 0) return cudaSuccess;
  const int64_t nb = (length + S - 1) / S;
  const int64_t blocks = (nb + 7) / 8;
  const int grid = (int)(blocks < 1 ? 1 : (blocks > (int64_t)sms * 8 ? (int64_t)sms * 8 : blocks));
  const auto* st = reinterpret_cast<const ulonglong4*>(states);
  if (f64) {
    if (inner) quantize_stream_kernel<double, 1><<<grid, 256, 0, s>>>((const double*)x, length, S, bits, st, scratch, meta);
    else quantize_stream_kernel<double, 0><<<grid, 256, 0, s>>>((const double*)x, length, S, bits, st, scratch, meta);
  } else {
    if (inner) quantize_stream_kernel<float, 1><<<grid, 256, 0, s>>>((const float*)x, length, S, bits, st, scratch, meta);
    else quantize_stream_kernel<float, 0><<<grid, 256, 0, s>>>((const float*)x, length, S, bits, st, scratch, meta);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_pack_codes(scratch, length, S, bits, codes, codes_bytes, sms, s);
}

}  // namespace qsdp
