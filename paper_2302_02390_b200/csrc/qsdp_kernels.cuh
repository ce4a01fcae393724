// qsdp_kernels.cuh -- K1/K2 (bucketed quantize), K3 (dequantize) and
// K4 (ordered dequantize-accumulate) for sm_100a.
//
// Reference semantics (pkg/src/qsdp, read-only):
//   K1  quantize_bucket(v, b, "shift", bucket_rng(...))          quantize.py:235-272
//   K2  quantize_bucket(v, b, "uniform_stochastic", ...)          quantize.py:273-274, 316-321
//   K3  dequantize(block)  = (lo + code*pitch) + shift            quantize.py:209-232
//   K4  acc = 0; acc = acc + vals_p (p = 0..P-1); acc / P         sharded.py:385-431
//   packing: LSB-first codes, each bucket padded to a byte         wire.py:78-95
//
// Layout in HBM (per segment): bucket j's packed codes at j*ceil(S*b/8),
// its metadata at meta[3j..3j+2] = {shift, lo, hi} (f32).
//
// Thread mapping: one "team" of TL lanes (TL = min(32, pow2ceil(S/4))) owns a
// bucket; lane t of the team owns element groups g*TL + t of 4 consecutive
// elements, so every warp-wide load is one fully coalesced 128-bit access per
// lane.  Min/max are team-reduced with xor shuffles; no shared memory.
//
// Exactness: the reference computes in IEEE binary64 (u = (v-lo)/(hi-lo),
// (u-r)/pitch, round-half-even; u*top, floor, d < frac).  Each element is first
// evaluated with a division-free fp64 fast path whose error is bounded
// (DESIGN.md "certified fast path"); the decision is accepted only when the
// bound proves it equals the correctly rounded chain, otherwise the element is
// recomputed with __ddiv_rn exactly.  No FMA contraction is possible: every
// operation on the parity path is an explicit _rn intrinsic.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "qsdp_device.cuh"

namespace qsdp {

// Each translation unit that instantiates quantize kernels owns a copy of the
// PCG64 jump table (no relocatable device code needed); see upload_jump_*.
static __device__ JumpEntry g_jump[kJumpTable];

// 1.5 * 2^20: adding it rounds to multiples of 2^-32, so the low mantissa bits
// hold round(w * 2^32) for |w| < 2^19 (32.32 fixed point, no F2I needed).
constexpr double kMagic32 = 1572864.0;
constexpr uint64_t kMantMask = (1ull << 52) - 1;
constexpr int64_t kMantBias = 1ll << 51;

__device__ __forceinline__ int64_t fixed32(double w) {
  const double y = __dadd_rn(w, kMagic32);
  return (int64_t)(__double_as_longlong(y) & kMantMask) - kMantBias;
}

__device__ __forceinline__ bool finite_f(float v) { return (__float_as_uint(v) & 0x7f800000u) != 0x7f800000u; }
__device__ __forceinline__ bool finite_d(double v) {
  return ((unsigned long long)__double_as_longlong(v) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}

// Min/max run on order-preserving integer keys of the IEEE bits (total order,
// -0.0 < +0.0): integer IMNMX instead of float compares, and a zero extremum
// keeps numpy's sign when the bucket's zero extremum has a single sign.
template <typename T>
struct InTraits;
template <>
struct InTraits<float> {
  using Key = int32_t;
  __device__ static __forceinline__ bool finite(float v) { return finite_f(v); }
  __device__ static __forceinline__ double to_d(float v) { return (double)v; }
  __device__ static __forceinline__ Key key(float v) {
    const int32_t b = __float_as_int(v);
    return b ^ ((b >> 31) & 0x7fffffff);
  }
  __device__ static __forceinline__ float from_key(Key k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }
  static constexpr Key kMax = 0x7fffffff, kMin = (int32_t)0x80000000;
};
template <>
struct InTraits<double> {
  using Key = long long;
  __device__ static __forceinline__ bool finite(double v) { return finite_d(v); }
  __device__ static __forceinline__ double to_d(double v) { return v; }
  __device__ static __forceinline__ Key key(double v) {
    const long long b = __double_as_longlong(v);
    return b ^ ((b >> 63) & 0x7fffffffffffffffll);
  }
  __device__ static __forceinline__ double from_key(Key k) {
    return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffll));
  }
  static constexpr Key kMax = 0x7fffffffffffffffll, kMin = (long long)0x8000000000000000ull;
};

// Streaming 128-bit loads (no L1 allocation) when the bucket stays in registers;
// cached loads when the bucket is re-read in a second pass.
template <bool STREAM>
__device__ __forceinline__ float4 ld4(const float* p) {
  float4 r;
  if (STREAM)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
  else
    r = __ldg(reinterpret_cast<const float4*>(p));
  return r;
}
template <bool STREAM>
__device__ __forceinline__ double2 ld2d(const double* p) {
  double2 r;
  if (STREAM)
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  else
    r = __ldg(reinterpret_cast<const double2*>(p));
  return r;
}

// Load elements [e, e+4) of a bucket holding n elements; masked lanes get 0.
template <typename T, bool VEC, bool STREAM>
__device__ __forceinline__ void load_group(const T* x, int e, int n, T v[4]) {
  if (VEC && e + 4 <= n) {
    if constexpr (sizeof(T) == 4) {
      float4 f = ld4<STREAM>(reinterpret_cast<const float*>(x) + e);
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
      double2 a = ld2d<STREAM>(reinterpret_cast<const double*>(x) + e);
      double2 b = ld2d<STREAM>(reinterpret_cast<const double*>(x) + e + 2);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (e + i < n) ? x[e + i] : T(0);
  }
}

// ---------------------------------------------------------------------------
// Exact (slow-path) element evaluation: the reference's fp64 chain, verbatim.
// ---------------------------------------------------------------------------
static __device__ __noinline__ uint32_t exact_shift_code(double a, double span, double r, double pitch, double top) {
  double u = __ddiv_rn(a, span);
  u = fmin(fmax(u, 0.0), 1.0);                    // np.clip(..., 0, 1)
  const double w = __ddiv_rn(__dsub_rn(u, r), pitch);
  long long k = __double2ll_rn(w);                // np.round: half to even
  k = k < 0 ? 0 : k;
  k = k > (long long)top ? (long long)top : k;    // np.clip(..., 0, top)
  return (uint32_t)k;
}

static __device__ __noinline__ uint32_t exact_stoch_code(double a, double span, double top, U128 st) {
  double u = __ddiv_rn(a, span);
  u = fmin(fmax(u, 0.0), 1.0);
  const double s = __dmul_rn(u, top);
  const double low = floor(s);
  const double frac = __dsub_rn(s, low);
  const double d = u64_to_unit_double(pcg_output(st));
  double c = low + (d < frac ? 1.0 : 0.0);
  c = fmin(fmax(c, 0.0), top);
  return (uint32_t)c;
}

template <int TL, typename K>
__device__ __forceinline__ K team_min_k(K v) {
#pragma unroll
  for (int o = TL / 2; o > 0; o >>= 1) v = min(v, (K)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int TL, typename K>
__device__ __forceinline__ K team_max_k(K v) {
#pragma unroll
  for (int o = TL / 2; o > 0; o >>= 1) v = max(v, (K)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int TL>
__device__ __forceinline__ int team_min_i(int v) {
#pragma unroll
  for (int o = TL / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ __forceinline__ bool direct_width(int bits) {
  return bits == 8 || bits == 4 || bits == 16 || bits == 2;
}

// Store the packed bits of element group gi (4 codes, LSB-first) of a bucket.
// `w` holds this lane's 4*bits bits; `other` the partner lane's (gi^1), used
// when a group of 4 codes does not fill whole bytes (8 codes = `bits` bytes).
// `pbytes` bounds the writes for the bucket's final partial group.
__device__ __forceinline__ void store_group(uint8_t* const* dst, int ndst, int64_t boff, int gi, uint64_t w,
                                            uint64_t other, int bits, int64_t pbytes, bool full) {
  if (direct_width(bits)) {
    const int nb = bits / 2;  // bytes per group of 4 codes
    const int64_t o = boff + (int64_t)gi * nb;
    if (full) {
      for (int d = 0; d < ndst; ++d) {
        uint8_t* p = dst[d] + o;
        if (bits == 8) *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
        else if (bits == 4) *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
        else if (bits == 16) *reinterpret_cast<unsigned long long*>(p) = w;
        else *p = (uint8_t)w;
      }
    } else {
      const int64_t lim = boff + pbytes;
      for (int d = 0; d < ndst; ++d)
        for (int k = 0; k < nb; ++k)
          if (o + k < lim) dst[d][o + k] = (uint8_t)(w >> (8 * k));
    }
    return;
  }
  if ((gi & 1) == 0) {
    const int sh = 4 * bits;  // < 64 for the widths routed here
    const uint64_t lo = w | (other << sh);
    const uint64_t hi = other >> (64 - sh);
    const int64_t o = boff + (int64_t)(gi >> 1) * bits;
    const int64_t lim = boff + pbytes;
    for (int d = 0; d < ndst; ++d)
      for (int k = 0; k < bits; ++k) {
        if (o + k >= lim) break;
        const uint64_t word = k < 8 ? lo : hi;
        dst[d][o + k] = (uint8_t)(word >> (8 * (k & 7)));
      }
  }
}

// ---------------------------------------------------------------------------
// K1/K2: batched bucket quantizer.
// INNER 0 = shift (weights), 1 = uniform_stochastic/flip (gradients).
// G = element groups per lane kept in registers (HOLD) or re-read (!HOLD).
// ---------------------------------------------------------------------------
// Per-element code: certified division-free fast path, exact fallback.
template <typename T, int INNER>
struct Coder {
  double lo, span, inv, pitch, top, r;
  U128 st, inc;

  __device__ __forceinline__ uint32_t code(T t) {
    const double a = __dsub_rn(InTraits<T>::to_d(t), lo);
    if (INNER == 0) {
      double u = __dmul_rn(a, inv);
      if constexpr (sizeof(T) == 8) u = fmin(fmax(u, 0.0), 1.0);
      const double wv = __dmul_rn(__dsub_rn(u, r), top);
      const int64_t q = fixed32(wv);
      const uint32_t fr = (uint32_t)q;
      if (fr - 0x7ffffffeu <= 3u) return exact_shift_code(a, span, r, pitch, top);  // |fr-2^31|<=2
      const int64_t k = (q >> 32) + (fr > 0x80000000u ? 1 : 0);
      return (uint32_t)(k < 0 ? 0 : (k > (int64_t)top ? (int64_t)top : k));
    } else {
      const bool at_hi = a >= span;
      const bool at_lo = a <= 0.0;
      const double u = at_hi ? 1.0 : (at_lo ? 0.0 : __dmul_rn(a, inv));
      const int64_t q = fixed32(__dmul_rn(u, top));
      const uint32_t fq = (uint32_t)q;
      const int64_t nfl = q >> 32;
      const uint32_t dh = pcg_output_hi32(st);
      uint32_t c;
      if (at_hi || at_lo) {
        c = (uint32_t)nfl;  // s is an exact integer, frac 0: d < 0 is false
      } else if (fq == 0u || fq - dh <= 1u) {
        c = exact_stoch_code(a, span, top, st);  // fq in {dh, dh+1} or floor uncertain
      } else {
        const int64_t cc = nfl + (fq > dh ? 1 : 0);
        c = (uint32_t)(cc > (int64_t)top ? (int64_t)top : cc);
      }
      return c;
    }
  }
};

template <typename T, int INNER, int TL, int G, bool HOLD, bool VEC>
__global__ void __launch_bounds__(256) quantize_kernel(const __grid_constant__ QJobTable tab) {
  constexpr int TEAMS = 32 / TL;
  const int lane = threadIdx.x & 31;
  const int lt = lane % TL;
  const int team = lane / TL;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket;
  const int bits = tab.bits;
  const bool pair = !direct_width(bits);
  const double top = (double)((1u << bits) - 1u);
  const int64_t pbs = payload_bytes(S, bits);
  const int groups = (S + 3) / 4;
  const int gl = (groups + TL - 1) / TL;  // groups per lane (<= G when HOLD)

  for (int64_t b0 = warp * TEAMS; b0 < tab.total_buckets; b0 += nwarps * TEAMS) {
    const int64_t b = b0 + team;
    const bool active = b < tab.total_buckets;
    const int j = active ? find_job_q(tab, b) : 0;
    const QJob& J = tab.jobs[j];
    const int64_t lb = active ? b - J.bucket_base : 0;
    const int64_t off = lb * S;
    const int n = active ? (int)min((int64_t)S, J.length - off) : 0;
    const T* x = reinterpret_cast<const T*>(J.x) + off;

    // ---- pass 1: load, finiteness, min/max (quantize.py:41-44, 251-252) ----
    using K = typename InTraits<T>::Key;
    T v[HOLD ? G : 1][4];
    K mnk = InTraits<T>::kMax, mxk = InTraits<T>::kMin;
    int bad = 0x7fffffff;
    auto scan = [&](const T t[4], int e) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (e + i < n) {
          if (InTraits<T>::finite(t[i])) {
            const K kk = InTraits<T>::key(t[i]);
            mnk = min(mnk, kk);
            mxk = max(mxk, kk);
          } else {
            bad = min(bad, e + i);
          }
        }
      }
    };
    if constexpr (HOLD) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int e = 4 * (g * TL + lt);
        if (g < gl && e < n) {
          load_group<T, VEC, true>(x, e, n, v[g]);
          scan(v[g], e);
        }
      }
    } else {
      for (int g = 0; g < gl; ++g) {
        const int e = 4 * (g * TL + lt);
        if (e < n) {
          T t[4];
          load_group<T, VEC, false>(x, e, n, t);
          scan(t, e);
        }
      }
    }
    mnk = team_min_k<TL>(mnk);
    mxk = team_max_k<TL>(mxk);
    bad = team_min_i<TL>(bad);

    // lo/hi = _f32(min/max)  (quantize.py:251-252)
    const float lof = (float)InTraits<T>::to_d(InTraits<T>::from_key(mnk));
    const float hif = (float)InTraits<T>::to_d(InTraits<T>::from_key(mxk));
    const bool nonfinite = bad != 0x7fffffff;
    const bool degenerate = nonfinite || !(lof < hif);  // quantize.py:254-264
    if (active && nonfinite && lt == 0 && tab.bad_index != nullptr)
      atomicMin(tab.bad_index, ((unsigned long long)j << 40) | (unsigned long long)(off + bad));

    Coder<T, INNER> cd;
    cd.lo = (double)lof;
    cd.span = __dsub_rn((double)hif, cd.lo);
    cd.inv = __drcp_rn(cd.span);
    cd.top = top;
    cd.pitch = __ddiv_rn(1.0, top);
    cd.r = 0.0;
    cd.st = U128{0, 0};
    cd.inc = U128{0, 0};
    U128 jmp_a{0, 0}, jmp_c{0, 0};
    float shift_f = 0.0f;
    if (active && !degenerate) {
      seed_bucket(J.seed, (uint64_t)(J.global_start + off), cd.st, cd.inc);
      if (INNER == 0) {
        // sample_shift(pitch): uniform(-p/2, p/2) = -p/2 + p*d, unfused (quantize.py:130-132)
        const U128 s1 = mad128(cd.st, pcg_mult(), cd.inc);
        const double d = u64_to_unit_double(pcg_output(s1));
        cd.r = __dadd_rn(__dmul_rn(cd.pitch, -0.5), __dmul_rn(cd.pitch, d));
        shift_f = __double2float_rn(__dmul_rn(cd.r, cd.span));  // _f32(r*(hi-lo))
      } else {
        // element e consumes draw e = out(state_{e+1}); lane starts at 4*lt, jumps 4*TL-3
        const JumpEntry e0 = g_jump[4 * lt + 1];
        cd.st = add128(mul128(e0.a, cd.st), mul128(e0.g, cd.inc));
        const JumpEntry ej = g_jump[4 * TL - 3];
        jmp_a = ej.a;
        jmp_c = mul128(ej.g, cd.inc);
      }
    }

    // ---- pass 2: codes + LSB-first packing --------------------------------
    auto emit = [&](const T t[4], int g) {
      const int gi = g * TL + lt;
      const int e = 4 * gi;
      uint64_t w = 0;
      if (!degenerate && e < n) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t c = cd.code(t[i]);
          if (INNER == 1 && i < 3) cd.st = mad128(cd.st, pcg_mult(), cd.inc);
          if (e + i >= n) c = 0;
          w |= (uint64_t)c << (i * bits);
        }
        if (INNER == 1) cd.st = add128(mul128(jmp_a, cd.st), jmp_c);
      }
      const uint64_t other = pair ? __shfl_xor_sync(0xffffffffu, w, 1) : 0ull;
      if (active && e < n) store_group(J.codes, J.ndst, lb * pbs, gi, w, other, bits, payload_bytes(n, bits), e + 4 <= n);
    };
    if constexpr (HOLD) {
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (g < gl) emit(v[g], g);
    } else {
      for (int g = 0; g < gl; ++g) {
        T t[4];
        const int e = 4 * (g * TL + lt);
        load_group<T, VEC, false>(x, e, n, t);
        emit(t, g);
      }
    }
    if (active && lt == 0) {
      const float sh = degenerate ? 0.0f : shift_f;
      const float l = nonfinite ? 0.0f : lof, h = nonfinite ? 0.0f : hif;
      for (int d = 0; d < J.ndst; ++d) {
        float* m = J.meta[d] + 3 * lb;
        m[0] = sh;
        m[1] = l;
        m[2] = h;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Generic quantizer for bucket sizes that are not a multiple of 8: one thread
// per bucket, exact fp64 chain for every element, bit-serial packing.
// ---------------------------------------------------------------------------
template <typename T, int INNER>
__global__ void __launch_bounds__(128) quantize_generic_kernel(const __grid_constant__ QJobTable tab) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int S = tab.bucket, bits = tab.bits;
  const double top = (double)((1u << bits) - 1u);
  const int64_t pbs = payload_bytes(S, bits);
  for (int64_t b = tid; b < tab.total_buckets; b += nth) {
    const int j = find_job_q(tab, b);
    const QJob& J = tab.jobs[j];
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    const T* x = reinterpret_cast<const T*>(J.x) + off;
    using K = typename InTraits<T>::Key;
    K mnk = InTraits<T>::kMax, mxk = InTraits<T>::kMin;
    int bad = -1;
    for (int i = 0; i < n; ++i) {
      const T t = x[i];
      if (!InTraits<T>::finite(t)) { bad = i; break; }
      mnk = min(mnk, InTraits<T>::key(t));
      mxk = max(mxk, InTraits<T>::key(t));
    }
    const float lof = (float)InTraits<T>::to_d(InTraits<T>::from_key(mnk));
    const float hif = (float)InTraits<T>::to_d(InTraits<T>::from_key(mxk));
    const double lo = lof, hi = hif;
    const bool degenerate = bad >= 0 || !(lo < hi);
    if (bad >= 0 && tab.bad_index != nullptr)
      atomicMin(tab.bad_index, ((unsigned long long)j << 40) | (unsigned long long)(off + bad));
    const double span = __dsub_rn(hi, lo), pitch = __ddiv_rn(1.0, top);
    U128 st{0, 0}, inc{0, 0};
    double r = 0.0;
    float shift_f = 0.0f;
    if (!degenerate) {
      seed_bucket(J.seed, (uint64_t)(J.global_start + off), st, inc);
      if (INNER == 0) {
        st = mad128(st, pcg_mult(), inc);
        const double d = u64_to_unit_double(pcg_output(st));
        r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
        shift_f = __double2float_rn(__dmul_rn(r, span));
      }
    }
    uint64_t acc = 0;
    int nacc = 0;
    int64_t o = lb * pbs;
    for (int i = 0; i < n; ++i) {
      uint32_t code = 0;
      if (!degenerate) {
        const double a = __dsub_rn(InTraits<T>::to_d(x[i]), lo);
        if (INNER == 0) {
          code = exact_shift_code(a, span, r, pitch, top);
        } else {
          st = mad128(st, pcg_mult(), inc);
          code = exact_stoch_code(a, span, top, st);
        }
      }
      acc |= (uint64_t)code << nacc;
      nacc += bits;
      while (nacc >= 8) {
        for (int d = 0; d < J.ndst; ++d) J.codes[d][o] = (uint8_t)acc;
        ++o;
        acc >>= 8;
        nacc -= 8;
      }
    }
    if (nacc > 0)
      for (int d = 0; d < J.ndst; ++d) J.codes[d][o] = (uint8_t)acc;
    for (int d = 0; d < J.ndst; ++d) {
      float* m = J.meta[d] + 3 * lb;
      m[0] = degenerate ? 0.0f : shift_f;
      m[1] = bad >= 0 ? 0.0f : lof;
      m[2] = bad >= 0 ? 0.0f : hif;
    }
  }
}

// ---------------------------------------------------------------------------
// K3 / K4: dequantize (one source) or ordered dequantize-accumulate (P sources).
// ---------------------------------------------------------------------------
// Bits [4*bits*gi, 4*bits*(gi+1)) of a bucket payload of pbytes bytes.
__device__ __forceinline__ uint64_t load_group_bits(const uint8_t* p, int gi, int bits, int64_t pbytes, bool full) {
  if (full) {
    if (bits == 8) return *reinterpret_cast<const uint32_t*>(p + 4 * (int64_t)gi);
    if (bits == 4) return *reinterpret_cast<const uint16_t*>(p + 2 * (int64_t)gi);
    if (bits == 16) return *reinterpret_cast<const unsigned long long*>(p + 8 * (int64_t)gi);
    if (bits == 2) return p[gi];
  }
  const int64_t bitoff = (int64_t)gi * 4 * bits;
  const int64_t b0 = bitoff >> 3;
  const int sh = (int)(bitoff & 7);
  const int nbytes = (sh + 4 * bits + 7) >> 3;
  unsigned __int128 acc = 0;
  for (int k = 0; k < nbytes; ++k)
    if (b0 + k < pbytes) acc |= (unsigned __int128)p[b0 + k] << (8 * k);
  const uint64_t v = (uint64_t)(acc >> sh);
  return bits == 16 ? v : (v & ((1ull << (4 * bits)) - 1ull));
}

__device__ __forceinline__ double code_to_double(uint32_t c) {
  // exact: 2^52 + c reinterpreted, minus 2^52
  return __dsub_rn(__longlong_as_double(0x4330000000000000ll | (long long)c), 4503599627370496.0);
}

template <int OUT, bool VEC>
__device__ __forceinline__ void store_out4(void* out, int64_t idx, int n_left, const double acc[4]) {
  if (OUT == 0) {
    float* o = reinterpret_cast<float*>(out) + idx;
    const float4 f = make_float4(__double2float_rn(acc[0]), __double2float_rn(acc[1]), __double2float_rn(acc[2]),
                                 __double2float_rn(acc[3]));
    if (VEC && n_left >= 4) {
      *reinterpret_cast<float4*>(o) = f;
    } else {
      const float fv[4] = {f.x, f.y, f.z, f.w};
      for (int i = 0; i < 4 && i < n_left; ++i) o[i] = fv[i];
    }
  } else if (OUT == 1) {
    double* o = reinterpret_cast<double*>(out) + idx;
    if (VEC && n_left >= 4) {
      reinterpret_cast<double2*>(o)[0] = make_double2(acc[0], acc[1]);
      reinterpret_cast<double2*>(o)[1] = make_double2(acc[2], acc[3]);
    } else {
      for (int i = 0; i < 4 && i < n_left; ++i) o[i] = acc[i];
    }
  } else {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + idx;
    __nv_bfloat16 h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __float2bfloat16_rn(__double2float_rn(acc[i]));
    if (VEC && n_left >= 4) {
      uint2 u;
      u.x = (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16);
      u.y = (uint32_t)__bfloat16_as_ushort(h[2]) | ((uint32_t)__bfloat16_as_ushort(h[3]) << 16);
      *reinterpret_cast<uint2*>(o) = u;
    } else {
      for (int i = 0; i < 4 && i < n_left; ++i) o[i] = h[i];
    }
  }
}

// K3: one source per job.  K4 (ACC): nsrc sources summed in order in fp64
// starting from +0.0, then divided by `divisor` (acc = zeros; acc = acc + vals;
// acc / P -- sharded.py:385-431).  Per-source scales of the current bucket are
// staged in shared memory (one row per team) by lanes 0..nsrc-1.
template <int TL, int OUT, bool VEC, bool ACC>
__global__ void __launch_bounds__(256) dequant_kernel(const __grid_constant__ DJobTable tab) {
  constexpr int TEAMS = 32 / TL;
  __shared__ double sm_meta[ACC ? 8 : 1][ACC ? TEAMS : 1][8][3];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int lt = lane % TL;
  const int team = lane / TL;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket, bits = tab.bits;
  const double top = (double)((1u << bits) - 1u);
  const int64_t pbs = payload_bytes(S, bits);
  const int groups = (S + 3) / 4;
  const int gl = (groups + TL - 1) / TL;
  const uint64_t cmask = (1ull << bits) - 1ull;

  for (int64_t b0 = warp * TEAMS; b0 < tab.total_buckets; b0 += nwarps * TEAMS) {
    const int64_t b = b0 + team;
    const bool active = b < tab.total_buckets;
    const int j = active ? find_job_d(tab, b) : 0;
    const DJob& J = tab.jobs[j];
    const int64_t lb = active ? b - J.bucket_base : 0;
    const int64_t off = lb * S;
    const int n = active ? (int)min((int64_t)S, J.length - off) : 0;
    const int64_t pb = payload_bytes(n, bits);
    if constexpr (!ACC) {
      double lo = 0.0, shift = 0.0, pitch = 0.0;
      if (active) {
        const float* m = J.meta[0] + 3 * lb;
        shift = (double)m[0];
        lo = (double)m[1];
        pitch = __ddiv_rn(__dsub_rn((double)m[2], lo), top);  // QuantizedBlock.pitch
      }
      const uint8_t* cp = J.codes[0] + lb * pbs;
      for (int g = 0; g < gl; ++g) {
        const int gi = g * TL + lt;
        const int e = 4 * gi;
        if (e >= n) break;
        const bool full = e + 4 <= n;
        const uint64_t w = load_group_bits(cp, gi, bits, pb, full && tab.codes_vec);
        double v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double c = code_to_double((uint32_t)((w >> (i * bits)) & cmask));
          v[i] = __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift);  // (lo + code*pitch) + shift
        }
        store_out4<OUT, VEC>(J.out, off + e, n - e, v);
      }
    } else {
      const int nsrc = J.nsrc;
      double(*row)[3] = sm_meta[wib][team];
      if (active && lt < nsrc) {
        const float* m = J.meta[lt] + 3 * lb;
        const double lo = (double)m[1];
        row[lt][0] = lo;
        row[lt][1] = __ddiv_rn(__dsub_rn((double)m[2], lo), top);
        row[lt][2] = (double)m[0];
      }
      __syncwarp();
      for (int g = 0; g < gl; ++g) {
        const int gi = g * TL + lt;
        const int e = 4 * gi;
        if (e >= n) break;
        const bool full = e + 4 <= n;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int p = 0; p < nsrc; ++p) {
          const double lo = row[p][0], pitch = row[p][1], shift = row[p][2];
          const uint64_t w = load_group_bits(J.codes[p] + lb * pbs, gi, bits, pb, full && tab.codes_vec);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double c = code_to_double((uint32_t)((w >> (i * bits)) & cmask));
            acc[i] = __dadd_rn(acc[i], __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift));
          }
        }
        if (tab.divisor != 1) {
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = __ddiv_rn(acc[i], (double)tab.divisor);
        }
        store_out4<OUT, VEC>(J.out, off + e, n - e, acc);
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Host-side launch helpers (instantiated per translation unit).
// ---------------------------------------------------------------------------
inline int team_lanes(int S) {
  int groups = (S + 3) / 4;
  int tl = 1;
  while (tl < groups && tl < 32) tl <<= 1;
  return tl;
}

inline int grid_for(int64_t total_buckets, int teams_per_warp, int sms) {
  const int64_t warps = (total_buckets + teams_per_warp - 1) / teams_per_warp;
  const int64_t blocks = (warps + 7) / 8;
  const int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM at most
  return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

template <typename T, int INNER, int TL>
cudaError_t launch_q_tl(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  // TL < 32 only when the bucket has <= TL groups of 4: one group per lane.
  constexpr int G = TL == 32 ? 8 : 1;
  const int S = tab.bucket;
  const int gl = ((S + 3) / 4 + TL - 1) / TL;
  const int grid = grid_for(tab.total_buckets, 32 / TL, sms);
  if (TL < 32 || gl <= G) {
    if (vec) quantize_kernel<T, INNER, TL, G, true, true><<<grid, 256, 0, s>>>(tab);
    else quantize_kernel<T, INNER, TL, G, true, false><<<grid, 256, 0, s>>>(tab);
  } else if constexpr (TL == 32) {
    if (vec) quantize_kernel<T, INNER, TL, 1, false, true><<<grid, 256, 0, s>>>(tab);
    else quantize_kernel<T, INNER, TL, 1, false, false><<<grid, 256, 0, s>>>(tab);
  }
  return cudaGetLastError();
}

template <typename T, int INNER>
cudaError_t launch_q_t(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  const int S = tab.bucket;
  if (S % 8 != 0) {
    const int64_t blocks = (tab.total_buckets + 127) / 128;
    const int64_t cap = (int64_t)sms * 16;
    quantize_generic_kernel<T, INNER><<<(int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks)), 128, 0, s>>>(tab);
    return cudaGetLastError();
  }
  switch (team_lanes(S)) {
    case 2: return launch_q_tl<T, INNER, 2>(tab, vec, sms, s);
    case 4: return launch_q_tl<T, INNER, 4>(tab, vec, sms, s);
    case 8: return launch_q_tl<T, INNER, 8>(tab, vec, sms, s);
    case 16: return launch_q_tl<T, INNER, 16>(tab, vec, sms, s);
    default: return launch_q_tl<T, INNER, 32>(tab, vec, sms, s);
  }
}

}  // namespace qsdp
