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
// elements, so every warp-wide access is fully coalesced.  Min/max are
// team-reduced with xor shuffles on order-preserving integer keys.
//
// Fast quantizer (quantize_tma_kernel, widths 2/4/8/16): every warp runs its
// own NST-stage pipeline -- one elected lane streams whole buckets into a
// shared-memory ring with cp.async.bulk (TMA bulk copies completing on an
// mbarrier) NST buckets ahead, so HBM reads overlap the code computation.
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
#include <cstdlib>

#include "qsdp_device.cuh"

namespace qsdp {

// Each translation unit that instantiates quantize kernels owns a copy of the
// PCG64 jump table (no relocatable device code needed); see upload_jump_*.
static __device__ JumpEntry g_jump[kJumpTable];

// 1.5 * 2^20: adding it rounds to multiples of 2^-32, so the low mantissa bits
// hold round(w * 2^32) for |w| < 2^19 (32.32 fixed point, no F2I needed).
constexpr double kMagic32 = 1572864.0;

struct Fixed32 {
  uint32_t frac;  // low 32 bits of round(w * 2^32)
  int32_t ip;     // floor of the rounded value (integer part), |ip| < 2^19
};
__device__ __forceinline__ Fixed32 fixed32(double w) {
  const double y = __dadd_rn(w, kMagic32);
  const uint32_t lo = (uint32_t)__double2loint(y);
  const uint32_t hi = (uint32_t)__double2hiint(y);
  // mantissa = 2^51 + round(w*2^32): integer part sits in hi bits [0, 20) offset by 2^19
  return Fixed32{lo, (int32_t)(hi & 0xFFFFFu) - (1 << 19)};
}

// Min/max run on order-preserving integer keys of the IEEE bits (total order,
// -0.0 < +0.0): integer IMNMX instead of float compares, and a zero extremum
// keeps numpy's sign when the bucket's zero extremum has a single sign.
// Non-finite values map outside [key(-inf), key(+inf)] exclusive bounds, so a
// bucket is finite iff key(-inf) < min_key and max_key < key(+inf).
template <typename T>
struct InTraits;
template <>
struct InTraits<float> {
  using Key = int32_t;
  __device__ static __forceinline__ double to_d(float v) { return (double)v; }
  __device__ static __forceinline__ bool finite(float v) {
    return (__float_as_uint(v) & 0x7f800000u) != 0x7f800000u;
  }
  __device__ static __forceinline__ Key key(float v) {
    const int32_t b = __float_as_int(v);
    return b ^ ((b >> 31) & 0x7fffffff);
  }
  __device__ static __forceinline__ float from_key(Key k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }
  static constexpr Key kMax = 0x7fffffff, kMin = (int32_t)0x80000000;
  static constexpr Key kPosInf = 0x7f800000, kNegInf = (int32_t)0x807fffff;
};
template <>
struct InTraits<double> {
  using Key = long long;
  __device__ static __forceinline__ double to_d(double v) { return v; }
  __device__ static __forceinline__ bool finite(double v) {
    return ((unsigned long long)__double_as_longlong(v) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
  }
  __device__ static __forceinline__ Key key(double v) {
    const long long b = __double_as_longlong(v);
    return b ^ ((b >> 63) & 0x7fffffffffffffffll);
  }
  __device__ static __forceinline__ double from_key(Key k) {
    return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffll));
  }
  static constexpr Key kMax = 0x7fffffffffffffffll, kMin = (long long)0x8000000000000000ull;
  static constexpr Key kPosInf = 0x7ff0000000000000ll, kNegInf = (long long)0x800fffffffffffffull;
};

// NaN-propagating 3-input min/max (FMNMX3.NAN) and warp reductions (CREDUX.*.F32.NAN), sm_100a.
// A NaN anywhere makes the result NaN, an infinity reaches the extremum, so the reduced pair alone
// says whether the bucket is finite.  The sign of a zero extremum is left to the key path.
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float d;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float warp_min_nan(float a) {
  float d;
  asm volatile("redux.sync.min.NaN.f32 %0, %1, 0xffffffff;" : "=f"(d) : "f"(a));
  return d;
}
__device__ __forceinline__ float warp_max_nan(float a) {
  float d;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(d) : "f"(a));
  return d;
}

// Streaming 128-bit loads (no L1 allocation) when a value is read once;
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

// 4 consecutive elements from shared memory (16-byte aligned group).
template <typename T>
__device__ __forceinline__ void lds_group(const T* s, int e, T v[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 f = *reinterpret_cast<const float4*>(s + e);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(s + e);
    const double2 b = *reinterpret_cast<const double2*>(s + e + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
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

static __device__ __noinline__ uint32_t exact_stoch_code_d(double a, double span, double top, uint64_t draw) {
  double u = __ddiv_rn(a, span);
  u = fmin(fmax(u, 0.0), 1.0);
  const double s = __dmul_rn(u, top);
  const double low = floor(s);
  const double frac = __dsub_rn(s, low);
  const double d = u64_to_unit_double(draw);
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
// Full-warp key reductions: redux.sync (one instruction) for 32-bit keys.
template <typename K>
__device__ __forceinline__ K warp_min_key(K v) {
  if constexpr (sizeof(K) == 4) return (K)__reduce_min_sync(0xffffffffu, (int)v);
  else return team_min_k<32>(v);
}
template <typename K>
__device__ __forceinline__ K warp_max_key(K v) {
  if constexpr (sizeof(K) == 4) return (K)__reduce_max_sync(0xffffffffu, (int)v);
  else return team_max_k<32>(v);
}

// Pack four codes of width BITS (LSB-first).
template <int BITS>
__device__ __forceinline__ uint64_t pack4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
  if constexpr (BITS == 8) {
    return __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
  } else {
    return (uint64_t)c0 | ((uint64_t)c1 << BITS) | ((uint64_t)c2 << (2 * BITS)) | ((uint64_t)c3 << (3 * BITS));
  }
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

// ---------------------------------------------------------------------------
// Per-bucket quantization context and the per-element certified fast path.
// ---------------------------------------------------------------------------
// NZ: the noise source -- 0 numpy PCG64 (bucket_rng, sequential stream with jumps),
// 1 numpy Philox4x64-10 (counter-based: st holds the key, a group's 4 draws are one block).
template <typename T, int INNER, int NZ = 0>
struct Coder {
  double lo, span, inv, pitch, top, r;
  U128 st, inc, jmp_a, jmp_c;

  // Bucket setup: scales, noise.  `lt` = lane in team, TL = team lanes.
  // noise: the table's qsdp_noise at run time -- Philox shift buckets (one draw) share the
  // PCG64 kernels; Philox stochastic buckets run the NZ == 1 instantiations.
  __device__ __forceinline__ void setup(float lof, float hif, int bits, const SeedPrefix& seed, uint64_t start,
                                        int lt, int TL, float& shift_f, int noise = 0) {
    top = (double)((1u << bits) - 1u);
    lo = (double)lof;
    span = __dsub_rn((double)hif, lo);
    inv = __drcp_rn(span);
    pitch = __ddiv_rn(1.0, top);
    r = 0.0;
    if (NZ == 1 || (INNER == 0 && noise == 1)) {
      philox_key(seed, start, st.lo, st.hi);
      if (INNER == 0) {  // sample_shift's single draw: word 0 of block 0
        const double d = u64_to_unit_double(philox_block(0, st.lo, st.hi).v[0]);
        r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
        shift_f = __double2float_rn(__dmul_rn(r, span));
      } else {
        shift_f = 0.0f;
      }
      return;
    }
    seed_bucket(seed, start, st, inc);
    if (INNER == 0) {
      // sample_shift(pitch): uniform(-p/2, p/2) = -p/2 + p*d, unfused (quantize.py:130-132)
      const U128 s1 = mad128(st, pcg_mult(), inc);
      const double d = u64_to_unit_double(pcg_output(s1));
      r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
      shift_f = __double2float_rn(__dmul_rn(r, span));  // _f32(r*(hi-lo))
    } else {
      // element e consumes draw e = out(state_{e+1}); lane starts at 4*lt, jumps 4*TL-3 per group
      const JumpEntry e0 = g_jump[4 * lt + 1];
      st = add128(mul128(e0.a, st), mul128(e0.g, inc));
      const JumpEntry ej = g_jump[4 * TL - 3];
      jmp_a = ej.a;
      jmp_c = mul128(ej.g, inc);
      shift_f = 0.0f;
    }
  }

  // Stochastic code of one element given its raw 64-bit draw (certified, exact fallback).
  __device__ __forceinline__ uint32_t code_draw(T t, uint64_t draw) {
    const double a = __dsub_rn(InTraits<T>::to_d(t), lo);
    const bool at_hi = a >= span;
    const bool at_lo = a <= 0.0;
    const double u = at_hi ? 1.0 : (at_lo ? 0.0 : __dmul_rn(a, inv));
    const Fixed32 q = fixed32(__dmul_rn(u, top));
    const uint32_t dh = (uint32_t)(draw >> 32);
    if (at_hi || at_lo) return (uint32_t)q.ip;
    if (q.frac - dh <= 1u) return exact_stoch_code_d(a, span, top, draw);
    const int c = q.ip + (q.frac > dh ? 1 : 0);
    return (uint32_t)min(c, (int)top);
  }

  // Code of one element; for INNER 1 uses the current state (caller steps it).
  __device__ __forceinline__ uint32_t code(T t) {
    const double a = __dsub_rn(InTraits<T>::to_d(t), lo);
    if (INNER == 0) {
      double u = __dmul_rn(a, inv);
      if constexpr (sizeof(T) == 8) u = fmin(fmax(u, 0.0), 1.0);
      const Fixed32 q = fixed32(__dmul_rn(__dsub_rn(u, r), top));
      // |w - w_fast| * 2^32 + rounding < 2: decided unless frac within 2 of 1/2
      if (q.frac - 0x7ffffffeu <= 3u) return exact_shift_code(a, span, r, pitch, top);
      const int k = q.ip + (q.frac > 0x80000000u ? 1 : 0);
      return (uint32_t)min(max(k, 0), (int)top);
    } else {
      const bool at_hi = a >= span;
      const bool at_lo = a <= 0.0;
      const double u = at_hi ? 1.0 : (at_lo ? 0.0 : __dmul_rn(a, inv));
      const Fixed32 q = fixed32(__dmul_rn(u, top));
      const uint32_t dh = pcg_output_hi32(st);
      if (at_hi || at_lo) return (uint32_t)q.ip;  // s exact integer, frac 0: d < 0 is false
      // uncertain iff (fq - dh) mod 2^32 <= 1 (covers fq == 0 too)
      if (q.frac - dh <= 1u) return exact_stoch_code(a, span, top, st);
      const int c = q.ip + (q.frac > dh ? 1 : 0);
      return (uint32_t)min(c, (int)top);
    }
  }

  // Bucket setup from a lane-parallel seed (seed_for): the same scales and noise as setup()
  // (PCG64 only) without every lane of the team re-running SeedSequence.
  template <typename SO>
  __device__ __forceinline__ void setup_seeded(float lof, float hif, int bits, const SO& sd, int lt, int TL,
                                               float& shift_f) {
    top = (double)((1u << bits) - 1u);
    lo = (double)lof;
    span = __dsub_rn((double)hif, lo);
    inv = __drcp_rn(span);
    pitch = __ddiv_rn(1.0, top);
    r = 0.0;
    if (INNER == 0) {
      r = sd.r;
      shift_f = __double2float_rn(__dmul_rn(r, span));  // _f32(r*(hi-lo))
      return;
    }
    inc = sd.inc;
    const JumpEntry e0 = g_jump[4 * lt + 1];
    st = add128(mul128(e0.a, sd.s0), mul128(e0.g, inc));
    const JumpEntry ej = g_jump[4 * TL - 3];
    jmp_a = ej.a;
    jmp_c = mul128(ej.g, inc);
    shift_f = 0.0f;
  }

  __device__ __forceinline__ void step() { st = pcg_step(st, inc); }
  __device__ __forceinline__ void jump() { st = add128(mul128(jmp_a, st), jmp_c); }

  // 4 codes of group starting at element e (elements >= n coded 0), packed LSB-first.
  __device__ __forceinline__ uint64_t group(const T v[4], int e, int n, int bits) {
    uint64_t w = 0;
    if constexpr (NZ == 1 && INNER == 1) {  // elements e..e+3 draw words 0..3 of block e / 4
      const Philox4 d = philox_block((uint64_t)(e >> 2), st.lo, st.hi);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t c = code_draw(v[i], d.v[i]);
        c = (e + i < n) ? c : 0u;
        w |= (uint64_t)c << (i * bits);
      }
      return w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t c = code(v[i]);
      if (INNER == 1 && i < 3) step();
      c = (e + i < n) ? c : 0u;
      w |= (uint64_t)c << (i * bits);
    }
    if (INNER == 1) jump();
    return w;
  }
};

// Store the packed bits (b/2 bytes) of group gi for the direct widths.
template <int BITS>
__device__ __forceinline__ void store_direct(uint8_t* base, int gi, uint64_t w, int64_t pbytes, bool full) {
  constexpr int NB = BITS / 2;
  uint8_t* p = base + (int64_t)gi * NB;
  if (full) {
    if (BITS == 8) *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
    else if (BITS == 4) *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
    else if (BITS == 16) *reinterpret_cast<unsigned long long*>(p) = w;
    else *p = (uint8_t)w;
  } else {
    const int64_t o = (int64_t)gi * NB;
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (o + k < pbytes) p[k] = (uint8_t)(w >> (8 * k));
  }
}

// First non-finite element of a bucket (rare path): team-serial scan.
template <typename T>
__device__ __noinline__ int first_nonfinite(const T* x, int n) {
  for (int i = 0; i < n; ++i)
    if (!InTraits<T>::finite(x[i])) return i;
  return n;
}

// ---------------------------------------------------------------------------
// mbarrier / TMA bulk-copy primitives (sm_90+ PTX, native on sm_100a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Resolve global bucket b of a job table.
struct BucketRef {
  int j;
  int n;
  int64_t lb, off;
};
__device__ __forceinline__ BucketRef resolve_q(const QJobTable& tab, int64_t b, int S) {
  BucketRef r;
  r.j = find_job_q(tab, b);
  const QJob& J = tab.jobs[r.j];
  r.lb = b - J.bucket_base;
  r.off = r.lb * S;
  r.n = (int)min((int64_t)S, J.length - r.off);
  return r;
}

struct SeedOut {
  U128 s0, inc;  // Philox stochastic (PH): s0 = the bucket's key (k0, k1)
  double r;
};

template <int INNER, int PH = 0>
__device__ __forceinline__ SeedOut seed_for(const QJobTable& tab, int64_t b, int S, double pitch) {
  SeedOut o;
  o.r = 0.0;
  o.s0 = U128{0, 0};
  o.inc = U128{0, 0};
  if (b < tab.total_buckets) {
    const BucketRef br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    if (INNER == 1 && PH) {  // numpy Philox keyed like bucket_rng (generate_state(2))
      philox_key(q_seed(tab, J), (uint64_t)(J.global_start + br.off), o.s0.lo, o.s0.hi);
      return o;
    }
    if (INNER == 0 && tab.noise == 1) {  // Philox: sample_shift's draw = word 0 of block 0
      uint64_t k0, k1;
      philox_key(q_seed(tab, J), (uint64_t)(J.global_start + br.off), k0, k1);
      const double d = u64_to_unit_double(philox_block(0, k0, k1).v[0]);
      o.r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
      return o;
    }
    seed_bucket(q_seed(tab, J), (uint64_t)(J.global_start + br.off), o.s0, o.inc);
    if (INNER == 0) {
      const U128 s1 = mad128(o.s0, pcg_mult(), o.inc);
      const double d = u64_to_unit_double(pcg_output(s1));
      o.r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));  // uniform(-p/2, p/2)
    }
  }
  return o;
}


// ---------------------------------------------------------------------------
// K1/K2 fast path: TMA-pipelined quantizer for the direct widths.
// Requirements (host-checked): BITS in {2,4,8,16}, S % 8 == 0, S*sizeof(T) <= 8 KB (16 KB for the TMA32 kernel).
// Dynamic smem: [warps][NST] stages of TEAMS*S elements, then [warps][NST] mbarriers.
// ---------------------------------------------------------------------------
template <typename T, int INNER, int BITS, int TL, int NST>
__global__ void __launch_bounds__(256) quantize_tma_kernel(const __grid_constant__ QJobTable tab, int vec) {
  const int64_t poff = q_parity_off(tab);
  constexpr int TEAMS = 32 / TL;
  extern __shared__ __align__(128) uint8_t smem[];
  const int S = tab.bucket;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int lt = lane % TL;
  const int team = lane / TL;
  const int64_t stage_elems = (int64_t)TEAMS * S;
  T* wbuf = reinterpret_cast<T*>(smem) + (int64_t)wib * NST * stage_elems;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)wpc * NST * stage_elems * sizeof(T)) + wib * NST;
  // seeds of the warp's next 32 buckets (32 / TEAMS iterations), one lane each: SeedSequence runs
  // once per bucket instead of once per team lane (a 64-element bucket is 16 lanes x 4 elements)
  SeedOut* seeds = reinterpret_cast<SeedOut*>(smem + (size_t)wpc * NST * stage_elems * sizeof(T) +
                                              (size_t)wpc * NST * sizeof(uint64_t)) + wib * 32;
  constexpr int ITS = 32 / TEAMS;  // iterations per seed batch
  const double seed_pitch = __ddiv_rn(1.0, (double)((1u << BITS) - 1u));
  const int64_t gw = (int64_t)blockIdx.x * wpc + wib;
  const int64_t nw = (int64_t)gridDim.x * wpc;
  const int64_t total = tab.total_buckets;
  const int64_t pbs = payload_bytes(S, BITS);
  const int gl = (S / 4 + TL - 1) / TL;
  using Tr = InTraits<T>;
  using K = typename Tr::Key;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], TEAMS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // Issue the bulk copy of iteration k into stage k % NST (team leaders).
  auto issue = [&](int64_t k) {
    const int64_t b = (gw + k * nw) * TEAMS + team;
    if (lt == 0) {
      uint64_t* bar = &bars[k % NST];
      uint32_t bytes = 0;
      const void* src = nullptr;
      if (b < total) {
        const BucketRef br = resolve_q(tab, b, S);
        if (vec && br.n == S) {
          bytes = (uint32_t)(S * sizeof(T));
          src = reinterpret_cast<const T*>(tab.jobs[br.j].x) + br.off;
        }
      }
      mbar_arrive_tx(bar, bytes);
      if (bytes) tma_load_1d(wbuf + (k % NST) * stage_elems + (int64_t)team * S, src, bytes, bar);
    }
  };

  for (int64_t k = 0; k < NST; ++k)
    if ((gw + k * nw) * TEAMS < total) issue(k);

  for (int64_t k = 0; (gw + k * nw) * TEAMS < total; ++k) {
    if (k % ITS == 0) {
      __syncwarp();
      seeds[lane] = seed_for<INNER>(tab, (gw + (k + lane / TEAMS) * nw) * TEAMS + lane % TEAMS, S, seed_pitch);
      __syncwarp();
    }
    const int stage = (int)(k % NST);
    mbar_wait(&bars[stage], (uint32_t)((k / NST) & 1));
    const T* sb = wbuf + stage * stage_elems + (int64_t)team * S;
    const int64_t b = (gw + k * nw) * TEAMS + team;
    const bool active = b < total;
    BucketRef br{0, 0, 0, 0};
    if (active) br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const bool in_smem = vec && n == S;
    const T* gx = reinterpret_cast<const T*>(J.x) + br.off;

    // ---- pass 1: min/max keys ------------------------------------------------
    K mnk = Tr::kMax, mxk = Tr::kMin;
    if (in_smem) {
      for (int g = 0; g < gl; ++g) {
        const int e = 4 * (g * TL + lt);
        if (e < n) {
          T v[4];
          lds_group(sb, e, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const K kk = Tr::key(v[i]);
            mnk = min(mnk, kk);
            mxk = max(mxk, kk);
          }
        }
      }
    } else {
      for (int g = 0; g < gl; ++g) {
        const int e = 4 * (g * TL + lt);
        if (e < n) {
          T v[4];
          load_group<T, false, false>(gx, e, n, v);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (e + i < n) {
              const K kk = Tr::key(v[i]);
              mnk = min(mnk, kk);
              mxk = max(mxk, kk);
            }
          }
        }
      }
    }
    mnk = team_min_k<TL>(mnk);
    mxk = team_max_k<TL>(mxk);
    const bool nonfinite = active && n > 0 && !(Tr::kNegInf < mnk && mxk < Tr::kPosInf);
    const float lof = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mnk));  // _f32(min)
    const float hif = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mxk));  // _f32(max)
    const bool degenerate = nonfinite || !(lof < hif);                        // quantize.py:254-264
    if (nonfinite && lt == 0 && tab.bad_index != nullptr) {
      const int i = first_nonfinite<T>(in_smem ? sb : gx, n);
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + i));
    }

    // ---- pass 2: codes ----------------------------------------------------------
    Coder<T, INNER> cd;
    float shift_f = 0.0f;
    if (active && !degenerate) cd.setup_seeded(lof, hif, BITS, seeds[(k % ITS) * TEAMS + team], lt, TL, shift_f);
    uint8_t* cbase = J.codes + poff + br.lb * pbs;
    const int64_t pb = payload_bytes(n, BITS);
    if (active && !degenerate && in_smem) {
      for (int g = 0; g < gl; ++g) {
        const int gi = g * TL + lt;
        const int e = 4 * gi;
        if (e < n) {
          T v[4];
          lds_group(sb, e, v);
          store_direct<BITS>(cbase, gi, cd.group(v, e, n, BITS), pb, true);
        }
      }
    } else if (active) {
      for (int g = 0; g < gl; ++g) {
        const int gi = g * TL + lt;
        const int e = 4 * gi;
        if (e < n) {
          uint64_t w = 0;
          if (!degenerate) {
            T v[4];
            load_group<T, false, false>(gx, e, n, v);
            w = cd.group(v, e, n, BITS);
          }
          store_direct<BITS>(cbase, gi, w, pb, e + 4 <= n);
        }
      }
    }
    if (active && lt == 0) {
      float* m = meta_at(J.meta, poff) + 3 * br.lb;
      m[0] = degenerate ? 0.0f : shift_f;
      m[1] = lof;
      m[2] = hif;
    }
    // release the stage to the async proxy, then refill it NST iterations ahead
    __syncwarp();
    fence_proxy_async();
    if ((gw + (k + NST) * nw) * TEAMS < total) issue(k + NST);
  }
}

// ---------------------------------------------------------------------------
// K1/K2 hot path for buckets of >= 128 elements (one warp per bucket).
// Same pipeline as quantize_tma_kernel, plus:
//  * per-bucket PCG64 seeding done lane-parallel, 32 future buckets at a time
//    (lane L seeds the warp's bucket k0+L), broadcast with shuffles;
//  * division-free certified codes with the fp64 chain folded into one DFMA:
//      shift:  y = (v-lo)*K1 + C,  K1 = fl(fl(1/span)*top),  C = fl(M+1/2 - fl(r*top))
//              -> code = clamp(floor(y - M), 0, top)  (the +1/2 makes floor == rint)
//      stoch:  y = (v-lo)*K1 + M  -> s in 32.32 fixed point: ip, fq
//              code = ip + (fq > d_hi)  with d_hi = top 32 bits of the draw
//    y's 32.32 fixed-point error is < 1.3 units of 2^-32, so a
//    code is certain unless (shift) |frac - 1/2| <= 2 units, or (stoch)
//    fq in {d_hi, d_hi+1} or fq == 0 off the bucket's extrema; those elements
//    are recomputed with the exact __ddiv_rn chain.
// ---------------------------------------------------------------------------
// COH: codes written by a peer in flight -- read at L2 (ld.global.cg), never
// through the non-coherent path.
template <int BITS, bool COH = false>
__device__ __forceinline__ uint64_t load_group_direct(const uint8_t* __restrict__ p, int gi) {
  if constexpr (COH) {
    if (BITS == 8) return __ldcg(reinterpret_cast<const unsigned int*>(p) + gi);
    if (BITS == 4) return __ldcg(reinterpret_cast<const unsigned short*>(p) + gi);
    if (BITS == 16) return __ldcg(reinterpret_cast<const unsigned long long*>(p) + gi);
    return __ldcg(reinterpret_cast<const unsigned char*>(p) + gi);
  } else {
    if (BITS == 8) return __ldg(reinterpret_cast<const uint32_t*>(p) + gi);
    if (BITS == 4) return __ldg(reinterpret_cast<const uint16_t*>(p) + gi);
    if (BITS == 16) return __ldg(reinterpret_cast<const unsigned long long*>(p) + gi);
    return __ldg(p + gi);
  }
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

// Fused dequant (the collective's own shard; world 1: the whole collective):
// the quantizer dequantizes its codes while they are in registers, exactly as
// K3 (or K4 with one source) would: v = (lo + code*pitch) + shift in fp64
// (quantize.py:209-232), K4: 0.0 + v (sharded.py:385-431, divisor 1).  The
// dequant launch and the code read-back from HBM disappear.
struct FusedDq {
  void* out;  // element 0 of the bucket, or nullptr
  double lo, pitch, shift;
  int dtype, add0;
};
// FDQ variants: 0 none; 1 fp32 out; 2 fp32 out with K4's 0.0 + v; 3 dtype / add0 read at run time.
template <int BITS, int FDQ>
__device__ __forceinline__ void dq_emit4(const FusedDq& f, int e, int n_left, uint64_t w) {
  double v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double c = code_to_double((uint32_t)((w >> (i * BITS)) & ((1ull << BITS) - 1ull)));
    v[i] = __dadd_rn(__dadd_rn(f.lo, __dmul_rn(c, f.pitch)), f.shift);
    if (FDQ == 2 || (FDQ == 3 && f.add0)) v[i] = __dadd_rn(0.0, v[i]);
  }
  if (FDQ == 1 || FDQ == 2 || f.dtype == 0) store_out4<0, true>(f.out, e, n_left, v);
  else if (f.dtype == 1) store_out4<1, true>(f.out, e, n_left, v);
  else store_out4<2, true>(f.out, e, n_left, v);
}
// The fused epilogue's per-bucket table (BITS <= 8, fp32 / bf16 output): entry c is code c's
// output value from dq_emit4's exact chain -- (lo + c*pitch) + shift in fp64, K4's 0.0 + v,
// one rounding to the output dtype -- so a lookup replaces the fp64 chain per element
// (2^BITS evaluations per bucket instead of S).  Warp-collective.
// Only the stochastic quantizer (issue-bound) takes it: the HBM-bound shift quantizer measured
// slower with the table's shared memory and registers (fused AG 0.53 -> 0.50 of peak).
__host__ __device__ constexpr bool dq_table_on(int INNER, int BITS, int FDQ) { return INNER == 1 && FDQ != 0 && BITS <= 8; }
template <int BITS, int FDQ>
__device__ __forceinline__ void dq_table_build(const FusedDq& f, uint32_t* tbl, int lane) {
  __syncwarp();  // the previous bucket's lookups are done
  for (int c = lane; c < (1 << BITS); c += 32) {
    double v = __dadd_rn(__dadd_rn(f.lo, __dmul_rn(code_to_double((uint32_t)c), f.pitch)), f.shift);
    if (FDQ == 2 || (FDQ == 3 && f.add0)) v = __dadd_rn(0.0, v);
    const float x = __double2float_rn(v);
    tbl[c] = (FDQ == 3 && f.dtype == 2) ? (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x)) : __float_as_uint(x);
  }
  __syncwarp();
}
// four full, aligned elements from the table (f.dtype 0 or 2; f64 output keeps dq_emit4)
template <int BITS, int FDQ>
__device__ __forceinline__ void dq_emit4_tab(const FusedDq& f, const uint32_t* tbl, int e, uint64_t w) {
  constexpr uint32_t M = (1u << BITS) - 1u;
  const uint32_t a = tbl[(uint32_t)w & M], b = tbl[(uint32_t)(w >> BITS) & M];
  const uint32_t c = tbl[(uint32_t)(w >> (2 * BITS)) & M], d = tbl[(uint32_t)(w >> (3 * BITS)) & M];
  if (FDQ == 3 && f.dtype == 2)
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(f.out) + e) = make_uint2(a | (b << 16), c | (d << 16));
  else
    *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(f.out) + e) = make_uint4(a, b, c, d);
}

template <int FDQ>
__device__ __forceinline__ FusedDq fused_dq(const QJobTable& tab, const QJob& J, int64_t off, float lof, float hif,
                                            float shift_f, int bits) {
  FusedDq f;
  f.out = nullptr;
  f.lo = f.pitch = f.shift = 0.0;
  f.dtype = tab.dq_dtype;
  f.add0 = tab.dq_add0;
  if (FDQ && J.dq_out != nullptr) {
    f.out = static_cast<uint8_t*>(J.dq_out) + off * (tab.dq_dtype == 1 ? 8 : tab.dq_dtype == 2 ? 2 : 4);
    f.lo = (double)lof;
    f.pitch = __ddiv_rn(__dsub_rn((double)hif, f.lo), (double)((1u << bits) - 1u));  // QuantizedBlock.pitch
    f.shift = (double)shift_f;
  }
  return f;
}

// Partial / unaligned / degenerate bucket (one per segment at most on the hot
// path): per-lane seeding and the Coder path; out of line to keep the fast
// loop's register budget.  Returns the bucket's f32 shift.
template <typename T, int INNER, int BITS, int FDQ = 0, int PH = 0>
static __device__ __forceinline__ float quantize_bucket_general(const SeedPrefix& seed, uint64_t start, const T* x, int n,
                                                             int gl, uint8_t* cbase, float lof, float hif,
                                                             bool degenerate, int lane, const QJobTable& tab,
                                                             const QJob& J, int64_t off) {
  Coder<T, INNER, PH> cd;
  float shift_f = 0.0f;
  if (!degenerate) cd.setup(lof, hif, BITS, seed, start, lane, 32, shift_f, tab.noise);
  const FusedDq fq = fused_dq<FDQ>(tab, J, off, lof, hif, degenerate ? 0.0f : shift_f, BITS);
  const int64_t pb = payload_bytes(n, BITS);
  for (int g = 0; g < gl; ++g) {
    const int gi = g * 32 + lane;
    const int e = 4 * gi;
    if (e < n) {
      uint64_t w = 0;
      if (!degenerate) {
        T v[4];
        load_group<T, false, false>(x, e, n, v);
        w = cd.group(v, e, n, BITS);
      }
      if (!FDQ || !tab.dq_nocodes) store_direct<BITS>(cbase, gi, w, pb, e + 4 <= n);
      if (fq.out != nullptr) dq_emit4<BITS, FDQ>(fq, e, n - e, w);
    }
  }
  return shift_f;
}

constexpr double kMagic = 1572864.0;  // 1.5 * 2^20

// Store the 8 packed codes of octet o (8*BITS bits = BITS bytes, aligned).
template <int BITS>
__device__ __forceinline__ void store_octet(uint8_t* base, int o, uint64_t w) {
  if (BITS == 8) reinterpret_cast<unsigned long long*>(base)[o] = w;
  else if (BITS == 4) reinterpret_cast<uint32_t*>(base)[o] = (uint32_t)w;
  else if (BITS == 2) reinterpret_cast<uint16_t*>(base)[o] = (uint16_t)w;
  else base[o] = (uint8_t)w;  // BITS == 16 never takes the octet path (64-bit word holds 4 codes)
}

// Push collectives: after the warp has written bucket codes (cb, nbytes) and its
// meta (m), copy both to the same offsets in every peer workspace
// (address + tab.mirror_delta[k], NVLink stores).  __syncwarp() has ordered the
// warp's own stores; the re-read comes from L2 (ld.cg), 16 bytes per lane.
__device__ __forceinline__ void mirror_bucket(const QJobTable& tab, uint8_t* cb, int64_t nbytes, float* m, int lane) {
  const int64_t head = ((uintptr_t)cb & 15) ? 0 : (nbytes >> 4);
  for (int64_t i = lane; i < head; i += 32) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(cb) + i);
    for (int k = 0; k < tab.mirror_n; ++k) reinterpret_cast<uint4*>(cb + tab.mirror_delta[k])[i] = v;
  }
  for (int64_t i = (head << 4) + lane; i < nbytes; i += 32) {
    const uint8_t v = __ldcg(cb + i);
    for (int k = 0; k < tab.mirror_n; ++k) cb[tab.mirror_delta[k] + i] = v;
  }
  if (lane < 3) {
    const float v = __ldcg(m + lane);
    for (int k = 0; k < tab.mirror_n; ++k) meta_at(m, tab.mirror_delta[k])[lane] = v;
  }
}

// Rare path of the octet loop: recompute the 8 codes, certifying each element
// again and falling back to the exact chain where the bound is not met.
template <typename T, int BITS>
static __device__ __noinline__ uint64_t stoch_octet_exact(const T* v, U128 st, U128 inc, double lo, double span,
                                                          double K1, double top) {
  using Tr = InTraits<T>;
  uint64_t w = 0;
  for (int i = 0; i < 8; ++i) {
    double a = __dsub_rn(Tr::to_d(v[i]), lo);
    if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);
    const double y = __fma_rn(a, K1, kMagic);
    const uint32_t fq = (uint32_t)__double2loint(y);
    const uint32_t ip = (uint32_t)__double2hiint(y) & 0x7FFFFu;
    const uint32_t dh = pcg_output_hi32(st);
    uint32_t c = ip + (fq > dh ? 1u : 0u);
    if ((fq - dh) <= 1u) c = exact_stoch_code(__dsub_rn(Tr::to_d(v[i]), lo), span, top, st);
    w |= (uint64_t)c << (i * BITS);
    st = pcg_step(st, inc);
  }
  return w;
}

// Rare path of the Philox octet loop: the 8 codes again, each element certified, the exact
// chain on the draw where the bound is not met.
template <typename T, int BITS>
static __device__ __noinline__ uint64_t philox_octet_exact(const T* v, Philox4 b0, Philox4 b1, double lo, double span,
                                                           double K1, double top) {
  using Tr = InTraits<T>;
  uint64_t w = 0;
  for (int i = 0; i < 8; ++i) {
    const uint64_t draw = i < 4 ? b0.v[i] : b1.v[i - 4];
    double a = __dsub_rn(Tr::to_d(v[i]), lo);
    if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);
    const double y = __fma_rn(a, K1, kMagic);
    const uint32_t fq = (uint32_t)__double2loint(y);
    const uint32_t ip = (uint32_t)__double2hiint(y) & 0x7FFFFu;
    const uint32_t dh = (uint32_t)(draw >> 32);
    uint32_t c = ip + (fq > dh ? 1u : 0u);
    if ((fq - dh) <= 1u) c = exact_stoch_code_d(__dsub_rn(Tr::to_d(v[i]), lo), span, top, draw);
    w |= (uint64_t)c << (i * BITS);
  }
  return w;
}

__device__ __forceinline__ U128 shfl_u128(const U128& v, int src) {
  U128 r;
  r.lo = __shfl_sync(0xffffffffu, v.lo, src);
  r.hi = __shfl_sync(0xffffffffu, v.hi, src);
  return r;
}

// Stateless job lookup for the TMA32 quantizer: one-job tables (every collective)
// resolve without a search, larger ones by binary search over the (param-space)
// bucket_base prefix.  Keeping no cursor state across buckets spares registers
// the per-bucket prologue would otherwise spill (ncu r2: LDL reloads of a cached
// cursor stalled ~9% of K2's samples on long scoreboard).
__device__ __forceinline__ BucketRef resolve_fast(const QJobTable& tab, int64_t b, int S) {
  int j = 0;
  if (tab.njobs > 1) {
    int lo = 0, hi = tab.njobs - 1;  // last job with bucket_base <= b
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tab.jobs[mid].bucket_base <= b) lo = mid;
      else hi = mid - 1;
    }
    j = lo;
  }
  BucketRef r;
  r.j = j;
  r.lb = b - tab.jobs[j].bucket_base;
  r.off = r.lb * S;
  r.n = (int)min((int64_t)S, tab.jobs[j].length - r.off);
  return r;
}

// PH (INNER 1 only): numpy Philox4x64-10 noise -- a lane's octet draws words 0..3 of blocks
// 2o and 2o+1 of the bucket's counter (no sequential stream, no jumps); octet buckets only
// (the launcher keeps other shapes on the team kernels).
template <typename T, int INNER, int BITS, int NST, int FDQ = 0, int PH = 0>
__device__ __forceinline__ void quantize_tma32_body(const QJobTable& tab, uint8_t* smem) {
  const int64_t poff = q_parity_off(tab);
  using Tr = InTraits<T>;
  using K = typename Tr::Key;
  constexpr uint32_t TOP = (1u << BITS) - 1u;
  const int S = tab.bucket;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  T* wbuf = reinterpret_cast<T*>(smem) + (int64_t)wib * NST * S;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)wpc * NST * S * sizeof(T)) + wib * NST;
  // lane-parallel seeds of the warp's next 32 buckets live in shared memory
  SeedOut* seeds = reinterpret_cast<SeedOut*>(smem + (size_t)wpc * NST * S * sizeof(T) +
                                              (size_t)wpc * NST * sizeof(uint64_t)) + wib * 32;
  // stochastic octet path: the per-lane jump A_{8 lane+1}, G_{8 lane+1} and the octet stride
  // A_{249}, G_{249}, copied once per CTA from the global table (a per-bucket LDG of them was
  // a long-scoreboard stall)
  JumpEntry* sjump = reinterpret_cast<JumpEntry*>(reinterpret_cast<uint8_t*>(seeds - wib * 32) +
                                                  (size_t)wpc * 32 * sizeof(SeedOut));
  // this warp's fused-dequant table (dq_table_on)
  uint32_t* dqt = reinterpret_cast<uint32_t*>(sjump + 33) + (size_t)wib * (1u << (BITS <= 8 ? BITS : 0));
  if (INNER == 1) {
    for (int t = threadIdx.x; t <= 32; t += blockDim.x) sjump[t] = g_jump[t < 32 ? 8 * t + 1 : 8 * 32 - 7];
    __syncthreads();
  }
  const int64_t gw = (int64_t)blockIdx.x * wpc + wib;
  const int64_t nw = (int64_t)gridDim.x * wpc;
  const int64_t total = tab.total_buckets;
  constexpr int PB8 = BITS;  // payload bytes per 8 elements: pbs = S * BITS / 8 (S % 8 == 0 here)
  const int gl = (S / 4 + 31) / 32;
  const double top = (double)TOP;
  const double pitch = __ddiv_rn(1.0, top);

  // per-lane jump constants: lane starts at element 4*lane, groups are 128 apart

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto bucket_of = [&](int64_t k) { return gw + k * nw; };
  auto issue = [&](int64_t k) {
    if (lane == 0) {
      const int64_t b = bucket_of(k);
      uint64_t* bar = &bars[k % NST];
      uint32_t bytes = 0;
      const T* src = nullptr;
      const BucketRef br = resolve_fast(tab, b, S);
      if (br.n == S) {
        src = reinterpret_cast<const T*>(tab.jobs[br.j].x) + br.off;
        if (((uintptr_t)src & 15u) == 0) bytes = (uint32_t)(S * sizeof(T));
      }
      mbar_arrive_tx(bar, bytes);
      if (bytes) tma_load_1d(wbuf + (k % NST) * S, src, bytes, bar);
    }
  };
  for (int64_t k = 0; k < NST; ++k)
    if (bucket_of(k) < total) issue(k);

  for (int64_t k = 0; bucket_of(k) < total; ++k) {
    if ((k & 31) == 0) {
      __syncwarp();
      seeds[lane] = seed_for<INNER, PH>(tab, bucket_of(k + lane), S, pitch);
      __syncwarp();
    }
    const int stage = (int)(k % NST);
    const int64_t b = bucket_of(k);
    const BucketRef br = resolve_fast(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const T* gx = reinterpret_cast<const T*>(J.x) + br.off;
    const bool in_smem = n == S && (((uintptr_t)gx & 15u) == 0);
    const T* sb = wbuf + stage * S;
    mbar_wait(&bars[stage], (uint32_t)((k / NST) & 1));

    // ---- pass 1: min/max keys (quantize.py:251-252) --------------------------
    K mnk = Tr::kMax, mxk = Tr::kMin;
    auto keys4 = [&](const T v[4]) {
      const K k0 = Tr::key(v[0]), k1 = Tr::key(v[1]), k2 = Tr::key(v[2]), k3 = Tr::key(v[3]);
      mnk = min(min(mnk, k0), min(k1, min(k2, k3)));
      mxk = max(max(mxk, k0), max(k1, max(k2, k3)));
    };
    if (in_smem && (S & 127) == 0) {
      const int gfull = S >> 7;
      bool keyed = true;
      if constexpr (sizeof(T) == 4) {
        // float min/max (1 FMNMX3 per 2 elements and bound), keys only for a zero extremum
        float mnf = __int_as_float(0x7f800000), mxf = __int_as_float(0xff800000);
#pragma unroll 4
        for (int g = 0; g < gfull; ++g) {
          T v[4];
          lds_group(sb, 4 * (g * 32 + lane), v);
          mnf = fmin3_nan(fmin3_nan(mnf, v[0], v[1]), v[2], v[3]);
          mxf = fmax3_nan(fmax3_nan(mxf, v[0], v[1]), v[2], v[3]);
        }
        mnf = warp_min_nan(mnf);
        mxf = warp_max_nan(mxf);
        keyed = mnf == 0.0f || mxf == 0.0f;  // -0 vs +0: total order on keys
        mnk = Tr::key(mnf);
        mxk = Tr::key(mxf);
        if (keyed) mnk = Tr::kMax, mxk = Tr::kMin;
      }
      if (keyed) {
#pragma unroll 4
        for (int g = 0; g < gfull; ++g) {
          T v[4];
          lds_group(sb, 4 * (g * 32 + lane), v);
          keys4(v);
        }
      }
    } else if (in_smem) {
      for (int g = 0; g < gl; ++g) {
        const int e = 4 * (g * 32 + lane);
        if (e < n) {
          T v[4];
          lds_group(sb, e, v);
          keys4(v);
        }
      }
    } else {
      for (int g = 0; g < gl; ++g) {
        const int e = 4 * (g * 32 + lane);
        if (e < n) {
          T v[4];
          load_group<T, false, false>(gx, e, n, v);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (e + i < n) {
              mnk = min(mnk, Tr::key(v[i]));
              mxk = max(mxk, Tr::key(v[i]));
            }
        }
      }
    }
    mnk = warp_min_key(mnk);
    mxk = warp_max_key(mxk);
    const bool nonfinite = n > 0 && !(Tr::kNegInf < mnk && mxk < Tr::kPosInf);
    const T mnv = Tr::from_key(mnk), mxv = Tr::from_key(mxk);
    const float lof = nonfinite ? 0.0f : (float)Tr::to_d(mnv);
    const float hif = nonfinite ? 0.0f : (float)Tr::to_d(mxv);
    const bool degenerate = nonfinite || !(lof < hif);  // quantize.py:254-264
    if (nonfinite && lane == 0 && tab.bad_index != nullptr) {
      const int i = first_nonfinite<T>(in_smem ? sb : gx, n);
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + i));
    }

    // ---- pass 2: codes --------------------------------------------------------
    const SeedOut& sd = seeds[k & 31];  // smem broadcast
    const double r = INNER == 0 ? sd.r : 0.0;
    const U128 s0 = INNER == 1 ? sd.s0 : U128{0, 0};
    const U128 inc = INNER == 1 ? sd.inc : U128{0, 0};
    uint8_t* cbase = J.codes + poff + br.lb * (int64_t)(S / 8 * PB8);
    const double lo = (double)lof;
    const double span = __dsub_rn((double)hif, lo);
    float shift_f = 0.0f;
    if (!degenerate && in_smem) {
      const double inv = __drcp_rn(span);
      const double K1 = __dmul_rn(inv, top);
      if (INNER == 0) {
        shift_f = __double2float_rn(__dmul_rn(r, span));  // _f32(r*(hi-lo))
        const FusedDq fq4 = fused_dq<FDQ>(tab, J, br.off, lof, hif, shift_f, BITS);
        const bool tab4 = dq_table_on(INNER, BITS, FDQ) && fq4.out != nullptr && fq4.dtype != 1;
        if (tab4) dq_table_build<BITS, FDQ>(fq4, dqt, lane);
        const double C = __dsub_rn(kMagic + 0.5, __dmul_rn(r, top));
        // A certified code lies in [0, top]: the low 19 integer bits are the code.
        auto code4 = [&](const T v[4], uint32_t c[4]) -> bool {
          bool unc = false;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            double a = __dsub_rn(Tr::to_d(v[i]), lo);
            if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);  // == np.clip of u
            const double y = __fma_rn(a, K1, C);
            const uint32_t fr = (uint32_t)__double2loint(y);
            unc |= (fr + 2u) <= 4u;  // |frac - 1/2| <= 2 units: not certified
            c[i] = (uint32_t)__double2hiint(y) & 0x7FFFFu;
          }
          return unc;
        };
        auto fix4 = [&](const T v[4], uint32_t c[4]) {
#pragma unroll
          for (int i = 0; i < 4; ++i) c[i] = exact_shift_code(__dsub_rn(Tr::to_d(v[i]), lo), span, r, pitch, top);
        };
        // fp32 certificate (float input, b <= 8, span in [2^-100, 2^100]):
        // t = fl(fl(fl(v-lo)*K1f + Cf) + 1536) with Cf = fl(1/2 - r*top + 2^-13) keeps 13 fraction
        // bits and |t - 1536 - 2^-13 - y| < 0.875 * 2^-13, so floor(t) - 1536 is the code unless t's
        // fraction is 0 or 1 units; those groups take the fp64 path above.
        const bool f32ok = sizeof(T) == 4 && BITS <= 8 && span >= 0x1p-100 && span <= 0x1p100;
        const float K1f = __double2float_rn(K1);
        const float Cf = __double2float_rn(__dadd_rn(__dsub_rn(0.5, __dmul_rn(r, top)), 0x1p-13));
        auto code4f = [&](const T v[4], uint32_t c[4]) -> bool {
          uint32_t m = 0xffffffffu;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float a = __fsub_rn((float)v[i], lof);
            const uint32_t b = __float_as_uint(__fadd_rn(__fmaf_rn(a, K1f, Cf), 1536.0f));
            m = min(m, b & 0x1ffeu);
            c[i] = BITS == 8 ? b >> 13 : (b >> 13) & TOP;  // pack4<8> takes the low byte
          }
          return m == 0u;
        };
        if ((S & 127) == 0 && f32ok) {  // every lane owns exactly S/128 full groups
          const int gfull = S >> 7;
#pragma unroll 2
          for (int g = 0; g < gfull; ++g) {
            const int gi = g * 32 + lane;
            T v[4];
            lds_group(sb, 4 * gi, v);
            uint32_t c[4];
            if (code4f(v, c) && code4(v, c)) fix4(v, c);  // rare: p ~ 2^-12 per element
            const uint64_t w = pack4<BITS>(c[0], c[1], c[2], c[3]);
            if (!FDQ || !tab.dq_nocodes) store_direct<BITS>(cbase, gi, w, 0, true);
            if (tab4) dq_emit4_tab<BITS, FDQ>(fq4, dqt, 4 * gi, w);
            else if (fq4.out != nullptr) dq_emit4<BITS, FDQ>(fq4, 4 * gi, 4, w);
          }
        } else if ((S & 127) == 0) {
          const int gfull = S >> 7;
#pragma unroll 2
          for (int g = 0; g < gfull; ++g) {
            const int gi = g * 32 + lane;
            T v[4];
            lds_group(sb, 4 * gi, v);
            uint32_t c[4];
            if (code4(v, c)) fix4(v, c);
            const uint64_t w = pack4<BITS>(c[0], c[1], c[2], c[3]);
            if (!FDQ || !tab.dq_nocodes) store_direct<BITS>(cbase, gi, w, 0, true);
            if (tab4) dq_emit4_tab<BITS, FDQ>(fq4, dqt, 4 * gi, w);
            else if (fq4.out != nullptr) dq_emit4<BITS, FDQ>(fq4, 4 * gi, 4, w);
          }
        } else {
          for (int g = 0; g < gl; ++g) {
            const int gi = g * 32 + lane;
            const int e = 4 * gi;
            if (e < n) {
              T v[4];
              lds_group(sb, e, v);
              uint32_t c[4];
              if (code4(v, c)) fix4(v, c);
              const uint64_t w = pack4<BITS>(c[0], c[1], c[2], c[3]);
              if (!FDQ || !tab.dq_nocodes) store_direct<BITS>(cbase, gi, w, 0, true);
              if (fq4.out != nullptr) dq_emit4<BITS, FDQ>(fq4, e, n - e, w);
            }
          }
        }
      } else if (BITS != 16 && (S & 255) == 0) {
        if constexpr (BITS != 16) {
        if constexpr (PH) {
          const int ol = S / 256;
          for (int g = 0; g < ol; ++g) {
            const int o = g * 32 + lane;
            T v[8];
            lds_group(sb, 8 * o, v);
            lds_group(sb, 8 * o + 4, v + 4);
            const Philox4 b0 = philox_block((uint64_t)(2 * o), s0.lo, s0.hi);
            const Philox4 b1 = philox_block((uint64_t)(2 * o + 1), s0.lo, s0.hi);
            uint64_t w = 0;
            bool unc = false;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              double a = __dsub_rn(Tr::to_d(v[i]), lo);
              if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);
              const double y = __fma_rn(a, K1, kMagic);
              const uint32_t fq = (uint32_t)__double2loint(y);
              const uint32_t ip = (uint32_t)__double2hiint(y) & 0x7FFFFu;
              const uint32_t dh = (uint32_t)((i < 4 ? b0.v[i] : b1.v[i - 4]) >> 32);
              unc |= (fq - dh) <= 1u;
              w |= (uint64_t)(ip + (fq > dh ? 1u : 0u)) << (i * BITS);
            }
            if (unc) w = philox_octet_exact<T, BITS>(sb + 8 * o, b0, b1, lo, span, K1, top);
            store_octet<BITS>(cbase, o, w);
          }
        } else {
        // octets: lane owns 8 consecutive elements 8*o (o = lane, lane+32, ...), so the
        // stream jumps once per 8 draws (by 256-7) instead of once per 4.
        // jump constants from the (L1-resident) table, per bucket: keeps registers for the loop
        const JumpEntry o0 = sjump[lane];
        U128 st = add128(mul128(o0.a, s0), mul128(o0.g, inc));  // state_{8*lane+1}
        const JumpEntry oj = sjump[32];
        const U128 OJa = oj.a;
        const U128 jc = mul128(oj.g, inc);
        const FusedDq fqs = fused_dq<FDQ>(tab, J, br.off, lof, hif, 0.0f, BITS);
        const bool tabs = dq_table_on(INNER, BITS, FDQ) && fqs.out != nullptr && fqs.dtype != 1;
        if (tabs) dq_table_build<BITS, FDQ>(fqs, dqt, lane);
        const int ol = S / 256;
        for (int g = 0; g < ol; ++g) {
          const int o = g * 32 + lane;
          T v[8];
          lds_group(sb, 8 * o, v);
          lds_group(sb, 8 * o + 4, v + 4);
          const U128 st0 = st;
          uint64_t w = 0;
          bool unc = false;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            double a = __dsub_rn(Tr::to_d(v[i]), lo);
            if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);
            const double y = __fma_rn(a, K1, kMagic);
            const uint32_t fq = (uint32_t)__double2loint(y);
            const uint32_t ip = (uint32_t)__double2hiint(y) & 0x7FFFFu;  // s >= 0: drop the 2^19 offset bit
            const uint32_t dh = pcg_output_hi32(st);
            unc |= (fq - dh) <= 1u;  // the only uncertain case
            w |= (uint64_t)(ip + (fq > dh ? 1u : 0u)) << (i * BITS);
            if (i < 7) st = FDQ == 0 ? add128_cc(mul128(st, pcg_mult()), inc) : pcg_step(st, inc);
          }
          if (unc) w = stoch_octet_exact<T, BITS>(sb + 8 * o, st0, inc, lo, span, K1, top);
          if (!FDQ || !tab.dq_nocodes) store_octet<BITS>(cbase, o, w);
          if (tabs) {
            dq_emit4_tab<BITS, FDQ>(fqs, dqt, 8 * o, w);
            dq_emit4_tab<BITS, FDQ>(fqs, dqt, 8 * o + 4, w >> (4 * BITS));
          } else if (fqs.out != nullptr) {
            dq_emit4<BITS, FDQ>(fqs, 8 * o, 4, w);
            dq_emit4<BITS, FDQ>(fqs, 8 * o + 4, 4, w >> (4 * BITS));
          }
          st = FDQ == 0 ? add128_cc(mul128(OJa, st), jc) : add128(mul128(OJa, st), jc);
        }
        }  // PCG64
        }
      } else if constexpr (!PH) {
        const JumpEntry e0 = g_jump[4 * lane + 1];
        U128 st = add128(mul128(e0.a, s0), mul128(e0.g, inc));  // state_{4*lane+1}
        const JumpEntry ej = g_jump[4 * 32 - 3];
        const U128 JA = ej.a;
        const U128 jc = mul128(ej.g, inc);
        const FusedDq fqq = fused_dq<FDQ>(tab, J, br.off, lof, hif, 0.0f, BITS);
#pragma unroll 2
        for (int g = 0; g < gl; ++g) {
          const int gi = g * 32 + lane;
          const int e = 4 * gi;
          if (e < n) {
            T v[4];
            lds_group(sb, e, v);
            uint64_t w = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              double a = __dsub_rn(Tr::to_d(v[i]), lo);
              if constexpr (sizeof(T) == 8) a = fmin(fmax(a, 0.0), span);
              const double y = __fma_rn(a, K1, kMagic);
              const uint32_t fq = (uint32_t)__double2loint(y);
              const uint32_t ip = (uint32_t)__double2hiint(y) & 0x7FFFFu;  // s >= 0: drop the 2^19 offset bit
              const uint32_t dh = pcg_output_hi32(st);
              uint32_t c = ip + (fq > dh ? 1u : 0u);
              const bool unc = (fq - dh) <= 1u;
              if (unc) c = exact_stoch_code(__dsub_rn(Tr::to_d(v[i]), lo), span, top, st);
              w |= (uint64_t)c << (i * BITS);
              if (i < 3) st = pcg_step(st, inc);
            }
            st = add128(mul128(JA, st), jc);
            if (!FDQ || !tab.dq_nocodes) store_direct<BITS>(cbase, gi, w, 0, true);
            if (fqq.out != nullptr) dq_emit4<BITS, FDQ>(fqq, e, n - e, w);
          }
        }
      }
    } else if (n > 0) {
      shift_f = quantize_bucket_general<T, INNER, BITS, FDQ, PH>(q_seed(tab, J), (uint64_t)(J.global_start + br.off), in_smem ? sb : gx,
                                                        n, gl, cbase, lof, hif, degenerate, lane, tab, J, br.off);
    }
    if (lane == 0) {
      float* m = meta_at(J.meta, poff) + 3 * br.lb;
      m[0] = degenerate ? 0.0f : shift_f;
      m[1] = lof;
      m[2] = hif;
    }
    __syncwarp();
    if (tab.mirror_n > 0) mirror_bucket(tab, cbase, payload_bytes(n, BITS), meta_at(J.meta, poff) + 3 * br.lb, lane);
    fence_proxy_async();
    if (bucket_of(k + NST) < total) issue(k + NST);
  }
}

template <typename T, int INNER, int BITS, int NST, int FDQ = 0, int PH = 0>
__global__ void __launch_bounds__(256, 2) quantize_tma32_kernel(const __grid_constant__ QJobTable tab) {
  extern __shared__ __align__(128) uint8_t smem[];
  quantize_tma32_body<T, INNER, BITS, NST, FDQ, PH>(tab, smem);
}

// ---------------------------------------------------------------------------
// K1/K2 for any width 1..16 (odd widths merge lane pairs into whole bytes),
// S % 8 == 0.  Registers hold up to G groups per lane (HOLD) or the bucket is
// re-read (second pass through L1/L2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store_pair(uint8_t* cbase, int gi, uint64_t w, uint64_t other, int bits,
                                           int64_t pbytes) {
  if (direct_width(bits)) {
    const int nb = bits / 2;
    const int64_t o = (int64_t)gi * nb;
    for (int k = 0; k < nb; ++k)
      if (o + k < pbytes) cbase[o + k] = (uint8_t)(w >> (8 * k));
    return;
  }
  if ((gi & 1) == 0) {
    const int sh = 4 * bits;  // < 64 for the widths routed here
    const uint64_t lo = w | (other << sh);
    const uint64_t hi = other >> (64 - sh);
    const int64_t o = (int64_t)(gi >> 1) * bits;
    for (int k = 0; k < bits; ++k) {
      if (o + k >= pbytes) break;
      const uint64_t word = k < 8 ? lo : hi;
      cbase[o + k] = (uint8_t)(word >> (8 * (k & 7)));
    }
  }
}

template <typename T, int INNER, int TL, int G, bool HOLD, bool VEC, int NZ = 0>
__global__ void __launch_bounds__(256) quantize_kernel(const __grid_constant__ QJobTable tab) {
  const int64_t poff = q_parity_off(tab);
  constexpr int TEAMS = 32 / TL;
  const int lane = threadIdx.x & 31;
  const int lt = lane % TL;
  const int team = lane / TL;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket;
  const int bits = tab.bits;
  const bool pair = !direct_width(bits);
  const int64_t pbs = payload_bytes(S, bits);
  const int groups = (S + 3) / 4;
  const int gl = (groups + TL - 1) / TL;
  using Tr = InTraits<T>;
  using K = typename Tr::Key;

  for (int64_t b0 = warp * TEAMS; b0 < tab.total_buckets; b0 += nwarps * TEAMS) {
    const int64_t b = b0 + team;
    const bool active = b < tab.total_buckets;
    BucketRef br{0, 0, 0, 0};
    if (active) br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const T* x = reinterpret_cast<const T*>(J.x) + br.off;

    T v[HOLD ? G : 1][4];
    K mnk = Tr::kMax, mxk = Tr::kMin;
    auto scan = [&](const T t[4], int e) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (e + i < n) {
          const K kk = Tr::key(t[i]);
          mnk = min(mnk, kk);
          mxk = max(mxk, kk);
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
    const bool nonfinite = active && n > 0 && !(Tr::kNegInf < mnk && mxk < Tr::kPosInf);
    const float lof = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mnk));
    const float hif = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mxk));
    const bool degenerate = nonfinite || !(lof < hif);
    if (nonfinite && lt == 0 && tab.bad_index != nullptr) {
      const int i = first_nonfinite<T>(x, n);
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + i));
    }

    Coder<T, INNER, NZ> cd;
    float shift_f = 0.0f;
    if (active && !degenerate)
      cd.setup(lof, hif, bits, q_seed(tab, J), (uint64_t)(J.global_start + br.off), lt, TL, shift_f, tab.noise);
    uint8_t* cbase = J.codes + poff + br.lb * pbs;
    const int64_t pb = payload_bytes(n, bits);
    auto emit = [&](const T t[4], int g) {
      const int gi = g * TL + lt;
      const int e = 4 * gi;
      uint64_t w = 0;
      if (!degenerate && e < n) w = cd.group(t, e, n, bits);
      const uint64_t other = pair ? __shfl_xor_sync(0xffffffffu, w, 1) : 0ull;
      if (active && e < n) {
        if (!pair && e + 4 <= n) {
          const int nb = bits / 2;
          uint8_t* p = cbase + (int64_t)gi * nb;
          if (bits == 8) *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
          else if (bits == 4) *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
          else if (bits == 16) *reinterpret_cast<unsigned long long*>(p) = w;
          else *p = (uint8_t)w;
        } else {
          store_pair(cbase, gi, w, other, bits, pb);
        }
      }
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
      float* m = meta_at(J.meta, poff) + 3 * br.lb;
      m[0] = degenerate ? 0.0f : shift_f;
      m[1] = lof;
      m[2] = hif;
    }
  }
}

// ---------------------------------------------------------------------------
// Generic quantizer for bucket sizes that are not a multiple of 8: one thread
// per bucket, exact fp64 chain for every element, bit-serial packing.
// ---------------------------------------------------------------------------
template <typename T, int INNER, int NZ = 0>
__global__ void __launch_bounds__(128) quantize_generic_kernel(const __grid_constant__ QJobTable tab) {
  const int64_t poff = q_parity_off(tab);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int S = tab.bucket, bits = tab.bits;
  const double top = (double)((1u << bits) - 1u);
  const int64_t pbs = payload_bytes(S, bits);
  using Tr = InTraits<T>;
  using K = typename Tr::Key;
  for (int64_t b = tid; b < tab.total_buckets; b += nth) {
    const BucketRef br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const T* x = reinterpret_cast<const T*>(J.x) + br.off;
    K mnk = Tr::kMax, mxk = Tr::kMin;
    int bad = -1;
    for (int i = 0; i < n; ++i) {
      const T t = x[i];
      if (!Tr::finite(t)) { bad = i; break; }
      mnk = min(mnk, Tr::key(t));
      mxk = max(mxk, Tr::key(t));
    }
    const float lof = bad >= 0 ? 0.0f : (float)Tr::to_d(Tr::from_key(mnk));
    const float hif = bad >= 0 ? 0.0f : (float)Tr::to_d(Tr::from_key(mxk));
    const bool degenerate = bad >= 0 || !(lof < hif);
    if (bad >= 0 && tab.bad_index != nullptr)
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + bad));
    const double lo = lof;
    const double span = __dsub_rn((double)hif, lo), pitch = __ddiv_rn(1.0, top);
    U128 st{0, 0}, inc{0, 0};
    double r = 0.0;
    float shift_f = 0.0f;
    if (!degenerate) {
      const bool ph = NZ == 1 || tab.noise == 1;
      if (ph) philox_key(q_seed(tab, J), (uint64_t)(J.global_start + br.off), st.lo, st.hi);
      else seed_bucket(q_seed(tab, J), (uint64_t)(J.global_start + br.off), st, inc);
      if (INNER == 0) {
        if (!ph) st = pcg_step(st, inc);
        const double d = u64_to_unit_double(ph ? philox_block(0, st.lo, st.hi).v[0] : pcg_output(st));
        r = __dadd_rn(__dmul_rn(pitch, -0.5), __dmul_rn(pitch, d));
        shift_f = __double2float_rn(__dmul_rn(r, span));
      }
    }
    uint64_t acc = 0;
    int nacc = 0;
    int64_t o = br.lb * pbs;
    for (int i = 0; i < n; ++i) {
      uint32_t code = 0;
      if (!degenerate) {
        const double a = __dsub_rn(Tr::to_d(x[i]), lo);
        if (INNER == 0) {
          code = exact_shift_code(a, span, r, pitch, top);
        } else if (NZ == 1) {
          code = exact_stoch_code_d(a, span, top, philox_block((uint64_t)(i >> 2), st.lo, st.hi).v[i & 3]);
        } else {
          st = pcg_step(st, inc);
          code = exact_stoch_code(a, span, top, st);
        }
      }
      acc |= (uint64_t)code << nacc;
      nacc += bits;
      while (nacc >= 8) {
        J.codes[poff + o++] = (uint8_t)acc;
        acc >>= 8;
        nacc -= 8;
      }
    }
    if (nacc > 0) J.codes[poff + o] = (uint8_t)acc;
    float* m = meta_at(J.meta, poff) + 3 * br.lb;
    m[0] = degenerate ? 0.0f : shift_f;
    m[1] = lof;
    m[2] = hif;
  }
}

// ---------------------------------------------------------------------------
// K3 / K4: dequantize (one source) or ordered dequantize-accumulate (P sources).
// ---------------------------------------------------------------------------
// Bits [4*bits*gi, 4*bits*(gi+1)) of a bucket payload of pbytes bytes (any width).
__device__ __forceinline__ uint64_t load_group_bits_any(const uint8_t* p, int gi, int bits, int64_t pbytes) {
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


// The lattice shift of this call: r = sample_shift(d, bucket_rng(key..., 0))
// = -d/2 + d * random() (quantize.py:130-132, numpy's unfused uniform).
static __device__ __noinline__ double lattice_shift(const DJobTable& tab) {
  const uint64_t step = tab.lat_key[1] + (tab.lat_step_ptr ? ld_dev_u64(tab.lat_step_ptr) : 0ull);
  const SeedPrefix pre = make_prefix(tab.lat_key[0], step, tab.lat_key[2], tab.lat_key[3], tab.lat_key[4]);
  U128 s0, inc;
  seed_bucket(pre, 0, s0, inc);
  const U128 s1 = mad128(s0, pcg_mult(), inc);
  const double u = u64_to_unit_double(pcg_output(s1));
  return __dadd_rn(__dmul_rn(tab.lat_d, -0.5), __dmul_rn(tab.lat_d, u));
}

// K4 epilogue: the averaged gradient g goes to J.out (when set) and, for a
// lattice step, the owner's iterate moves to d * rint((x - c*g - r)/d) + r
// (qsdp_step, optimizer.py:212-216; np.round = half to even), in fp64.
template <int OUT, bool VEC, bool LAT>
__device__ __forceinline__ void acc_store4(const DJobTable& tab, const DJob& J, int64_t idx, int n_left,
                                           const double g[4], double lat_r) {
  if (!LAT || J.out != nullptr) store_out4<OUT, VEC>(J.out, idx, n_left, g);
  if constexpr (LAT) {
    const double c = tab.lat_c, d = tab.lat_d, inv_d = tab.lat_inv_d;
    const bool vx = VEC && n_left >= 4 && (((uintptr_t)J.lat_x & 15) == 0);
    double x[4];
    if (tab.lat_xdtype == 1) {
      const double* xp = reinterpret_cast<const double*>(J.lat_x) + idx;
      if (vx) {
        const double2 a = reinterpret_cast<const double2*>(xp)[0], b = reinterpret_cast<const double2*>(xp)[1];
        x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
      } else {
        for (int i = 0; i < 4; ++i) x[i] = i < n_left ? xp[i] : 0.0;
      }
    } else {
      const float* xp = reinterpret_cast<const float*>(J.lat_x) + idx;
      if (vx) {
        const float4 a = *reinterpret_cast<const float4*>(xp);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      } else {
        for (int i = 0; i < 4; ++i) x[i] = i < n_left ? (double)xp[i] : 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // z = (y - r) / d in fp64; rint(z) from z' = (y - r) * fl(1/d) (|z' - z| < 3.5e-16 |z|)
      // unless z' is within 4e-16 |z'| of a half-integer or too large for the test
      const double a = __dsub_rn(__dsub_rn(x[i], __dmul_rn(c, g[i])), lat_r);
      const double z1 = __dmul_rn(a, inv_d);
      const double fz = floor(z1), t = __dsub_rn(z1, fz);
      double q = t < 0.5 ? fz : __dadd_rn(fz, 1.0);
      if (fabs(__dsub_rn(t, 0.5)) <= 4e-16 * fabs(z1) || !(fabs(z1) < 0x1p51)) q = rint(__ddiv_rn(a, d));
      x[i] = __dadd_rn(__dmul_rn(d, q), lat_r);
    }
    if (tab.lat_xdtype == 1) {
      double* xp = reinterpret_cast<double*>(J.lat_x) + idx;
      if (vx) {
        reinterpret_cast<double2*>(xp)[0] = make_double2(x[0], x[1]);
        reinterpret_cast<double2*>(xp)[1] = make_double2(x[2], x[3]);
      } else {
        for (int i = 0; i < 4 && i < n_left; ++i) xp[i] = x[i];
      }
    } else {
      float* xp = reinterpret_cast<float*>(J.lat_x) + idx;
      if (vx) {
        *reinterpret_cast<float4*>(xp) = make_float4(__double2float_rn(x[0]), __double2float_rn(x[1]),
                                                     __double2float_rn(x[2]), __double2float_rn(x[3]));
      } else {
        for (int i = 0; i < 4 && i < n_left; ++i) xp[i] = __double2float_rn(x[i]);
      }
    }
  }
}

// Lattice move of 4 iterate values already in registers (see acc_store4).
__device__ __forceinline__ void lat_move4(const DJobTable& tab, double x[4], const double g[4], double lat_r) {
  const double c = tab.lat_c, d = tab.lat_d, inv_d = tab.lat_inv_d;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double a = __dsub_rn(__dsub_rn(x[i], __dmul_rn(c, g[i])), lat_r);
    const double z1 = __dmul_rn(a, inv_d);
    const double fz = floor(z1), t = __dsub_rn(z1, fz);
    double q = t < 0.5 ? fz : __dadd_rn(fz, 1.0);
    if (fabs(__dsub_rn(t, 0.5)) <= 4e-16 * fabs(z1) || !(fabs(z1) < 0x1p51)) q = rint(__ddiv_rn(a, d));
    x[i] = __dadd_rn(__dmul_rn(d, q), lat_r);
  }
}

template <typename XT>
__device__ __forceinline__ void lat_load4(const void* base, int64_t idx, int n_left, XT x[4]) {
  const XT* p = reinterpret_cast<const XT*>(base) + idx;
  if (n_left >= 4 && (((uintptr_t)p & 15) == 0)) {
    if constexpr (sizeof(XT) == 4) {
      const float4 a = *reinterpret_cast<const float4*>(p);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    } else {
      const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
      x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
    }
  } else {
    for (int i = 0; i < 4; ++i) x[i] = i < n_left ? p[i] : XT(0);
  }
}

template <typename XT>
__device__ __forceinline__ void lat_store4(void* base, int64_t idx, int n_left, const double x[4]) {
  XT* p = reinterpret_cast<XT*>(base) + idx;
  if (n_left >= 4 && (((uintptr_t)p & 15) == 0)) {
    if constexpr (sizeof(XT) == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(__double2float_rn(x[0]), __double2float_rn(x[1]),
                                                  __double2float_rn(x[2]), __double2float_rn(x[3]));
    } else {
      reinterpret_cast<double2*>(p)[0] = make_double2(x[0], x[1]);
      reinterpret_cast<double2*>(p)[1] = make_double2(x[2], x[3]);
    }
  } else {
    for (int i = 0; i < 4 && i < n_left; ++i) p[i] = (XT)x[i];
  }
}

// K3: one source per job.  K4 (ACC): nsrc sources summed in order in fp64
// starting from +0.0, then divided by `divisor` (acc = zeros; acc = acc + vals;
// acc / P -- sharded.py:385-431).  Per-source scales of the current bucket are
// staged in shared memory (one row per team) by lanes 0..nsrc-1.
// BITS > 0: direct width with aligned group loads on full buckets; BITS == 0: any width.
// One warp per bucket, S % 128 == 0 (every lane owns S/128 full groups of 4).
// ADD0: K4 with a single source and divisor 1 -- out = (0.0 + val) / 1 (the
// reference's zeros + vals; only the sign of a zero can differ from val).
template <int BITS, int OUT, bool COH, bool ADD0 = false, bool LAT = false>
__device__ __forceinline__ void dequant_fast32(const DJobTable& tab, int64_t poff, int64_t warp, int64_t nwarps,
                                               double lat_r = 0.0) {
  constexpr int UMAX = 8;
  const int lane = threadIdx.x & 31;
  const int S = tab.bucket;
  const int G = S >> 7;  // groups per lane
  const double top = (double)((1u << BITS) - 1u);
  const int64_t pbs = payload_bytes(S, BITS);
  struct Pre {
    uint32_t w[UMAX];
    float m0, m1, m2;
    int j, n;
    int64_t lb;
  };
  auto fetch = [&](int64_t b, Pre& p) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    p.j = j;
    p.lb = b - J.bucket_base;
    p.n = (int)min((int64_t)S, J.length - p.lb * S);
    const float* m = meta_at(J.meta[0], poff) + 3 * p.lb;
    p.m0 = COH ? __ldcg(m) : m[0];
    p.m1 = COH ? __ldcg(m + 1) : m[1];
    p.m2 = COH ? __ldcg(m + 2) : m[2];
    const uint8_t* __restrict__ cp = J.codes[0] + poff + p.lb * pbs;
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      const int gi = u * 32 + lane;
      p.w[u] = (u < G && 4 * gi < p.n) ? (uint32_t)load_group_direct<BITS, COH>(cp, gi) : 0u;
    }
  };
  int64_t b = warp;
  if (b >= tab.total_buckets) return;
  Pre cur;
  fetch(b, cur);
  while (b < tab.total_buckets) {
    const int64_t bn = b + nwarps;
    Pre nxt;
    if (bn < tab.total_buckets) fetch(bn, nxt);  // issued before the current bucket's math
    const DJob& J = tab.jobs[cur.j];
    const double lo = (double)cur.m1, shift = (double)cur.m0;
    const double pitch = __ddiv_rn(__dsub_rn((double)cur.m2, lo), top);  // QuantizedBlock.pitch
    const int64_t off = cur.lb * S;
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      const int gi = u * 32 + lane;
      const int e = 4 * gi;
      if (u < G && e < cur.n) {
        double v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double c = code_to_double((cur.w[u] >> (i * BITS)) & ((1u << BITS) - 1u));
          v[i] = __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift);  // (lo + code*pitch) + shift
          if (ADD0) v[i] = __dadd_rn(0.0, v[i]);
        }
        if (ADD0) acc_store4<OUT, true, LAT>(tab, J, off + e, cur.n - e, v, lat_r);
        else store_out4<OUT, true>(J.out, off + e, cur.n - e, v);
      }
    }
    b = bn;
    cur = nxt;
  }
}

// K4 fast path for nsrc in [2, NSMAX]: one warp per bucket (S % 128 == 0,
// S <= 1024, direct widths 8 / 4, aligned buffers).  The code words of ALL
// sources for a chunk of UC groups per lane are issued together (NSMAX * UC = 16
// loads in flight per lane) before the ordered fp64 accumulation
// (acc = 0.0; acc = acc + val_p for p = 0..nsrc-1; acc / divisor, sharded.py:385-431).
// Per-source scales live in shared memory rows (lanes < nsrc fill them).
// A power-of-two divisor is applied as a multiply by its exact reciprocal
// (bit-identical to the division); other divisors divide.
template <int BITS, int OUT, bool COH, int NSMAX, bool LAT>
__device__ __forceinline__ void dequant_acc_fast32(const DJobTable& tab, int64_t poff, int64_t warp, int64_t nwarps,
                                                   double (*row)[3], double lat_r) {
  constexpr int UC = 16 / NSMAX;
  const int lane = threadIdx.x & 31;
  const int S = tab.bucket;
  const int G = S >> 7;  // groups per lane
  const double top = (double)((1u << BITS) - 1u);
  const int64_t pbs = payload_bytes(S, BITS);
  const int dv = tab.divisor;
  const bool pow2 = (dv & (dv - 1)) == 0;
  const double rdiv = 1.0 / (double)dv;  // exact for powers of two
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    const int nsrc = J.nsrc;
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    __syncwarp();
    if (lane < nsrc) {
      const float* m = meta_at(J.meta[lane], poff) + 3 * lb;
      const float m0 = COH ? __ldcg(m) : m[0], m1 = COH ? __ldcg(m + 1) : m[1], m2 = COH ? __ldcg(m + 2) : m[2];
      const double lo = (double)m1;
      row[lane][0] = lo;
      row[lane][1] = __ddiv_rn(__dsub_rn((double)m2, lo), top);  // QuantizedBlock.pitch
      row[lane][2] = (double)m0;
    }
    __syncwarp();
    for (int g0 = 0; g0 < G; g0 += UC) {
      uint32_t w[NSMAX][UC];
#pragma unroll
      for (int p = 0; p < NSMAX; ++p) {
        const uint8_t* __restrict__ cp = J.codes[p < nsrc ? p : 0] + poff + lb * pbs;
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int gi = (g0 + u) * 32 + lane;
          w[p][u] = (p < nsrc && g0 + u < G && 4 * gi < n) ? (uint32_t)load_group_direct<BITS, COH>(cp, gi) : 0u;
        }
      }
      double acc[UC][4];
#pragma unroll
      for (int u = 0; u < UC; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[u][i] = 0.0;
#pragma unroll
      for (int p = 0; p < NSMAX; ++p) {
        if (p < nsrc) {
          const double lo = row[p][0], pitch = row[p][1], shift = row[p][2];
#pragma unroll
          for (int u = 0; u < UC; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double c = code_to_double((w[p][u] >> (i * BITS)) & ((1u << BITS) - 1u));
              acc[u][i] = __dadd_rn(acc[u][i], __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift));
            }
        }
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int gi = (g0 + u) * 32 + lane;
        const int e = 4 * gi;
        if (g0 + u < G && e < n) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            acc[u][i] = pow2 ? __dmul_rn(acc[u][i], rdiv) : __ddiv_rn(acc[u][i], (double)dv);
          acc_store4<OUT, true, LAT>(tab, J, off + e, n - e, acc[u], lat_r);
        }
      }
    }
  }
}

// K4 + lattice step (fast configuration): as dequant_acc_fast32, with the
// iterate's values of a chunk loaded together with its code words, so one
// memory round trip per chunk serves both (XT = iterate dtype).
template <int BITS, int OUT, int NSMAX, typename XT>
__device__ __forceinline__ void dequant_lat_fast32(const DJobTable& tab, int64_t poff, int64_t warp, int64_t nwarps,
                                                   double (*row)[3], double lat_r) {
  constexpr int UC = 16 / NSMAX < 4 ? 16 / NSMAX : 4;  // groups per chunk (wider measured slower: registers)
  const int lane = threadIdx.x & 31;
  const int S = tab.bucket;
  const int G = S >> 7;
  const double top = (double)((1u << BITS) - 1u);
  const int64_t pbs = payload_bytes(S, BITS);
  const int dv = tab.divisor;
  const bool pow2 = (dv & (dv - 1)) == 0;
  const double rdiv = 1.0 / (double)dv;
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    const int nsrc = J.nsrc;
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    __syncwarp();
    if (lane < nsrc) {
      const float* m = meta_at(J.meta[lane], poff) + 3 * lb;
      const double lo = (double)m[1];
      row[lane][0] = lo;
      row[lane][1] = __ddiv_rn(__dsub_rn((double)m[2], lo), top);
      row[lane][2] = (double)m[0];
    }
    __syncwarp();
    for (int g0 = 0; g0 < G; g0 += UC) {
      uint32_t w[NSMAX][UC];
      XT xv[UC][4];  // the iterate in its own type until used
#pragma unroll
      for (int p = 0; p < NSMAX; ++p) {
        const uint8_t* __restrict__ cp = J.codes[p < nsrc ? p : 0] + poff + lb * pbs;
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int gi = (g0 + u) * 32 + lane;
          w[p][u] = (p < nsrc && g0 + u < G && 4 * gi < n) ? (uint32_t)load_group_direct<BITS, false>(cp, gi) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int e = 4 * ((g0 + u) * 32 + lane);
        if (g0 + u < G && e < n) lat_load4<XT>(J.lat_x, off + e, n - e, xv[u]);
      }
      double acc[UC][4];
#pragma unroll
      for (int u = 0; u < UC; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[u][i] = 0.0;
#pragma unroll
      for (int p = 0; p < NSMAX; ++p) {
        if (p < nsrc) {
          const double lo = row[p][0], pitch = row[p][1], shift = row[p][2];
#pragma unroll
          for (int u = 0; u < UC; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double c = code_to_double((w[p][u] >> (i * BITS)) & ((1u << BITS) - 1u));
              acc[u][i] = __dadd_rn(acc[u][i], __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift));
            }
        }
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int e = 4 * ((g0 + u) * 32 + lane);
        if (g0 + u < G && e < n) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            acc[u][i] = pow2 ? __dmul_rn(acc[u][i], rdiv) : __ddiv_rn(acc[u][i], (double)dv);
          if (J.out != nullptr) store_out4<OUT, true>(J.out, off + e, n - e, acc[u]);
          double xd[4] = {(double)xv[u][0], (double)xv[u][1], (double)xv[u][2], (double)xv[u][3]};
          lat_move4(tab, xd, acc[u], lat_r);
          lat_store4<XT>(J.lat_x, off + e, n - e, xd);
        }
      }
    }
  }
}

template <int BITS, int TL, int OUT, bool VEC, bool ACC, bool COH = false, bool LAT = false>
__device__ __forceinline__ void dequant_body(const DJobTable& tab, double* sm_meta_base, double lat_r = 0.0) {
  const int64_t poff = d_parity_off(tab);
  constexpr int TEAMS = 32 / TL;
  constexpr int U = 8;  // groups whose code words are loaded before use
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int lt = lane % TL;
  const int team = lane / TL;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket;
  const int bits = BITS > 0 ? BITS : tab.bits;
  const double top = (double)((1u << bits) - 1u);
  const int64_t pbs = payload_bytes(S, bits);
  const int groups = (S + 3) / 4;
  const int gl = (groups + TL - 1) / TL;
  const uint64_t cmask = (1ull << bits) - 1ull;
  const bool cvec = BITS > 0 && tab.codes_vec;

  if constexpr (TL == 32 && (BITS == 8 || BITS == 4) && VEC) {
    // K3 hot path: a bucket's code words are loaded one bucket AHEAD (software
    // pipelining across the warp's buckets), so HBM / NVLink latency overlaps the
    // previous bucket's fp64 dequantization.  K4 with one source takes it too.
    bool single = !ACC || tab.divisor == 1;
    if constexpr (ACC) {
      for (int j = 0; j < tab.njobs && single; ++j) single = tab.jobs[j].nsrc == 1;
    }
    if (single && cvec && (S & 127) == 0 && S <= 1024) {
      dequant_fast32<BITS, OUT, COH, ACC, LAT>(tab, poff, warp, nwarps, lat_r);
      return;
    }
    if constexpr (ACC) {
      int ns = 0;
      for (int j = 0; j < tab.njobs; ++j) ns = max(ns, tab.jobs[j].nsrc);
      if (cvec && (S & 127) == 0 && S <= 1024 && ns <= 8) {
        double(*row)[3] = reinterpret_cast<double(*)[3]>(sm_meta_base + ((size_t)wib * TEAMS * 8) * 3);
        if (ns <= 2) dequant_acc_fast32<BITS, OUT, COH, 2, LAT>(tab, poff, warp, nwarps, row, lat_r);
        else if (ns <= 4) dequant_acc_fast32<BITS, OUT, COH, 4, LAT>(tab, poff, warp, nwarps, row, lat_r);
        else dequant_acc_fast32<BITS, OUT, COH, 8, LAT>(tab, poff, warp, nwarps, row, lat_r);
        return;
      }
    }
  }

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
        const float* m = meta_at(J.meta[0], poff) + 3 * lb;
        const float m0 = COH ? __ldcg(m) : m[0], m1 = COH ? __ldcg(m + 1) : m[1], m2 = COH ? __ldcg(m + 2) : m[2];
        shift = (double)m0;
        lo = (double)m1;
        pitch = __ddiv_rn(__dsub_rn((double)m2, lo), top);  // QuantizedBlock.pitch
      }
      const uint8_t* __restrict__ cp = J.codes[0] + poff + lb * pbs;
      if (cvec && n == S) {
        for (int g0 = 0; g0 < gl; g0 += U) {
          uint64_t w[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int gi = (g0 + u) * TL + lt;
            w[u] = (g0 + u < gl && 4 * gi < n) ? load_group_direct<BITS, COH>(cp, gi) : 0ull;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int gi = (g0 + u) * TL + lt;
            if (g0 + u < gl && 4 * gi < n) {
              double v[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const double c = code_to_double((uint32_t)((w[u] >> (i * bits)) & cmask));
                v[i] = __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift);  // (lo + code*pitch) + shift
              }
              store_out4<OUT, VEC>(J.out, off + 4 * gi, 4, v);
            }
          }
        }
      } else {
        for (int g = 0; g < gl; ++g) {
          const int gi = g * TL + lt;
          const int e = 4 * gi;
          if (e >= n) break;
          const uint64_t w = load_group_bits_any(cp, gi, bits, pb);
          double v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double c = code_to_double((uint32_t)((w >> (i * bits)) & cmask));
            v[i] = __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift);
          }
          store_out4<OUT, VEC>(J.out, off + e, n - e, v);
        }
      }
    } else {
      const int nsrc = J.nsrc;
      double(*row)[3] = reinterpret_cast<double(*)[3]>(sm_meta_base + ((size_t)(wib * TEAMS + team) * 8) * 3);
      if (active && lt < nsrc) {
        const float* m = meta_at(J.meta[lt], poff) + 3 * lb;
        const float m0 = COH ? __ldcg(m) : m[0], m1 = COH ? __ldcg(m + 1) : m[1], m2 = COH ? __ldcg(m + 2) : m[2];
        const double lo = (double)m1;
        row[lt][0] = lo;
        row[lt][1] = __ddiv_rn(__dsub_rn((double)m2, lo), top);
        row[lt][2] = (double)m0;
      }
      __syncwarp();
      constexpr int UA = 4;  // groups accumulated together (their code loads are in flight together)
      for (int g0 = 0; g0 < gl; g0 += UA) {
        double acc[UA][4];
#pragma unroll
        for (int u = 0; u < UA; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[u][i] = 0.0;
        for (int p = 0; p < nsrc; ++p) {
          const uint8_t* __restrict__ cp = J.codes[p] + poff + lb * pbs;
          uint64_t w[UA];
#pragma unroll
          for (int u = 0; u < UA; ++u) {
            const int gi = (g0 + u) * TL + lt;
            const int e = 4 * gi;
            w[u] = 0;
            if (g0 + u < gl && e < n)
              w[u] = (cvec && e + 4 <= n) ? load_group_direct<BITS, COH>(cp, gi) : load_group_bits_any(cp, gi, bits, pb);
          }
          const double lo = row[p][0], pitch = row[p][1], shift = row[p][2];
#pragma unroll
          for (int u = 0; u < UA; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const double c = code_to_double((uint32_t)((w[u] >> (i * bits)) & cmask));
              acc[u][i] = __dadd_rn(acc[u][i], __dadd_rn(__dadd_rn(lo, __dmul_rn(c, pitch)), shift));
            }
        }
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          const int gi = (g0 + u) * TL + lt;
          const int e = 4 * gi;
          if (g0 + u < gl && e < n) {
            if (tab.divisor != 1) {
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[u][i] = __ddiv_rn(acc[u][i], (double)tab.divisor);
            }
            acc_store4<OUT, VEC, LAT>(tab, J, off + e, n - e, acc[u], lat_r);
          }
        }
      }
      __syncwarp();
    }
  }
}

template <int BITS, int TL, int OUT, bool VEC, bool ACC, bool LAT = false>
__global__ void __launch_bounds__(256) dequant_kernel(const __grid_constant__ DJobTable tab) {
  __shared__ double sm_meta[ACC ? 8 * (32 / TL) * 8 * 3 : 1];
  double lat_r = 0.0;
  if constexpr (LAT) {  // one keyed draw per warp (lane 0), broadcast by shuffle
    double r = 0.0;
    if ((threadIdx.x & 31) == 0) r = lattice_shift(tab);
    lat_r = __shfl_sync(0xffffffffu, r, 0);
  }
  dequant_body<BITS, TL, OUT, VEC, ACC, false, LAT>(tab, sm_meta, lat_r);
}

// K4 + lattice step, fast configuration only (TL 32, widths 8 / 4, S % 128 == 0,
// S <= 1024, aligned buffers, nsrc <= NSMAX): its own kernel so its register
// budget is that of this path alone (the general kernel's paths share one).
template <int BITS, int OUT, int NSMAX, typename XT>
__global__ void __launch_bounds__(256) dequant_lat_fast_kernel(const __grid_constant__ DJobTable tab) {
  __shared__ double sm_meta[8 * 8 * 3];
  double r = 0.0;
  if ((threadIdx.x & 31) == 0) r = lattice_shift(tab);
  const double lat_r = __shfl_sync(0xffffffffu, r, 0);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double(*row)[3] = reinterpret_cast<double(*)[3]>(sm_meta + (size_t)(threadIdx.x >> 5) * 8 * 3);
  dequant_lat_fast32<BITS, OUT, NSMAX, XT>(tab, d_parity_off(tab), warp, nwarps, row, lat_r);
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

inline int grid_for(int64_t total_buckets, int teams_per_warp, int sms, int warps_per_cta = 8, int ctas_per_sm = 8) {
  const int64_t warps = (total_buckets + teams_per_warp - 1) / teams_per_warp;
  const int64_t blocks = (warps + warps_per_cta - 1) / warps_per_cta;
  const int64_t cap = (int64_t)sms * ctas_per_sm;
  return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

// Persistent grid: exactly the CTAs that are co-resident (one wave), fewer if
// the work is smaller.  Every kernel grid-strides over buckets, so a partial
// second wave would only add a tail.
template <typename F>
inline int persistent_grid(F kern, int threads, size_t smem, int64_t total_buckets, int teams_per_warp, int sms,
                           int max_per_sm = 0) {
  // one cached occupancy answer per (kernel, block size, smem size): every quantizer
  // instantiation has the same function type, so the kernel address is part of the key
  struct Entry { const void* k; size_t smem; int threads, per_sm; };
  static thread_local Entry cache[16] = {};
  static thread_local int next = 0;
  const void* kp = reinterpret_cast<const void*>(kern);
  int per_sm = 0;
  for (const Entry& e : cache)
    if (e.k == kp && e.smem == smem && e.threads == threads) per_sm = e.per_sm;
  if (per_sm == 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem) != cudaSuccess || v < 1) v = 1;
    per_sm = v;
    cache[next] = Entry{kp, smem, threads, v};
    next = (next + 1) & 15;
  }
  if (max_per_sm > 0 && per_sm > max_per_sm) per_sm = max_per_sm;
  return grid_for(total_buckets, teams_per_warp, sms, threads / 32, per_sm);
}


// Opt a kernel into more than 48 KB of dynamic shared memory.  The attribute is
// per device context, so the cache (one per kernel instantiation, passed in) is
// indexed by the current device.
template <typename F>
inline cudaError_t ensure_smem_attr(F kern, size_t smem, size_t (&cache)[64]) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  size_t& done = cache[dev & 63];
  if (smem <= done || smem <= 48 * 1024) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done = smem;
  return e;
}

// Fast TMA path.  Returns false when the configuration needs the general kernel.
template <typename T, int INNER, int BITS, int FDQ, int PH = 0>
cudaError_t launch_q_tma32_v(const QJobTable& tab, int sms, cudaStream_t s) {
  constexpr int NST = 2;
  const size_t stage = (size_t)tab.bucket * sizeof(T);
  int wpc = 8;
  if (stage <= 8192) {
    while (wpc > 2 && (size_t)wpc * NST * stage > 64 * 1024) wpc >>= 1;
  } else {  // 16 KB buckets (S = 4096 fp32): two CTAs per SM, each as many warps' rings as fit in
            // ~100 KB (3 warps: measured 3.7 / 1.4 TB/s K1 / K2 vs 3.3 / 1.2 with one 6-warp CTA)
    const size_t per_warp = NST * stage + NST * sizeof(uint64_t) + 32 * sizeof(SeedOut);
    wpc = (int)((100 * 1024 - 33 * sizeof(JumpEntry)) / per_warp);
    wpc = wpc < 1 ? 1 : (wpc > 8 ? 8 : wpc);
  }
  const size_t smem = (size_t)wpc * NST * stage + (size_t)wpc * NST * sizeof(uint64_t) +
                      (size_t)wpc * 32 * sizeof(SeedOut) + 33 * sizeof(JumpEntry) +
                      (dq_table_on(INNER, BITS, FDQ) ? (size_t)wpc * (1u << BITS) * sizeof(uint32_t) : 0);
  auto kern = quantize_tma32_kernel<T, INNER, BITS, NST, FDQ, PH>;
  static thread_local size_t smem_set[64] = {};  // per instantiation and device
  if (cudaError_t e = ensure_smem_attr(kern, smem, smem_set); e != cudaSuccess) return e;
  // tab.cta_cap (qsdp_comm_set_ctas_per_sm): leave CTA slots on every SM to a concurrent
  // collective (an HBM-bound all-gather beside an issue-bound reduce-scatter)
  const int grid = persistent_grid(kern, wpc * 32, smem, tab.total_buckets, 1, sms, tab.cta_cap);
  kern<<<grid, wpc * 32, smem, s>>>(tab);
  return cudaGetLastError();
}

// Fast TMA path; the fused-dequant variant only when a job asks for it.
template <typename T, int INNER, int BITS>
cudaError_t launch_q_tma32(const QJobTable& tab, int sms, cudaStream_t s) {
  bool fdq = false;
  for (int j = 0; j < tab.njobs; ++j) fdq = fdq || tab.jobs[j].dq_out != nullptr;
  if (!fdq) return launch_q_tma32_v<T, INNER, BITS, 0>(tab, sms, s);
  if (sizeof(T) == 4 && tab.dq_dtype == 0)  // fp32 out: dtype and K4's 0.0 + v fixed at compile time
    return tab.dq_add0 ? launch_q_tma32_v<T, INNER, BITS, 2>(tab, sms, s) : launch_q_tma32_v<T, INNER, BITS, 1>(tab, sms, s);
  return launch_q_tma32_v<T, INNER, BITS, 3>(tab, sms, s);
}

template <typename T, int INNER, int BITS, int TL>
cudaError_t launch_q_tma(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  if constexpr (TL == 32) {
    (void)vec;
    return launch_q_tma32<T, INNER, BITS>(tab, sms, s);
  } else {
    constexpr int NST = 2;
    constexpr int TEAMS = 32 / TL;
    const size_t stage = (size_t)TEAMS * tab.bucket * sizeof(T);
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * NST * stage > 64 * 1024) wpc >>= 1;
    const size_t smem = (size_t)wpc * NST * stage + (size_t)wpc * NST * sizeof(uint64_t) +
                        (size_t)wpc * 32 * sizeof(SeedOut);
    auto kern = quantize_tma_kernel<T, INNER, BITS, TL, NST>;
    static thread_local size_t smem_set[64] = {};
    if (cudaError_t e = ensure_smem_attr(kern, smem, smem_set); e != cudaSuccess) return e;
    const int grid = persistent_grid(kern, wpc * 32, smem, tab.total_buckets, TEAMS, sms);
    kern<<<grid, wpc * 32, smem, s>>>(tab, vec ? 1 : 0);
    return cudaGetLastError();
  }
}

template <typename T, int INNER, int TL>
cudaError_t launch_q_tl(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  const int S = tab.bucket;
  if (S * (int)sizeof(T) <= (TL == 32 ? 16384 : 8192)) {
    switch (tab.bits) {
      case 8: return launch_q_tma<T, INNER, 8, TL>(tab, vec, sms, s);
      case 4: return launch_q_tma<T, INNER, 4, TL>(tab, vec, sms, s);
      case 2: return launch_q_tma<T, INNER, 2, TL>(tab, vec, sms, s);
      case 16: return launch_q_tma<T, INNER, 16, TL>(tab, vec, sms, s);
      default: break;
    }
  }
  // TL < 32 only when the bucket has <= TL groups of 4: one group per lane.
  constexpr int G = TL == 32 ? 8 : 1;
  const int gl = ((S + 3) / 4 + TL - 1) / TL;
  auto go = [&](auto kern) {
    kern<<<persistent_grid(kern, 256, 0, tab.total_buckets, 32 / TL, sms), 256, 0, s>>>(tab);
  };
  if (TL < 32 || gl <= G) {
    if (vec) go(quantize_kernel<T, INNER, TL, G, true, true>);
    else go(quantize_kernel<T, INNER, TL, G, true, false>);
  } else if constexpr (TL == 32) {
    if (vec) go(quantize_kernel<T, INNER, TL, 1, false, true>);
    else go(quantize_kernel<T, INNER, TL, 1, false, false>);
  }
  return cudaGetLastError();
}

// Philox noise (qsdp_noise 1): the team kernels with the counter-based Coder (any width,
// S % 8 == 0), or the generic kernel; the TMA fast paths are PCG64-only.
template <typename T, int INNER, int TL>
cudaError_t launch_q_philox_tl(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  const int S = tab.bucket;
  constexpr int G = TL == 32 ? 8 : 1;
  const int gl = ((S + 3) / 4 + TL - 1) / TL;
  auto go = [&](auto kern) {
    kern<<<persistent_grid(kern, 256, 0, tab.total_buckets, 32 / TL, sms), 256, 0, s>>>(tab);
  };
  if (TL < 32 || gl <= G) {
    if (vec) go(quantize_kernel<T, INNER, TL, G, true, true, 1>);
    else go(quantize_kernel<T, INNER, TL, G, true, false, 1>);
  } else if constexpr (TL == 32) {
    if (vec) go(quantize_kernel<T, INNER, TL, 1, false, true, 1>);
    else go(quantize_kernel<T, INNER, TL, 1, false, false, 1>);
  }
  return cudaGetLastError();
}

template <typename T, int INNER>
cudaError_t launch_q_philox(const QJobTable& tab, bool vec, int sms, cudaStream_t s) {
  const int S = tab.bucket;
  // K2 with octet buckets: the TMA32 quantizer with counter-based draws (no fused epilogue:
  // the comm's push / fused paths are PCG64-only)
  bool fdq = false;
  for (int j = 0; j < tab.njobs; ++j) fdq = fdq || tab.jobs[j].dq_out != nullptr;
  if (INNER == 1 && !fdq && S % 256 == 0 && S * (int)sizeof(T) <= 16384) {
    switch (tab.bits) {
      case 8: return launch_q_tma32_v<T, 1, 8, 0, 1>(tab, sms, s);
      case 4: return launch_q_tma32_v<T, 1, 4, 0, 1>(tab, sms, s);
      case 2: return launch_q_tma32_v<T, 1, 2, 0, 1>(tab, sms, s);
      default: break;
    }
  }
  if (S % 8 != 0) {
    const int64_t blocks = (tab.total_buckets + 127) / 128;
    const int64_t cap = (int64_t)sms * 16;
    quantize_generic_kernel<T, INNER, 1><<<(int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks)), 128, 0, s>>>(tab);
    return cudaGetLastError();
  }
  switch (team_lanes(S)) {
    case 2: return launch_q_philox_tl<T, INNER, 2>(tab, vec, sms, s);
    case 4: return launch_q_philox_tl<T, INNER, 4>(tab, vec, sms, s);
    case 8: return launch_q_philox_tl<T, INNER, 8>(tab, vec, sms, s);
    case 16: return launch_q_philox_tl<T, INNER, 16>(tab, vec, sms, s);
    default: return launch_q_philox_tl<T, INNER, 32>(tab, vec, sms, s);
  }
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
  int tl = team_lanes(S);
  const bool direct = tab.bits == 2 || tab.bits == 4 || tab.bits == 8 || tab.bits == 16;
  // S in (32, 64], whole-byte groups: 8 buckets per warp, 4 groups per lane (the per-bucket work
  // is shared by more buckets per warp instruction; odd widths keep their lane-pair packing)
  if (tl == 16 && direct) tl = 4;
  switch (tl) {
    case 2: return launch_q_tl<T, INNER, 2>(tab, vec, sms, s);
    case 4: return launch_q_tl<T, INNER, 4>(tab, vec, sms, s);
    case 8: return launch_q_tl<T, INNER, 8>(tab, vec, sms, s);
    case 16: return launch_q_tl<T, INNER, 16>(tab, vec, sms, s);
    default: return launch_q_tl<T, INNER, 32>(tab, vec, sms, s);
  }
}

}  // namespace qsdp
