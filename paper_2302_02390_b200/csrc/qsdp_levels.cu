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
  const int64_t poff = d_parity_off(tab);  // communicator slot parity (0 outside collectives)
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    const float* m = meta_at(J.meta[0], poff) + 3 * lb;
    const double lo = (double)m[1];
    const double span = __dsub_rn((double)m[2], lo);  // scale_hi - scale_lo
    const uint8_t* cp = J.codes[0] + poff + lb * pbs;
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

// ---------------------------------------------------------------------------
// Fast paths (tables of <= 2^12 levels, S % 256 == 0 and aligned buffers).
//
// Code search: a per-CTA index of kCells + 1 cells centred on t/kCells,
// t = 0..kCells.  The cell of u in [0, 1] is round(u * kCells), read from the
// low word of u + 1.5*2^40 (one DADD; the ulp there is 2^-12 = 1/kCells);
// a tie may pick either neighbour, and both windows contain u.  Cell t covers
// the window W = [(t - 1/2)/kCells - 8e-16, (t + 1/2)/kCells + 8e-16)
// (8e-16 > the 4e-16 certification radius plus one rounding of the bounds)
// and stores
//   base[t] = #{mids < lower end of W}   (| kMulti when W holds two or more mids)
//   cmid[t] = the single mid in W, or +inf when W holds none.
// For u' in cell t and the exact u (|u - u'| < 4e-16, both in W), with
// d = u' - cmid:  #{mids < u} = base + (d > 0)  unless |d| <= 4e-16, so a code
// costs two independent smem loads, one DADD and two compares; multi-mid cells
// and near-mid values take the searched + exact-division path.
// ---------------------------------------------------------------------------
constexpr int kCells = 4096;
constexpr uint16_t kMulti = 0x8000;
constexpr double kCellMagic = 1649267441664.0;  // 1.5 * 2^40

// #{mids[0..nm) < t}
__device__ __forceinline__ int count_below(const double* mids, int nm, double t) {
  int lo_i = 0, hi_i = nm;
  while (lo_i < hi_i) {
    const int m = (lo_i + hi_i) >> 1;
    if (mids[m] < t) lo_i = m + 1;
    else hi_i = m;
  }
  return lo_i;
}

struct LevelIndex {
  const double* mids;
  const double* cmid;    // fp64 index (f64 inputs)
  const float* cmid32;   // fp32 prefilter index (f32 inputs): float2 {cmid, base bits}, same smem
  const uint16_t* base;
  int nm;         // number of mids = nl - 1
  double ulo, uhi;  // clip(clip(u, 0, 1), q0, qL) == clip(u, ulo, uhi)
  float ulo32, uhi32;
  int fixed;      // >= 0: every u clips to one value (table outside [0, 1]); its code
  // no NaN can reach here (non-finite buckets are degenerate): plain selects
  __device__ __forceinline__ double clip(double u) const {
    u = u < ulo ? ulo : u;
    return u > uhi ? uhi : u;
  }
  __device__ __forceinline__ uint32_t search(double u) const { return (uint32_t)count_below(mids, nm, u); }
  __device__ __forceinline__ uint32_t code_slow(double a, double inv, double span) const {
    const double u1 = clip(__dmul_rn(a, inv));
    uint32_t c = search(u1);
    const bool near = (c > 0 && fabs(u1 - mids[c - 1]) <= 4e-16) || ((int)c < nm && fabs(mids[c] - u1) <= 4e-16);
    if (near) c = search(clip(__ddiv_rn(a, span)));
    return c;
  }
  // branch-free candidate code of one element, u' = (v - lo) * fl(1/span);
  // *slow is set when it is not certified (then code_slow decides).  fixed < 0.
  __device__ __forceinline__ uint32_t code_fast(double a, double inv, bool& slow) const {
    const double u1 = clip(__dmul_rn(a, inv));
    const int t = __double2loint(__dadd_rn(u1, kCellMagic));
    const uint16_t b = base[t];
    const double d = __dsub_rn(u1, cmid[t]);
    slow = (b & kMulti) || fabs(d) <= 4e-16;
    return (uint32_t)(b & 0x7fff) + (d > 0.0 ? 1u : 0u);
  }
  __device__ __forceinline__ uint32_t code(double a, double inv, double span) const {
    bool slow;
    const uint32_t c = code_fast(a, inv, slow);
    return slow ? code_slow(a, inv, span) : c;
  }
  // f32 inputs: lo and hi are the bucket's own min / max (exact), so
  // u32 = fl(fl(x - lo) * fl(1/fl(hi - lo))) is within 2.4e-7 of u, 3.6e-7
  // after the f32 clip bounds; cells carry a 2e-6 window and f32 mids (error
  // <= 6e-8).  |u32 - cmid32| > 1e-6 therefore certifies the comparison;
  // otherwise the element takes code_slow (fp64, exact).
  __device__ __forceinline__ uint32_t code_fast32(float x, float lof, float inv32, bool& slow) const {
    float u = __fmul_rn(__fsub_rn(x, lof), inv32);
    u = fminf(fmaxf(u, ulo32), uhi32);
    const int t = __float_as_int(__fadd_rn(u, 3072.0f)) & 0x3FFFFF;  // round(u * 4096): ulp(3072) = 2^-12
    const float2 e = reinterpret_cast<const float2*>(cmid32)[t];     // {cmid (NaN: multi-mid cell), base}
    const float d = __fsub_rn(u, e.x);
    slow = !(fabsf(d) > 1e-6f);
    return (uint32_t)__float_as_int(e.y) + (d > 0.0f ? 1u : 0u);
  }
};

// The index in smem (built by build_level_index) seen as a LevelIndex.
template <bool F32>
__device__ __forceinline__ LevelIndex level_index_view(double* sm, const double* levels, int nl) {
  double* cmid = sm + nl;
  const uint16_t* base = reinterpret_cast<const uint16_t*>(cmid + kCells + 1);
  const int nm = nl - 1;
  const double q0 = levels[0], qL = levels[nl - 1];
  LevelIndex ix{sm, cmid, reinterpret_cast<const float*>(cmid), base, nm, fmax(0.0, q0), fmin(1.0, qL), 0.f, 0.f, -1};
  if (q0 > 1.0) ix.ulo = ix.uhi = q0;  // np.clip(clip(u, 0, 1), q0, qL) is constant
  if (qL < 0.0) ix.ulo = ix.uhi = qL;
  if (ix.ulo > 1.0 || ix.uhi < 0.0) ix.fixed = count_below(sm, nm, ix.ulo);
  ix.ulo32 = __double2float_rn(ix.ulo);
  ix.uhi32 = __double2float_rn(ix.uhi);
  return ix;
}

// smem: mids[nl] doubles, then cmid[kCells + 1] doubles + base[kCells + 1] uint16
// (f64 inputs) or {cmid, base} float2 entries (F32: the prefilter index)
template <bool F32>
__device__ __forceinline__ LevelIndex build_level_index(double* sm, const double* levels, int nl) {
  double* cmid = sm + nl;
  uint16_t* base = reinterpret_cast<uint16_t*>(cmid + kCells + 1);
  const int nm = nl - 1;
  for (int i = threadIdx.x; i < nm; i += blockDim.x) sm[i] = __dmul_rn(__dadd_rn(levels[i], levels[i + 1]), 0.5);
  __syncthreads();
  // each thread walks a run of consecutive cells; the window ends only grow,
  // so two forward pointers replace per-cell binary searches
  constexpr double h = 1.0 / (double)kCells;
  const double margin = F32 ? 2e-6 : 8e-16;
  const int per = (kCells + 1 + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per, c1 = min(c0 + per, kCells + 1);
  if (c0 < c1) {
    int plo = count_below(sm, nm, __dsub_rn(((double)c0 - 0.5) * h, margin));
    int phi = count_below(sm, nm, __dadd_rn(((double)c0 + 0.5) * h, margin));
    for (int c = c0; c < c1; ++c) {
      const double wlo = __dsub_rn(((double)c - 0.5) * h, margin), whi = __dadd_rn(((double)c + 0.5) * h, margin);
      while (plo < nm && sm[plo] < wlo) ++plo;  // plo = #{mids < wlo}
      while (phi < nm && sm[phi] < whi) ++phi;  // phi = #{mids < whi}
      if (F32) {
        const float cm = phi - plo == 1 ? __double2float_rn(sm[plo]) : (phi - plo == 0 ? INFINITY : __int_as_float(0x7fc00000));
        reinterpret_cast<float2*>(cmid)[c] = make_float2(cm, __int_as_float(plo));
      } else {
        base[c] = (uint16_t)plo | (phi - plo >= 2 ? kMulti : 0);
        cmid[c] = phi - plo == 1 ? sm[plo] : INFINITY;
      }
    }
  }
  __syncthreads();
  return level_index_view<F32>(sm, levels, nl);
}

inline size_t level_index_smem(int nl) {
  return sizeof(double) * (nl + kCells + 1) + sizeof(uint16_t) * (kCells + 1);
}

template <typename T>
__device__ __forceinline__ void load_octet(const T* p, T v[8]) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = ld4<true>(reinterpret_cast<const float*>(p));
    const float4 b = ld4<true>(reinterpret_cast<const float*>(p) + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 d = ld2d<true>(reinterpret_cast<const double*>(p) + 2 * k);
      v[2 * k] = d.x;
      v[2 * k + 1] = d.y;
    }
  }
}

// One warp per bucket; full buckets (n == S == 256*G) are held in registers
// (G octets per lane, vector loads), short tail buckets take the octet loop
// with scalar loads.
// Pack / store the 8 codes of one octet (8*bits bits = `bits` bytes at byte o*bits).
__device__ __forceinline__ void store_packed(uint8_t* base, int64_t o, unsigned __int128 w, int bits) {
  uint8_t* p = base + o * bits;
  if (bits == 8) *reinterpret_cast<unsigned long long*>(p) = (unsigned long long)w;
  else if (bits == 4) *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
  else if (bits == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
  else if (bits == 1) *p = (uint8_t)w;
  else if (bits == 16) {
    reinterpret_cast<unsigned long long*>(p)[0] = (unsigned long long)w;
    reinterpret_cast<unsigned long long*>(p)[1] = (unsigned long long)(w >> 64);
  } else {
    for (int k = 0; k < bits; ++k) p[k] = (uint8_t)(w >> (8 * k));
  }
}

// One bucket element by element on the exact route: short tail buckets, and
// f32 buckets whose 1/span overflows the prefilter.  Rare; kept out of line so
// the unrolled hot loop stays small in the instruction cache.
template <typename T>
static __device__ __noinline__ void levels_bucket_generic(double* smx, const double* levels, int nl, const T* x, int n, uint8_t* cbase,
                                                          int bits, float lof, float inv32, bool pf, double lo,
                                                          double inv, double span, bool degenerate, bool constant,
                                                          int lane) {
  using Tr = InTraits<T>;
  const LevelIndex ix = level_index_view<sizeof(T) == 4>(smx, levels, nl);
  const int64_t lim = payload_bytes(n, bits);
  for (int o = lane; 8 * o < n; o += 32) {
    unsigned __int128 w = 0;
    for (int i = 0; i < 8; ++i) {
      const int e = 8 * o + i;
      uint32_t c = 0;
      if (!degenerate && e < n) {
        const double a = __dsub_rn(Tr::to_d(x[e]), lo);
        if (constant) {
          c = (uint32_t)ix.fixed;
        } else if constexpr (sizeof(T) == 8) {
          c = ix.code(a, inv, span);
        } else {
          bool sl = true;
          if (pf) c = ix.code_fast32((float)x[e], lof, inv32, sl);
          if (sl) c = ix.code_slow(a, inv, span);
        }
      }
      w |= (unsigned __int128)c << (i * bits);
    }
    const int64_t ob = (int64_t)o * bits;
    if (ob + bits <= lim && 8 * o + 8 <= n) {
      store_packed(cbase, o, w, bits);
    } else {
      for (int k = 0; k < bits && ob + k < lim; ++k) cbase[ob + k] = (uint8_t)(w >> (8 * k));
    }
  }
}

// One warp per bucket; full buckets (n == S == 256*G) are held in registers
// (G octets per lane, vector loads) and coded branch-free (f32 prefilter for
// f32 inputs, fp64 cells for f64); uncertified elements are re-coded exactly and
// patched into the packed word.
template <typename T, int G, int BITS>
__global__ void __launch_bounds__(256) quantize_levels_hold_kernel(const __grid_constant__ QJobTable tab,
                                                                   const double* __restrict__ levels, int nl) {
  extern __shared__ double smx[];
  const LevelIndex ix = build_level_index<sizeof(T) == 4>(smx, levels, nl);
  const int64_t poff = q_parity_off(tab);
  using Tr = InTraits<T>;
  using K = typename Tr::Key;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket, bits = BITS ? BITS : tab.bits;
  const uint32_t cmask = (1u << bits) - 1u;
  const int64_t pbs = payload_bytes(S, bits);
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const BucketRef br = resolve_q(tab, b, S);
    const QJob& J = tab.jobs[br.j];
    const int n = br.n;
    const T* x = reinterpret_cast<const T*>(J.x) + br.off;
    uint8_t* cbase = J.codes + poff + br.lb * pbs;
    const bool full = n == S;
    T v[G][8];
    K mnk = Tr::kMax, mxk = Tr::kMin;
    if (full) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        load_octet<T>(x + 256 * g + 8 * lane, v[g]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const K kk = Tr::key(v[g][i]);
          mnk = min(mnk, kk);
          mxk = max(mxk, kk);
        }
      }
    } else {
      for (int i = lane; i < n; i += 32) {
        const K kk = Tr::key(x[i]);
        mnk = min(mnk, kk);
        mxk = max(mxk, kk);
      }
    }
    mnk = team_min_k<32>(mnk);
    mxk = team_max_k<32>(mxk);
    const bool nonfinite = n > 0 && !(Tr::kNegInf < mnk && mxk < Tr::kPosInf);
    const float lof = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mnk));
    const float hif = nonfinite ? 0.0f : (float)Tr::to_d(Tr::from_key(mxk));
    const bool degenerate = nonfinite || !(lof < hif) || nl == 1;
    const bool constant = !degenerate && ix.fixed >= 0;  // every element clips to one level
    if (nonfinite && lane == 0 && tab.bad_index != nullptr) {
      const int i = first_nonfinite<T>(x, n);
      atomicMin(tab.bad_index, ((unsigned long long)br.j << 40) | (unsigned long long)(br.off + i));
    }
    const double lo = (double)lof;
    const double span = __dsub_rn((double)hif, lo);
    const double inv = __drcp_rn(span);
    const float inv32 = __frcp_rn(__fsub_rn(hif, lof));
    const bool pf = sizeof(T) == 4 && isfinite(inv32) && inv32 != 0.0f;  // f32 prefilter representable
    if (full && !degenerate && !constant && (sizeof(T) == 8 || pf)) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        unsigned __int128 w = 0;
        uint32_t slow = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          bool sl;
          uint32_t c;
          if constexpr (sizeof(T) == 4) c = ix.code_fast32(v[g][i], lof, inv32, sl);
          else c = ix.code_fast(__dsub_rn(v[g][i], lo), inv, sl);
          slow |= (uint32_t)sl << i;
          w |= (unsigned __int128)c << (i * bits);
        }
        while (slow) {  // rare: near a mid or in a multi-mid cell; re-read x (L1 hit)
          const int i = __ffs(slow) - 1;
          slow &= slow - 1;
          const uint32_t c = ix.code_slow(__dsub_rn(Tr::to_d(x[256 * g + 8 * lane + i]), lo), inv, span);
          w = (w & ~((unsigned __int128)cmask << (i * bits))) | ((unsigned __int128)c << (i * bits));
        }
        store_packed(cbase, 32 * g + lane, w, bits);
      }
    } else if (full && (degenerate || constant)) {
      const uint32_t c = degenerate ? 0u : (uint32_t)ix.fixed;
      unsigned __int128 w = 0;
      for (int i = 0; i < 8; ++i) w |= (unsigned __int128)c << (i * bits);
#pragma unroll
      for (int g = 0; g < G; ++g) store_packed(cbase, 32 * g + lane, w, bits);
    } else {
      levels_bucket_generic<T>(smx, levels, nl, x, n, cbase, bits, lof, inv32, pf, lo, inv, span, degenerate, constant,
                               lane);
    }
    if (lane == 0) {
      float* m = meta_at(J.meta, poff) + 3 * br.lb;
      m[0] = 0.0f;
      m[1] = lof;
      m[2] = hif;
    }
  }
}

// Dequant fast path: lane per octet, codes read as one `bits`-byte word, the
// table in smem, vector stores.  S % 8 == 0 and aligned buffers (host-checked).
template <int OUT>
__global__ void __launch_bounds__(256) dequant_levels_vec_kernel(const __grid_constant__ DJobTable tab,
                                                                 const double* __restrict__ levels) {
  extern __shared__ double sq[];
  const int nl = 1 << tab.bits;
  for (int i = threadIdx.x; i < nl; i += blockDim.x) sq[i] = levels[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int S = tab.bucket, bits = tab.bits;
  const uint32_t mask = (1u << bits) - 1u;
  const int64_t pbs = payload_bytes(S, bits);
  const int64_t poff = d_parity_off(tab);  // communicator slot parity (0 outside collectives)
  for (int64_t b = warp; b < tab.total_buckets; b += nwarps) {
    const int j = find_job_d(tab, b);
    const DJob& J = tab.jobs[j];
    const int64_t lb = b - J.bucket_base, off = lb * S;
    const int n = (int)min((int64_t)S, J.length - off);
    const float* m = meta_at(J.meta[0], poff) + 3 * lb;
    const double lo = (double)m[1];
    const double span = __dsub_rn((double)m[2], lo);
    const uint8_t* cp = J.codes[0] + poff + lb * pbs;
    const int64_t lim = payload_bytes(n, bits);
    for (int o = lane; 8 * o < n; o += 32) {
      const uint8_t* p = cp + (int64_t)o * bits;
      unsigned __int128 w = 0;
      if (8 * o + 8 <= n) {
        if (bits == 8) w = *reinterpret_cast<const unsigned long long*>(p);
        else if (bits == 4) w = *reinterpret_cast<const uint32_t*>(p);
        else if (bits == 2) w = *reinterpret_cast<const uint16_t*>(p);
        else if (bits == 1) w = *p;
        else if (bits == 16)
          w = (unsigned __int128)reinterpret_cast<const unsigned long long*>(p)[0] |
              ((unsigned __int128)reinterpret_cast<const unsigned long long*>(p)[1] << 64);
        else
          for (int k = 0; k < bits; ++k) w |= (unsigned __int128)p[k] << (8 * k);
      } else {
        for (int k = 0; k < bits && (int64_t)o * bits + k < lim; ++k) w |= (unsigned __int128)p[k] << (8 * k);
      }
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t c = (uint32_t)(w >> (i * bits)) & mask;
        v[i] = __dadd_rn(lo, __dmul_rn(sq[c], span));  // lo + levels[codes] * span
      }
      const int64_t e0 = off + 8 * o;
      if (8 * o + 8 <= n) {
        if (OUT == 0) {
          float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(J.out) + e0);
          d[0] = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]),
                             __double2float_rn(v[3]));
          d[1] = make_float4(__double2float_rn(v[4]), __double2float_rn(v[5]), __double2float_rn(v[6]),
                             __double2float_rn(v[7]));
        } else if (OUT == 1) {
          double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(J.out) + e0);
#pragma unroll
          for (int k = 0; k < 4; ++k) d[k] = make_double2(v[2 * k], v[2 * k + 1]);
        } else {
          __nv_bfloat16 h[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) h[i] = __float2bfloat16_rn(__double2float_rn(v[i]));
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(J.out) + e0) = *reinterpret_cast<uint4*>(h);
        }
      } else {
        for (int i = 0; i < 8 && 8 * o + i < n; ++i) {
          if (OUT == 0) reinterpret_cast<float*>(J.out)[e0 + i] = __double2float_rn(v[i]);
          else if (OUT == 1) reinterpret_cast<double*>(J.out)[e0 + i] = v[i];
          else reinterpret_cast<__nv_bfloat16*>(J.out)[e0 + i] = __float2bfloat16_rn(__double2float_rn(v[i]));
        }
      }
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

template <typename T, int G, int BITS>
static void launch_hold_b(const QJobTable& tab, const double* levels, int nl, int sms, cudaStream_t s) {
  auto k = quantize_levels_hold_kernel<T, G, BITS>;
  const size_t sm = level_index_smem(nl);
  static thread_local size_t attr[64] = {};  // opt in above the default once per instantiation and device
  ensure_smem_attr(k, sm, attr);
  k<<<persistent_grid(k, 256, sm, tab.total_buckets, 1, sms), 256, sm, s>>>(tab, levels, nl);
}

template <typename T, int G>
static void launch_hold(const QJobTable& tab, const double* levels, int nl, int sms, cudaStream_t s) {
  if (tab.bits == 8) launch_hold_b<T, G, 8>(tab, levels, nl, sms, s);
  else if (tab.bits == 4) launch_hold_b<T, G, 4>(tab, levels, nl, sms, s);
  else launch_hold_b<T, G, 0>(tab, levels, nl, sms, s);
}

template <typename T>
static bool launch_q_hold(const QJobTable& tab, const double* levels, int nl, int sms, cudaStream_t s) {
  switch (tab.bucket) {
    case 256: launch_hold<T, 1>(tab, levels, nl, sms, s); return true;
    case 512: launch_hold<T, 2>(tab, levels, nl, sms, s); return true;
    case 1024: launch_hold<T, 4>(tab, levels, nl, sms, s); return true;
    case 2048:
      if constexpr (sizeof(T) == 4) {
        launch_hold<T, 8>(tab, levels, nl, sms, s);
        return true;
      }
      return false;
    default: return false;
  }
}

cudaError_t launch_quantize_levels(const QJobTable& tab, int in_f64, const double* levels, int nl, bool vec, int sms,
                                   cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  if (vec && nl <= (1 << kSmemLevelBits)) {
    const bool done = in_f64 ? launch_q_hold<double>(tab, levels, nl, sms, s) : launch_q_hold<float>(tab, levels, nl, sms, s);
    if (done) return cudaGetLastError();
  }
  const int grid = grid_for(tab.total_buckets, 1, sms);
  const size_t sm = nl <= (1 << kSmemLevelBits) ? sizeof(double) * nl : 0;
  if (in_f64) quantize_levels_kernel<double><<<grid, 256, sm, s>>>(tab, levels, nl);
  else quantize_levels_kernel<float><<<grid, 256, sm, s>>>(tab, levels, nl);
  return cudaGetLastError();
}

cudaError_t launch_dequant_levels(const DJobTable& tab, const double* levels, bool vec, int sms, cudaStream_t s) {
  if (tab.total_buckets == 0) return cudaSuccess;
  if (vec && tab.bits <= kSmemLevelBits && tab.bucket % 8 == 0) {
    const size_t sm = sizeof(double) << tab.bits;
    if (tab.out_dtype == 0) {
      auto k = dequant_levels_vec_kernel<0>;
      k<<<persistent_grid(k, 256, sm, tab.total_buckets, 1, sms), 256, sm, s>>>(tab, levels);
    } else if (tab.out_dtype == 1) {
      auto k = dequant_levels_vec_kernel<1>;
      k<<<persistent_grid(k, 256, sm, tab.total_buckets, 1, sms), 256, sm, s>>>(tab, levels);
    } else {
      auto k = dequant_levels_vec_kernel<2>;
      k<<<persistent_grid(k, 256, sm, tab.total_buckets, 1, sms), 256, sm, s>>>(tab, levels);
    }
    return cudaGetLastError();
  }
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
