// qsdp_device.cuh -- device-side building blocks shared by the sm_100a kernels.
//
//  * numpy SeedSequence -> PCG64 restated on the device, keyed exactly like the
//    reference's bucket_rng (pkg/src/qsdp/sharded.py:235-240).  The four
//    prefix key fields (root_seed, step, layer, phase) plus the worker field
//    are absorbed on the host once per segment (SeedPrefix); the device absorbs
//    only the per-bucket `start` word(s) and runs generate_state + PCG64 seeding.
//  * 128-bit LCG arithmetic for PCG64 stepping and O(1) jump-ahead:
//    state_{k} = A_k * state_0 + G_k * inc  (mod 2^128).
//  * the job tables the batched kernels take as __grid_constant__ parameters.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qsdp {

// ---------------------------------------------------------------------------
// SeedSequence constants (numpy/random/bit_generator.pyx).
// ---------------------------------------------------------------------------
constexpr uint32_t SS_INIT_A = 0x43b0d7e5u;
constexpr uint32_t SS_MULT_A = 0x931e8875u;
constexpr uint32_t SS_INIT_B = 0x8b51f9ddu;
constexpr uint32_t SS_MULT_B = 0x58f38dedu;
constexpr uint32_t SS_MIX_L = 0xca01f9ddu;
constexpr uint32_t SS_MIX_R = 0x4973f715u;

constexpr uint64_t PCG_MULT_HI = 0x2360ED051FC65DA4ull;
constexpr uint64_t PCG_MULT_LO = 0x4385DF649FCCF645ull;

// Pool state after absorbing the segment-constant key words.
struct SeedPrefix {
  uint32_t pool[4];
  uint32_t hash_const;
  uint32_t _pad;
};

struct U128 {
  uint64_t lo, hi;
};

__host__ __device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= SS_MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__host__ __device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

__host__ __device__ __forceinline__ void ss_absorb(uint32_t pool[4], uint32_t& hc, uint32_t w) {
#pragma unroll
  for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(w, hc));
}

// Absorb an integer key field (_int_to_uint32_array: LE 32-bit chunks, 0 -> [0]).
__host__ __device__ __forceinline__ void ss_absorb_u64(uint32_t pool[4], uint32_t& hc, uint64_t v) {
  ss_absorb(pool, hc, (uint32_t)v);
  if (v >> 32) ss_absorb(pool, hc, (uint32_t)(v >> 32));
}

// generate_state(4, uint64) -> v[0..3]; then PCG64 seeding
// (pcg_setseq_128_srandom_r): inc = (seq<<1)|1, state = (inc+init)*M + inc.
__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
#ifdef __CUDACC__
// add128 with the carry through the flag (IADD3 carry chain instead of a 64-bit compare +
// select): 7% fewer SASS in K2's octet loop; used where it measured faster (K2 without the
// fused epilogue -- with it the loop's schedule got worse)
__device__ __forceinline__ U128 add128_cc(U128 a, U128 b) {
  U128 r;
  asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;" : "=l"(r.lo), "=l"(r.hi) : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
  return r;
}
#endif
// a*b + c (mod 2^128)
__host__ __device__ __forceinline__ U128 mad128(U128 a, U128 b, U128 c) { return add128(mul128(a, b), c); }

__host__ __device__ __forceinline__ U128 pcg_mult() { return U128{PCG_MULT_LO, PCG_MULT_HI}; }

// One PCG64 LCG step  s <- s*M + inc (mod 2^128).  (A hand-written 32-bit-limb
// mad.cc carry chain was measured no faster: SASS has no carry-out IMAD, so each
// partial product becomes IMAD + IADD3; the 64-bit form below lets ptxas use
// IMAD.WIDE.U32 pairs.)
__host__ __device__ __forceinline__ U128 pcg_step(U128 s, U128 inc) { return add128(mul128(s, pcg_mult()), inc); }

// Finish SeedSequence for one bucket and seed PCG64; returns (state, inc).
__host__ __device__ __forceinline__ void seed_bucket(const SeedPrefix& pre, uint64_t start, U128& state,
                                                     U128& inc) {
  uint32_t pool[4] = {pre.pool[0], pre.pool[1], pre.pool[2], pre.pool[3]};
  uint32_t hc = pre.hash_const;
  ss_absorb_u64(pool, hc, start);
  uint32_t st[8];
  uint32_t hb = SS_INIT_B;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  const uint64_t v0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  const uint64_t v1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  const uint64_t v2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  const uint64_t v3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
  const U128 init{v1, v0};
  inc.lo = (v3 << 1) | 1ull;
  inc.hi = (v2 << 1) | (v3 >> 63);
  state = mad128(add128(inc, init), pcg_mult(), inc);
}

// SeedSequence prefix: absorb root, step, layer, phase, worker (each coerced to
// LE uint32 words, 0 -> [0]) -- numpy mix_entropy with pool size 4.  The
// bucket's `start` is absorbed last by seed_bucket.
__host__ __device__ __forceinline__ SeedPrefix make_prefix(uint64_t root, uint64_t step, uint64_t layer,
                                                           uint64_t phase, uint64_t worker) {
  uint32_t words[10];
  int n = 0;
  const uint64_t f[5] = {root, step, layer, phase, worker};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    words[n++] = (uint32_t)f[i];
    if (f[i] >> 32) words[n++] = (uint32_t)(f[i] >> 32);
  }
  SeedPrefix p{};
  uint32_t hc = SS_INIT_A;
#pragma unroll
  for (int i = 0; i < 4; ++i) p.pool[i] = ss_hashmix(words[i], hc);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) p.pool[d] = ss_mix(p.pool[d], ss_hashmix(p.pool[s], hc));
  for (int s = 4; s < n; ++s) ss_absorb(p.pool, hc, words[s]);
  p.hash_const = hc;
  return p;
}

// ---------------------------------------------------------------------------
// Counter-based noise: numpy's Philox (Philox4x64-10, numpy/random/src/philox),
// the generator np.random.Generator(np.random.Philox(SeedSequence(key6))).  Its
// key is SeedSequence.generate_state(2, uint64) -- the first four words of the same
// pool the PCG64 seeding draws -- and draw i is word i % 4 of the block with
// counter i / 4 + 1 (numpy increments the counter before its first block), so any
// element's draw is computed directly: no sequential state.
// ---------------------------------------------------------------------------
constexpr uint64_t PHILOX_M0 = 0xD2E7470EE14C6C93ull, PHILOX_M1 = 0xCA5A826395121157ull;
constexpr uint64_t PHILOX_W0 = 0x9E3779B97F4A7C15ull, PHILOX_W1 = 0xBB67AE8584CAA73Bull;
struct Philox4 {
  uint64_t v[4];
};
__host__ __device__ __forceinline__ Philox4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                                          uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    const uint64_t lo0 = PHILOX_M0 * c0, hi0 = mulhi64(PHILOX_M0, c0);
    const uint64_t lo1 = PHILOX_M1 * c2, hi1 = mulhi64(PHILOX_M1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return Philox4{{c0, c1, c2, c3}};
}
// Block `blk` (0-based) of a fresh numpy Philox: counter blk + 1 (256-bit, carry into word 1).
__host__ __device__ __forceinline__ Philox4 philox_block(uint64_t blk, uint64_t k0, uint64_t k1) {
  const uint64_t c0 = blk + 1ull;
  return philox4x64_10(c0, c0 == 0 ? 1ull : 0ull, 0, 0, k0, k1);
}
// SeedSequence(prefix + start).generate_state(2, uint64) -> (k0, k1)
__host__ __device__ __forceinline__ void philox_key(const SeedPrefix& pre, uint64_t start, uint64_t& k0,
                                                    uint64_t& k1) {
  uint32_t pool[4] = {pre.pool[0], pre.pool[1], pre.pool[2], pre.pool[3]};
  uint32_t hc = pre.hash_const;
  ss_absorb_u64(pool, hc, start);
  uint32_t st[4];
  uint32_t hb = SS_INIT_B;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  k0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  k1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

// One PCG64 step (state <- state*M + inc) and XSL-RR output of the new state.
__host__ __device__ __forceinline__ uint64_t pcg_output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
// High 32 bits of the XSL-RR output only (one funnel shift instead of two).
__device__ __forceinline__ uint32_t pcg_output_hi32(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  // rotr64(x, rot) >> 32 == funnel of (xh:xl) by rot, taking the high word.
  // bits [rot+32, rot+64) of the 128-bit word (x:x).
  const uint32_t lo_w = rot < 32 ? xh : xl;
  const uint32_t hi_w = rot < 32 ? xl : xh;
  return __funnelshift_r(lo_w, hi_w, rot & 31);
}

// numpy next_double: (x >> 11) * 2^-53
__host__ __device__ __forceinline__ double u64_to_unit_double(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------------------
// PCG64 jump-ahead table: entry k holds (A_k, G_k) with
//   state_k = A_k * state_0 + G_k * inc,  A_k = M^k,  G_k = sum_{j<k} M^j.
// Entries 0..kJumpTable-1 are filled at library load.
// ---------------------------------------------------------------------------
constexpr int kJumpTable = 256;
struct JumpEntry {
  U128 a, g;
};

// ---------------------------------------------------------------------------
// Job tables for the batched kernels.
// ---------------------------------------------------------------------------
constexpr int kMaxJobs = 64;
#define QSDP_FUSE_MAX_WORLD 8

struct QJob {
  const void* x;          // segment input (element 0 of the segment)
  uint8_t* codes;         // packed-code output (parity-0 slot when the table has a parity source)
  float* meta;            // per-bucket {shift, lo, hi}
  int64_t length;         // elements in the segment
  int64_t global_start;   // key `start` of bucket 0 (sharded.py:243-248)
  int64_t bucket_base;    // prefix: global bucket index of this job's bucket 0
  SeedPrefix seed;        // root, step, layer, phase, worker already absorbed (static step)
  uint64_t key[5];        // raw (root, step, layer, phase, worker) for a device step source
  void* dq_out;           // fused dequant of this segment (element 0), or nullptr (TMA32 path only)
};

struct QJobTable {
  QJob jobs[kMaxJobs];
  int32_t njobs;
  int32_t bits;
  int32_t bucket;
  int32_t inner;
  int64_t total_buckets;
  unsigned long long* bad_index;  // atomicMin target: (job << 40) | element, or nullptr
  // CUDA-graph support: if step_ptr is set, the key's step is key[1] + *step_ptr
  // (read on the device at run time); if parity_ptr is set, outputs move by
  // ((*parity_ptr + parity_adj) & 1) * parity_stride bytes (double-buffered slots).
  const unsigned long long* step_ptr;
  const unsigned long long* parity_ptr;
  int64_t parity_stride;
  int32_t parity_adj;
  // push collectives: every bucket's codes + meta are also copied to
  // (its address + mirror_delta[k]) -- the same slot in a peer's workspace
  int32_t mirror_n;
  int64_t mirror_delta[QSDP_FUSE_MAX_WORLD - 1];
  // fused dequant epilogue (jobs with dq_out): K3's value (lo + code*pitch) + shift,
  // or K4's single-source 0.0 + value (dq_add0), stored as dq_dtype (0 f32, 1 f64, 2 bf16)
  int32_t dq_dtype;
  int32_t dq_add0;
  int32_t dq_nocodes;  // world 1: the fused dequant is the only consumer -> codes not stored
  int32_t noise;       // qsdp_noise: 0 PCG64 (bucket_rng), 1 Philox4x64-10 (counter-based)
  int32_t cta_cap;     // launch only: > 0 caps the TMA32 quantizer's CTAs per SM
};

struct DJob {
  const uint8_t* codes[8];  // sources (1 for plain dequant; P for dequant-accumulate)
  const float* meta[8];
  void* out;                // may be nullptr for a lattice step (then only x moves)
  void* lat_x;              // lattice step: this job's iterate (in / out)
  int64_t length;
  int64_t bucket_base;
  int32_t nsrc;
  int32_t _pad;
};

struct DJobTable {
  DJob jobs[kMaxJobs];
  int32_t njobs;
  int32_t bits;
  int32_t bucket;
  int32_t out_dtype;  // 0 f32, 1 f64, 2 bf16
  int64_t total_buckets;
  int32_t accumulate;  // 0: out = dequant(src0)  1: out = (0.0 + sum_p dequant(src_p)) / divisor
  int32_t divisor;     // K4 divides the fp64 sum by this (the reference's `acc / P`)
  int32_t codes_vec;   // 1: code groups may be read with aligned 2/4/8-byte loads
  int32_t parity_adj;
  const unsigned long long* parity_ptr;  // sources move by ((*p + adj) & 1) * parity_stride bytes
  int64_t parity_stride;
  // Lattice-projected step fused into K4 (optimizer.py:194-229): with the averaged
  // gradient g, x <- d * rint((x - c*g - r) / d) + r, r = uniform(-d/2, d/2) drawn
  // from the keyed stream lat_key (step += *lat_step_ptr when set), start 0.
  int32_t lat_on;
  int32_t lat_xdtype;  // 0 f32, 1 f64
  double lat_c, lat_d, lat_inv_d;  // lat_inv_d = fl(1/d) (certified rounding, exact fallback)
  uint64_t lat_key[5];
  const unsigned long long* lat_step_ptr;
};

// Geometry of one wire message (qsdp_wire.cu).
struct WireGeom {
  int64_t length;      // total elements
  int64_t nb;          // blocks
  int64_t pbs;         // payload bytes of a full block
  int64_t last_n;      // elements of the last block
  int64_t last_pb;     // payload bytes of the last block
  int64_t blk;         // 12 + pbs: wire bytes of a full block
  int64_t msg_bytes;   // 14 + sum over blocks
  int64_t codes_bytes; // (nb-1)*pbs + last_pb
  int32_t bits, bucket;
  uint8_t header[16];  // the 14 header bytes (host-built)
};

__host__ __device__ __forceinline__ int64_t payload_bytes(int64_t len, int bits) { return (len * bits + 7) / 8; }

__device__ __forceinline__ int find_job_q(const QJobTable& t, int64_t b) {
  int j = 0;
  while (j + 1 < t.njobs && t.jobs[j + 1].bucket_base <= b) ++j;
  return j;
}
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long ld_dev_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ int64_t q_parity_off(const QJobTable& t) {
  return t.parity_ptr ? (int64_t)((ld_dev_u64(t.parity_ptr) + (unsigned long long)t.parity_adj) & 1ull) * t.parity_stride
                      : 0;
}
__device__ __forceinline__ int64_t d_parity_off(const DJobTable& t) {
  return t.parity_ptr ? (int64_t)((ld_dev_u64(t.parity_ptr) + (unsigned long long)t.parity_adj) & 1ull) * t.parity_stride
                      : 0;
}
__device__ __forceinline__ SeedPrefix q_seed(const QJobTable& t, const QJob& J) {
  if (t.step_ptr == nullptr) return J.seed;
  return make_prefix(J.key[0], J.key[1] + ld_dev_u64(t.step_ptr), J.key[2], J.key[3], J.key[4]);
}
__device__ __forceinline__ float* meta_at(float* m, int64_t byte_off) {
  return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(m) + byte_off);
}
__device__ __forceinline__ const float* meta_at(const float* m, int64_t byte_off) {
  return reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(m) + byte_off);
}
#endif

__device__ __forceinline__ int find_job_d(const DJobTable& t, int64_t b) {
  int j = 0;
  while (j + 1 < t.njobs && t.jobs[j + 1].bucket_base <= b) ++j;
  return j;
}

}  // namespace qsdp
