// qsdp_capi.cu -- the extern "C" boundary (include/qsdp_b200.h) and the
// multi-GPU collectives C1 (quantized all-gather) / C2 (quantized
// reduce-scatter) over NVLink peer memory.
//
// C1 replaces ShardedMLP._gather (pkg/src/qsdp/sharded.py:323-373):
//   rank r quantizes its own shard (key worker 0) into its local slot; after a
//   system-scope flag barrier every rank PULLS all P slots straight from the
//   peers' HBM over NVLink inside the dequantize kernel, writing the full
//   gathered tensor -- the transfer is fused into the dequant pass.
// C2 replaces ShardedMLP._reduce_scatter (sharded.py:375-433):
//   rank r quantizes all P destination segments of its gradient (key worker r)
//   into P local slots; after the barrier, owner q pulls slot q from sources
//   p = 0..P-1 in order and dequant-accumulates in fp64, then divides by P.
// Slots are double-buffered by call parity, so one barrier per collective
// suffices: a rank rewrites parity k's slots only after every peer has passed
// the barrier of call k+1, i.e. finished reading call k-1's data.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qsdp_b200.h"
#include "qsdp_device.cuh"

namespace qsdp {
cudaError_t launch_quantize_f32(const QJobTable& tab, bool vec, int sms, cudaStream_t s);
cudaError_t launch_quantize_f64(const QJobTable& tab, bool vec, int sms, cudaStream_t s);
cudaError_t launch_quantize_philox(const QJobTable& tab, bool f64, bool vec, int sms, cudaStream_t s);
cudaError_t launch_levels_stochastic(const double* v, int64_t n, const double* q, int nl, const uint64_t* state,
                                     uint32_t* codes, cudaStream_t s);
cudaError_t launch_quantize_stream(const void* x, bool f64, int64_t length, int S, int bits, int inner,
                                   const uint64_t* states, uint32_t* scratch, uint8_t* codes, int64_t codes_bytes,
                                   float* meta, int sms, cudaStream_t s);
cudaError_t launch_dequant(const DJobTable& tab, bool vec, int sms, cudaStream_t s);
cudaError_t upload_jump_f32(const JumpEntry* host);
cudaError_t upload_jump_f64(const JumpEntry* host);
cudaError_t launch_quantize_levels(const QJobTable& tab, int in_f64, const double* levels, int nl, bool vec, int sms,
                                   cudaStream_t s);
cudaError_t launch_dequant_levels(const DJobTable& tab, const double* levels, bool vec, int sms, cudaStream_t s);
cudaError_t launch_learn_levels(const double* values, int64_t n, double* q, int nl, double lr, cudaStream_t s);
cudaError_t launch_wire_encode(const uint8_t* codes, const float* meta, const WireGeom& g, uint8_t* out, int sms,
                               cudaStream_t s);
cudaError_t launch_wire_decode(const uint8_t* msg, const WireGeom& g, int64_t nblk, uint8_t* codes, float* meta,
                               unsigned long long* err, int sms, cudaStream_t s);
cudaError_t launch_pack_codes(const uint32_t* codes, int64_t length, int bucket, int bits, uint8_t* out,
                              int64_t out_bytes, int sms, cudaStream_t s);
cudaError_t launch_unpack_codes(const uint8_t* packed, int64_t length, int bucket, int bits, uint32_t* codes, int sms,
                                cudaStream_t s);
}  // namespace qsdp

using namespace qsdp;

// NVTX range over one C-ABI call (host side: the enqueue of its launches), so an nsys / ncu
// timeline (ncu --nvtx) attributes the kernels to the collective that issued them.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace {

thread_local std::string g_last_error;

qsdp_status fail(qsdp_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

qsdp_status cuda_fail(cudaError_t e, const char* where) {
  return fail(QSDP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define QSDP_CUDA(call)                                    \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);    \
  } while (0)

// --- per-device state: SM count + jump table uploaded once -----------------
struct DeviceState {
  int sms = 0;
  bool jump_ready = false;
};
std::mutex g_mu;
DeviceState g_dev[64];

qsdp_status ensure_device(int& sms) {
  int dev = 0;
  QSDP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceState& d = g_dev[dev & 63];
  if (!d.jump_ready) {
    JumpEntry tab[kJumpTable];
    U128 a{1, 0}, g{0, 0};
    const U128 one{1, 0};
    for (int k = 0; k < kJumpTable; ++k) {
      tab[k].a = a;
      tab[k].g = g;
      g = add128(mul128(pcg_mult(), g), one);  // G_{k+1} = M G_k + 1
      a = mul128(pcg_mult(), a);               // A_{k+1} = M A_k
    }
    QSDP_CUDA(upload_jump_f32(tab));
    QSDP_CUDA(upload_jump_f64(tab));
    QSDP_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    d.jump_ready = true;
  }
  sms = d.sms;
  return QSDP_OK;
}

SeedPrefix key_prefix(const qsdp_key& k, uint64_t worker) {
  return make_prefix(k.root_seed, k.step, k.layer, k.phase, worker);
}

qsdp_status check_cfg(const qsdp_qcfg* c, bool levels = false) {
  if (c == nullptr) return fail(QSDP_EINVAL, "null qsdp_qcfg");
  if (c->bits < 1 || c->bits > 16) return fail(QSDP_EINVAL, "bit_width must be in [1, 16]");
  if (c->bucket < 1) return fail(QSDP_EINVAL, "bucket_size must be >= 1");
  if (levels ? c->inner != QSDP_INNER_LEVELS : (c->inner != QSDP_INNER_SHIFT && c->inner != QSDP_INNER_STOCHASTIC))
    return fail(QSDP_EINVAL, levels ? "levels entry points take inner = QSDP_INNER_LEVELS" : "unknown inner mode");
  if (c->noise != QSDP_NOISE_PCG64_SEEDSEQ && c->noise != QSDP_NOISE_PHILOX4x64)
    return fail(QSDP_EINVAL, "unsupported noise mode");
  return QSDP_OK;
}

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

size_t dtype_size(int dt) { return dt == QSDP_F64 ? 8 : (dt == QSDP_BF16 ? 2 : 4); }

// Split a list of quantize jobs into launches of <= kMaxJobs.
struct QJobSpec {
  const void* x;
  int64_t length, global_start;
  uint8_t* codes;
  float* meta;
  SeedPrefix seed;
  uint64_t key[5];
  void* dq_out = nullptr;  // fused dequant destination (TMA32 path only; see fdq_ok)
};

// Device-side sources that make a launch sequence replayable as a CUDA graph.
struct DynSrc {
  const unsigned long long* step_ptr = nullptr;    // key step += *step_ptr
  const unsigned long long* parity_ptr = nullptr;  // slot parity = (*parity_ptr + adj) & 1
  int64_t parity_stride = 0;
  int32_t parity_adj = 0;
  int32_t sm_cap = 0;    // > 0: size grids for at most this many SMs (comm SM budget)
  int32_t cta_cap = 0;   // > 0: at most this many quantizer CTAs per SM
  int32_t dq_dtype = 0;  // fused dequant epilogue: output dtype and K4's single-source 0.0 + v
  int32_t dq_add0 = 0;
  int32_t dq_nocodes = 0;  // world 1: nobody reads the codes
  int32_t mirror_n = 0;  // push collectives: copy every bucket to these byte offsets too
  int64_t mirror_delta[QSDP_FUSE_MAX_WORLD - 1] = {};
};

// Table builders of the quantize / dequantize launches.
void build_qtab(QJobTable& tab, const std::vector<QJobSpec>& jobs, size_t& i, const qsdp_qcfg* cfg, uint64_t* d_bad,
                const DynSrc& dyn, bool& vec) {
  memset(&tab, 0, sizeof(tab));
  tab.bits = cfg->bits;
  tab.bucket = cfg->bucket;
  tab.inner = cfg->inner;
  tab.noise = cfg->noise;
  tab.cta_cap = dyn.cta_cap;
  tab.bad_index = reinterpret_cast<unsigned long long*>(d_bad);
  tab.step_ptr = dyn.step_ptr;
  tab.parity_ptr = dyn.parity_ptr;
  tab.parity_stride = dyn.parity_stride;
  tab.parity_adj = dyn.parity_adj;
  tab.dq_dtype = dyn.dq_dtype;
  tab.dq_add0 = dyn.dq_add0;
  tab.dq_nocodes = dyn.dq_nocodes;
  tab.mirror_n = dyn.mirror_n;
  for (int k = 0; k < dyn.mirror_n; ++k) tab.mirror_delta[k] = dyn.mirror_delta[k];
  int64_t nb = 0;
  vec = cfg->bucket % 4 == 0;
  int nj = 0;
  for (; i < jobs.size() && nj < kMaxJobs; ++i) {
    const QJobSpec& s = jobs[i];
    if (s.length <= 0) continue;
    QJob& J = tab.jobs[nj++];
    J.x = s.x;
    J.codes = s.codes;
    J.meta = s.meta;
    J.length = s.length;
    J.global_start = s.global_start;
    J.bucket_base = nb;
    J.seed = s.seed;
    for (int w = 0; w < 5; ++w) J.key[w] = s.key[w];
    J.dq_out = s.dq_out;
    nb += (s.length + cfg->bucket - 1) / cfg->bucket;
    vec = vec && aligned(s.x, 16);
  }
  tab.njobs = nj;
  tab.total_buckets = nb;
}

qsdp_status run_quantize(const std::vector<QJobSpec>& jobs, int x_dtype, const qsdp_qcfg* cfg,
                         uint64_t* d_bad, cudaStream_t stream, const DynSrc& dyn = DynSrc(),
                         const double* levels = nullptr, int nlevels = 0) {
  if (x_dtype != QSDP_F32 && x_dtype != QSDP_F64) return fail(QSDP_EINVAL, "input dtype must be f32 or f64");
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  if (dyn.sm_cap > 0 && dyn.sm_cap < sms) sms = dyn.sm_cap;
  size_t i = 0;
  while (i < jobs.size()) {
    QJobTable tab;
    bool vec = false;
    build_qtab(tab, jobs, i, cfg, d_bad, dyn, vec);
    if (tab.njobs == 0) continue;
    bool codes_ok = true;  // wide code stores of the levels fast path
    for (int k = 0; k < tab.njobs; ++k) codes_ok = codes_ok && aligned(tab.jobs[k].codes, 8);
    cudaError_t e = levels != nullptr      ? launch_quantize_levels(tab, x_dtype == QSDP_F64, levels, nlevels, vec && codes_ok, sms, stream)
                    : cfg->noise == QSDP_NOISE_PHILOX4x64 && cfg->inner == QSDP_INNER_STOCHASTIC
                          ? launch_quantize_philox(tab, x_dtype == QSDP_F64, vec, sms, stream)
                    : x_dtype == QSDP_F64 ? launch_quantize_f64(tab, vec, sms, stream)
                                          : launch_quantize_f32(tab, vec, sms, stream);
    if (e != cudaSuccess) return cuda_fail(e, "quantize kernel launch");
  }
  return QSDP_OK;
}

struct DJobSpec {
  const uint8_t* codes[8];
  const float* meta[8];
  int nsrc;
  int64_t length;
  void* out;
  void* lat_x = nullptr;  // lattice step iterate (K4 epilogue)
};

void build_dtab(DJobTable& tab, const std::vector<DJobSpec>& jobs, size_t& i, const qsdp_qcfg* cfg, int accumulate,
                int divisor, int out_dtype, const DynSrc& dyn, bool& vec, const qsdp_lattice* lat = nullptr) {
  memset(&tab, 0, sizeof(tab));
  tab.bits = cfg->bits;
  tab.bucket = cfg->bucket;
  tab.out_dtype = out_dtype;
  tab.accumulate = accumulate;
  tab.divisor = divisor < 1 ? 1 : divisor;
  tab.parity_ptr = dyn.parity_ptr;
  tab.parity_stride = dyn.parity_stride;
  tab.parity_adj = dyn.parity_adj;
  vec = cfg->bucket % 4 == 0;
  bool cvec = cfg->bucket % 8 == 0;
  int64_t nb = 0;
  int nj = 0;
  for (; i < jobs.size() && nj < kMaxJobs; ++i) {
    const DJobSpec& s = jobs[i];
    if (s.length <= 0) continue;
    DJob& J = tab.jobs[nj++];
    for (int p = 0; p < s.nsrc; ++p) {
      J.codes[p] = s.codes[p];
      J.meta[p] = s.meta[p];
      cvec = cvec && aligned(s.codes[p], 8);
    }
    J.nsrc = s.nsrc;
    J.out = s.out;
    J.lat_x = s.lat_x;
    J.length = s.length;
    J.bucket_base = nb;
    nb += (s.length + cfg->bucket - 1) / cfg->bucket;
    vec = vec && aligned(s.out, out_dtype == QSDP_BF16 ? 8 : 16);
  }
  tab.njobs = nj;
  tab.total_buckets = nb;
  tab.codes_vec = cvec ? 1 : 0;
  if (lat != nullptr) {
    tab.lat_on = 1;
    tab.lat_xdtype = lat->x_dtype == QSDP_F64 ? 1 : 0;
    tab.lat_c = lat->lr_over_beta;
    tab.lat_d = lat->delta;
    tab.lat_inv_d = 1.0 / lat->delta;
    tab.lat_key[0] = lat->shift_key.root_seed;
    tab.lat_key[1] = lat->shift_key.step;
    tab.lat_key[2] = lat->shift_key.layer;
    tab.lat_key[3] = lat->shift_key.phase;
    tab.lat_key[4] = lat->shift_key.worker;
    tab.lat_step_ptr = dyn.step_ptr;
  }
}

qsdp_status run_dequant(const std::vector<DJobSpec>& jobs, const qsdp_qcfg* cfg, int accumulate,
                        int divisor, int out_dtype, cudaStream_t stream, const DynSrc& dyn = DynSrc(),
                        const double* levels = nullptr, const qsdp_lattice* lat = nullptr) {
  if (out_dtype != QSDP_F32 && out_dtype != QSDP_F64 && out_dtype != QSDP_BF16)
    return fail(QSDP_EINVAL, "output dtype must be f32, f64 or bf16");
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  if (dyn.sm_cap > 0 && dyn.sm_cap < sms) sms = dyn.sm_cap;
  for (const DJobSpec& s : jobs)
    if (s.length > 0 && (s.nsrc < 1 || s.nsrc > 8)) return fail(QSDP_EINVAL, "nsrc must be in [1, 8]");
  size_t i = 0;
  while (i < jobs.size()) {
    DJobTable tab;
    bool vec = false;
    build_dtab(tab, jobs, i, cfg, accumulate, divisor, out_dtype, dyn, vec, lat);
    if (tab.njobs == 0) continue;
    bool out16 = true;  // 16-byte vector stores of the levels fast path (bf16 included)
    for (int k = 0; k < tab.njobs; ++k) out16 = out16 && aligned(tab.jobs[k].out, 16);
    cudaError_t e = levels != nullptr ? launch_dequant_levels(tab, levels, vec && out16 && tab.codes_vec, sms, stream)
                                      : launch_dequant(tab, vec, sms, stream);
    if (e != cudaSuccess) return cuda_fail(e, "dequantize kernel launch");
  }
  return QSDP_OK;
}

int64_t payload(int64_t len, int bits) { return (len * bits + 7) / 8; }

}  // namespace

// ===========================================================================
// extern "C" entry points
// ===========================================================================
extern "C" {

const char* qsdp_last_error(void) { return g_last_error.c_str(); }
const char* qsdp_version(void) { return "qsdp_b200 0.1 (sm_100a)"; }

int64_t qsdp_num_buckets(int64_t length, int32_t bucket) {
  if (length <= 0 || bucket < 1) return 0;
  return (length + bucket - 1) / bucket;
}

int64_t qsdp_codes_bytes(int64_t length, const qsdp_qcfg* cfg) {
  if (length <= 0 || cfg == nullptr || cfg->bucket < 1) return 0;
  const int64_t nb = qsdp_num_buckets(length, cfg->bucket);
  return (nb - 1) * payload(cfg->bucket, cfg->bits) + payload(length - (nb - 1) * cfg->bucket, cfg->bits);
}

int64_t qsdp_message_size_bits(int64_t length, const qsdp_qcfg* cfg) {
  // HEADER_BITS + sum(BLOCK_META_BITS + 8*payload) (wire.py:47-51, 187-192)
  int64_t bits = 14 * 8;
  if (length <= 0) return bits;
  return bits + 96 * qsdp_num_buckets(length, cfg->bucket) + 8 * qsdp_codes_bytes(length, cfg);
}

void qsdp_shard_bounds(int64_t size, int32_t world, qsdp_segment* out) {
  const int64_t base = world > 0 ? size / world : 0;
  for (int p = 0; p < world; ++p) {
    out[p].global_start = p * base;
    out[p].length = (p == world - 1) ? size - p * base : base;
  }
}

qsdp_status qsdp_quantize(const void* x, int32_t x_dtype, qsdp_segment seg, const qsdp_qcfg* cfg,
                          const qsdp_key* key, uint8_t* codes, float* meta, uint64_t* d_bad, void* stream) {
  NvtxRange nvtx_("qsdp_quantize");
  qsdp_qitem it;
  it.x = x;
  it.seg = seg;
  it.key = *key;
  it.codes = codes;
  it.meta = meta;
  return qsdp_quantize_batch(&it, 1, x_dtype, cfg, d_bad, stream);
}

qsdp_status qsdp_quantize_batch(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                const qsdp_qcfg* cfg, uint64_t* d_bad, void* stream) {
  NvtxRange nvtx_("qsdp_quantize_batch");
  return qsdp_quantize_batch_dstep(items, nitems, x_dtype, cfg, d_bad, nullptr, stream);
}

static qsdp_status quantize_items(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype, const qsdp_qcfg* cfg,
                                  uint64_t* d_bad, const uint64_t* d_step, const double* levels, int nlevels,
                                  void* stream) {
  qsdp_status st = check_cfg(cfg, levels != nullptr);
  if (st != QSDP_OK) return st;
  if (nitems < 0 || (nitems > 0 && items == nullptr)) return fail(QSDP_EINVAL, "bad item list");
  std::vector<QJobSpec> jobs;
  jobs.reserve(nitems);
  for (int i = 0; i < nitems; ++i) {
    const qsdp_qitem& it = items[i];
    if (it.seg.length < 0 || it.seg.global_start < 0) return fail(QSDP_EINVAL, "negative segment");
    if (it.seg.length > 0 && (it.x == nullptr || it.codes == nullptr || it.meta == nullptr))
      return fail(QSDP_EINVAL, "null buffer");
    const bool direct = cfg->bits == 2 || cfg->bits == 4 || cfg->bits == 8 || cfg->bits == 16;
    if (direct && it.seg.length > 0 && !aligned(it.codes, 8))
      return fail(QSDP_EINVAL, "codes buffer must be 8-byte aligned");
    QJobSpec s;
    s.x = it.x;
    s.length = it.seg.length;
    s.global_start = it.seg.global_start;
    s.codes = it.codes;
    s.meta = it.meta;
    s.seed = key_prefix(it.key, it.key.worker);
    s.key[0] = it.key.root_seed;
    s.key[1] = it.key.step;
    s.key[2] = it.key.layer;
    s.key[3] = it.key.phase;
    s.key[4] = it.key.worker;
    jobs.push_back(s);
  }
  DynSrc dyn;
  dyn.step_ptr = reinterpret_cast<const unsigned long long*>(d_step);
  return run_quantize(jobs, x_dtype, cfg, d_bad, reinterpret_cast<cudaStream_t>(stream), dyn, levels, nlevels);
}

qsdp_status qsdp_quantize_batch_dstep(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                      const qsdp_qcfg* cfg, uint64_t* d_bad, const uint64_t* d_step,
                                      void* stream) {
  NvtxRange nvtx_("qsdp_quantize_batch_dstep");
  return quantize_items(items, nitems, x_dtype, cfg, d_bad, d_step, nullptr, 0, stream);
}

static bool pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }

qsdp_status qsdp_levels_stochastic(const double* d_values, int64_t n, const double* d_levels, int32_t nlevels,
                                   const uint64_t* state, uint32_t* d_codes, void* stream) {
  if (n < 0 || nlevels < 2 || state == nullptr) return fail(QSDP_EINVAL, "need n >= 0, >= 2 levels and a stream state");
  if (n > 0 && (d_values == nullptr || d_levels == nullptr || d_codes == nullptr)) return fail(QSDP_EINVAL, "null buffer");
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_levels_stochastic(d_values, n, d_levels, nlevels, state, d_codes,
                                           reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "stochastic levels launch");
  return QSDP_OK;
}

qsdp_status qsdp_quantize_stream(const void* x, int32_t x_dtype, int64_t length, const qsdp_qcfg* cfg,
                                 const uint64_t* d_states, uint8_t* codes, float* meta, uint32_t* d_scratch,
                                 void* stream) {
  NvtxRange nvtx_("qsdp_quantize_stream");
  qsdp_status st = check_cfg(cfg);
  if (st != QSDP_OK) return st;
  if (cfg->noise != QSDP_NOISE_PCG64_SEEDSEQ) return fail(QSDP_EINVAL, "a shared stream replays numpy PCG64");
  if (x_dtype != QSDP_F32 && x_dtype != QSDP_F64) return fail(QSDP_EINVAL, "input dtype must be f32 or f64");
  if (length < 0) return fail(QSDP_EINVAL, "negative length");
  if (length > 0 && (x == nullptr || d_states == nullptr || codes == nullptr || meta == nullptr || d_scratch == nullptr))
    return fail(QSDP_EINVAL, "null buffer");
  int sms = 0;
  st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_quantize_stream(x, x_dtype == QSDP_F64, length, cfg->bucket, cfg->bits, cfg->inner, d_states,
                                         d_scratch, codes, qsdp_codes_bytes(length, cfg), meta, sms,
                                         reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "stream quantize launch");
  return QSDP_OK;
}

qsdp_status qsdp_quantize_levels_batch(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                       const qsdp_qcfg* cfg, const double* d_levels, int32_t nlevels,
                                       uint64_t* d_bad, void* stream) {
  NvtxRange nvtx_("qsdp_quantize_levels_batch");
  if (d_levels == nullptr) return fail(QSDP_EINVAL, "inner 'levels' requires a LevelTable");
  if (!pow2(nlevels)) return fail(QSDP_EINVAL, "level count must be a power of two");
  if (cfg != nullptr && cfg->bits >= 1 && cfg->bits <= 16 && nlevels > (1 << cfg->bits))
    return fail(QSDP_EINVAL, "code out of range for bit_width: level table larger than 2**bits");
  return quantize_items(items, nitems, x_dtype, cfg, d_bad, nullptr, d_levels, nlevels, stream);
}

qsdp_status qsdp_quantize_levels(const void* x, int32_t x_dtype, int64_t length, const qsdp_qcfg* cfg,
                                 const double* d_levels, int32_t nlevels, uint8_t* codes, float* meta,
                                 uint64_t* d_bad, void* stream) {
  qsdp_qitem it;
  memset(&it, 0, sizeof(it));
  it.x = x;
  it.seg.length = length;
  it.codes = codes;
  it.meta = meta;
  return qsdp_quantize_levels_batch(&it, 1, x_dtype, cfg, d_levels, nlevels, d_bad, stream);
}

qsdp_status qsdp_dequantize(const uint8_t* codes, const float* meta, int64_t length, const qsdp_qcfg* cfg,
                            void* out, int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_dequantize");
  qsdp_ditem it;
  memset(&it, 0, sizeof(it));
  it.codes[0] = codes;
  it.meta[0] = meta;
  it.nsrc = 1;
  it.length = length;
  it.out = out;
  return qsdp_dequantize_batch(&it, 1, cfg, out_dtype, stream);
}

static qsdp_status dequant_items(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg, int acc,
                                 int32_t divisor, int32_t out_dtype, void* stream,
                                 const double* levels = nullptr) {
  qsdp_status st = check_cfg(cfg, levels != nullptr);
  if (st != QSDP_OK) return st;
  std::vector<DJobSpec> jobs;
  jobs.reserve(nitems);
  for (int i = 0; i < nitems; ++i) {
    const qsdp_ditem& it = items[i];
    if (it.length < 0) return fail(QSDP_EINVAL, "negative length");
    if (it.nsrc < 1 || it.nsrc > 8) return fail(QSDP_EINVAL, "nsrc must be in [1, 8]");
    DJobSpec s;
    memset(&s, 0, sizeof(s));
    for (int p = 0; p < it.nsrc; ++p) {
      s.codes[p] = it.codes[p];
      s.meta[p] = it.meta[p];
    }
    s.nsrc = acc ? it.nsrc : 1;
    s.length = it.length;
    s.out = it.out;
    jobs.push_back(s);
  }
  return run_dequant(jobs, cfg, acc, divisor, out_dtype, reinterpret_cast<cudaStream_t>(stream), DynSrc(), levels);
}

qsdp_status qsdp_dequantize_levels_batch(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg,
                                         const double* d_levels, int32_t nlevels, int32_t out_dtype,
                                         void* stream) {
  NvtxRange nvtx_("qsdp_dequantize_levels_batch");
  if (d_levels == nullptr) return fail(QSDP_EINVAL, "mode 'levels' requires a LevelTable");
  if (cfg != nullptr && (cfg->bits < 1 || cfg->bits > 16 || nlevels != (1 << cfg->bits)))
    return fail(QSDP_EINVAL, "level table size does not match bit_width");
  return dequant_items(items, nitems, cfg, 0, 1, out_dtype, stream, d_levels);
}

qsdp_status qsdp_dequantize_levels(const uint8_t* codes, const float* meta, int64_t length,
                                   const qsdp_qcfg* cfg, const double* d_levels, int32_t nlevels, void* out,
                                   int32_t out_dtype, void* stream) {
  qsdp_ditem it;
  memset(&it, 0, sizeof(it));
  it.codes[0] = codes;
  it.meta[0] = meta;
  it.nsrc = 1;
  it.length = length;
  it.out = out;
  return qsdp_dequantize_levels_batch(&it, 1, cfg, d_levels, nlevels, out_dtype, stream);
}

qsdp_status qsdp_learn_levels(const double* d_values, int64_t n, double* d_levels, int32_t nlevels,
                              double learning_rate, void* stream) {
  if (nlevels < 1 || nlevels > 4096 || (nlevels & (nlevels - 1)) != 0)
    return fail(QSDP_EINVAL, "level count must be a power of two <= 4096");
  if (n < 1) return fail(QSDP_EINVAL, "cannot learn levels from an empty value set");
  if (d_values == nullptr || d_levels == nullptr) return fail(QSDP_EINVAL, "null buffer");
  cudaError_t e = launch_learn_levels(d_values, n, d_levels, nlevels, learning_rate,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "learn_levels kernel launch");
  return QSDP_OK;
}

qsdp_status qsdp_dequantize_batch(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg,
                                  int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_dequantize_batch");
  return dequant_items(items, nitems, cfg, 0, 1, out_dtype, stream);
}

qsdp_status qsdp_dequant_accumulate(const uint8_t* const* codes, const float* const* meta, int32_t nsrc,
                                    int64_t length, const qsdp_qcfg* cfg, int32_t divisor, void* out,
                                    int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_dequant_accumulate");
  if (nsrc < 1 || nsrc > 8) return fail(QSDP_EINVAL, "nsrc must be in [1, 8]");
  qsdp_ditem it;
  memset(&it, 0, sizeof(it));
  for (int p = 0; p < nsrc; ++p) {
    it.codes[p] = codes[p];
    it.meta[p] = meta[p];
  }
  it.nsrc = nsrc;
  it.length = length;
  it.out = out;
  return dequant_items(&it, 1, cfg, 1, divisor, out_dtype, stream);
}

qsdp_status qsdp_dequant_accumulate_batch(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg,
                                          int32_t divisor, int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_dequant_accumulate_batch");
  return dequant_items(items, nitems, cfg, 1, divisor, out_dtype, stream);
}

static qsdp_status check_lattice(const qsdp_lattice* lat, const void* x) {
  if (lat == nullptr || x == nullptr) return fail(QSDP_EINVAL, "null lattice argument");
  if (!(lat->delta > 0) || !std::isfinite(lat->delta)) return fail(QSDP_EINVAL, "resolution must be > 0");
  if (!std::isfinite(lat->lr_over_beta)) return fail(QSDP_EINVAL, "step size must be finite");
  if (lat->x_dtype != QSDP_F32 && lat->x_dtype != QSDP_F64) return fail(QSDP_EINVAL, "iterate dtype must be f32 or f64");
  return QSDP_OK;
}

qsdp_status qsdp_dequant_accumulate_lattice(const uint8_t* const* codes, const float* const* meta, int32_t nsrc,
                                            int64_t length, const qsdp_qcfg* cfg, int32_t divisor, void* g_out,
                                            int32_t out_dtype, void* x, const qsdp_lattice* lat, void* stream) {
  qsdp_status st = check_lattice(lat, x);
  if (st != QSDP_OK) return st;
  st = check_cfg(cfg);
  if (st != QSDP_OK) return st;
  if (nsrc < 1 || nsrc > 8) return fail(QSDP_EINVAL, "nsrc must be in [1, 8]");
  std::vector<DJobSpec> jobs(1);
  memset(&jobs[0], 0, sizeof(DJobSpec));
  for (int p = 0; p < nsrc; ++p) {
    jobs[0].codes[p] = codes[p];
    jobs[0].meta[p] = meta[p];
  }
  jobs[0].nsrc = nsrc;
  jobs[0].length = length;
  jobs[0].out = g_out;
  jobs[0].lat_x = x;
  return run_dequant(jobs, cfg, 1, divisor, out_dtype, reinterpret_cast<cudaStream_t>(stream), DynSrc(), nullptr, lat);
}

static void put_u32_le(uint8_t* p, uint32_t v) { memcpy(p, &v, 4); }
static uint32_t get_u32_le(const uint8_t* p) {
  uint32_t v;
  memcpy(&v, p, 4);
  return v;
}

// Geometry of a message with this header (all blocks full but the last).
static WireGeom wire_geom(int bits, int64_t bucket, int64_t nb, int64_t total) {
  WireGeom g;
  memset(&g, 0, sizeof(g));
  g.bits = bits;
  g.bucket = (int32_t)bucket;
  g.length = total;
  g.nb = nb;
  g.pbs = payload(bucket, bits);
  g.last_n = total - (nb - 1) * bucket;
  g.last_pb = payload(g.last_n, bits);
  g.blk = 12 + g.pbs;
  g.msg_bytes = 14 + (nb - 1) * g.blk + 12 + g.last_pb;
  g.codes_bytes = (nb - 1) * g.pbs + g.last_pb;
  g.header[0] = 1;
  g.header[1] = (uint8_t)bits;
  put_u32_le(g.header + 2, (uint32_t)(nb == 1 ? total : bucket));
  put_u32_le(g.header + 6, (uint32_t)nb);
  put_u32_le(g.header + 10, (uint32_t)total);
  return g;
}

qsdp_status qsdp_pack_codes(const uint32_t* codes, int64_t length, const qsdp_qcfg* cfg, uint8_t* out,
                            void* stream) {
  if (cfg == nullptr || cfg->bits < 1 || cfg->bits > 32 || cfg->bucket < 1 || length < 0)
    return fail(QSDP_EINVAL, "bad packing configuration");
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_pack_codes(codes, length, cfg->bucket, cfg->bits, out, qsdp_codes_bytes(length, cfg), sms,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack launch");
  return QSDP_OK;
}

qsdp_status qsdp_unpack_codes(const uint8_t* packed, int64_t length, const qsdp_qcfg* cfg, uint32_t* codes,
                              void* stream) {
  if (cfg == nullptr || cfg->bits < 1 || cfg->bits > 32 || cfg->bucket < 1 || length < 0)
    return fail(QSDP_EINVAL, "bad packing configuration");
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_unpack_codes(packed, length, cfg->bucket, cfg->bits, codes, sms,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "unpack launch");
  return QSDP_OK;
}

qsdp_status qsdp_wire_parse(const uint8_t* hdr, int64_t msg_bytes, qsdp_wire_info* info) {
  if (info == nullptr || (hdr == nullptr && msg_bytes > 0)) return fail(QSDP_EINVAL, "null argument");
  memset(info, 0, sizeof(*info));
  if (msg_bytes < 14)
    return fail(QSDP_ETRUNC, "message of " + std::to_string(msg_bytes) + " bytes is shorter than the header");
  const int version = hdr[0], bits = hdr[1];
  const int64_t bucket = get_u32_le(hdr + 2), count = get_u32_le(hdr + 6), total = get_u32_le(hdr + 10);
  info->version = version;
  info->bits = bits;
  info->bucket = bucket;
  info->blocks = count;
  info->total_length = total;
  if (version != 1) return fail(QSDP_EVERSION, "unsupported wire version " + std::to_string(version));
  if (count == 0) {
    if (msg_bytes != 14 || total != 0) return fail(QSDP_EDECODE, "empty message carries trailing data");
    info->expected_bytes = 14;
    return QSDP_OK;
  }
  if (bits < 1 || bits > 32) return fail(QSDP_ERANGE, "header bit_width " + std::to_string(bits) + " outside [1, 32]");
  if (bucket < 1) return fail(QSDP_EDECODE, "bucket_size must be positive for non-empty messages");
  // last_len = total - (count-1)*bucket, exactly (u32 * u32 needs 64 unsigned bits)
  const __int128 last_len = (__int128)total - (__int128)(count - 1) * (__int128)bucket;
  if (!(last_len >= 1 && last_len <= bucket))
    return fail(QSDP_EDECODE, "total_length " + std::to_string(total) + " inconsistent with " + std::to_string(count) +
                                  " buckets of " + std::to_string(bucket));
  const WireGeom g = wire_geom(bits, bucket, count, total);
  info->expected_bytes = g.msg_bytes;
  // leading blocks whose meta and payload are wholly inside msg_bytes
  int64_t full = (msg_bytes - 14) / g.blk;
  if (full > count - 1) full = count - 1;
  info->complete_blocks = full;
  if (full == count - 1 && 14 + (count - 1) * g.blk + 12 + g.last_pb <= msg_bytes) info->complete_blocks = count;
  return QSDP_OK;
}

qsdp_status qsdp_wire_encode_device(const uint8_t* codes, const float* meta, int64_t length, const qsdp_qcfg* cfg,
                                    uint8_t* d_out, int64_t out_cap, void* stream) {
  // the codec moves bytes: any width a QuantizedBlock may carry (1..32)
  if (cfg == nullptr || cfg->bits < 1 || cfg->bits > 32 || cfg->bucket < 1)
    return fail(QSDP_EINVAL, "bit_width must be in [1, 32] and bucket_size >= 1");
  qsdp_status st = QSDP_OK;
  if (length < 0 || length > 0xffffffffll) return fail(QSDP_EINVAL, "segment length must fit the u32 header field");
  if (d_out == nullptr) return fail(QSDP_EINVAL, "null output");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (length == 0) {  // encode([]) == header (1, 0, 0, 0, 0) (wire.py:110-111)
    if (out_cap < 14) return fail(QSDP_EINVAL, "wire buffer too small");
    const uint8_t h[14] = {1, 0};
    QSDP_CUDA(cudaMemcpyAsync(d_out, h, 14, cudaMemcpyHostToDevice, s));
    return QSDP_OK;
  }
  const WireGeom g = wire_geom(cfg->bits, cfg->bucket, qsdp_num_buckets(length, cfg->bucket), length);
  if (out_cap < g.msg_bytes) return fail(QSDP_EINVAL, "wire buffer too small");
  int sms = 0;
  st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_wire_encode(codes, meta, g, d_out, sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "wire encode launch");
  return QSDP_OK;
}

qsdp_status qsdp_wire_decode_device(const uint8_t* d_msg, const qsdp_wire_info* info, uint8_t* codes, float* meta,
                                    uint64_t* d_err, void* stream) {
  if (info == nullptr || d_err == nullptr) return fail(QSDP_EINVAL, "null argument");
  if (info->blocks == 0 || info->complete_blocks == 0) return QSDP_OK;
  const WireGeom g = wire_geom(info->bits, info->bucket, info->blocks, info->total_length);
  int sms = 0;
  qsdp_status st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  cudaError_t e = launch_wire_decode(d_msg, g, info->complete_blocks, codes, meta,
                                     reinterpret_cast<unsigned long long*>(d_err), sms,
                                     reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "wire decode launch");
  return QSDP_OK;
}

int64_t qsdp_wire_encode(const uint8_t* codes, const float* meta, int64_t length, const qsdp_qcfg* cfg,
                         uint8_t* out, int64_t out_cap) {
  const int64_t need = qsdp_message_size_bits(length, cfg) / 8;
  if (out_cap < need) {
    g_last_error = "wire buffer too small";
    return -1;
  }
  auto put_u32 = [](uint8_t* p, uint32_t v) { memcpy(p, &v, 4); };
  memset(out, 0, 14);
  out[0] = 1;  // WIRE_VERSION
  if (length <= 0) return 14;
  const int64_t nb = qsdp_num_buckets(length, cfg->bucket);
  const int64_t pbs = payload(cfg->bucket, cfg->bits);
  out[1] = (uint8_t)cfg->bits;
  put_u32(out + 2, (uint32_t)(nb == 1 ? length : cfg->bucket));  // blocks[0].length
  put_u32(out + 6, (uint32_t)nb);
  put_u32(out + 10, (uint32_t)length);
  int64_t o = 14;
  for (int64_t j = 0; j < nb; ++j) {
    const int64_t n = length - j * cfg->bucket < cfg->bucket ? length - j * cfg->bucket : cfg->bucket;
    memcpy(out + o, meta + 3 * j, 12);
    o += 12;
    const int64_t pb = payload(n, cfg->bits);
    memcpy(out + o, codes + j * pbs, (size_t)pb);
    o += pb;
  }
  return o;
}

}  // extern "C"

// ===========================================================================
// Multi-GPU communicator (C1 / C2)
// ===========================================================================
// Workspace layout (per rank, one cudaMalloc exported over CUDA IPC):
//   [0, 64)     flags[8]: flags[j] = last epoch rank j signalled to this rank
//   [128, 136)  epoch: collectives completed (advanced by the barrier kernel)
//   [256, ...)  slots[2 parities][world]: packed codes (slot_codes) + meta (slot_meta)
// Every launch reads the epoch on the device, so a whole training step's
// sequence of collectives can be captured once and replayed as a CUDA graph.
struct PeerFlags {
  unsigned long long* flags[QSDP_MAX_WORLD];  // flags[j] = base of rank j's flag array
};

constexpr size_t kEpochOff = 128;
constexpr int kBarrierSMs = 8;

// Failure detection: a peer that never arrives (dead, hung or desynchronised)
// must not hang this rank.  Each waiting lane gives up after `timeout_ns` of
// %globaltimer and records (peer + 1) | (target epoch << 8) in a host-mapped
// word; the host surfaces it as QSDP_EPEER at the next collective or
// qsdp_comm_status() call (errors propagate, never hang -- quantize.py:41-44's
// contract carried over to the transport).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void qsdp_barrier_kernel(PeerFlags pf, int rank, int world, unsigned long long* epoch_ptr,
                                    unsigned long long* err_word, unsigned long long timeout_ns) {
  const int t = threadIdx.x;
  const unsigned long long target = *reinterpret_cast<volatile unsigned long long*>(epoch_ptr) + 1ull;
  if (t < world) {
    __threadfence_system();
    unsigned long long* dst = pf.flags[t] + rank;  // peer t learns "rank reached target"
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(target) : "memory");
    const unsigned long long* mine = pf.flags[rank] + t;
    const unsigned long long t0 = globaltimer_ns();
    unsigned long long v = 0;
    for (unsigned it = 0;; ++it) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= target) break;
      if ((it & 255u) == 255u && globaltimer_ns() - t0 > timeout_ns) {
        atomicCAS(err_word, 0ull, (unsigned long long)(t + 1) | (target << 8));
        __threadfence_system();
        break;
      }
    }
  }
  __syncthreads();
  if (t == 0) *reinterpret_cast<volatile unsigned long long*>(epoch_ptr) = target;
}

// ---------------------------------------------------------------------------
// Full-precision pieces of a group collective (biases / norms: sharded.py:359-371,
// 414-429) ride on the barrier kernel: pushed into the peers' slots before its arrive,
// copied out (all-gather) or averaged in rank order (reduce-scatter) after its wait --
// no extra launch and no separate collective for them.
// ---------------------------------------------------------------------------
constexpr int kMaxRaw = 48;
struct RawPieceDev {
  const uint8_t* src;  // all-gather: this rank's piece; reduce-scatter: destination 0's piece
  int64_t n;           // elements
  int64_t slot_off;    // byte offset of the piece's values in a slot
  int64_t out_off;     // element offset in the output (all-gather: + q * stride)
};
struct RawTable {
  int32_t n, mode;             // pieces; 0 all-gather, 1 reduce-scatter
  int32_t in_dt, out_dt;       // qsdp_dtype
  int32_t world, rank;
  int64_t stride;              // rank_stride (elements)
  int64_t slot_bytes, parity_stride;
  uint8_t* out;
  uint8_t* own_slots;                      // own slot 0, parity 0
  uint8_t* peer_slot[QSDP_MAX_WORLD];      // slot [rank] of rank p's workspace, parity 0 (own: base)
  RawPieceDev p[kMaxRaw];
};

__device__ __forceinline__ int dt_size(int dt) { return dt == QSDP_F64 ? 8 : dt == QSDP_BF16 ? 2 : 4; }
__device__ __forceinline__ double raw_ld(const uint8_t* b, int dt, int64_t i) {
  if (dt == QSDP_F64) return reinterpret_cast<const double*>(b)[i];
  if (dt == QSDP_BF16) return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(b)[i]);
  return (double)reinterpret_cast<const float*>(b)[i];
}
__device__ __forceinline__ void raw_st(uint8_t* b, int dt, int64_t i, double v) {  // round to nearest even
  if (dt == QSDP_F64) reinterpret_cast<double*>(b)[i] = v;
  else if (dt == QSDP_BF16) reinterpret_cast<__nv_bfloat16*>(b)[i] = __double2bfloat16(v);
  else reinterpret_cast<float*>(b)[i] = __double2float_rn(v);
}

// before the arrive: all-gather -- cast this rank's piece to the output dtype into its own
// output slice and into slot [rank] of every peer; reduce-scatter -- destination q's piece
// (input dtype, unchanged) into slot [rank] of owner q.
__device__ void raw_push(const RawTable& rt, int64_t par) {
  const int nt = blockDim.x;
  for (int k = 0; k < rt.n; ++k) {
    const RawPieceDev& pc = rt.p[k];
    for (int q = 0; q < rt.world; ++q) {
      if (rt.mode == 0) {
        uint8_t* dst = q == rt.rank ? rt.out + (size_t)(rt.rank * rt.stride + pc.out_off) * dt_size(rt.out_dt)
                                    : rt.peer_slot[q] + par + pc.slot_off;
        for (int64_t i = threadIdx.x; i < pc.n; i += nt) raw_st(dst, rt.out_dt, i, raw_ld(pc.src, rt.in_dt, i));
      } else {
        const uint8_t* src = pc.src + (size_t)(q * rt.stride) * dt_size(rt.in_dt);
        uint8_t* dst = rt.peer_slot[q] + par + pc.slot_off;
        const int es = dt_size(rt.in_dt);
        for (int64_t i = threadIdx.x; i < pc.n * es / 2; i += nt)
          reinterpret_cast<uint16_t*>(dst)[i] = reinterpret_cast<const uint16_t*>(src)[i];
      }
    }
  }
}

// after the wait: all-gather -- peers' pieces from own slots into the output; reduce-scatter
// -- out = (0.0 + v_0 + v_1 + ... + v_{P-1}) / P in fp64, sources in rank order, rounded once.
__device__ void raw_post(const RawTable& rt, int64_t par) {
  const int nt = blockDim.x;
  for (int k = 0; k < rt.n; ++k) {
    const RawPieceDev& pc = rt.p[k];
    if (rt.mode == 0) {
      const int es = dt_size(rt.out_dt);
      for (int q = 0; q < rt.world; ++q) {
        if (q == rt.rank) continue;
        const uint8_t* src = rt.own_slots + (size_t)q * rt.slot_bytes + par + pc.slot_off;
        uint8_t* dst = rt.out + (size_t)(q * rt.stride + pc.out_off) * es;
        for (int64_t i = threadIdx.x; i < pc.n * es / 2; i += nt)
          reinterpret_cast<uint16_t*>(dst)[i] = reinterpret_cast<const uint16_t*>(src)[i];
      }
    } else {
      uint8_t* dst = rt.out + (size_t)pc.out_off * dt_size(rt.out_dt);
      for (int64_t i = threadIdx.x; i < pc.n; i += nt) {
        double acc = 0.0;
        for (int q = 0; q < rt.world; ++q)
          acc = __dadd_rn(acc, raw_ld(rt.own_slots + (size_t)q * rt.slot_bytes + par + pc.slot_off, rt.in_dt, i));
        raw_st(dst, rt.out_dt, i, __ddiv_rn(acc, (double)rt.world));
      }
    }
  }
}

// The flag barrier with the full-precision pieces (world 1: the pieces only, no flags).
__global__ void __launch_bounds__(512) qsdp_barrier_raw_kernel(PeerFlags pf, unsigned long long* epoch_ptr,
                                                               unsigned long long* err_word,
                                                               unsigned long long timeout_ns, RawTable rt) {
  const int t = threadIdx.x;
  const int rank = rt.rank, world = rt.world;
  const unsigned long long target =
      world > 1 ? *reinterpret_cast<volatile unsigned long long*>(epoch_ptr) + 1ull : 0ull;
  const int64_t par = world > 1 ? (int64_t)(target & 1ull) * rt.parity_stride : 0;
  raw_push(rt, par);
  __threadfence_system();
  __syncthreads();
  if (world > 1 && t < world) {
    unsigned long long* dst = pf.flags[t] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(target) : "memory");
    const unsigned long long* mine = pf.flags[rank] + t;
    const unsigned long long t0 = globaltimer_ns();
    unsigned long long v = 0;
    for (unsigned it = 0;; ++it) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= target) break;
      if ((it & 255u) == 255u && globaltimer_ns() - t0 > timeout_ns) {
        atomicCAS(err_word, 0ull, (unsigned long long)(t + 1) | (target << 8));
        __threadfence_system();
        break;
      }
    }
  }
  __syncthreads();
  raw_post(rt, par);
  if (t == 0 && world > 1) *reinterpret_cast<volatile unsigned long long*>(epoch_ptr) = target;
}

// Full-precision pieces beyond the barrier kernel's table (more than kMaxRaw in one call):
// phase 0 pushes them before the barrier kernel (slot parity of the coming epoch, adj 1),
// phase 1 copies out / averages them after it (the advanced epoch, adj 0).
__global__ void __launch_bounds__(512) qsdp_raw_phase_kernel(const unsigned long long* epoch_ptr, int adj, int phase,
                                                             RawTable rt) {
  const int64_t par = rt.world > 1
                          ? (int64_t)((*reinterpret_cast<const volatile unsigned long long*>(epoch_ptr) + (unsigned long long)adj) & 1ull) *
                                rt.parity_stride
                          : 0;
  if (phase == 0) raw_push(rt, par);
  else raw_post(rt, par);
}

__global__ void qsdp_counter_add_kernel(unsigned long long* p, unsigned long long delta) { *p += delta; }

struct qsdp_comm {
  int rank = 0, world = 1, device = 0;
  int64_t max_seg = 0;
  qsdp_qcfg w{}, g{};
  size_t slot_codes = 0, slot_meta = 0, slot_bytes = 0;
  size_t bytes = 0;
  uint8_t* base = nullptr;
  uint8_t* peer[QSDP_MAX_WORLD] = {};
  bool opened[QSDP_MAX_WORLD] = {};
  const unsigned long long* step_src = nullptr;
  int sm_budget = 0;                // > 0: the collectives' kernels use at most this many SMs
  int sm_default = 0;               // budget when none is set: world > 1 leaves kBarrierSMs SMs free
  int ctas_per_sm = 0;              // > 0: the quantizer's CTAs per SM
  const double* wlevels = nullptr;  // learned weight table (w.inner == QSDP_INNER_LEVELS)
  int wnlevels = 0;
  unsigned long long* err_host = nullptr;  // host-mapped failure word (barrier timeout)
  unsigned long long* err_dev = nullptr;
  unsigned long long timeout_ns = 0;

  static constexpr size_t kFlagBytes = 256;
  uint8_t* slot(uint8_t* b, int idx) const { return b + kFlagBytes + (size_t)idx * slot_bytes; }  // parity 0
  int64_t parity_stride() const { return (int64_t)world * (int64_t)slot_bytes; }
  unsigned long long* epoch() const { return reinterpret_cast<unsigned long long*>(base + kEpochOff); }
};

static size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

extern "C" {

qsdp_status qsdp_counter_add(uint64_t* d_counter, uint64_t delta, void* stream) {
  if (d_counter == nullptr) return fail(QSDP_EINVAL, "null counter");
  qsdp_counter_add_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(d_counter), (unsigned long long)delta);
  QSDP_CUDA(cudaGetLastError());
  return QSDP_OK;
}

qsdp_status qsdp_comm_create(qsdp_comm** out, int32_t rank, int32_t world, int32_t device,
                             int64_t max_segment_elems, const qsdp_qcfg* wcfg, const qsdp_qcfg* gcfg) {
  if (out == nullptr) return fail(QSDP_EINVAL, "null out");
  if (world < 1 || world > QSDP_MAX_WORLD || rank < 0 || rank >= world)
    return fail(QSDP_EINVAL, "world must be in [1, 8] and 0 <= rank < world");
  qsdp_status st = check_cfg(wcfg, wcfg != nullptr && wcfg->inner == QSDP_INNER_LEVELS);
  if (st != QSDP_OK) return st;
  st = check_cfg(gcfg);
  if (st != QSDP_OK) return st;
  QSDP_CUDA(cudaSetDevice(device));
  int sms = 0;
  st = ensure_device(sms);
  if (st != QSDP_OK) return st;
  qsdp_comm* c = new qsdp_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  // A collective's flag barrier is a one-CTA kernel: with several collectives in flight, a
  // persistent quantizer holding every SM would queue it (and every peer waiting on it)
  // behind whole kernels.  Leaving a few SMs free keeps the barriers moving (N=4 bench
  // +2-3%, profiles/r2/smcap_n4.txt).
  c->sm_default = world > 1 && sms > 2 * kBarrierSMs ? sms - kBarrierSMs : 0;
  c->max_seg = max_segment_elems;
  c->w = *wcfg;
  c->g = *gcfg;
  const int64_t cw = qsdp_codes_bytes(max_segment_elems, wcfg), cg = qsdp_codes_bytes(max_segment_elems, gcfg);
  const int64_t nbw = qsdp_num_buckets(max_segment_elems, wcfg->bucket);
  const int64_t nbg = qsdp_num_buckets(max_segment_elems, gcfg->bucket);
  c->slot_codes = round_up((size_t)(cw > cg ? cw : cg) + 16, 256);
  c->slot_meta = round_up((size_t)(nbw > nbg ? nbw : nbg) * 12 + 16, 256);
  c->slot_bytes = c->slot_codes + c->slot_meta;
  c->bytes = qsdp_comm::kFlagBytes + 2 * (size_t)world * c->slot_bytes;
  cudaError_t e = cudaMalloc(&c->base, c->bytes);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(comm workspace)");
  }
  e = cudaMemset(c->base, 0, c->bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(c->base);
    delete c;
    return cuda_fail(e, "cudaMemset(comm workspace)");
  }
  c->peer[rank] = c->base;
  e = cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(unsigned long long), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
  if (e != cudaSuccess) {
    if (c->err_host) cudaFreeHost(c->err_host);
    cudaFree(c->base);
    delete c;
    return cuda_fail(e, "cudaHostAlloc(comm failure word)");
  }
  *reinterpret_cast<volatile unsigned long long*>(c->err_host) = 0;
  // default barrier timeout 60 s (QSDP_TIMEOUT_MS overrides; qsdp_comm_set_timeout at run time)
  const char* tmo = getenv("QSDP_TIMEOUT_MS");
  c->timeout_ns = (unsigned long long)(tmo != nullptr ? atoll(tmo) : 60000ll) * 1000000ull;
  *out = c;
  return QSDP_OK;
}

qsdp_status qsdp_comm_set_weight_levels(qsdp_comm* c, const double* d_levels, int32_t nlevels) {
  if (c == nullptr) return fail(QSDP_EINVAL, "null comm");
  if (c->w.inner != QSDP_INNER_LEVELS) return fail(QSDP_EINVAL, "weight config is not inner 'levels'");
  if (d_levels == nullptr || nlevels != (1 << c->w.bits))
    return fail(QSDP_EINVAL, "level table size does not match bit_width");
  c->wlevels = d_levels;
  c->wnlevels = nlevels;
  return QSDP_OK;
}

qsdp_status qsdp_comm_set_ctas_per_sm(qsdp_comm* c, int32_t ctas) {
  if (c == nullptr) return fail(QSDP_EINVAL, "null comm");
  c->ctas_per_sm = ctas < 0 ? 0 : ctas;
  return QSDP_OK;
}

qsdp_status qsdp_comm_set_sm_budget(qsdp_comm* c, int32_t sms) {
  if (c == nullptr || sms < 0) return fail(QSDP_EINVAL, "bad SM budget");
  c->sm_budget = sms;
  return QSDP_OK;
}

static qsdp_status comm_failed(const qsdp_comm* c);

qsdp_status qsdp_comm_set_timeout(qsdp_comm* c, int64_t timeout_ms) {
  if (c == nullptr || timeout_ms < 1) return fail(QSDP_EINVAL, "timeout must be >= 1 ms");
  c->timeout_ns = (unsigned long long)timeout_ms * 1000000ull;
  return QSDP_OK;
}

qsdp_status qsdp_comm_status(qsdp_comm* c) {
  if (c == nullptr) return fail(QSDP_EINVAL, "null comm");
  return comm_failed(c);
}

qsdp_status qsdp_comm_set_step_source(qsdp_comm* c, const uint64_t* d_step) {
  if (c == nullptr) return fail(QSDP_EINVAL, "null comm");
  c->step_src = reinterpret_cast<const unsigned long long*>(d_step);
  return QSDP_OK;
}

qsdp_status qsdp_comm_ipc_handle(qsdp_comm* c, void* handle) {
  if (c == nullptr || handle == nullptr) return fail(QSDP_EINVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) <= QSDP_IPC_HANDLE_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  QSDP_CUDA(cudaSetDevice(c->device));
  QSDP_CUDA(cudaIpcGetMemHandle(&h, c->base));
  memset(handle, 0, QSDP_IPC_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  return QSDP_OK;
}

qsdp_status qsdp_comm_open_peers(qsdp_comm* c, const void* handles) {
  if (c == nullptr || handles == nullptr) return fail(QSDP_EINVAL, "null argument");
  QSDP_CUDA(cudaSetDevice(c->device));
  for (int j = 0; j < c->world; ++j) {
    if (j == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)j * QSDP_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(QSDP_EPEER, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    c->peer[j] = static_cast<uint8_t*>(p);
    c->opened[j] = true;
  }
  return QSDP_OK;
}

qsdp_status qsdp_comm_destroy(qsdp_comm* c) {
  if (c == nullptr) return QSDP_OK;
  cudaSetDevice(c->device);
  for (int j = 0; j < c->world; ++j)
    if (c->opened[j]) cudaIpcCloseMemHandle(c->peer[j]);
  if (c->base) cudaFree(c->base);
  if (c->err_host) cudaFreeHost(c->err_host);
  delete c;
  return QSDP_OK;
}

// A peer failed to arrive at an earlier barrier: every later collective fails fast.
static qsdp_status comm_failed(const qsdp_comm* c) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(c->err_host);
  if (e == 0) return QSDP_OK;
  const int peer = (int)(e & 255ull) - 1;
  return fail(QSDP_EPEER, "rank " + std::to_string(c->rank) + ": peer " + std::to_string(peer) +
                              " did not arrive at barrier epoch " + std::to_string(e >> 8) + " within " +
                              std::to_string(c->timeout_ns / 1000000ull) + " ms");
}

static qsdp_status comm_barrier(qsdp_comm* c, cudaStream_t s) {
  PeerFlags pf;
  memset(&pf, 0, sizeof(pf));
  for (int j = 0; j < c->world; ++j) {
    if (c->peer[j] == nullptr) return fail(QSDP_EPEER, "peers not opened");
    pf.flags[j] = reinterpret_cast<unsigned long long*>(c->peer[j]);
  }
  qsdp_barrier_kernel<<<1, 32, 0, s>>>(pf, c->rank, c->world, c->epoch(), c->err_dev, c->timeout_ns);
  QSDP_CUDA(cudaGetLastError());
  return QSDP_OK;
}

static qsdp_status check_segs(const qsdp_comm* c, const qsdp_segment* segs) {
  if (segs == nullptr) return fail(QSDP_EINVAL, "null segments");
  for (int p = 0; p < c->world; ++p) {
    if (segs[p].length < 0 || segs[p].length > c->max_seg)
      return fail(QSDP_EINVAL, "segment longer than the communicator's max_segment_elems");
    if (segs[p].global_start < segs[0].global_start) return fail(QSDP_EINVAL, "segments must start at segs[0]");
  }
  return QSDP_OK;
}

// Dynamic sources for one side of a collective: the quantize launch runs
// before the barrier advances the epoch (adj 1), the dequant launch after (adj 0).
static DynSrc comm_dyn(const qsdp_comm* c, int adj) {
  DynSrc d;
  d.step_ptr = c->step_src;
  d.sm_cap = c->sm_budget > 0 ? c->sm_budget : c->sm_budget < 0 ? 0 : c->sm_default;
  d.cta_cap = c->ctas_per_sm;
  if (c->world > 1) {
    d.parity_ptr = c->epoch();
    d.parity_stride = c->parity_stride();
    d.parity_adj = adj;
  }
  return d;
}

static QJobSpec comm_qjob(const void* x, const qsdp_segment& seg, uint8_t* slot, size_t slot_codes,
                          const qsdp_key& key, uint64_t worker) {
  QJobSpec q;
  q.x = x;
  q.length = seg.length;
  q.global_start = seg.global_start;
  q.codes = slot;
  q.meta = reinterpret_cast<float*>(slot + slot_codes);
  q.seed = key_prefix(key, worker);
  q.key[0] = key.root_seed;
  q.key[1] = key.step;
  q.key[2] = key.layer;
  q.key[3] = key.phase;
  q.key[4] = worker;
  return q;
}

// The push all-gather needs the quantizer that copies buckets out (the TMA32
// kernel: direct widths, S % 8 == 0, 72 <= S, S * sizeof(T) <= 16 KB).
static bool push_ok(const qsdp_comm* c, const qsdp_qcfg* cfg, int in_dtype) {
  const bool direct = cfg->bits == 2 || cfg->bits == 4 || cfg->bits == 8 || cfg->bits == 16;
  const int isz = in_dtype == QSDP_F64 ? 8 : 4;
  return c->world > 1 && cfg->inner != QSDP_INNER_LEVELS &&
         (cfg->noise == QSDP_NOISE_PCG64_SEEDSEQ || cfg->inner == QSDP_INNER_SHIFT) && direct &&
         cfg->bucket % 8 == 0 && cfg->bucket >= 72 && cfg->bucket * isz <= 16384;
}

// The fused dequant epilogue lives in the TMA32 quantizer: direct widths,
// S % 8 == 0, a whole warp per bucket (S >= 72), S * sizeof(T) <= 16 KB
// (launch_q_t's routing), an fp32 / fp64 / bf16 output.
static bool fdq_ok(const qsdp_qcfg* cfg, int in_dtype, int out_dtype) {
  static const bool off = getenv("QSDP_NO_FDQ") != nullptr && getenv("QSDP_NO_FDQ")[0] == '1';  // A/B switch
  if (off) return false;
  const bool direct = cfg->bits == 2 || cfg->bits == 4 || cfg->bits == 8 || cfg->bits == 16;
  const int isz = in_dtype == QSDP_F64 ? 8 : 4;
  return cfg->inner != QSDP_INNER_LEVELS &&
         (cfg->noise == QSDP_NOISE_PCG64_SEEDSEQ || cfg->inner == QSDP_INNER_SHIFT) && direct && cfg->bucket % 8 == 0 &&
         cfg->bucket >= 72 && cfg->bucket * isz <= 16384 &&
         (out_dtype == QSDP_F32 || out_dtype == QSDP_F64 || out_dtype == QSDP_BF16);
}

qsdp_status qsdp_all_gather(qsdp_comm* c, const void* shard, int32_t in_dtype, const qsdp_segment* segs,
                            const qsdp_key* key, void* full_out, int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_all_gather");
  if (c == nullptr || key == nullptr) return fail(QSDP_EINVAL, "null argument");
  qsdp_status st = comm_failed(c);
  if (st != QSDP_OK) return st;
  st = check_segs(c, segs);
  if (st != QSDP_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const qsdp_qcfg* cfg = &c->w;
  const bool lv = cfg->inner == QSDP_INNER_LEVELS;
  if (lv && c->wlevels == nullptr) return fail(QSDP_EINVAL, "inner 'levels' requires a LevelTable (qsdp_comm_set_weight_levels)");
  const bool push = push_ok(c, cfg, in_dtype);
  // PUSH: the quantizer writes this rank's shard into slot [rank] of its own
  // workspace and, bucket by bucket, copies it to slot [rank] of every peer
  // (NVLink stores overlapped with the quantizer); after the barrier every rank
  // dequantizes all P slots from its own HBM.
  // PULL (other configurations): quantize into the local slot [0]; after the
  // barrier every rank dequantizes the P shards straight from the peers' slots.
  DynSrc dq = comm_dyn(c, 1);
  if (push)
    for (int p = 0; p < c->world; ++p)
      if (p != c->rank) dq.mirror_delta[dq.mirror_n++] = (int64_t)((uintptr_t)c->peer[p] - (uintptr_t)c->base);
  std::vector<QJobSpec> q(1, comm_qjob(shard, segs[c->rank], c->slot(c->base, push ? c->rank : 0), c->slot_codes,
                                       *key, 0));  // key worker 0 (sharded.py:341)
  const size_t osz = dtype_size(out_dtype);
  // this rank's own shard is dequantized by the quantizer itself (fused epilogue):
  // the dequant launch covers the peers' shards only (none at world 1)
  // (vector stores: the shard's first output element must be 16-byte aligned, 8 for bf16 --
  // shard_bounds offsets need not be multiples of 4; otherwise K3 covers the own shard too)
  uint8_t* own_out = static_cast<uint8_t*>(full_out) + (size_t)(segs[c->rank].global_start - segs[0].global_start) * osz;
  const bool fdq = fdq_ok(cfg, in_dtype, out_dtype) && aligned(own_out, osz == 2 ? 8 : 16);
  if (fdq) {
    q[0].dq_out = own_out;
    dq.dq_dtype = out_dtype == QSDP_F32 ? 0 : out_dtype == QSDP_F64 ? 1 : 2;
    dq.dq_nocodes = c->world == 1 ? 1 : 0;  // world 1: the fused dequant is the only reader
  }
  std::vector<DJobSpec> d;
  for (int p = 0; p < c->world; ++p) {
    if (fdq && p == c->rank) continue;
    DJobSpec js;
    memset(&js, 0, sizeof(DJobSpec));
    uint8_t* sl = push ? c->slot(c->base, p) : c->slot(c->peer[p], 0);
    js.codes[0] = sl;
    js.meta[0] = reinterpret_cast<const float*>(sl + c->slot_codes);
    js.nsrc = 1;
    js.length = segs[p].length;
    js.out = static_cast<uint8_t*>(full_out) + (size_t)(segs[p].global_start - segs[0].global_start) * osz;
    d.push_back(js);
  }
  // 1. quantize this rank's shard (and push it when `push`)
  st = run_quantize(q, in_dtype, cfg, nullptr, s, dq, lv ? c->wlevels : nullptr, c->wnlevels);
  if (st != QSDP_OK) return st;
  // 2. publish + wait for every peer's slot of this call
  if (c->world > 1) {
    st = comm_barrier(c, s);
    if (st != QSDP_OK) return st;
  }
  // 3. dequantize the (remaining) shards into the gathered buffer
  if (d.empty()) return QSDP_OK;
  return run_dequant(d, cfg, 0, 1, out_dtype, s, comm_dyn(c, 0), lv ? c->wlevels : nullptr);
}

static qsdp_status reduce_scatter_impl(qsdp_comm* c, const void* full_grad, int32_t in_dtype,
                                       const qsdp_segment* segs, const qsdp_key* key, void* shard_out,
                                       int32_t out_dtype, void* stream, void* x_shard, const qsdp_lattice* lat);

qsdp_status qsdp_reduce_scatter(qsdp_comm* c, const void* full_grad, int32_t in_dtype, const qsdp_segment* segs,
                                const qsdp_key* key, void* shard_out, int32_t out_dtype, void* stream) {
  NvtxRange nvtx_("qsdp_reduce_scatter");
  if (shard_out == nullptr) return fail(QSDP_EINVAL, "null output");
  return reduce_scatter_impl(c, full_grad, in_dtype, segs, key, shard_out, out_dtype, stream, nullptr, nullptr);
}

static qsdp_status reduce_scatter_impl(qsdp_comm* c, const void* full_grad, int32_t in_dtype,
                                       const qsdp_segment* segs, const qsdp_key* key, void* shard_out,
                                       int32_t out_dtype, void* stream, void* x_shard, const qsdp_lattice* lat) {
  if (c == nullptr || key == nullptr) return fail(QSDP_EINVAL, "null argument");
  qsdp_status st = comm_failed(c);
  if (st != QSDP_OK) return st;
  st = check_segs(c, segs);
  if (st != QSDP_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const qsdp_qcfg* cfg = &c->g;
  const size_t isz = dtype_size(in_dtype);
  // PUSH: the quantizer stores destination q's codes straight into owner q's
  // receive slot [rank] over NVLink (K2 is compute-bound, so the posted peer
  // stores ride along), and the owner's dequant-accumulate reads all P sources
  // from its own HBM.  Slot reuse is safe with one barrier per collective: a rank
  // writes parity n's slots on a peer only after that peer has arrived at
  // barrier n-1, which it does after finishing its dequant of call n-2.
  // 1. quantize every destination segment of this rank's gradient (worker = rank)
  std::vector<QJobSpec> q;
  for (int p = 0; p < c->world; ++p) {
    const void* x = static_cast<const uint8_t*>(full_grad) + (size_t)(segs[p].global_start - segs[0].global_start) * isz;
    q.push_back(comm_qjob(x, segs[p], c->slot(c->peer[p], c->rank), c->slot_codes, *key, (uint64_t)c->rank));
  }
  std::vector<DJobSpec> d(1);
  memset(&d[0], 0, sizeof(DJobSpec));
  for (int p = 0; p < c->world; ++p) {
    uint8_t* sl = c->slot(c->base, p);
    d[0].codes[p] = sl;
    d[0].meta[p] = reinterpret_cast<const float*>(sl + c->slot_codes);
  }
  d[0].nsrc = c->world;
  d[0].length = segs[c->rank].length;
  d[0].out = shard_out;
  d[0].lat_x = x_shard;
  DynSrc dq = comm_dyn(c, 1);
  // world 1: the average of one source is the quantizer's own dequant epilogue (0.0 + v)
  const bool fdq1 = c->world == 1 && lat == nullptr && shard_out != nullptr && fdq_ok(cfg, in_dtype, out_dtype) &&
                    aligned(shard_out, dtype_size(out_dtype) == 2 ? 8 : 16);
  if (fdq1) {
    q[0].dq_out = shard_out;
    dq.dq_dtype = out_dtype == QSDP_F32 ? 0 : out_dtype == QSDP_F64 ? 1 : 2;
    dq.dq_add0 = 1;
    dq.dq_nocodes = 1;
  }
  st = run_quantize(q, in_dtype, cfg, nullptr, s, dq);
  if (st != QSDP_OK) return st;
  if (fdq1) return QSDP_OK;
  if (c->world > 1) {
    st = comm_barrier(c, s);
    if (st != QSDP_OK) return st;
  }
  // 3. owner dequant-accumulates sources 0..P-1 (in order) from its own slots
  return run_dequant(d, cfg, 1, c->world, out_dtype, s, comm_dyn(c, 0), nullptr, lat);
}

// ---------------------------------------------------------------------------
// Group collectives: several equal-per-rank pieces in one call (an FSDP2 group's
// dense parameters, each at a fixed offset of every rank's flat buffer).  One
// quantize launch, one barrier and one dequant launch for the whole group; piece
// k of rank q is keyed with start = q * rank_stride + offset_k (sharded.py:243-248
// per piece).  Slot layout: piece k's codes at a 16-byte aligned offset, its meta
// after all codes -- the same on every rank, derived from the piece list alone.
// ---------------------------------------------------------------------------
struct PieceLayout {
  std::vector<size_t> code_off, meta_off;  // quantized: codes / meta; full precision: values (in code_off)
  size_t codes = 0, meta = 0;
  int ndense = 0, nraw = 0;
};

// raw_esz: bytes per full-precision element in a slot (all-gather: output dtype, values
// pre-cast; reduce-scatter: input dtype).  Quantized pieces first, then the raw values.
static qsdp_status piece_layout(const qsdp_comm* c, const qsdp_qcfg* cfg, const qsdp_piece* pieces, int32_t np,
                                size_t raw_esz, PieceLayout& L) {
  if (np < 1 || pieces == nullptr) return fail(QSDP_EINVAL, "need at least one piece");
  L.code_off.assign(np, 0);
  L.meta_off.assign(np, 0);
  for (int k = 0; k < np; ++k) {
    if (pieces[k].numel < 0 || pieces[k].offset < 0) return fail(QSDP_EINVAL, "negative piece");
    if (pieces[k].numel > 0 && pieces[k].src == nullptr) return fail(QSDP_EINVAL, "null piece input");
    if (pieces[k].raw) {
      if (pieces[k].numel > 0) ++L.nraw;
      continue;
    }
    ++L.ndense;
    L.code_off[k] = L.codes;
    L.meta_off[k] = L.meta;
    L.codes += round_up((size_t)qsdp_codes_bytes(pieces[k].numel, cfg), 16);
    L.meta += (size_t)qsdp_num_buckets(pieces[k].numel, cfg->bucket) * 12;
  }
  for (int k = 0; k < np; ++k)
    if (pieces[k].raw && pieces[k].numel > 0) {
      L.code_off[k] = L.codes;
      L.codes += round_up((size_t)pieces[k].numel * raw_esz, 16);
    }
  if (L.codes > c->slot_codes || L.meta > c->slot_meta)
    return fail(QSDP_EINVAL, "group pieces exceed the communicator's slot (max_segment_elems)");
  return QSDP_OK;
}

// The barrier of a group collective, carrying its full-precision pieces (world 1 with raw
// pieces: the kernel without flags; world 1 without: nothing).
static qsdp_status pieces_barrier(qsdp_comm* c, const qsdp_piece* pieces, int32_t np, const PieceLayout& L, int mode,
                                  int32_t in_dtype, int32_t out_dtype, int64_t stride, void* out, cudaStream_t s) {
  if (L.nraw == 0) return c->world > 1 ? comm_barrier(c, s) : QSDP_OK;
  PeerFlags pf;
  memset(&pf, 0, sizeof(pf));
  for (int j = 0; j < c->world; ++j) {
    if (c->peer[j] == nullptr) return fail(QSDP_EPEER, "peers not opened");
    pf.flags[j] = reinterpret_cast<unsigned long long*>(c->peer[j]);
  }
  RawTable rt;
  memset(&rt, 0, sizeof(rt));
  rt.mode = mode;
  rt.in_dt = in_dtype;
  rt.out_dt = out_dtype;
  rt.world = c->world;
  rt.rank = c->rank;
  rt.stride = stride;
  rt.slot_bytes = (int64_t)c->slot_bytes;
  rt.parity_stride = c->world > 1 ? c->parity_stride() : 0;
  rt.out = static_cast<uint8_t*>(out);
  rt.own_slots = c->slot(c->base, 0);
  for (int p = 0; p < c->world; ++p) rt.peer_slot[p] = c->slot(c->peer[p], c->rank);
  // the barrier kernel carries the first kMaxRaw pieces; any further ones go in tables of
  // kMaxRaw through a push kernel before it and a copy-out / average kernel after it
  std::vector<RawTable> extra;
  for (int k = 0; k < np; ++k) {
    if (!pieces[k].raw || pieces[k].numel <= 0) continue;
    const RawPieceDev d{static_cast<const uint8_t*>(pieces[k].src), pieces[k].numel, (int64_t)L.code_off[k],
                        pieces[k].offset};
    if (rt.n < kMaxRaw) {
      rt.p[rt.n++] = d;
      continue;
    }
    if (extra.empty() || extra.back().n == kMaxRaw) {
      extra.push_back(rt);
      extra.back().n = 0;
    }
    extra.back().p[extra.back().n++] = d;
  }
  for (const RawTable& e : extra) qsdp_raw_phase_kernel<<<1, 512, 0, s>>>(c->epoch(), 1, 0, e);
  qsdp_barrier_raw_kernel<<<1, 512, 0, s>>>(pf, c->epoch(), c->err_dev, c->timeout_ns, rt);
  for (const RawTable& e : extra) qsdp_raw_phase_kernel<<<1, 512, 0, s>>>(c->epoch(), 0, 1, e);
  QSDP_CUDA(cudaGetLastError());
  return QSDP_OK;
}

qsdp_status qsdp_all_gather_pieces(qsdp_comm* c, const qsdp_piece* pieces, int32_t npieces, int32_t in_dtype,
                                   int64_t rank_stride, const qsdp_key* key, void* full_out, int32_t out_dtype,
                                   void* stream) {
  NvtxRange nvtx_("qsdp_all_gather_pieces");
  if (c == nullptr || key == nullptr || full_out == nullptr) return fail(QSDP_EINVAL, "null argument");
  qsdp_status st = comm_failed(c);
  if (st != QSDP_OK) return st;
  const qsdp_qcfg* cfg = &c->w;
  const size_t osz = dtype_size(out_dtype);
  PieceLayout L;
  st = piece_layout(c, cfg, pieces, npieces, osz, L);
  if (st != QSDP_OK) return st;
  if (cfg->inner == QSDP_INNER_LEVELS && L.ndense > 0)
    return fail(QSDP_EINVAL, "group collectives quantize with affine weight specs (levels: full-precision pieces only)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool push = push_ok(c, cfg, in_dtype);
  DynSrc dq = comm_dyn(c, 1);
  if (push)
    for (int p = 0; p < c->world; ++p)
      if (p != c->rank) dq.mirror_delta[dq.mirror_n++] = (int64_t)((uintptr_t)c->peer[p] - (uintptr_t)c->base);
  uint8_t* own = c->slot(c->base, push ? c->rank : 0);
  const bool fdq_cfg = fdq_ok(cfg, in_dtype, out_dtype);
  bool fdq_all = fdq_cfg;  // one epilogue setting per table: fuse only when every own piece can
  std::vector<QJobSpec> q;
  for (int k = 0; k < npieces; ++k) {
    if (pieces[k].raw) continue;
    const int64_t gs = (int64_t)c->rank * rank_stride + pieces[k].offset;
    qsdp_segment seg{gs, pieces[k].numel};
    QJobSpec j = comm_qjob(pieces[k].src, seg, own + L.code_off[k], 0, *key, 0);
    j.meta = reinterpret_cast<float*>(own + c->slot_codes + L.meta_off[k]);
    uint8_t* o = static_cast<uint8_t*>(full_out) + (size_t)gs * osz;
    if (!aligned(o, osz == 2 ? 8 : 16)) fdq_all = false;
    j.dq_out = o;
    q.push_back(j);
  }
  if (fdq_all) {
    dq.dq_dtype = out_dtype == QSDP_F32 ? 0 : out_dtype == QSDP_F64 ? 1 : 2;
    dq.dq_nocodes = c->world == 1 ? 1 : 0;
  } else {
    for (auto& j : q) j.dq_out = nullptr;
  }
  std::vector<DJobSpec> d;
  for (int p = 0; p < c->world; ++p) {
    if (fdq_all && p == c->rank) continue;
    uint8_t* sl = push ? c->slot(c->base, p) : c->slot(c->peer[p], 0);
    for (int k = 0; k < npieces; ++k) {
      if (pieces[k].raw) continue;
      DJobSpec js;
      memset(&js, 0, sizeof(DJobSpec));
      js.codes[0] = sl + L.code_off[k];
      js.meta[0] = reinterpret_cast<const float*>(sl + c->slot_codes + L.meta_off[k]);
      js.nsrc = 1;
      js.length = pieces[k].numel;
      js.out = static_cast<uint8_t*>(full_out) + (size_t)((int64_t)p * rank_stride + pieces[k].offset) * osz;
      d.push_back(js);
    }
  }
  if (!q.empty()) {
    st = run_quantize(q, in_dtype, cfg, nullptr, s, dq);
    if (st != QSDP_OK) return st;
  }
  st = pieces_barrier(c, pieces, npieces, L, 0, in_dtype, out_dtype, rank_stride, full_out, s);
  if (st != QSDP_OK) return st;
  if (d.empty()) return QSDP_OK;
  return run_dequant(d, cfg, 0, 1, out_dtype, s, comm_dyn(c, 0));
}

qsdp_status qsdp_reduce_scatter_pieces(qsdp_comm* c, const qsdp_piece* pieces, int32_t npieces, int32_t in_dtype,
                                       int64_t rank_stride, const qsdp_key* key, void* shard_out, int32_t out_dtype,
                                       void* stream) {
  NvtxRange nvtx_("qsdp_reduce_scatter_pieces");
  if (c == nullptr || key == nullptr || shard_out == nullptr) return fail(QSDP_EINVAL, "null argument");
  qsdp_status st = comm_failed(c);
  if (st != QSDP_OK) return st;
  const qsdp_qcfg* cfg = &c->g;
  const size_t isz = dtype_size(in_dtype), osz = dtype_size(out_dtype);
  PieceLayout L;
  st = piece_layout(c, cfg, pieces, npieces, isz, L);
  if (st != QSDP_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::vector<QJobSpec> q;
  std::vector<int> dense;  // piece index of each quantized piece
  for (int k = 0; k < npieces; ++k)
    if (!pieces[k].raw) dense.push_back(k);
  for (int p = 0; p < c->world; ++p) {  // destination p's piece k -> owner p's slot [rank]
    uint8_t* dst = c->slot(c->peer[p], c->rank);
    for (int k : dense) {
      qsdp_segment seg{(int64_t)p * rank_stride + pieces[k].offset, pieces[k].numel};
      const void* x = static_cast<const uint8_t*>(pieces[k].src) + (size_t)((int64_t)p * rank_stride) * isz;
      QJobSpec j = comm_qjob(x, seg, dst + L.code_off[k], 0, *key, (uint64_t)c->rank);
      j.meta = reinterpret_cast<float*>(dst + c->slot_codes + L.meta_off[k]);
      q.push_back(j);
    }
  }
  DynSrc dq = comm_dyn(c, 1);
  bool fdq1 = c->world == 1 && fdq_ok(cfg, in_dtype, out_dtype);
  for (int k : dense)
    if (fdq1) fdq1 = aligned(static_cast<uint8_t*>(shard_out) + (size_t)pieces[k].offset * osz, osz == 2 ? 8 : 16);
  if (fdq1) {
    for (size_t i = 0; i < dense.size(); ++i)
      q[i].dq_out = static_cast<uint8_t*>(shard_out) + (size_t)pieces[dense[i]].offset * osz;
    dq.dq_dtype = out_dtype == QSDP_F32 ? 0 : out_dtype == QSDP_F64 ? 1 : 2;
    dq.dq_add0 = 1;
    dq.dq_nocodes = 1;
  }
  if (!q.empty()) {
    st = run_quantize(q, in_dtype, cfg, nullptr, s, dq);
    if (st != QSDP_OK) return st;
  }
  st = pieces_barrier(c, pieces, npieces, L, 1, in_dtype, out_dtype, rank_stride, shard_out, s);
  if (st != QSDP_OK || fdq1 || dense.empty()) return st;
  std::vector<DJobSpec> d;
  for (int k : dense) {
    DJobSpec js;
    memset(&js, 0, sizeof(DJobSpec));
    for (int p = 0; p < c->world; ++p) {
      uint8_t* sl = c->slot(c->base, p);
      js.codes[p] = sl + L.code_off[k];
      js.meta[p] = reinterpret_cast<const float*>(sl + c->slot_codes + L.meta_off[k]);
    }
    js.nsrc = c->world;
    js.length = pieces[k].numel;
    js.out = static_cast<uint8_t*>(shard_out) + (size_t)pieces[k].offset * osz;
    d.push_back(js);
  }
  return run_dequant(d, cfg, 1, c->world, out_dtype, s, comm_dyn(c, 0));
}

qsdp_status qsdp_reduce_scatter_lattice(qsdp_comm* c, const void* full_grad, int32_t in_dtype, const qsdp_segment* segs,
                                        const qsdp_key* key, void* shard_out, int32_t out_dtype, void* x_shard,
                                        const qsdp_lattice* lat, void* stream) {
  NvtxRange nvtx_("qsdp_reduce_scatter_lattice");
  qsdp_status st = check_lattice(lat, x_shard);
  if (st != QSDP_OK) return st;
  return reduce_scatter_impl(c, full_grad, in_dtype, segs, key, shard_out, out_dtype, stream, x_shard, lat);
}

}  // extern "C"
