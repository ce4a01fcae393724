/*
 * qsdp_b200.h -- C ABI of the B200-native QSDP communication hot path.
 *
 * Drop-in boundary for the reference's quantizer and FSDP-hook API
 * (reference = arxiv/paper_2302_02390 artifact, pkg/src/qsdp; paths below are
 * relative to that package).  Every entry point is extern "C", takes plain
 * device pointers and sizes, and is stream-ordered on the caller's
 * cudaStream_t (passed as void*) with no hidden device synchronisation.
 *
 *   reference (Python/NumPy)                         replaced by
 *   ------------------------------------------------ ---------------------------------
 *   quantize_bucket / _segment_blocks (shift)         qsdp_quantize / qsdp_quantize_batch
 *     quantize.py:235-272, sharded.py:243-248            (inner = QSDP_INNER_SHIFT)
 *   quantize_bucket (uniform_stochastic | flip)       qsdp_quantize / qsdp_quantize_batch
 *     quantize.py:273-274, 316-321                       (inner = QSDP_INNER_STOCHASTIC)
 *   bucket_rng / sample_shift / rng.random            device SeedSequence->PCG64 (no entry point;
 *     sharded.py:235-240, quantize.py:130-132            keyed by qsdp_key + bucket start)
 *   _pack_codes / _unpack_codes  wire.py:82-95         packed code layout of every entry point
 *   dequantize  quantize.py:209-232                    qsdp_dequantize / qsdp_dequantize_batch
 *   acc = acc + vals ... acc / P  sharded.py:385-431   qsdp_dequant_accumulate
 *   message_size_bits  wire.py:187-192                 qsdp_message_size_bits
 *   encode  wire.py:108-131                            qsdp_wire_encode_device (device) /
 *                                                        qsdp_wire_encode (host buffers)
 *   decode  wire.py:134-184                            qsdp_wire_parse + qsdp_wire_decode_device
 *   ShardedMLP._gather  sharded.py:323-373             qsdp_all_gather (one process per GPU)
 *   ShardedMLP._reduce_scatter  sharded.py:375-433     qsdp_reduce_scatter
 *   qsdp_step (lattice projection)  optimizer.py:194-229  qsdp_reduce_scatter_lattice /
 *                                                        qsdp_dequant_accumulate_lattice (K4 epilogue)
 *   quantize_bucket (levels) + quantize_with_levels    qsdp_quantize_levels / _batch
 *     quantize.py:235-286, 400-416                       (inner = QSDP_INNER_LEVELS)
 *   dequantize(block, "levels", table)  quantize.py:225-231  qsdp_dequantize_levels / _batch
 *   learn_levels  quantize.py:366-397                  qsdp_learn_levels (one sequential pass)
 *
 * Device layout of one quantized segment (length L, bucket S, width b):
 *   codes: bucket j's LSB-first packed codes at byte j*ceil(S*b/8), each bucket
 *          zero-padded to a whole byte (exactly the wire payload, wire.py:14-20);
 *   meta:  float[nb][3] = {shift, scale_lo, scale_hi} per bucket (the wire's
 *          per-block field order).
 *
 * Error behaviour mirrors the reference exception types:
 *   QSDP_EINVAL     ValueError for bad arguments (bit width, bucket size, ...)
 *   QSDP_ENONFINITE ValueError("non-finite ... at index i") -- reported through
 *                   the optional device word *d_bad (see qsdp_quantize)
 *   QSDP_ERANGE     CodeRangeError (wire.py:74; header bit width outside [1, 32])
 *   QSDP_EDECODE / QSDP_ETRUNC / QSDP_EVERSION   DecodeError / TruncatedMessageError /
 *                   UnsupportedVersionError (qsdp_wire_parse / qsdp_wire_decode_device)
 *   QSDP_ECUDA      CUDA runtime failure (message in qsdp_last_error())
 *   QSDP_EPEER      peer-memory / IPC setup failure, or a peer missed a barrier (timeout)
 */
#ifndef QSDP_B200_H_
#define QSDP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QSDP_OK = 0,
  QSDP_EINVAL = 1,
  QSDP_ENONFINITE = 2,
  QSDP_ERANGE = 3,
  QSDP_ECUDA = 4,
  QSDP_ENCCL = 5,
  QSDP_EPEER = 6,
  QSDP_EDECODE = 7,   /* DecodeError (wire.py:62) */
  QSDP_ETRUNC = 8,    /* TruncatedMessageError (wire.py:66) */
  QSDP_EVERSION = 9   /* UnsupportedVersionError (wire.py:70) */
} qsdp_status;

typedef enum { QSDP_INNER_SHIFT = 0, QSDP_INNER_STOCHASTIC = 1, QSDP_INNER_LEVELS = 2 } qsdp_inner;
/* Noise of the quantizers' draws, keyed per bucket by (root, step, layer, phase, worker,
 * start) through numpy's SeedSequence:
 *   QSDP_NOISE_PCG64_SEEDSEQ  np.random.default_rng(SeedSequence(key)) == bucket_rng
 *                             (sharded.py:235-240): sequential 128-bit LCG stream;
 *   QSDP_NOISE_PHILOX4x64     np.random.Generator(np.random.Philox(SeedSequence(key))):
 *                             counter-based Philox4x64-10 (key = generate_state(2, uint64)),
 *                             draw i = word i%4 of block i/4 + 1 -- any generator the
 *                             reference's quantize_bucket accepts (quantize.py:235-241). */
typedef enum { QSDP_NOISE_PCG64_SEEDSEQ = 0, QSDP_NOISE_PHILOX4x64 = 1 } qsdp_noise;
typedef enum { QSDP_F32 = 0, QSDP_F64 = 1, QSDP_BF16 = 2 } qsdp_dtype;

/* mirrors QuantConfig (sharded.py:76-93) for one tensor class */
typedef struct {
  int32_t bits;   /* 1..16 */
  int32_t bucket; /* >= 1 (BucketSpec.bucket_size, quantize.py:64-75) */
  int32_t inner;  /* qsdp_inner */
  int32_t noise;  /* qsdp_noise */
} qsdp_qcfg;

/* bucket_rng(root_seed, step, layer_idx, phase, worker, start): the bucket start
   is implicit (segment global_start + j*bucket). */
typedef struct {
  uint64_t root_seed, step, layer, phase, worker;
} qsdp_key;

/* a shard / reduce-scatter segment: buckets are cut from its own start and keyed
   with start = global_start + j*bucket (sharded.py:243-248, 334-343). */
typedef struct {
  int64_t global_start, length;
} qsdp_segment;

/* One entry of a batched quantize: input segment -> packed codes + meta. */
typedef struct {
  const void* x;       /* device, dtype given by the call */
  qsdp_segment seg;
  qsdp_key key;
  uint8_t* codes;      /* device, qsdp_codes_bytes(seg.length, cfg) bytes */
  float* meta;         /* device, 3*qsdp_num_buckets(seg.length, cfg->bucket) floats */
} qsdp_qitem;

/* One entry of a batched dequantize / dequant-accumulate. */
typedef struct {
  const uint8_t* codes[8]; /* nsrc sources with identical bucket structure */
  const float* meta[8];
  int32_t nsrc;
  int64_t length;
  void* out;               /* device, dtype given by the call */
} qsdp_ditem;

#define QSDP_IPC_HANDLE_BYTES 64
#define QSDP_MAX_WORLD 8

typedef struct qsdp_comm qsdp_comm;

/* ---- sizes & accounting (pure host functions) ---- */
int64_t qsdp_num_buckets(int64_t length, int32_t bucket);
int64_t qsdp_codes_bytes(int64_t length, const qsdp_qcfg* cfg);
/* encoded message size of one segment incl. header/meta/padding (wire.py:187-192) */
int64_t qsdp_message_size_bits(int64_t length, const qsdp_qcfg* cfg);
/* shard_bounds(size, P) (sharded.py:193-200): writes P segments */
void qsdp_shard_bounds(int64_t size, int32_t world, qsdp_segment* out);
const char* qsdp_last_error(void);
const char* qsdp_version(void);

/* ---- K1/K2: quantize ----
 * x: device fp32 or fp64 (x_dtype).  d_bad (optional device uint64, initialise
 * to UINT64_MAX) receives min over non-finite elements of (item<<40 | index in
 * segment); buckets containing one are emitted as zero codes / zero meta. */
qsdp_status qsdp_quantize(const void* x, int32_t x_dtype, qsdp_segment seg, const qsdp_qcfg* cfg,
                          const qsdp_key* key, uint8_t* codes, float* meta, uint64_t* d_bad,
                          void* stream);
qsdp_status qsdp_quantize_batch(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                const qsdp_qcfg* cfg, uint64_t* d_bad, void* stream);
/* Same, with the keys' step offset read on the device at run time
 * (step = key.step + *d_step): a captured CUDA graph replays with fresh noise. */
qsdp_status qsdp_quantize_batch_dstep(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                      const qsdp_qcfg* cfg, uint64_t* d_bad, const uint64_t* d_step,
                                      void* stream);
/* Shared-generator bucketing (bucketed_quantize with one rng, quantize.py:289-313; the theory
 * side's UniformStochasticGradientQuantizer, optimizer.py:177-191): bucket j's draws continue
 * ONE numpy PCG64 stream.  d_states[4*j..4*j+3] = (state_lo, state_hi, inc_lo, inc_hi) of the
 * stream before bucket j's first draw (the caller's prefix sum: 1 draw per non-degenerate
 * shift bucket, n per non-degenerate stochastic bucket, 0 for a degenerate one).  Input must
 * be finite (the caller raises first, as the reference does).  d_scratch: length uint32. */
qsdp_status qsdp_quantize_stream(const void* x, int32_t x_dtype, int64_t length, const qsdp_qcfg* cfg,
                                 const uint64_t* d_states, uint8_t* codes, float* meta, uint32_t* d_scratch,
                                 void* stream);
/* quantize_with_levels(v, table, stochastic=True, rng) (quantize.py:400-422) on device fp64
 * values: element i draws the i-th double of the numpy PCG64 stream whose state before the
 * first draw is state[4] = (state_lo, state_hi, inc_lo, inc_hi) (host memory); nlevels >= 2. */
qsdp_status qsdp_levels_stochastic(const double* d_values, int64_t n, const double* d_levels, int32_t nlevels,
                                   const uint64_t* state, uint32_t* d_codes, void* stream);
/* *d_counter += delta on the stream (advances a device step counter inside a graph). */
qsdp_status qsdp_counter_add(uint64_t* d_counter, uint64_t delta, void* stream);

/* ---- K3: dequantize one segment (fp32 out == float32(reference fp64); bf16 == RNE of that) ---- */
qsdp_status qsdp_dequantize(const uint8_t* codes, const float* meta, int64_t length,
                            const qsdp_qcfg* cfg, void* out, int32_t out_dtype, void* stream);
qsdp_status qsdp_dequantize_batch(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg,
                                  int32_t out_dtype, void* stream);

/* ---- K4: out = (0 + sum_{p<nsrc} dequant(src_p)) / divisor, fp64 ordered sum ---- */
qsdp_status qsdp_dequant_accumulate(const uint8_t* const* codes, const float* const* meta,
                                    int32_t nsrc, int64_t length, const qsdp_qcfg* cfg,
                                    int32_t divisor, void* out, int32_t out_dtype, void* stream);
qsdp_status qsdp_dequant_accumulate_batch(const qsdp_ditem* items, int32_t nitems,
                                          const qsdp_qcfg* cfg, int32_t divisor,
                                          int32_t out_dtype, void* stream);

/* ---- learned levels ----
 * d_levels: device float64[nlevels], strictly increasing (LevelTable,
 * quantize.py:344-363).  cfg->inner must be QSDP_INNER_LEVELS; the keys are not
 * used (levels mode draws no noise); meta shift is 0.  Codes are bit-exact with
 * quantize_with_levels(clip((v-lo)/(hi-lo), 0, 1), table) (searchsorted over the
 * level mids, side="left").  Quantize takes any power-of-two table with
 * nlevels <= 2^bits (a wider table is EINVAL: its codes could not be stored). */
qsdp_status qsdp_quantize_levels_batch(const qsdp_qitem* items, int32_t nitems, int32_t x_dtype,
                                       const qsdp_qcfg* cfg, const double* d_levels, int32_t nlevels,
                                       uint64_t* d_bad, void* stream);
qsdp_status qsdp_quantize_levels(const void* x, int32_t x_dtype, int64_t length, const qsdp_qcfg* cfg,
                                 const double* d_levels, int32_t nlevels, uint8_t* codes, float* meta,
                                 uint64_t* d_bad, void* stream);
/* lo + levels[code] * (hi - lo) in fp64, stored as out_dtype; nlevels == 2^bits
   ("level table size does not match bit_width" otherwise) */
qsdp_status qsdp_dequantize_levels_batch(const qsdp_ditem* items, int32_t nitems, const qsdp_qcfg* cfg,
                                         const double* d_levels, int32_t nlevels, int32_t out_dtype,
                                         void* stream);
qsdp_status qsdp_dequantize_levels(const uint8_t* codes, const float* meta, int64_t length,
                                   const qsdp_qcfg* cfg, const double* d_levels, int32_t nlevels, void* out,
                                   int32_t out_dtype, void* stream);
/* One pass of learn_levels over device float64 values[n] (in order), updating
 * d_levels[nlevels] in place, including the re-sort / collision nudge.  The
 * caller performs the reference's empty / non-finite / distinct-count checks.
 * nlevels: a power of two <= 4096. */
qsdp_status qsdp_learn_levels(const double* d_values, int64_t n, double* d_levels, int32_t nlevels,
                              double learning_rate, void* stream);

/* ---- wire codec: byte-exact reference messages ---- */
typedef struct {
  int32_t version, bits;
  int64_t bucket, blocks, total_length;
  int64_t expected_bytes;   /* size of a well-formed message with this header */
  int64_t complete_blocks;  /* leading blocks wholly present in msg_bytes */
} qsdp_wire_info;
/* Header parse with decode's header-level checks, in its order (wire.py:136-158):
 * hdr = the first min(14, msg_bytes) bytes (host).  QSDP_OK with blocks == 0 for the
 * empty message.  Truncation / trailing bytes are reported by the caller after the
 * complete blocks were validated (info->complete_blocks, info->expected_bytes). */
qsdp_status qsdp_wire_parse(const uint8_t* hdr, int64_t msg_bytes, qsdp_wire_info* info);
/* Device encode: one segment in the device layout -> the message
 * (qsdp_message_size_bits(length, cfg) / 8 bytes at d_out). */
qsdp_status qsdp_wire_encode_device(const uint8_t* codes, const float* meta, int64_t length,
                                    const qsdp_qcfg* cfg, uint8_t* d_out, int64_t out_cap, void* stream);
/* Device decode of info->complete_blocks blocks into the device layout (any
 * width 1..32; the quantizers / dequantizers use 1..16).  d_err[2] (device, init UINT64_MAX) receive the first block with nonzero
 * padding bits (DecodeError) and the first with !(scale_lo <= scale_hi) (ValueError). */
qsdp_status qsdp_wire_decode_device(const uint8_t* d_msg, const qsdp_wire_info* info, uint8_t* codes,
                                    float* meta, uint64_t* d_err, void* stream);

/* uint32 codes (one per element, < 2^bits) <-> the packed device layout
 * (_pack_codes / _unpack_codes per bucket, wire.py:82-95), widths 1..32. */
qsdp_status qsdp_pack_codes(const uint32_t* codes, int64_t length, const qsdp_qcfg* cfg, uint8_t* out,
                            void* stream);
qsdp_status qsdp_unpack_codes(const uint8_t* packed, int64_t length, const qsdp_qcfg* cfg, uint32_t* codes,
                              void* stream);

/* ---- lattice-projected step fused with the reduce-scatter epilogue ----
 * With g = the K4 average (fp64, before any rounding): x <- d*rint((x - c*g - r)/d) + r
 * (qsdp_step, optimizer.py:212-216), r = sample_shift(d, bucket_rng(shift_key..., 0)), the
 * first draw of the keyed stream (its step also advances with the comm's device step). */
typedef struct {
  double lr_over_beta;  /* c = eta / beta */
  double delta;         /* d: fine lattice pitch (> 0) */
  qsdp_key shift_key;
  int32_t x_dtype;      /* QSDP_F32 | QSDP_F64 (fp64 iterates are bit-exact with the reference) */
} qsdp_lattice;
qsdp_status qsdp_dequant_accumulate_lattice(const uint8_t* const* codes, const float* const* meta, int32_t nsrc,
                                            int64_t length, const qsdp_qcfg* cfg, int32_t divisor, void* g_out,
                                            int32_t out_dtype, void* x, const qsdp_lattice* lat, void* stream);

/* ---- host wire export (wire.py:108-131): codes/meta already on the host ---- */
int64_t qsdp_wire_encode(const uint8_t* codes, const float* meta, int64_t length,
                         const qsdp_qcfg* cfg, uint8_t* out, int64_t out_cap);

/* ---- C1/C2: multi-GPU collectives over NVLink peer memory (one process per GPU) ----
 * create -> export this rank's IPC handle -> exchange handles out of band
 * (any transport; the Python host uses torch.distributed) -> open peers. */
qsdp_status qsdp_comm_create(qsdp_comm** out, int32_t rank, int32_t world, int32_t device,
                             int64_t max_segment_elems, const qsdp_qcfg* wcfg,
                             const qsdp_qcfg* gcfg);
qsdp_status qsdp_comm_ipc_handle(qsdp_comm* c, void* handle /* QSDP_IPC_HANDLE_BYTES */);
qsdp_status qsdp_comm_open_peers(qsdp_comm* c, const void* handles /* world*QSDP_IPC_HANDLE_BYTES */);
/* Keys' step = key.step + *d_step for every later collective (NULL: key.step).
 * With it, and the communicator's device-side epoch, a sequence of
 * qsdp_all_gather / qsdp_reduce_scatter calls can be captured in a CUDA graph. */
qsdp_status qsdp_comm_set_step_source(qsdp_comm* c, const uint64_t* d_step);
/* Learned weight levels for the all-gather (w.inner == QSDP_INNER_LEVELS): a
 * device float64[2^w.bits] table that stays valid while the comm uses it. */
qsdp_status qsdp_comm_set_weight_levels(qsdp_comm* c, const double* d_levels, int32_t nlevels);
/* Size the collectives' grids for at most `sms` SMs: leaves the rest of the GPU to compute
 * kernels that run concurrently (FSDP2 overlaps comm streams with compute).  0 = the
 * default (world 1: all SMs; world > 1: all but 8, so the one-CTA flag barriers of other
 * in-flight collectives always find an SM); < 0 = all SMs. */
qsdp_status qsdp_comm_set_sm_budget(qsdp_comm* c, int32_t sms);
/* At most `ctas` quantizer CTAs per SM (0 = as many as fit): an HBM-bound all-gather capped
 * at one CTA per SM leaves the other slot to a concurrent, issue-bound reduce-scatter on
 * another stream (the backward phase), instead of taking turns with it. */
qsdp_status qsdp_comm_set_ctas_per_sm(qsdp_comm* c, int32_t ctas);
/* Failure detection.  A barrier whose peer does not arrive within the timeout
 * (default 60 s; env QSDP_TIMEOUT_MS at creation) gives up instead of hanging and
 * records the peer in a host-mapped word: qsdp_comm_status() -- and every later
 * qsdp_all_gather / qsdp_reduce_scatter -- then returns QSDP_EPEER naming the peer
 * and epoch (the data of that collective is undefined).  qsdp_comm_status() does
 * not synchronise: call it after the stream has completed the collectives to check. */
qsdp_status qsdp_comm_set_timeout(qsdp_comm* c, int64_t timeout_ms);
qsdp_status qsdp_comm_status(qsdp_comm* c);
/* Quantized all-gather (ShardedMLP._gather): this rank's shard = segs[rank];
 * every rank writes the dequantized full tensor (sum of segs lengths) to full_out.
 * key->worker is forced to 0 (sharded.py:341). */
qsdp_status qsdp_all_gather(qsdp_comm* c, const void* shard, int32_t in_dtype,
                            const qsdp_segment* segs, const qsdp_key* key, void* full_out,
                            int32_t out_dtype, void* stream);
/* Quantized reduce-scatter (ShardedMLP._reduce_scatter): full_grad holds this
 * rank's whole gradient; segs[q] is destination q's shard; shard_out receives
 * (sum_p dequant(Q_p(grad_p[segs[rank]]))) / world.  key->worker = this rank. */
qsdp_status qsdp_reduce_scatter(qsdp_comm* c, const void* full_grad, int32_t in_dtype,
                                const qsdp_segment* segs, const qsdp_key* key, void* shard_out,
                                int32_t out_dtype, void* stream);
/* C2 with the lattice step on the owner's shard: shard_out (may be NULL) receives the
 * average gradient, x_shard (lat->x_dtype) the projected iterate.  Never fused. */
qsdp_status qsdp_reduce_scatter_lattice(qsdp_comm* c, const void* full_grad, int32_t in_dtype,
                                        const qsdp_segment* segs, const qsdp_key* key, void* shard_out,
                                        int32_t out_dtype, void* x_shard, const qsdp_lattice* lat, void* stream);
/* Group collectives: npieces equal-per-rank pieces in one call -- e.g. an FSDP2 group's
 * dense parameters, piece k at element offset_k of every rank's flat buffer of
 * rank_stride elements.  Piece k of rank q is keyed with start = q*rank_stride + offset_k;
 * one quantize launch, one barrier and one dequant launch per call.
 *   all-gather:     src = this rank's piece (numel elements); full_out[q*rank_stride + offset_k ...]
 *                   receives rank q's dequantized piece.
 *   reduce-scatter: src = piece k of destination 0 in this rank's rank-major gradient
 *                   (destination q's piece at src + q*rank_stride elements); shard_out[offset_k ...]
 *                   receives the fp64-ordered average over ranks.
 * The pieces' codes + meta must fit the communicator's slot (max_segment_elems). */
typedef struct {
  const void* src;
  int64_t offset, numel;
  int32_t raw;       /* non-zero: a full-precision piece (bias / norm, sharded.py:359-371, 414-429):
                        all-gather -- every rank's piece cast (RNE) to out_dtype; reduce-scatter --
                        out = (0.0 + v_0 + ... + v_{P-1}) / P in fp64, ranks in order, rounded once.
                        Carried by the collective's barrier kernel (beyond 48 pieces, by a push
                        kernel before it and a copy-out kernel after it). */
  int32_t reserved;
} qsdp_piece;
qsdp_status qsdp_all_gather_pieces(qsdp_comm* c, const qsdp_piece* pieces, int32_t npieces, int32_t in_dtype,
                                   int64_t rank_stride, const qsdp_key* key, void* full_out, int32_t out_dtype,
                                   void* stream);
qsdp_status qsdp_reduce_scatter_pieces(qsdp_comm* c, const qsdp_piece* pieces, int32_t npieces, int32_t in_dtype,
                                       int64_t rank_stride, const qsdp_key* key, void* shard_out, int32_t out_dtype,
                                       void* stream);
qsdp_status qsdp_comm_destroy(qsdp_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* QSDP_B200_H_ */
