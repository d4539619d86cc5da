/*
 * dcomp_b200.h -- C ABI of the B200-native hot path of arXiv 2502.15443
 * ("LLM double compression": compression-aware INT8 quantization, pruning,
 * chunked static-table rANS in the DCC1 container, fused decode->W8A8 GEMM).
 *
 * The reference (`dcomp`, /root/reference/pkg/src/dcomp) is a CPU Python
 * package whose only natively compiled code is four numba kernels; every
 * entry point below replaces one of those kernels or a numpy hot loop, cited
 * as "replaces <file>:<line>".  The reference has no FFI of its own: the
 * Python host layer (paper_2502_15443_b200/) binds these symbols with ctypes
 * exactly as a maintainer would bind them from the reference.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every pointer argument is a DEVICE
 *    pointer unless its name ends in `_host`.  `stream` is a cudaStream_t
 *    passed as void*.  Calls are asynchronous on `stream` unless noted.
 *  - Return value: 0 = ok, negative = argument / CUDA error (message via
 *    dc_last_error()).  Data errors never become return codes: they are
 *    written per chunk into a device `status` array (DC_CHUNK_* below), and
 *    the host maps them to the reference's exception classes and messages.
 *  - The library never allocates long-lived device memory; callers own all
 *    buffers (the Python layer uses the torch caching allocator).
 *  - Buffers that stream bytes are read from must have DC_READ_SLACK readable
 *    bytes past their end (corrupt streams may over-read; verdicts stay exact).
 */
#ifndef DCOMP_B200_H
#define DCOMP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DC_OK 0
#define DC_ERR_ARG (-1)
#define DC_ERR_CUDA (-2)
#define DC_ERR_UNSUPPORTED (-3)

#define DC_READ_SLACK 16384

/* Per-chunk status codes (device int32 arrays).  Map 1:1 onto the reference
 * exceptions raised by ans.split_blob / _prepare_payload / decode_blobs_into
 * (ans.py:333-343, 364-367, 375-430) and container.unpack (container.py:327-331). */
#define DC_CHUNK_OK 0
#define DC_CHUNK_TRUNC_TABLE 1 /* TruncatedError "truncated stream: missing table header" */
#define DC_CHUNK_BAD_TABLE 2   /* CorruptStreamError "corrupt stream: invalid frequency table" */
#define DC_CHUNK_STATE_RANGE 3 /* CorruptStreamError "corrupt stream: final state out of range" */
#define DC_CHUNK_EMPTY_BAD 4   /* CorruptStreamError "corrupt stream" (zero-length output) */
#define DC_CHUNK_CORRUPT 5     /* CorruptStreamError "corrupt stream" (decode verdict) */
#define DC_CHUNK_CHAIN 6       /* internal: split-point chain mismatch -> exact serial re-decode */

/* ---------------------------------------------------------------- info */
int dc_version(void);
const char *dc_last_error(void);
int dc_device_sm_count(int device);

/* ------------------------------------------------------- rANS decoding
 * A decode "job list" describes n chunks inside one device byte buffer:
 *   blob_off[i]  u64  offset of chunk i's bytes in `base` (ANS blob: u12 table | u32 state | stream)
 *   blob_len[i]  u64  comp_len of chunk i
 *   out_off[i]   u64  where its decoded bytes go in `out`
 *   out_len[i]   u64  uncomp_len
 *   codec[i]     u8   0 = store (raw copy), 1 = ANS
 * Split-point ("segment") index: for ANS chunk i, segments of 2^seg_shift
 * symbols start at seg_base[i]; seg_state[j] / seg_off[j] hold the decoder
 * state and stream byte offset (relative to blob+388) at each segment start.
 */

/* Prologue checks of every ANS chunk: blob length, u12 table validity,
 * start-state range, zero-length outputs.  replaces ans.py:284-299 (from_bytes),
 * ans.py:333-343 (_prepare_payload), ans.py:364-367 (split_blob), ans.py:382-392. */
int dc_ans_validate(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                    const uint64_t *out_len, const uint8_t *codec, int64_t n_chunks,
                    int32_t *status, void *stream);

/* Exact serial decode of the listed chunks, one CTA per chunk: the
 * reference verdict rule (final state == 2^20 and every stream byte
 * consumed; bytes past the stream read as zero) and, when seg_state is
 * non-null, the split points of every segment.  Skips chunks whose status
 * is a prologue error.  replaces ans.py:71-94 (_dec1) and ans.py:413-430
 * (the lone re-run of flagged lanes). */
int dc_ans_decode_serial(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                         const uint64_t *out_off, const uint64_t *out_len, const int32_t *chunk_ids,
                         int64_t n_ids, uint8_t *out, uint32_t seg_shift, const int64_t *seg_base,
                         uint32_t *seg_state, uint32_t *seg_off, int32_t *status, void *stream);

/* Segment-parallel decode (the hot kernel): each lane decodes one segment
 * from its split point; every segment's end state/offset must meet the next
 * split point (or 2^20 / stream end), else the chunk is flagged
 * DC_CHUNK_CHAIN for an exact serial re-decode.  tasks: int32 quads
 * (chunk, first segment (relative), segment count, 0), at most
 * dc_decode_task_segments() segments each, sorted by chunk.
 * replaces ans.py:97-200 (_dec2/_dec4 multi-lane interleave) with
 * thousands of lanes per chunk. */
int dc_decode_task_segments(void);
int dc_ans_decode_segments(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                           const uint64_t *out_off, const uint64_t *out_len, uint32_t seg_shift,
                           const int64_t *seg_base, const uint32_t *seg_state, const uint32_t *seg_off,
                           const int32_t *tasks, int64_t n_tasks, uint8_t *out, int32_t *status,
                           void *stream);
/* Narrow-CTA variant (4 warps, 3 CTAs/SM, 45 KB staging) for chunks of a few
 * hundred segments (e.g. 64 KiB): tasks of dc_decode_narrow_segments() segments
 * keep two interleaved chains per lane.  Task stream spans must fit
 * dc_decode_stage_cap(1) bytes (dc_decode_stage_cap(0) for the wide kernel). */
int dc_ans_decode_segments_narrow(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                                  const uint64_t *out_off, const uint64_t *out_len, uint32_t seg_shift,
                                  const int64_t *seg_base, const uint32_t *seg_state, const uint32_t *seg_off,
                                  const int32_t *tasks, int64_t n_tasks, uint8_t *out, int32_t *status,
                                  void *stream);
int dc_decode_narrow_segments(void);
int dc_decode_stage_cap(int narrow);

/* Small-chunk variant (every chunk <= dc_decode_small_max_chunk() bytes):
 * warp tasks of <= dc_decode_small_segments() segments, a compact per-warp
 * table (u8 slot->symbol + per-symbol update), stream read through L1.
 * Same arguments, task format, outputs and chain checks as
 * dc_ans_decode_segments.  replaces ans.py:97-200 at small chunk sizes. */
int dc_decode_small_segments(void);
int dc_decode_small_max_chunk(void);
int dc_ans_decode_small(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                        const uint64_t *out_off, const uint64_t *out_len, uint32_t seg_shift,
                        const int64_t *seg_base, const uint32_t *seg_state, const uint32_t *seg_off,
                        const int32_t *tasks, int64_t n_tasks, uint8_t *out, int32_t *status, void *stream);

/* Raw copy of store chunks (codec 0).  replaces container.py:309-310. */
int dc_store_copy(const uint8_t *base, const uint64_t *blob_off, const uint64_t *out_off,
                  const uint64_t *out_len, const uint8_t *codec, int64_t n_chunks, uint8_t *out,
                  void *stream);

/* --------------------------------------------------------------- CRC32
 * CRC-32/ISO-HDLC (zlib.crc32) of n byte ranges data[off[i] .. off[i]+len[i]);
 * max_len >= every len[i] (sizes the grid); data_bytes = the size of the
 * buffer at `data` (enables the TMA lane kernel for whole 64 KB spans of
 * ranges whose end is 128-byte aligned; 0 = piece kernel only).
 * replaces container.py:169 and :327-331 (zlib.crc32 per chunk). */
int dc_crc32_ranges(const uint8_t *data, uint64_t data_bytes, const uint64_t *off, const uint64_t *len, int64_t n,
                    uint64_t max_len, uint32_t *crc_out, void *stream);

/* ------------------------------------------------------- rANS encoding
 * Payload = `total` bytes split every `chunk_size` bytes (last may be short).
 */

/* Per-chunk 256-bin byte histograms (hist: n_chunks*256 u32, zeroed by the
 * call).  replaces ans.py:282 (np.bincount in AnsTable.for_data). */
int dc_hist_chunks(const uint8_t *data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                   uint32_t *hist, void *stream);

/* Largest-remainder normalization to 4096 with the reference's exact
 * tie-breaks, plus the packed 384-byte u12 wire table of every chunk.
 * replaces ans.py:213-243 (_normalize) and ans.py:246-253 (_pack_u12). */
int dc_normalize_tables(const uint32_t *hist, int64_t n_chunks, uint32_t *freq, uint8_t *table_bytes,
                        void *stream);

/* Reverse rANS encode of every chunk with todo[i] != 0: pass 1 runs each
 * chunk's serial state chain (one warp per chunk), pass 2 writes the
 * renormalization bytes in parallel from the recorded states (see
 * dc_ans_encode_work_bytes).  Emitted bytes are written BACKWARDS from the end of the chunk's slot in
 * `scratch` (slot i = [i*chunk_size, i*chunk_size + len_i)), so the decoder-
 * order stream is scratch[slot_end - stream_len[i] .. slot_end).  Encoding
 * stops early once the blob could not beat raw storage (388 + emitted >=
 * len_i; stream_len = UINT64_MAX then), since container.pack stores such
 * chunks.  flags bit 0 = standalone blob: never stop early (the caller
 * leaves 2*len_i + 8 writable bytes below the slot end).  When seg_state is
 * non-null, records the encoder state and emitted byte count at every
 * 2^seg_shift-th symbol (the decoder split points).
 * replaces ans.py:55-68 (_enc_kernel) and ans.py:316-325 (ans_compress). */
int dc_ans_encode_chunks(const uint8_t *data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                         const uint8_t *todo, const uint32_t *freq, uint8_t *scratch,
                         uint32_t *final_state, uint64_t *stream_len, uint32_t seg_shift,
                         const int64_t *seg_base, uint32_t *seg_state, uint32_t *seg_emitted,
                         uint32_t flags, void *work, uint64_t work_bytes, void *stream);

/* Device work space dc_ans_encode_chunks needs (caller-owned): the per-symbol
 * encoder states of pass 1 (4 B/symbol) and the byte counts every 256
 * symbols that let pass 2 emit the stream bytes in parallel.  flags bit 0:
 * standalone blob (never abort to store); bit 1: lengths only (skip pass 2). */
int dc_ans_encode_work_bytes(uint64_t total, uint64_t chunk_size, int64_t n_chunks, uint64_t *out);

/* Assemble chunk payloads into the container byte image: chunk i goes to
 * dst[file_off[i]]: ANS = table_bytes[i] | u32 LE final_state | stream;
 * store = raw bytes.  replaces container.py:160-177 (payload join). */
int dc_assemble_payloads(const uint8_t *data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                         const uint8_t *codec, const uint8_t *table_bytes, const uint32_t *final_state,
                         const uint64_t *stream_len, const uint8_t *scratch, const uint64_t *file_off,
                         uint8_t *dst, void *stream);

/* ------------------------------------------------ quantization (kernel 1)
 * dtype: 0 = f64 (the reference's type), 1 = f32, 2 = bf16, 3 = f16; widened
 * to f64 exactly.  s (f64 [cols]) may be NULL (identity scale).
 */

/* max |W[r,c] * s[c]| as the bits of a non-negative f64 (exact: max is
 * order-free), plus a non-finite flag.  f32 / bf16 / f16 inputs with cols % 8
 * == 0 take a streaming column-max pass: max|W*s| = max_c RN(max_r |W[r,c]| *
 * s[c]) since IEEE rounding is monotone and s > 0.  replaces scaling.py:78-81
 * (W*s) and :99 (np.abs(v).max()); WeightTensor's isfinite check
 * (tensors.py:33-34). */
int dc_quant_absmax(const void *w, int dtype, const double *s, int64_t rows, int64_t cols,
                    unsigned long long *absmax_bits, int *nonfinite, void *stream);

/* q = clip(sign(x) * floor(|x| + 0.5), -127, 127), x = (W*s) / w_scale in IEEE
 * f64.  replaces scaling.py:84-105 (_round_half_away, quantize). */
int dc_quantize(const void *w, int dtype, const double *s, int64_t rows, int64_t cols, double w_scale,
                int8_t *q, void *stream);

/* out = q * w_scale / s[c].  replaces scaling.py:114-117 (dequantize). */
int dc_dequantize(const int8_t *q, double w_scale, const double *s, int64_t rows, int64_t cols, double *out,
                  void *stream);

/* W8A8 activation prologue (scaling.py:143-149 on decode activations): for each
 * of n_tensors records {const void *x; const double *s; int8_t *q; double *sx;
 * double *xp; uint64_t *mbits; int64_t k} (dc_act_quant_bytes() each, device
 * array; xp = [ntok][k] f64 scratch, *mbits zeroed by the caller): X' = X / s
 * (IEEE f64), *sx = max|X'| / 127, q = clip(sign * floor(|X'| / sx + 0.5), +-127)
 * over [ntok][k] activations of `dtype` (as dc_quantize); max_k >= every k.
 * status[i] (zeroed by the caller) = 1 non-finite input, 2 zero dynamic range
 * (q = 0, sx = 0).  Two launches (scale + max, then round), all tensors each. */
int dc_act_quant_bytes(void);
int dc_act_quant(const void *tensors, int n_tensors, int dtype, int64_t ntok, int64_t max_k, int32_t *status,
                 void *stream);

/* Calibration statistics: acc_bits[c] = max(acc_bits[c], bits(|x[r, c]| as f64))
 * over rows x cols activations x (dtype as dc_quantize), i.e. a running
 * per-input-channel max|x| kept as f64 bit patterns (zero-initialise once).
 * replaces the exporter's forward pre-hook (exporter export.py:85-90). */
int dc_channel_absmax(const void *x, int dtype, int64_t rows, int64_t cols, uint64_t *acc_bits, void *stream);

/* out = W * s[c].  replaces scaling.py:78-81 (scale_weights). */
int dc_scale_weights(const double *w, const double *s, int64_t rows, int64_t cols, double *out, void *stream);

/* ------------------------------------------------------ pruning (kernel 1)
 * Zero the k lowest scores cm[c]*|q| (f64), ties by row-major index (rows*cols < 2^32).
 * replaces pruning.py:37-64 (prune_scores, _lowest_k, prune). */
/* score[r, c] = cm[c] * |q[r, c]| as f64 (rows x cols, row-major).
 * replaces pruning.py:37-40 (prune_scores). */
int dc_prune_scores(const int8_t *q, const double *cm, int64_t rows, int64_t cols, double *out, void *stream);
int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t *out_host);
int dc_prune_tensor(const int8_t *q, const double *cm, int64_t rows, int64_t cols, int64_t k, int8_t *out,
                    uint8_t *scratch, void *stream);
int dc_prune_rows(const int8_t *q, const double *cm, int64_t rows, int64_t cols, int64_t k_per_row, int8_t *out,
                  void *stream);

/* ------------------------------------------- W8A8 GEMM (kernel 3 core)
 * acc[t, n] (+)= sum_k x[t, k] * w[n, k], int8 x int8 -> exact int32 on
 * tcgen05 (kind::i8) with TMA-fed SWIZZLE_128B tiles and a TMEM accumulator.
 * w: [n_rows][k], x: [ntok <= 32][k] row-major int8, k % 128 == 0; kslice
 * (multiple of 128 dividing k) splits K across CTAs -- then results are
 * atomically added into acc (caller zeroes it), else stored.
 * replaces the integer product of scaling.py:148-151 (simulate_layer). */
int dc_w8a8_gemm(const int8_t *w, int64_t n_rows, int64_t k, const int8_t *x, int64_t ntok, int32_t *acc,
                 int64_t kslice, void *stream);

/* ------------------------------------- grouped + fused GEMMs (kernel 3)
 * A "layer table" is a device array of 32-byte records
 *   { const int8_t *x; int32_t *acc; int64_t t_off; int32_t n_rows; int32_t k; }
 * (x: [ntok][k] int8 activations, acc: [ntok][n_rows] int32 accumulators the
 * caller zeroes, t_off: the layer's byte offset in the DCC1 payload) and a
 * unit table is int32 quads (layer, m0, k0, kslice): 128 weight rows x a
 * K-slice each.  Every layer of a model runs in ONE launch.  ntok <= 16. */
int dc_gemm_tensor_bytes(void);
int dc_tmap_bytes(void);
/* Host helper: 2 CUtensorMaps per layer (W box 128x128, X box 128x16, SW128)
 * into maps_host (64-byte aligned). */
int dc_w8a8_grouped_maps(const int8_t *const *w_host, const int8_t *const *x_host, const int64_t *rows_host,
                         const int64_t *k_host, int n, int ntok, void *maps_host);
/* Uncompressed INT8 weights: TMA -> smem -> tcgen05.mma.kind::i8 -> TMEM. */
int dc_w8a8_grouped(const void *maps, const void *layers, const int32_t *units, int64_t n_units, int ntok,
                    void *stream);
/* Persistent grouped W8A8: one CTA per SM looping over the unit table (TMA
 * stream continuous across units, double-buffered TMEM accumulators);
 * `max_ctas` > 0 caps the grid (= SMs used), 0 = every SM. */
int dc_w8a8_grouped_persist(const void *maps, const void *tens, const int32_t *units, int64_t n_units, int ntok,
                            int max_ctas, void *stream);

/* Fused decompress -> W8A8 straight from DCC1 chunks (north-star kernel 3):
 * one persistent 16-warp CTA per SM; items (layer, m0, k0, klen) of
 * dc_fused_item_rows() rows x klen <= dc_fused_item_k() bytes; 1024 decode
 * chains (each from its split point, seg_shift 8) write 16-byte groups into a
 * 6-deep TMEM ring of 32-byte K-steps; the last warp to finish a K-step issues
 * its tcgen05.mma (A from TMEM) for all 8 row tiles -- decoded weights never
 * reach HBM.  chunk_size, layer offsets and k multiples of 256.  Broken chains
 * (or split points outside the stream) set status[chunk] = DC_CHUNK_CHAIN
 * (caller falls back to decode + GEMM).  Replaces scaling.py:148-151 on
 * weights decoded by ans.py:71-94. */
int dc_fused_item_rows(void);
int dc_fused_item_k(void);
/* `epi` (nullable): per layer {float *y; uint32_t *cnt; float scale; int32 n_slices;
 * const double *sx; double sw} -- y = acc * (sx ? (float)(*sx * sw) : scale)
 * (dc_fused_epi_bytes() each): the fused dequant epilogue y = acc * scale written
 * by the last K-slice item of each 1024-row block (cnt zeroed before first use).
 * `max_ctas` > 0 caps the persistent grid (one CTA per SM) so a concurrent INT8
 * GEMM on another stream gets the remaining SMs; 0 = every SM. */
int dc_fused_epi_bytes(void);
int dc_fused_ring_gemm(const uint8_t *base, const uint64_t *blob_off, const uint64_t *blob_len,
                       const uint64_t *out_len, const uint8_t *codec, uint64_t chunk_size, const int64_t *seg_base,
                       const uint32_t *seg_state, const uint32_t *seg_off, const void *layers, const int32_t *items,
                       int64_t n_items, int ntok, int32_t *status, const void *epi, int max_ctas,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DCOMP_B200_H */
