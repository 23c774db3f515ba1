/*
 * fzb200.h -- C ABI of the B200 (sm_100a) FZModules hot path.
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * Every entry point is asynchronous on `stream` and returns 0 or a negative
 * FZB_E_* launch/argument error.  Data-dependent failures (corrupt streams,
 * malformed codes, ...) are OR-ed as FZB_ERR_* bits into a caller-provided
 * device status word (uint32_t*), which the host reads once per pipeline
 * run and maps 1:1 onto the reference's FZError classes.
 *
 * Each function names the reference routine it replaces (fzpipe,
 * /root/reference/pkg/src/fzpipe).  The reference is Python + numba; these
 * are the calls its stage dispatchers (pipeline.py:269-297, 415-436) would
 * bind through ctypes -- see INTEGRATION.md.
 *
 * Device layout conventions: quantization codes are u16 (radius <= 32768,
 * the bitshuffle limit of encode.py:336-337); outlier flags are a u32
 * bitmap with bit (t & 31) of word t >> 5; eb_abs lives in device memory
 * (double*) so no host sync is needed between min/max and the predictor.
 */
#ifndef FZB200_H
#define FZB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FZB_API __attribute__((visibility("default")))

/* negative return codes (argument / launch errors) */
#define FZB_E_WORKSPACE (-1001) /* workspace too small */
#define FZB_E_RADIUS (-1002)    /* radius outside [1, 32768] (RadiusTooLarge) */
#define FZB_E_ARG (-1003)       /* invalid argument */

FZB_API int fzb_abi_version(void);
/* Record a CUDA event on a stream; external = 1 makes it an event-record node
 * when the stream is being captured into a CUDA graph (per-kernel timing of
 * replayed graphs). */
FZB_API int fzb_event_create(void **event);
FZB_API int fzb_event_destroy(void *event);
FZB_API int fzb_event_record(void *event, void *stream, int external);
FZB_API int fzb_event_elapsed_ms(void *start, void *stop, float *ms);

/* ---- a1: bound resolution (pipeline.py:360-364, core.py:155-170) ------- */
/* Exact f32 min/max of d_in[0..n) -> d_lohi[0..1]; sets FZB_ERR_NONFINITE. */
FZB_API size_t fzb_minmax_workspace_bytes(uint64_t n);
FZB_API int fzb_minmax_f32(const float *d_in, uint64_t n, float *d_lohi, void *d_ws, size_t ws_bytes,
                           uint32_t *d_status, void *stream);
/* d_eb = eb_mode ? magnitude * (hi - lo) : magnitude, in f64 exactly as core.py:167. */
FZB_API int fzb_resolve_bound(const float *d_lohi, int eb_mode, double magnitude, double *d_eb, void *stream);

/* Codes per chunk of the encoder's "holds a code != R" flags (fzb_histogram_chunks,
 * fzb_lorenzo1d_walk_f32, fzb_huffman_encode_chunks). */
#define FZB_HF_CHUNK 4096

/* ---- a2-a4: Lorenzo (predict.py:93-144, 221-253) ------------------------ */
/* The workspace carries a launch epoch and tagged halo slots across calls:
 * zero-fill it once when it is allocated, then pass it unchanged (any later
 * geometry that fits may reuse it; never share one between two streams). */
FZB_API size_t fzb_lorenzo_workspace_bytes(uint32_t n0, uint32_t n1, uint32_t n2);
/* codes u16[n]; d_bitmap u32[ceil(n/32)] zeroed by caller; outliers set bits.
 * Inputs must be finite, as fzpipe's Field enforces (core.py:98-100). */
FZB_API int fzb_lorenzo_encode_f32(const float *d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double *d_eb,
                                   uint32_t radius, uint16_t *d_codes, uint32_t *d_bitmap, void *d_ws,
                                   size_t ws_bytes, void *stream);
/* 1D fields in two steps, so the field is read once before its bound is
 * known (same result as fzb_lorenzo_encode_f32, which runs both):
 * prepare writes the walker's min-max summaries into d_ws (workspace of
 * fzb_lorenzo_workspace_bytes(1, 1, n)), fills d_codes with radius and, with
 * d_lohi, stores the field's (min, max) and FZB_ERR_NONFINITE exactly as
 * fzb_minmax_f32 (replaces pipeline.py:360-361's min/max pass); walk then
 * runs the event walker with the resolved d_eb. */
FZB_API int fzb_lorenzo1d_prepare_f32(const float *d_in, uint64_t n, uint32_t radius, uint16_t *d_codes,
                                      float *d_lohi, void *d_ws, size_t ws_bytes, uint32_t *d_status,
                                      void *stream);
/* d_notr (optional, u8[ceil(n / FZB_HF_CHUNK)]): zeroed here, then 1 for every
 * chunk that gets a code != radius -- the flags of fzb_histogram_chunks. */
FZB_API int fzb_lorenzo1d_walk_f32(const float *d_in, uint64_t n, const double *d_eb, uint32_t radius,
                                   uint16_t *d_codes, uint32_t *d_bitmap, uint8_t *d_notr, void *d_ws,
                                   size_t ws_bytes, void *stream);
/* d_recon holds the outlier values (fzb_outlier_scatter) and is completed in place. */
FZB_API int fzb_lorenzo_decode_f32(const uint16_t *d_codes, const uint32_t *d_bitmap, float *d_recon, uint32_t n0,
                                   uint32_t n1, uint32_t n2, const double *d_eb, uint32_t radius, void *d_ws,
                                   size_t ws_bytes, void *stream);

/* Batches of nf same-shaped fields in one wavefront launch (fields
 * in flight per GPU).  Field f: d_in/d_codes/d_recon + f * field_stride
 * elements, d_bitmap + f * bitmap_stride_words, bound d_eb[f].  Same outputs
 * as nf single-field calls; the workspace rules above apply. */
FZB_API size_t fzb_lorenzo_batch_workspace_bytes(uint32_t nf, uint32_t n0, uint32_t n1, uint32_t n2);
FZB_API int fzb_lorenzo_encode_batch_f32(const float *d_in, uint32_t nf, uint64_t field_stride, uint32_t n0,
                                         uint32_t n1, uint32_t n2, const double *d_eb, uint32_t radius,
                                         uint16_t *d_codes, uint32_t *d_bitmap, uint64_t bitmap_stride_words,
                                         void *d_ws, size_t ws_bytes, void *stream);
FZB_API int fzb_lorenzo_decode_batch_f32(const uint16_t *d_codes, const uint32_t *d_bitmap,
                                         uint64_t bitmap_stride_words, float *d_recon, uint32_t nf,
                                         uint64_t field_stride, uint32_t n0, uint32_t n1, uint32_t n2,
                                         const double *d_eb, uint32_t radius, void *d_ws, size_t ws_bytes,
                                         void *stream);

/* ---- a5-a6: G-Interp (predict.py:147-201, 270-344) ---------------------- */
/* d_recon: f32[n] workspace (encode) / output (decode); d_anchors f32[prod((d-1)/stride+1)]. */
FZB_API int fzb_interp_encode_f32(const float *d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double *d_eb,
                                  uint32_t radius, uint32_t anchor_stride, const double *h_weights4,
                                  uint16_t *d_codes, float *d_recon, uint32_t *d_bitmap, float *d_anchors,
                                  void *stream);
FZB_API int fzb_interp_decode_f32(const uint16_t *d_codes, const uint32_t *d_bitmap, const float *d_anchors,
                                  float *d_recon, uint32_t n0, uint32_t n1, uint32_t n2, const double *d_eb,
                                  uint32_t radius, uint32_t anchor_stride, const double *h_weights4, void *stream);

/* ---- outliers (predict.py:212-214, pipeline.py:300-304, 402-412) ------- */
FZB_API size_t fzb_outlier_workspace_bytes(uint64_t n);
/* bitmap -> sorted u64 indices + f32 values (gathered from d_in); *d_count = k. */
FZB_API int fzb_outlier_compact(const uint32_t *d_bitmap, uint64_t n, const float *d_in, uint64_t *d_idx,
                                float *d_vals, uint64_t *d_count, void *d_ws, size_t ws_bytes, void *stream);
/* Scatter k outliers into d_recon + d_bitmap (zeroed by caller) and check the
 * QuantOutput invariants (core.py:207-215) against d_codes.  d_codes may be
 * NULL: the sentinel check is then left to fzb_outlier_check, so the scatter
 * can run beside the codec decode (the reference's decompress graph,
 * pipeline.py:490-580: huffman-decode || outlier-scatter). */
FZB_API int fzb_outlier_scatter(const uint64_t *d_idx, const float *d_vals, uint64_t k, uint64_t n,
                                const uint16_t *d_codes, uint32_t radius, float *d_recon, uint32_t *d_bitmap,
                                uint32_t *d_status, void *stream);
/* core.py:214-215: every outlier position must hold the sentinel code. */
FZB_API int fzb_outlier_check(const uint64_t *d_idx, uint64_t k, uint64_t n, const uint16_t *d_codes,
                              uint32_t radius, uint32_t *d_status, void *stream);

/* ---- a7: histogram (encode.py:79-111) ----------------------------------- */
/* d_bins u64[nbins] is zeroed here; codes >= nbins set FZB_ERR_CODE_RANGE. */
FZB_API int fzb_histogram(const uint16_t *d_codes, uint64_t n, uint32_t nbins, uint64_t *d_bins,
                          uint32_t *d_status, void *stream);
/* Same, plus d_notr u8[ceil(n / FZB_HF_CHUNK)]: 1 iff that chunk of codes holds
 * a code other than nbins / 2 (the zero-code R).  fzb_huffman_encode_chunks
 * uses it to skip re-reading chunks that are all R (low-entropy fields). */
FZB_API int fzb_histogram_chunks(const uint16_t *d_codes, uint64_t n, uint32_t nbins, uint64_t *d_bins,
                                 uint8_t *d_notr, uint32_t *d_status, void *stream);
/* Same bins from flags already known (fzb_lorenzo1d_walk_f32's): full
 * chunks whose flag is clear are counted as FZB_HF_CHUNK codes R without
 * being read. */
FZB_API int fzb_histogram_flagged(const uint16_t *d_codes, uint64_t n, uint32_t nbins, uint64_t *d_bins,
                                  const uint8_t *d_notr, uint32_t *d_status, void *stream);

/* ---- a8: codebook (encode.py:118-217) ----------------------------------- */
FZB_API size_t fzb_huffman_build_workspace_bytes(uint32_t nsym);
/* Length-limited (32) package-merge with the reference's tie-breaking,
 * canonical codewords, and d_bit_count = sum(bins * len). */
FZB_API int fzb_huffman_build(const uint64_t *d_bins, uint32_t nsym, uint8_t *d_lengths, uint32_t *d_codewords,
                              uint64_t *d_bit_count, void *d_ws, size_t ws_bytes, void *stream);

/* ---- a9: Huffman encode (encode.py:220-231, 279-291) -------------------- */
FZB_API size_t fzb_huffman_encode_workspace_bytes(uint64_t n);
/* MSB-first stream written as d_out bytes (capacity out_cap >= ceil(bits/8)
 * rounded up to 4); sets FZB_ERR_HF_MISMATCH if the packed length differs
 * from *d_bit_count. */
FZB_API int fzb_huffman_encode(const uint16_t *d_codes, uint64_t n, const uint8_t *d_lengths,
                               const uint32_t *d_codewords, uint32_t nsym, const uint64_t *d_bit_count,
                               uint8_t *d_out, uint64_t out_cap, void *d_ws, size_t ws_bytes, uint32_t *d_status,
                               void *stream);
/* Same stream; d_notr from fzb_histogram_chunks over the same codes (NULL =
 * read every chunk). */
FZB_API int fzb_huffman_encode_chunks(const uint16_t *d_codes, uint64_t n, const uint8_t *d_lengths,
                                      const uint32_t *d_codewords, uint32_t nsym, const uint64_t *d_bit_count,
                                      const uint8_t *d_notr, uint8_t *d_out, uint64_t out_cap, void *d_ws,
                                      size_t ws_bytes, uint32_t *d_status, void *stream);

/* ---- a10: Huffman decode (encode.py:234-317) ----------------------------- */
FZB_API size_t fzb_huffman_decode_workspace_bytes(uint64_t nbytes, uint32_t nsym);
FZB_API int fzb_huffman_decode(const uint8_t *d_stream, uint64_t nbytes, uint64_t n, const uint8_t *d_lengths,
                               uint32_t nsym, uint16_t *d_codes, void *d_ws, size_t ws_bytes, uint32_t *d_status,
                               void *stream);

/* ---- a11-a12: bitshuffle (encode.py:324-391) ----------------------------- */
FZB_API size_t fzb_bitshuffle_workspace_bytes(uint64_t n);
/* d_bitmap: nblocks*16 bytes; d_payload: capacity nblocks*128 words; *d_nwords = payload words. */
FZB_API int fzb_bitshuffle_encode(const uint16_t *d_codes, uint64_t n, uint8_t *d_bitmap, uint32_t *d_payload,
                                  uint64_t *d_nwords, void *d_ws, size_t ws_bytes, void *stream);
FZB_API int fzb_bitshuffle_decode(const uint8_t *d_bitmap, const uint32_t *d_payload, uint64_t payload_words,
                                  uint64_t n, uint32_t radius, uint16_t *d_codes, void *d_ws, size_t ws_bytes,
                                  uint32_t *d_status, void *stream);

/* ---- utilities ----------------------------------------------------------- */
FZB_API int fzb_fill_u16(uint16_t *d_dst, uint64_t n, uint16_t value, void *stream);

/* opt-in pipeline 5: sampled profiling of the G-Interp (anchor stride, weights)
 * candidates (16|8) x (cubic, linear, natural cubic); u64 costs into d_scores[6] */
FZB_API int fzb_interp_profile(const float *d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double *d_eb,
                               uint64_t *d_scores, void *stream);

/* ---- opt-in dual-quant Lorenzo (pipeline ids 3/4; no reference counterpart:
 * north_star items 1 and 4).  p = rint(x / 2eb) with |x / 2eb| < 2^27 (else
 * status bit 15), deltas = integer Lorenzo difference of p (zero padding),
 * codes = delta + R or R for an outlier (|delta| >= R or |RN32(2eb p) - x| > eb,
 * flag set in d_bitmap).  Decode = prefix sums along k, j, i. */
FZB_API int fzb_dualquant_encode_f32(const float *d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double *d_eb,
                                     uint32_t radius, uint16_t *d_codes, uint32_t *d_bitmap, uint32_t *d_status,
                                     void *stream);
/* deltas of the *d_k compacted outliers (fzb_outlier_compact indices) */
FZB_API int fzb_dualquant_outlier_deltas(const float *d_in, uint32_t n0, uint32_t n1, uint32_t n2,
                                         const uint64_t *d_idx, const uint64_t *d_k, const double *d_eb,
                                         uint32_t radius, int32_t *d_deltas, uint32_t *d_status, void *stream);
FZB_API size_t fzb_dualquant_decode_workspace_bytes(uint32_t n0, uint32_t n1, uint32_t n2);
/* codes + k outliers (indices, deltas, values) -> d_out; d_bitmap zeroed by the caller */
FZB_API int fzb_dualquant_decode_f32(const uint16_t *d_codes, const uint64_t *d_idx, const int32_t *d_deltas,
                                     const float *d_vals, uint64_t k, uint32_t n0, uint32_t n1, uint32_t n2,
                                     const double *d_eb, uint32_t radius, uint32_t *d_bitmap, float *d_out,
                                     void *d_ws, size_t ws_bytes, uint32_t *d_status, void *stream);

/* ---- verification: metrics.quality (metrics.py:49-75) bit-identical ------ */
/* Sums the leaves of numpy's pairwise-sum tree of d*d (d = f64(orig) -
 * f64(recon)); d_leaf_len <= 128.  d_red[0] = bits of max|d|, d_red[1] /
 * d_red[2] = order-preserving keys of min / max(orig); initialise to
 * {0, ~0ull, 0}.  The host folds the leaf sums up the same tree. */
FZB_API int fzb_quality_leaves(const float *d_orig, const float *d_recon, const uint64_t *d_leaf_off,
                               const uint16_t *d_leaf_len, uint64_t nleaves, double *d_leaf_sum,
                               unsigned long long *d_red, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FZB200_H */
