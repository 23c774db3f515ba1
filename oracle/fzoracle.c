/*
 * fzoracle.c -- CPU restatement of the fzpipe hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for the B200 kernels.  It is NOT product
 * code: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or the timed
 * CPU baseline.  The product path (paper_2509_20563_b200) never calls it.
 *
 * Every routine restates one reference routine from
 * /root/reference/pkg/src/fzpipe (cited file:line), keeping the reference's
 * exact floating-point operation order: f64 arithmetic, no FMA contraction
 * (build with -ffp-contract=off), IEEE division, round-to-nearest f64->f32.
 * Pinned against the reference itself: tests/golden/*.npz were produced by
 * importing fzpipe (scripts/make_golden.py) and tests/test_oracle_golden.py
 * checks this file against them bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FZO_EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------- min/max */

/* pipeline.py:360-361 / core.py:162-163: exact f32 min and max. */
FZO_EXPORT void fzo_minmax(const float *x, int64_t n, float *lo, float *hi) {
    float a = x[0], b = x[0];
    for (int64_t i = 1; i < n; i++) {
        float v = x[i];
        if (v < a) a = v;
        if (v > b) b = v;
    }
    *lo = a;
    *hi = b;
}

/* ------------------------------------------------------------- quantizer */

/* predict.py:70-90 (_quant_store). */
static inline void quant_store(double v, double pred, double two_eb, double eb, int64_t radius,
                               uint32_t *codes, float *recon, uint8_t *flags, int64_t t) {
    double q = (v - pred) / two_eb;
    double aq = fabs(q);
    double f = floor(aq);
    double r = (aq - f >= 0.5) ? f + 1.0 : f;
    if (r < (double)radius) {
        int64_t s = (int64_t)r;
        if (q < 0.0) s = -s;
        float rec = (float)(pred + two_eb * (double)s);
        if (fabs((double)rec - v) <= eb) {
            codes[t] = (uint32_t)(s + radius);
            recon[t] = rec;
            return;
        }
    }
    codes[t] = (uint32_t)radius;
    recon[t] = (float)v;
    flags[t] = 1;
}

/* ---------------------------------------------------------------- Lorenzo */

/* predict.py:93-115 (_lorenzo_encode).  recon must be zero-initialised. */
FZO_EXPORT void fzo_lorenzo_encode(const float *orig, uint32_t *codes, float *recon, uint8_t *flags,
                                   int64_t n0, int64_t n1, int64_t n2, double eb, int64_t radius) {
    const double two_eb = 2.0 * eb;
    const int64_t p = n1 * n2;
    for (int64_t i = 0; i < n0; i++)
        for (int64_t j = 0; j < n1; j++)
            for (int64_t k = 0; k < n2; k++) {
                int64_t t = (i * n1 + j) * n2 + k;
                double pred = 0.0;
                if (i > 0) pred += recon[t - p];
                if (j > 0) pred += recon[t - n2];
                if (k > 0) pred += recon[t - 1];
                if (i > 0 && j > 0) pred -= recon[t - p - n2];
                if (i > 0 && k > 0) pred -= recon[t - p - 1];
                if (j > 0 && k > 0) pred -= recon[t - n2 - 1];
                if (i > 0 && j > 0 && k > 0) pred += recon[t - p - n2 - 1];
                quant_store((double)orig[t], pred, two_eb, eb, radius, codes, recon, flags, t);
            }
}

/* predict.py:118-144 (_lorenzo_decode).  Outliers pre-scattered into recon/flags. */
FZO_EXPORT void fzo_lorenzo_decode(const uint32_t *codes, const uint8_t *flags, float *recon,
                                   int64_t n0, int64_t n1, int64_t n2, double eb, int64_t radius) {
    const double two_eb = 2.0 * eb;
    const int64_t p = n1 * n2;
    for (int64_t i = 0; i < n0; i++)
        for (int64_t j = 0; j < n1; j++)
            for (int64_t k = 0; k < n2; k++) {
                int64_t t = (i * n1 + j) * n2 + k;
                if (flags[t]) continue;
                double pred = 0.0;
                if (i > 0) pred += recon[t - p];
                if (j > 0) pred += recon[t - n2];
                if (k > 0) pred += recon[t - 1];
                if (i > 0 && j > 0) pred -= recon[t - p - n2];
                if (i > 0 && k > 0) pred -= recon[t - p - 1];
                if (j > 0 && k > 0) pred -= recon[t - n2 - 1];
                if (i > 0 && j > 0 && k > 0) pred += recon[t - p - n2 - 1];
                int64_t s = (int64_t)codes[t] - radius;
                recon[t] = (float)(pred + two_eb * (double)s);
            }
}

/* ------------------------------------------------------------ interpolation */

/* predict.py:147-160 (_interp_predict). */
static inline double interp_predict(const float *recon, int64_t t, int64_t c, int64_t n, int64_t sh,
                                    int64_t s3h, int64_t h, const double *w) {
    if (c - 3 * h >= 0 && c + 3 * h < n)
        return w[0] * (double)recon[t - s3h] + w[1] * (double)recon[t - sh] +
               w[2] * (double)recon[t + sh] + w[3] * (double)recon[t + s3h];
    if (c + h < n) return 0.5 * (double)recon[t - sh] + 0.5 * (double)recon[t + sh];
    return (double)recon[t - sh];
}

static inline void interp_visit(const float *orig, uint32_t *codes, float *recon, uint8_t *flags,
                                int64_t t, double pred, double two_eb, double eb, int64_t radius,
                                int encode) {
    if (encode) {
        quant_store((double)orig[t], pred, two_eb, eb, radius, codes, recon, flags, t);
    } else if (!flags[t]) {
        int64_t s = (int64_t)codes[t] - radius;
        recon[t] = (float)(pred + two_eb * (double)s);
    }
}

/* predict.py:163-201 (_interp_pass): one (level h, axis) pass. */
FZO_EXPORT void fzo_interp_pass(const float *orig, uint32_t *codes, float *recon, uint8_t *flags,
                                int64_t n0, int64_t n1, int64_t n2, int64_t h, int axis, double eb,
                                int64_t radius, const double *w, int encode) {
    const double two_eb = 2.0 * eb;
    const int64_t h2 = 2 * h;
    if (axis == 0) {
        for (int64_t i = h; i < n0; i += h2)
            for (int64_t j = 0; j < n1; j += h2)
                for (int64_t k = 0; k < n2; k += h2) {
                    int64_t t = (i * n1 + j) * n2 + k;
                    double pred = interp_predict(recon, t, i, n0, h * n1 * n2, 3 * h * n1 * n2, h, w);
                    interp_visit(orig, codes, recon, flags, t, pred, two_eb, eb, radius, encode);
                }
    } else if (axis == 1) {
        for (int64_t i = 0; i < n0; i += h)
            for (int64_t j = h; j < n1; j += h2)
                for (int64_t k = 0; k < n2; k += h2) {
                    int64_t t = (i * n1 + j) * n2 + k;
                    double pred = interp_predict(recon, t, j, n1, h * n2, 3 * h * n2, h, w);
                    interp_visit(orig, codes, recon, flags, t, pred, two_eb, eb, radius, encode);
                }
    } else {
        for (int64_t i = 0; i < n0; i += h)
            for (int64_t j = 0; j < n1; j += h)
                for (int64_t k = h; k < n2; k += h2) {
                    int64_t t = (i * n1 + j) * n2 + k;
                    double pred = interp_predict(recon, t, k, n2, h, 3 * h, h, w);
                    interp_visit(orig, codes, recon, flags, t, pred, two_eb, eb, radius, encode);
                }
    }
}

/* predict.py:309-319 (_run_interp): levels h = stride/2 .. 1, axes 0,1,2. */
FZO_EXPORT void fzo_interp_run(const float *orig, uint32_t *codes, float *recon, uint8_t *flags,
                               int64_t n0, int64_t n1, int64_t n2, double eb, int64_t radius,
                               int64_t anchor_stride, const double *w, int encode) {
    for (int64_t h = anchor_stride / 2; h >= 1; h /= 2)
        for (int axis = 0; axis < 3; axis++)
            fzo_interp_pass(orig, codes, recon, flags, n0, n1, n2, h, axis, eb, radius, w, encode);
}

/* -------------------------------------------------------------- histogram */

/* encode.py:79-84 (histogram_exact); topk (87-111) is identical by contract.
 * Returns -1 (CodeOutOfRange) if any code >= nbins. */
FZO_EXPORT int fzo_histogram(const uint32_t *codes, int64_t n, int64_t nbins, uint64_t *bins) {
    memset(bins, 0, (size_t)nbins * sizeof(uint64_t));
    for (int64_t i = 0; i < n; i++) {
        if ((int64_t)codes[i] >= nbins) return -1;
        bins[codes[i]]++;
    }
    return 0;
}

/* ------------------------------------------------------------ Huffman book */

typedef struct { uint64_t w; uint32_t tb; } pm_item;

static int pm_item_less(const pm_item *a, const pm_item *b) {
    return a->w < b->w || (a->w == b->w && a->tb < b->tb);
}

static int pm_cmp(const void *x, const void *y) {
    const pm_item *a = (const pm_item *)x, *b = (const pm_item *)y;
    if (pm_item_less(a, b)) return -1;
    if (pm_item_less(b, a)) return 1;
    return 0;
}

/* encode.py:174-213 (_package_merge_lengths), restated without coin trees.
 * Levels: M_0 = base; P_l = pairwise packages of M_{l-1}; M_l = merge(base,
 * P_l) by (weight, tiebreak) exactly as heapq.merge's two-head comparison
 * (cross-list key ties are impossible: a package with tiebreak s contains
 * leaf s plus positive weight).  The selected items of every M_l form a
 * prefix, so each leaf's length is the number of levels whose selected
 * prefix contains it.  Returns 0, or -2 on allocation failure. */
FZO_EXPORT int fzo_package_merge(const uint64_t *counts, int64_t nsym, int limit, uint8_t *lengths) {
    memset(lengths, 0, (size_t)nsym);
    int64_t m = 0;
    for (int64_t s = 0; s < nsym; s++) m += counts[s] != 0;
    if (m == 0) return 0;
    if (m == 1) {
        for (int64_t s = 0; s < nsym; s++)
            if (counts[s]) lengths[s] = 1;
        return 0;
    }
    pm_item *base = malloc(sizeof(pm_item) * m);
    pm_item *pk = malloc(sizeof(pm_item) * m);
    pm_item *merged = malloc(sizeof(pm_item) * 2 * m);
    uint8_t *isbase = malloc((size_t)limit * 2 * m); /* isbase[l][pos] for M_l */
    int64_t *mlen = malloc(sizeof(int64_t) * limit);
    if (!base || !pk || !merged || !isbase || !mlen) {
        free(base); free(pk); free(merged); free(isbase); free(mlen);
        return -2;
    }
    int64_t b = 0;
    for (int64_t s = 0; s < nsym; s++)
        if (counts[s]) { base[b].w = counts[s]; base[b].tb = (uint32_t)s; b++; }
    qsort(base, m, sizeof(pm_item), pm_cmp);
    /* M_0 = base */
    memcpy(merged, base, sizeof(pm_item) * m);
    int64_t mcur = m;
    memset(isbase, 1, (size_t)m);
    mlen[0] = m;
    for (int l = 1; l < limit; l++) {
        int64_t np = mcur / 2;
        for (int64_t t = 0; t < np; t++) {
            pk[t].w = merged[2 * t].w + merged[2 * t + 1].w;
            pk[t].tb = merged[2 * t].tb;
        }
        int64_t i = 0, j = 0, o = 0;
        uint8_t *ib = isbase + (size_t)l * 2 * m;
        while (i < m || j < np) {
            if (j >= np || (i < m && !pm_item_less(&pk[j], &base[i]))) {
                merged[o] = base[i++]; ib[o++] = 1;
            } else {
                merged[o] = pk[j++]; ib[o++] = 0;
            }
        }
        mcur = o;
        mlen[l] = o;
    }
    /* take = M_{limit-1}[:2(m-1)]; walk levels down. */
    int64_t L = 2 * (m - 1);
    for (int l = limit - 1; l >= 1; l--) {
        const uint8_t *ib = isbase + (size_t)l * 2 * m;
        int64_t nb = 0;
        for (int64_t p = 0; p < L; p++) nb += ib[p];
        for (int64_t p = 0; p < nb; p++) lengths[base[p].tb]++;
        L = 2 * (L - nb);
    }
    for (int64_t p = 0; p < L; p++) lengths[base[p].tb]++;
    free(base); free(pk); free(merged); free(isbase); free(mlen);
    return 0;
}

/* encode.py:155-171 (canonical_codewords): by (length asc, symbol asc). */
FZO_EXPORT void fzo_canonical_codewords(const uint8_t *cl, int64_t nsym, uint32_t *cw) {
    memset(cw, 0, sizeof(uint32_t) * nsym);
    uint64_t code = 0;
    int prev = 0;
    for (int l = 1; l <= 32; l++)
        for (int64_t s = 0; s < nsym; s++) {
            if (cl[s] != l) continue;
            code <<= (l - prev);
            cw[s] = (uint32_t)code;
            code += 1;
            prev = l;
        }
}

/* encode.py:220-231 (_hf_pack).  out must be zeroed; returns bit count. */
FZO_EXPORT int64_t fzo_huffman_pack(const uint32_t *sym, int64_t n, const uint32_t *cw,
                                    const uint8_t *cl, uint8_t *out) {
    int64_t bitpos = 0;
    for (int64_t i = 0; i < n; i++) {
        uint32_t c = cw[sym[i]];
        int l = cl[sym[i]];
        for (int b = l - 1; b >= 0; b--) {
            if ((c >> b) & 1) out[bitpos >> 3] |= (uint8_t)(1u << (7 - (bitpos & 7)));
            bitpos++;
        }
    }
    return bitpos;
}

/* encode.py:234-276 (_decode_tables + _hf_unpack).  Returns the final bit
 * position, -1 on truncation, -2 on a pattern matching no codeword. */
FZO_EXPORT int64_t fzo_huffman_unpack(const uint8_t *stream, int64_t nbytes, int64_t n,
                                      const uint8_t *cl, int64_t nsym, uint32_t *out) {
    int maxlen = 0;
    int64_t cnt[34] = {0};
    for (int64_t s = 0; s < nsym; s++) {
        if (cl[s] > maxlen) maxlen = cl[s];
        if (cl[s]) cnt[cl[s]]++;
    }
    int64_t first_code[34] = {0}, first_idx[34] = {0}, limit[34] = {0};
    int64_t code = 0, idx = 0;
    for (int l = 1; l <= maxlen; l++) {
        code <<= 1;
        first_code[l] = code;
        first_idx[l] = idx;
        limit[l] = code + cnt[l];
        code += cnt[l];
        idx += cnt[l];
    }
    uint32_t *sym_sorted = malloc(sizeof(uint32_t) * (idx ? idx : 1));
    int64_t q = 0;
    for (int l = 1; l <= maxlen; l++)
        for (int64_t s = 0; s < nsym; s++)
            if (cl[s] == l) sym_sorted[q++] = (uint32_t)s;
    const int64_t total_bits = nbytes * 8;
    int64_t bitpos = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t c = 0;
        int l = 0;
        for (;;) {
            if (bitpos >= total_bits) { free(sym_sorted); return -1; }
            int bit = (stream[bitpos >> 3] >> (7 - (bitpos & 7))) & 1;
            bitpos++;
            c = (c << 1) | bit;
            l++;
            if (l > maxlen) { free(sym_sorted); return -2; }
            if (c < limit[l]) {
                out[i] = sym_sorted[first_idx[l] + c - first_code[l]];
                break;
            }
        }
    }
    free(sym_sorted);
    return bitpos;
}

/* ------------------------------------------------------------- bitshuffle */

/* encode.py:329-353: 256-code blocks, 16 bit planes of 8 LE u32 words,
 * word index blk*128 + p*8 + w; bitmap LSB-first; payload = nonzero words.
 * bitmap must hold nblocks*16 bytes (zeroed by callee); payload nblocks*128
 * words.  Returns the payload word count. */
FZO_EXPORT int64_t fzo_bitshuffle_encode(const uint32_t *codes, int64_t n, uint8_t *bitmap,
                                         uint32_t *payload) {
    int64_t nblocks = (n + 255) / 256;
    memset(bitmap, 0, (size_t)nblocks * 16);
    int64_t np = 0;
    for (int64_t blk = 0; blk < nblocks; blk++)
        for (int p = 0; p < 16; p++)
            for (int w = 0; w < 8; w++) {
                uint32_t word = 0;
                for (int j = 0; j < 32; j++) {
                    int64_t t = blk * 256 + 32 * w + j;
                    uint32_t c = t < n ? (codes[t] & 0xFFFFu) : 0u;
                    word |= ((c >> p) & 1u) << j;
                }
                int64_t wi = blk * 128 + p * 8 + w;
                if (word) {
                    bitmap[wi >> 3] |= (uint8_t)(1u << (wi & 7));
                    payload[np++] = word;
                }
            }
    return np;
}

/* encode.py:356-391 (bitshuffle_decode), after the host-side length checks.
 * Returns 0, -3 for nonzero padding bits, -4 for a decoded code >= 2R. */
FZO_EXPORT int fzo_bitshuffle_decode(const uint8_t *bitmap, const uint32_t *payload, int64_t n,
                                     int64_t radius, uint32_t *out) {
    int64_t nblocks = (n + 255) / 256;
    int64_t pi = 0;
    uint32_t words[128];
    for (int64_t blk = 0; blk < nblocks; blk++) {
        for (int i = 0; i < 128; i++) {
            int64_t wi = blk * 128 + i;
            words[i] = (bitmap[wi >> 3] >> (wi & 7)) & 1 ? payload[pi++] : 0u;
        }
        for (int w = 0; w < 8; w++)
            for (int j = 0; j < 32; j++) {
                uint32_t c = 0;
                for (int p = 0; p < 16; p++) c |= ((words[p * 8 + w] >> j) & 1u) << p;
                int64_t t = blk * 256 + 32 * w + j;
                if (t < n) out[t] = c;
                else if (c) return -3;
            }
    }
    for (int64_t t = 0; t < n; t++)
        if ((int64_t)out[t] >= 2 * radius) return -4;
    return 0;
}
