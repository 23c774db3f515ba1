// lorenzo.cu -- exact (bit-for-bit) Lorenzo predictor-quantizer for sm_100a.
//
// Reference: fzpipe predict.py:93-144 (_lorenzo_encode / _lorenzo_decode),
// a row-major sweep in which every element is predicted from the f32
// *reconstructed* values of its 7 preceding corner neighbours.  The
// recurrence cannot be reassociated (SURVEY.md findings 3-4), so the B200
// design keeps the reference order and extracts parallelism from the
// dependency DAG instead:
//
//  * 2D/3D: a tiled hyperplane wavefront.  A CTA owns PI x 32 "rows"
//    (i, j) and marches along k; thread (a, b) handles element
//    (i0+a, j0+b, s-a-b) at step s, so all dependencies inside the tile are
//    one step old.  Neighbour recon values move through a 4-slot shared
//    ring; the first i-row / j-column read halos (faces) written by the
//    upstream tiles through L2, guarded by per-tile progress counters
//    (st.release / ld.acquire).  Tiles are handed out by an atomic ticket in
//    row-major (A, B) order so that every tile only waits on tiles that are
//    already resident: no deadlock for any grid size.
//    Inputs (orig or codes) and outputs (codes or recon) are staged through
//    shared rings in "step" coordinates so that global traffic is coalesced
//    row segments of G elements.
//  * 1D: a single serial chain.  Zero-code stretches keep the recon value
//    bitwise constant, so the encoder walks events (nonzero code or
//    outlier) with one warp, skipping 1024-element blocks whose [min, max]
//    lies inside the zero-code interval (the predicate is convex in v).
//    The decoder compacts events, replays the chain per outlier-delimited
//    segment, and broadcast-fills recon in parallel.
#include "common.cuh"

namespace {

constexpr int G = 8;        // steps per group (staging / progress granularity)
constexpr int RING = 32;    // ring slots (steps)
constexpr int PITCH = 33;   // words per row in f32/u32 rings (conflict-free)
constexpr int CPITCH = 34;  // u16 per row in the encoder code ring
constexpr uint32_t MARK = 0xFFFFFFFFu;

template <int PI>
struct Tile {
    static constexpr int NT = PI * 32;
    static constexpr int HROWS = 33 + PI + 1;                   // HU (33) + HL (PI+1)
    static constexpr int HITER = (HROWS * G + NT - 1) / NT;     // halo loads per thread
    static constexpr int OITER = G;                             // ring loads per thread
};

template <int PI>
FZB_DEV void tile_sync() {
    if constexpr (PI == 1) __syncwarp(); else __syncthreads();
}

FZB_DEV void wait_progress(const uint32_t* p, uint32_t need) {
    if (!p) return;
    if (ld_acquire(p) >= need) return;
    unsigned ns = 32;
    while (ld_acquire(p) < need) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

struct Geo {
    int n0, n1, n2, nA, nB;
};

// Shared-memory carve-up for a PI x 32 tile.
template <int PI, bool DEC>
struct Smem {
    static constexpr int NT = PI * 32;
    // input ring: ENC f32 orig, DEC u32 code/mark      [NT][PITCH]
    // output ring: ENC u16 codes [NT][CPITCH], DEC f32 recon [NT][PITCH]
    // RR: recon exchange ring [4][NT]; HU [33][PITCH]; HL [PI+1][PITCH]
    static constexpr size_t in_words = (size_t)NT * PITCH;
    static constexpr size_t out_bytes = DEC ? (size_t)NT * PITCH * 4 : (size_t)NT * CPITCH * 2;
    static constexpr size_t rr_words = 4 * NT;
    static constexpr size_t hu_words = 33 * PITCH;
    static constexpr size_t hl_words = (PI + 1) * PITCH;
    static constexpr size_t bytes = in_words * 4 + ((out_bytes + 15) / 16) * 16 + (rr_words + hu_words + hl_words) * 4 + 16;
};

// One kernel body for both directions.
//   ENC: in = orig (f32), out_codes (u16), bitmap |= outliers
//   DEC: in = codes (u16) + bitmap (outliers) + recon (pre-scattered outlier values), out = recon
template <int PI, bool DEC>
__global__ void __launch_bounds__(PI * 32)
lz_wave_kernel(const float* __restrict__ orig, const uint16_t* __restrict__ codes_in,
               uint16_t* __restrict__ codes_out, uint32_t* __restrict__ bitmap, float* __restrict__ recon,
               float* __restrict__ faceI, float* __restrict__ faceJ, uint32_t* __restrict__ progress,
               uint32_t* __restrict__ ticket, Geo geo, const double* __restrict__ d_eb, int radius) {
    using T = Tile<PI>;
    using SM = Smem<PI, DEC>;
    constexpr int NT = T::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* IN = reinterpret_cast<uint32_t*>(smem_raw);
    unsigned char* OUTB = smem_raw + SM::in_words * 4;
    float* RR = reinterpret_cast<float*>(OUTB + ((SM::out_bytes + 15) / 16) * 16);
    float* HU = RR + SM::rr_words;
    float* HL = HU + SM::hu_words;
    int* s_tile = reinterpret_cast<int*>(HL + SM::hl_words);
    uint16_t* CR = reinterpret_cast<uint16_t*>(OUTB);  // ENC
    float* OR = reinterpret_cast<float*>(OUTB);        // DEC

    const int n0 = geo.n0, n1 = geo.n1, n2 = geo.n2, nB = geo.nB;
    const int tid = threadIdx.x, a = tid >> 5, b = tid & 31;
    if (tid == 0) *s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int tile = *s_tile;
    const int A = tile / nB, B = tile % nB;
    const int i0 = A * PI, j0 = B * 32;
    const int i = i0 + a, j = j0 + b;
    const bool row_ok = (i < n0) && (j < n1);
    const QParams P = make_qparams(*d_eb, radius);
    const int S = n2 + PI - 1 + 31;
    const int NGRP = (S + G - 1) / G;
    const uint32_t* progI = (A > 0) ? progress + (tile - nB) : nullptr;
    const uint32_t* progJ = (B > 0) ? progress + (tile - 1) : nullptr;
    const bool writeI = (a == PI - 1) && (A < geo.nA - 1);
    const bool writeJ = (b == 31) && (B < nB - 1);
    const long long rowbase = ((long long)i * n1 + j) * n2;

    // ---- staging helpers -------------------------------------------------
    uint32_t st_in[T::OITER];
    float st_val[DEC ? T::OITER : 1];
    float st_h[T::HITER];

    auto load_group = [&](int gg) {
        // ring input for steps [gg*G, gg*G+G)
#pragma unroll
        for (int e = 0; e < T::OITER; e++) {
            const int flat = e * NT + tid;
            const int row = flat / G, off = flat % G;
            const int ra = row >> 5, rb = row & 31;
            const int ii = i0 + ra, jj = j0 + rb;
            const int k = gg * G + off - ra - rb;
            st_in[e] = 0u;
            if constexpr (DEC) st_val[e] = 0.f;
            if (ii < n0 && jj < n1 && k >= 0 && k < n2) {
                const long long t = ((long long)ii * n1 + jj) * n2 + k;
                if constexpr (DEC) {
                    const uint32_t flag = (__ldg(bitmap + (t >> 5)) >> (t & 31)) & 1u;
                    if (flag) {
                        st_in[e] = MARK;
                        st_val[e] = recon[t];
                    } else {
                        st_in[e] = __ldg(codes_in + t);
                    }
                } else {
                    st_in[e] = __float_as_uint(__ldg(orig + t));
                }
            }
        }
        // halos for steps [gg*G, gg*G+G)
#pragma unroll
        for (int e = 0; e < T::HITER; e++) {
            const int h = e * NT + tid;
            st_h[e] = 0.f;
            if (h < 33 * G) {
                const int jj = h / G - 1, off = h % G;
                const int k = gg * G + off - jj;
                const int jg = j0 + jj;
                if (A > 0 && jg >= 0 && jg < n1 && k >= 0 && k < n2)
                    st_h[e] = __ldcg(faceI + ((long long)(A - 1) * n1 + jg) * n2 + k);
            } else if (h < T::HROWS * G) {
                const int hh = h - 33 * G;
                const int aa = hh / G - 1, off = hh % G;
                const int k = gg * G + off - aa;
                const int ig = i0 + aa;
                if (B > 0 && ig >= 0 && ig < n0 && k >= 0 && k < n2)
                    st_h[e] = __ldcg(faceJ + ((long long)(B - 1) * n0 + ig) * n2 + k);
            }
        }
    };
    auto store_group = [&](int gg) {
#pragma unroll
        for (int e = 0; e < T::OITER; e++) {
            const int flat = e * NT + tid;
            const int row = flat / G, off = flat % G;
            const int slot = (gg * G + off) & (RING - 1);
            IN[row * PITCH + slot] = st_in[e];
            if constexpr (DEC) {
                if (st_in[e] == MARK) OR[row * PITCH + slot] = st_val[e];
            }
        }
#pragma unroll
        for (int e = 0; e < T::HITER; e++) {
            const int h = e * NT + tid;
            if (h < 33 * G) {
                const int r = h / G, off = h % G;
                HU[r * PITCH + ((gg * G + off) & (RING - 1))] = st_h[e];
            } else if (h < T::HROWS * G) {
                const int hh = h - 33 * G;
                const int r = hh / G, off = hh % G;
                HL[r * PITCH + ((gg * G + off) & (RING - 1))] = st_h[e];
            }
        }
    };
    auto need_for = [&](int gg, int lag) -> uint32_t {
        long long v = (long long)(gg + 1) * G + lag;
        return (uint32_t)(v < S ? v : S);
    };

    // ---- prologue: group 0 ------------------------------------------------
    if (tid == 0) {
        wait_progress(progI, need_for(0, PI));
        wait_progress(progJ, need_for(0, 32));
    }
    __syncthreads();
    load_group(0);
    store_group(0);
    // The corner value r[i0-1, j0-1, 0] lives at step -1 of halo row jj = -1
    // (slot 31); no group covers negative steps, so load it here.
    if (tid == 0 && A > 0 && B > 0 && j0 - 1 < n1)
        HU[RING - 1] = __ldcg(faceI + ((long long)(A - 1) * n1 + (j0 - 1)) * n2);

    float up_prev = 0.f, left_prev = 0.f, diag_prev = 0.f, self_prev = 0.f;

    for (int g = 0; g < NGRP; g++) {
        const bool more = (g + 1) < NGRP;
        if (tid == 0 && more) {
            wait_progress(progI, need_for(g + 1, PI));
            wait_progress(progJ, need_for(g + 1, 32));
        }
        __syncthreads();
        if (more) load_group(g + 1);

#pragma unroll
        for (int st = 0; st < G; st++) {
            const int s = g * G + st;
            const int k = s - a - b;
            if (row_ok && k >= 0 && k < n2) {
                const int slot = s & (RING - 1);
                const int ks = (k & 3) * NT;
                float up = 0.f, left = 0.f, diag = 0.f;
                if (i > 0) up = (a > 0) ? RR[ks + tid - 32] : HU[(b + 1) * PITCH + slot];
                if (j > 0) left = (b > 0) ? RR[ks + tid - 1] : HL[(a + 1) * PITCH + slot];
                if (i > 0 && j > 0) {
                    const int ps = (s - 1) & (RING - 1);
                    diag = (a > 0 && b > 0) ? RR[ks + tid - 33]
                                            : (a == 0 ? HU[b * PITCH + ps] : HL[a * PITCH + ps]);
                }
                // predict.py:100-114 -- ordered f64 inclusion-exclusion
                double pred = 0.0;
                if (i > 0) pred = __dadd_rn(pred, (double)up);
                if (j > 0) pred = __dadd_rn(pred, (double)left);
                if (k > 0) pred = __dadd_rn(pred, (double)self_prev);
                if (i > 0 && j > 0) pred = __dsub_rn(pred, (double)diag);
                if (i > 0 && k > 0) pred = __dsub_rn(pred, (double)up_prev);
                if (j > 0 && k > 0) pred = __dsub_rn(pred, (double)left_prev);
                if (i > 0 && j > 0 && k > 0) pred = __dadd_rn(pred, (double)diag_prev);
                float rec;
                if constexpr (DEC) {
                    const uint32_t c = IN[tid * PITCH + slot];
                    if (c == MARK) {
                        rec = OR[tid * PITCH + slot];
                    } else {
                        rec = dequantize(pred, (int)c, P);
                        OR[tid * PITCH + slot] = rec;
                    }
                } else {
                    const double v = (double)__uint_as_float(IN[tid * PITCH + slot]);
                    bool outl;
                    const int code = quantize(v, pred, P, rec, outl);
                    CR[tid * CPITCH + slot] = (uint16_t)code;
                    if (outl) {
                        const long long t = rowbase + k;
                        atomicOr(bitmap + (t >> 5), 1u << (t & 31));
                    }
                }
                RR[ks + tid] = rec;
                if (writeI) faceI[((long long)A * n1 + j) * n2 + k] = rec;
                if (writeJ) faceJ[((long long)B * n0 + i) * n2 + k] = rec;
                up_prev = up;
                left_prev = left;
                diag_prev = diag;
                self_prev = rec;
            }
            tile_sync<PI>();
        }
        if (tid == 0) st_release(progress + tile, (uint32_t)min((g + 1) * G, S));
        // flush group g (all steps of the group are complete)
#pragma unroll
        for (int e = 0; e < T::OITER; e++) {
            const int flat = e * NT + tid;
            const int row = flat / G, off = flat % G;
            const int ra = row >> 5, rb = row & 31;
            const int ii = i0 + ra, jj = j0 + rb;
            const int s = g * G + off;
            const int k = s - ra - rb;
            if (ii < n0 && jj < n1 && k >= 0 && k < n2) {
                const long long t = ((long long)ii * n1 + jj) * n2 + k;
                if constexpr (DEC) recon[t] = OR[row * PITCH + (s & (RING - 1))];
                else codes_out[t] = CR[row * CPITCH + (s & (RING - 1))];
            }
        }
        if (more) store_group(g + 1);
    }
}

// ------------------------------------------------------------------- 1D ---

constexpr int BS1 = 1024;  // elements per summary block

// codes := R everywhere (zero-code default) and per-block [min, max].
__global__ void lz1d_summary_kernel(const float* __restrict__ x, long long n, uint16_t* __restrict__ codes,
                                    int radius, float* __restrict__ bmin, float* __restrict__ bmax,
                                    long long nblk) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long blk = warp; blk < nblk; blk += nw) {
        const long long base = blk * BS1;
        float lo = INFINITY, hi = -INFINITY;
#pragma unroll 4
        for (int e = 0; e < BS1 / 32; e++) {
            const long long t = base + e * 32 + lane;
            if (t < n) {
                const float v = __ldg(x + t);
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
                codes[t] = (uint16_t)radius;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            bmin[blk] = lo;
            bmax[blk] = hi;
        }
    }
}

// Zero-code predicate for fixed predictor value pred: code R, not an outlier.
FZB_DEV bool zero_code(double v, double pred, const QParams& P) {
    float rec;
    bool outl;
    const int c = quantize(v, pred, P, rec, outl);
    return c == P.radius && !outl;
}

// One warp walks the whole chain.
__global__ void __launch_bounds__(32) lz1d_walk_kernel(const float* __restrict__ x, long long n,
                                                        uint16_t* __restrict__ codes, uint32_t* __restrict__ bitmap,
                                                        const float* __restrict__ bmin, const float* __restrict__ bmax,
                                                        long long nblk, const double* __restrict__ d_eb, int radius) {
    const int lane = threadIdx.x;
    const QParams P = make_qparams(*d_eb, radius);
    long long t = 0;
    float r = 0.f;
    while (t < n) {
        // process event t (every lane computes the same thing)
        {
            const double v = (double)__ldg(x + t);
            const double pred = (t == 0) ? 0.0 : __dadd_rn(0.0, (double)r);
            float rec;
            bool outl;
            const int c = quantize(v, pred, P, rec, outl);
            if (lane == 0) {
                if (c != radius) codes[t] = (uint16_t)c;
                if (outl) atomicOr(bitmap + (t >> 5), 1u << (t & 31));
            }
            r = rec;
            t++;
        }
        const double pred = __dadd_rn(0.0, (double)r);
        // find next t' >= t with !zero_code(x[t'])
        for (;;) {
            if (t >= n) break;
            long long blk = t / BS1;
            if (t % BS1 != 0) {
                // finish the current block: each lane takes 32 contiguous elements
                const long long bend = min((blk + 1) * BS1, n);
                long long found = -1;
                for (long long c0 = t; c0 < bend && found < 0; c0 += 32 * 32) {
                    long long mine = -1;
                    const long long lb = c0 + (long long)lane * 32;
                    for (int e = 0; e < 32; e++) {
                        const long long tt = lb + e;
                        if (tt >= bend) break;
                        if (!zero_code((double)__ldg(x + tt), pred, P)) { mine = tt; break; }
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, mine >= 0);
                    if (m) found = __shfl_sync(0xffffffffu, mine, __ffs(m) - 1);
                }
                if (found >= 0) { t = found; break; }
                t = bend;
                continue;
            }
            // block-aligned: probe 32 block summaries at once
            const long long bb = blk + lane;
            bool skip = false;
            if (bb < nblk) {
                skip = zero_code((double)__ldg(bmin + bb), pred, P) && zero_code((double)__ldg(bmax + bb), pred, P);
            }
            const unsigned nonskip = __ballot_sync(0xffffffffu, !skip);  // lanes past nblk count as non-skip
            if (nonskip == 0) { t = (blk + 32) * BS1; continue; }
            const int first = __ffs(nonskip) - 1;
            const long long fb = blk + first;
            if (fb >= nblk) { t = n; break; }
            // scan block fb entirely (32 lanes x 32 elements)
            const long long lb = fb * BS1 + (long long)lane * 32;
            long long mine = -1;
            for (int e = 0; e < 32; e++) {
                const long long tt = lb + e;
                if (tt >= n) break;
                if (!zero_code((double)__ldg(x + tt), pred, P)) { mine = tt; break; }
            }
            const unsigned m = __ballot_sync(0xffffffffu, mine >= 0);
            if (m) { t = __shfl_sync(0xffffffffu, mine, __ffs(m) - 1); break; }
            t = min((fb + 1) * BS1, n);
        }
    }
}

// ---- 1D decode: events = nonzero code or outlier --------------------------
// Between events the recon value is bitwise constant, so the decoder
// (1) compacts event positions, (2) replays the chain per segment that
// starts at event 0 or at an outlier (outliers reset the state), writing
// each event's value into recon[pos], and (3) fills every other element
// with the value of the last event at or before it.
constexpr int EV_CHUNK = 4096;  // elements per counting CTA

FZB_DEV bool is_event(const uint16_t* codes, const uint32_t* bitmap, long long t, int radius) {
    return codes[t] != radius || ((bitmap[t >> 5] >> (t & 31)) & 1u);
}
FZB_DEV bool is_outlier(const uint32_t* bitmap, long long t) { return (bitmap[t >> 5] >> (t & 31)) & 1u; }

__global__ void lz1d_event_count_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap,
                                        long long n, int radius, uint32_t* __restrict__ counts) {
    __shared__ uint32_t tmp[33];
    const long long base = (long long)blockIdx.x * EV_CHUNK;
    uint32_t c = 0;
    for (int e = threadIdx.x; e < EV_CHUNK; e += blockDim.x) {
        const long long t = base + e;
        if (t < n && is_event(codes, bitmap, t, radius)) c++;
    }
    uint32_t tot;
    block_exclusive_scan(c, tmp, &tot);
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void lz1d_event_compact_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap,
                                          long long n, int radius, const unsigned long long* __restrict__ offs,
                                          long long* __restrict__ evpos) {
    __shared__ uint32_t tmp[33];
    const long long base = (long long)blockIdx.x * EV_CHUNK;
    unsigned long long o = offs[blockIdx.x];
    for (int e0 = 0; e0 < EV_CHUNK; e0 += blockDim.x) {
        const long long t = base + e0 + threadIdx.x;
        const bool evt = (t < n) && is_event(codes, bitmap, t, radius);
        uint32_t tot;
        const uint32_t p = block_exclusive_scan(evt ? 1u : 0u, tmp, &tot);
        if (evt) evpos[o + p] = t;
        o += tot;
    }
}

__global__ void lz1d_event_chain_kernel(const long long* __restrict__ evpos, const unsigned long long* __restrict__ nev_p,
                                        const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap,
                                        float* __restrict__ recon, const double* __restrict__ d_eb, int radius) {
    const unsigned long long nev = *nev_p;
    const QParams P = make_qparams(*d_eb, radius);
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < nev;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const long long p0 = evpos[e];
        if (!(e == 0 || is_outlier(bitmap, p0))) continue;
        float r = 0.f;
        for (unsigned long long q = e; q < nev; q++) {
            const long long p = evpos[q];
            const bool outl = is_outlier(bitmap, p);
            if (q != e && outl) break;
            if (outl) {
                r = recon[p];  // pre-scattered outlier value
            } else {
                const double pred = (p == 0) ? 0.0 : __dadd_rn(0.0, (double)r);
                r = dequantize(pred, (int)codes[p], P);
                recon[p] = r;
            }
        }
    }
}

__global__ void lz1d_fill_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap, long long n,
                                 int radius, const unsigned long long* __restrict__ offs,
                                 const long long* __restrict__ evpos, float* __restrict__ recon) {
    __shared__ long long wmax[32];
    const long long base = (long long)blockIdx.x * EV_CHUNK;
    const unsigned long long o = offs[blockIdx.x];
    long long carry = o > 0 ? evpos[o - 1] : -1;  // last event before this chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int e0 = 0; e0 < EV_CHUNK; e0 += blockDim.x) {
        const long long t = base + e0 + threadIdx.x;
        const bool evt = (t < n) && is_event(codes, bitmap, t, radius);
        long long m = evt ? t : -1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, m, d);
            if (lane >= d) m = max(m, y);
        }
        if (lane == 31) wmax[warp] = m;
        __syncthreads();
        long long pre = carry;
        for (int w = 0; w < warp; w++) pre = max(pre, wmax[w]);
        m = max(m, pre);
        long long blockmax = carry;
        for (int w = 0; w < nw; w++) blockmax = max(blockmax, wmax[w]);
        __syncthreads();
        if (t < n && !evt) recon[t] = m >= 0 ? recon[m] : 0.f;
        carry = blockmax;
    }
}

// exclusive scan of u32 counts into u64 offsets (single CTA), total -> *tot
__global__ void scan_counts_kernel(const uint32_t* __restrict__ cnt, long long m, unsigned long long* __restrict__ offs,
                                   unsigned long long* __restrict__ tot) {
    __shared__ unsigned long long tmp[33];
    unsigned long long carry = 0;
    for (long long b0 = 0; b0 < m; b0 += blockDim.x) {
        const long long q = b0 + threadIdx.x;
        const unsigned long long x = q < m ? cnt[q] : 0ull;
        unsigned long long t;
        const unsigned long long p = block_exclusive_scan64(x, tmp, &t);
        if (q < m) offs[q] = carry + p;
        carry += t;
    }
    if (threadIdx.x == 0) *tot = carry;
}

template <int PI, bool DEC>
int launch_wave(const float* orig, const uint16_t* codes_in, uint16_t* codes_out, uint32_t* bitmap, float* recon,
                int n0, int n1, int n2, const double* d_eb, int radius, void* ws, size_t ws_bytes, cudaStream_t st) {
    Geo g;
    g.n0 = n0; g.n1 = n1; g.n2 = n2;
    g.nA = (n0 + PI - 1) / PI;
    g.nB = (n1 + 31) / 32;
    const size_t ntile = (size_t)g.nA * g.nB;
    const size_t fI = (size_t)g.nA * n1 * n2, fJ = (size_t)g.nB * n0 * n2;
    const size_t need = 256 + ntile * 4 + (fI + fJ) * 4;
    if (ws_bytes < need) return FZB_E_WORKSPACE;
    unsigned char* w = static_cast<unsigned char*>(ws);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(w);
    uint32_t* progress = reinterpret_cast<uint32_t*>(w + 256);
    float* faceI = reinterpret_cast<float*>(w + 256 + ((ntile * 4 + 255) / 256) * 256);
    float* faceJ = faceI + fI;
    cudaMemsetAsync(w, 0, 256 + ntile * 4, st);
    const size_t smem = Smem<PI, DEC>::bytes;
    auto kfn = lz_wave_kernel<PI, DEC>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<(unsigned)ntile, PI * 32, smem, st>>>(orig, codes_in, codes_out, bitmap, recon, faceI, faceJ, progress,
                                               ticket, g, d_eb, radius);
    return fzb_check_launch();
}

template <int PI>
size_t wave_ws(int n0, int n1, int n2) {
    const size_t nA = (n0 + PI - 1) / PI, nB = (n1 + 31) / 32;
    const size_t ntile = nA * nB;
    return 256 + ((ntile * 4 + 255) / 256) * 256 + (nA * n1 * n2 + nB * n0 * n2) * 4 + 256;
}

// Collapse unit extents (the recurrence with a unit axis is the lower-dim one).
void canon(uint32_t& n0, uint32_t& n1, uint32_t& n2) {
    uint32_t d[3] = {n0, n1, n2}, o[3] = {1, 1, 1};
    int q = 2;
    for (int x = 2; x >= 0; x--)
        if (d[x] > 1) o[q--] = d[x];
    n0 = o[0]; n1 = o[1]; n2 = o[2];
}

int pick_pi(uint32_t n0) { return n0 >= 8 ? 8 : (n0 >= 4 ? 4 : (n0 >= 2 ? 2 : 1)); }

}  // namespace

extern "C" {

FZB_API size_t fzb_lorenzo_workspace_bytes(uint32_t n0, uint32_t n1, uint32_t n2) {
    canon(n0, n1, n2);
    const long long n = (long long)n0 * n1 * n2;
    if (n0 == 1 && n1 == 1) {
        // encode: block summaries; decode: counts + offsets + event records + event recon
        const long long nblk = (n + BS1 - 1) / BS1, nch = (n + EV_CHUNK - 1) / EV_CHUNK;
        const size_t enc = (size_t)nblk * 8 + 512;
        const size_t dec = 1024 + (size_t)nch * 4 + (size_t)nch * 8 + (size_t)n * 8;
        return enc > dec ? enc : dec;
    }
    switch (pick_pi(n0)) {
        case 8: return wave_ws<8>(n0, n1, n2);
        case 4: return wave_ws<4>(n0, n1, n2);
        case 2: return wave_ws<2>(n0, n1, n2);
        default: return wave_ws<1>(n0, n1, n2);
    }
}

// Reference: predict.py:93-115 (_lorenzo_encode) + the outlier flags of
// predict.py:212-214.  codes: u16[n]; bitmap: u32[ceil(n/32)] zeroed by the
// caller; receives one bit per outlier.
FZB_API int fzb_lorenzo_encode_f32(const float* d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb,
                                   uint32_t radius, uint16_t* d_codes, uint32_t* d_bitmap, void* d_ws,
                                   size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    canon(n0, n1, n2);
    const long long n = (long long)n0 * n1 * n2;
    if (n == 0) return 0;
    if (n0 == 1 && n1 == 1) {
        const long long nblk = (n + BS1 - 1) / BS1;
        if (ws_bytes < (size_t)nblk * 8) return FZB_E_WORKSPACE;
        float* bmin = static_cast<float*>(d_ws);
        float* bmax = bmin + nblk;
        lz1d_summary_kernel<<<kNumSMs * 8, 256, 0, st>>>(d_in, n, d_codes, (int)radius, bmin, bmax, nblk);
        lz1d_walk_kernel<<<1, 32, 0, st>>>(d_in, n, d_codes, d_bitmap, bmin, bmax, nblk, d_eb, (int)radius);
        return fzb_check_launch();
    }
    switch (pick_pi(n0)) {
        case 8: return launch_wave<8, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 4: return launch_wave<4, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 2: return launch_wave<2, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        default: return launch_wave<1, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
    }
}

// Reference: predict.py:242-253 / 118-144.  d_recon must already hold the
// outlier values at their positions and d_bitmap their flags
// (fzb_outlier_scatter); every other element is reconstructed in place.
FZB_API int fzb_lorenzo_decode_f32(const uint16_t* d_codes, const uint32_t* d_bitmap, float* d_recon, uint32_t n0,
                                   uint32_t n1, uint32_t n2, const double* d_eb, uint32_t radius, void* d_ws,
                                   size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    canon(n0, n1, n2);
    const long long n = (long long)n0 * n1 * n2;
    if (n == 0) return 0;
    if (n0 == 1 && n1 == 1) {
        const long long nch = (n + EV_CHUNK - 1) / EV_CHUNK;
        if (ws_bytes < fzb_lorenzo_workspace_bytes(1, 1, (uint32_t)n)) return FZB_E_WORKSPACE;
        unsigned char* w = static_cast<unsigned char*>(d_ws);
        unsigned long long* nev = reinterpret_cast<unsigned long long*>(w);
        uint32_t* counts = reinterpret_cast<uint32_t*>(w + 256);
        unsigned long long* offs = reinterpret_cast<unsigned long long*>(w + 256 + ((nch * 4 + 255) / 256) * 256);
        long long* evpos = reinterpret_cast<long long*>(reinterpret_cast<unsigned char*>(offs) + ((nch * 8 + 255) / 256) * 256);
        lz1d_event_count_kernel<<<(unsigned)nch, 256, 0, st>>>(d_codes, d_bitmap, n, (int)radius, counts);
        scan_counts_kernel<<<1, 1024, 0, st>>>(counts, nch, offs, nev);
        lz1d_event_compact_kernel<<<(unsigned)nch, 256, 0, st>>>(d_codes, d_bitmap, n, (int)radius, offs, evpos);
        lz1d_event_chain_kernel<<<kNumSMs * 4, 128, 0, st>>>(evpos, nev, d_codes, d_bitmap, d_recon, d_eb, (int)radius);
        lz1d_fill_kernel<<<(unsigned)nch, 256, 0, st>>>(d_codes, d_bitmap, n, (int)radius, offs, evpos, d_recon);
        return fzb_check_launch();
    }
    switch (pick_pi(n0)) {
        case 8: return launch_wave<8, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 4: return launch_wave<4, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 2: return launch_wave<2, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        default: return launch_wave<1, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
    }
}

}  // extern "C"
