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
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "scan.cuh"

namespace {

constexpr int G = 8;        // steps per group (staging / progress granularity)
constexpr int RING = 32;    // ring slots (steps)
constexpr int PITCH = 33;   // words per row in f32/u32 rings (conflict-free)
constexpr int CPITCH = 34;  // u16 per row in the encoder code ring
constexpr uint32_t MARK = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xffffffffu;

FZB_DEV void wait_progress(const uint32_t* p, uint32_t need) {
    if (!p) return;
    if (ld_acquire(p) >= need) return;
    unsigned ns = 32;
    while (ld_acquire(p) < need) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

FZB_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct Geo {
    int n0, n1, n2, nA, nB;
};

// Workspace header: the first WS_HDR bytes of every Lorenzo workspace, shared
// by all paths that run on it (an Engine reuses one workspace across shapes,
// dimensionalities and directions).
//   word 0     v7 launch epoch = the LL tag of the faces; only ever incremented
//   word 1     v7 tile ticket
//   words 2-3  u64 signature of the v7 face layout the workspace holds (0 = none)
//   word 4     v7: this launch must clear the faces (layout changed)
//   words 6-7  1D walker: the walking CTA's current block, read by its prefetch CTA
//   word 32    v4 tile ticket (v4 progress counters start at WS_HDR)
// v7 faces are only trusted under the layout that wrote them: every other
// path lays its data out from WS_HDR on and resets the signature, and a v7
// launch whose layout differs from the signature zeroes its faces first, so
// a stale word (another shape's faces, tile order, event counts, summaries)
// can never carry the current epoch.
constexpr size_t WS_HDR = 256;
void invalidate_faces(void* ws, cudaStream_t st) {
    cudaMemsetAsync(static_cast<unsigned char*>(ws) + 8, 0, 8, st);
}

// ---------------------------------------------------------------- v4
// Warp-specialised wavefront.  Warps 0..PI-1 compute (thread (a, b) owns row
// (i0+a, j0+b), element k = s-a-b at step s); warp PI is the producer: it
// waits on upstream progress, stages the input ring (cp.async, zero-filled
// outside the field) and the halos one group ahead, flushes finished
// groups and publishes progress (the gpu-scope fences stay off the compute
// warps).  Inputs of steps before a row's k == 0 are exact zeros, so those
// steps compute exact zeros and the 7-term history needs no masking.
// Lane 0's left/diagonal halo values ride the same rotated shuffle as the
// in-warp neighbours (lane 31 forwards them), so there is no divergence.
// Barriers: 1 = per-step among compute warps, 2 = FULL (producer ->
// compute, group staged), 3 = DONE (compute -> producer, group finished).
FZB_DEV void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
FZB_DEV void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
FZB_DEV void cp_async4_zfill(void* smem, const void* gmem, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = ok ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

template <int PI, bool DEC>
struct Smem4 {
    static constexpr int NT = PI * 32;
    static constexpr size_t in_words = (size_t)NT * PITCH;
    static constexpr size_t out_bytes = DEC ? (size_t)NT * PITCH * 4 : (size_t)NT * CPITCH * 2;
    static constexpr size_t rr_words = PI > 1 ? 8 * NT : 0;
    static constexpr size_t hu_words = 33 * PITCH;
    static constexpr size_t hl_words = (PI + 1) * PITCH;
    static constexpr size_t bytes = in_words * 4 + ((out_bytes + 15) / 16) * 16 + (rr_words + hu_words + hl_words) * 4 + 16;
};

template <int PI>
struct Blocks4 {
    static constexpr int MINB = PI >= 8 ? 3 : (PI >= 4 ? 5 : (PI >= 2 ? 8 : 12));
};

template <int PI, bool DEC>
__global__ void __launch_bounds__((PI + 1) * 32, Blocks4<PI>::MINB)
lz_wave4_kernel(const float* __restrict__ orig, const uint16_t* __restrict__ codes_in,
                uint16_t* __restrict__ codes_out, uint32_t* __restrict__ bitmap, float* __restrict__ recon,
                float* __restrict__ faceI, float* __restrict__ faceJ, uint32_t* __restrict__ progress,
                uint32_t* __restrict__ ticket, const int* __restrict__ order, Geo geo,
                const double* __restrict__ d_eb, int radius) {
    constexpr int NT = PI * 32;           // compute threads
    constexpr int HROWS = 33 + PI + 1;
    using SM = Smem4<PI, DEC>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* IN = reinterpret_cast<uint32_t*>(smem_raw);
    unsigned char* OUTB = smem_raw + SM::in_words * 4;
    float* RR = reinterpret_cast<float*>(OUTB + ((SM::out_bytes + 15) / 16) * 16);
    float* HU = RR + SM::rr_words;
    float* HL = HU + SM::hu_words;
    int* s_tile = reinterpret_cast<int*>(HL + SM::hl_words);
    uint16_t* CR = reinterpret_cast<uint16_t*>(OUTB);
    float* OR = reinterpret_cast<float*>(OUTB);

    const int n0 = geo.n0, n1 = geo.n1, n2 = geo.n2, nB = geo.nB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // exact zeros everywhere a step before k == 0 can look (RR, HU, HL rings)
    for (int q = tid; q < (int)(SM::rr_words + SM::hu_words + SM::hl_words); q += blockDim.x) RR[q] = 0.f;
    if (tid == 0) *s_tile = order[atomicAdd(ticket, 1u)];
    __syncthreads();
    const int tile = *s_tile;
    const int A = tile / nB, B = tile % nB;
    const int i0 = A * PI, j0 = B * 32;
    const int S = n2 + PI - 1 + 31;
    const int NGRP = (S + G - 1) / G;
    const long long plane = (long long)n1 * n2;
    const long long tile_base = (long long)i0 * plane + (long long)j0 * n2;

    if (warp == PI) {
        // ============ producer: upstream waits, halos, progress fences ============
        const uint32_t* progI = (A > 0) ? progress + (tile - nB) : nullptr;
        const uint32_t* progJ = (B > 0) ? progress + (tile - 1) : nullptr;
        const bool has_dep = (A < geo.nA - 1) || (B < nB - 1);
        constexpr int HE = (HROWS * G + 31) / 32;
        float hreg[HE];
        auto need = [&](int gg, int lag) -> uint32_t {
            const long long v = (long long)(gg + 1) * G + lag;
            return (uint32_t)(v < S ? v : S);
        };
        auto stage = [&](int gg) {
            if (progI) wait_progress(progI, need(gg, PI));
            if (progJ) wait_progress(progJ, need(gg, 32));
#pragma unroll
            for (int e = 0; e < HE; e++) {
                const int h = e * 32 + lane;
                hreg[e] = 0.f;
                if (h < 33 * G) {
                    const int jj = h / G - 1, off = h % G;
                    const int k = gg * G + off - jj;
                    const int jg = j0 + jj;
                    if (A > 0 && jg >= 0 && jg < n1 && k >= 0 && k < n2)
                        hreg[e] = __ldcg(faceI + ((long long)(A - 1) * n1 + jg) * n2 + k);
                } else if (h < HROWS * G) {
                    const int hh = h - 33 * G;
                    const int aa = hh / G - 1, off = hh % G;
                    const int k = gg * G + off - aa;
                    const int ig = i0 + aa;
                    if (B > 0 && ig >= 0 && ig < n0 && k >= 0 && k < n2)
                        hreg[e] = __ldcg(faceJ + ((long long)(B - 1) * n0 + ig) * n2 + k);
                }
            }
        };
        auto commit = [&](int gg) {
#pragma unroll
            for (int e = 0; e < HE; e++) {
                const int h = e * 32 + lane;
                if (h < 33 * G) HU[(h / G) * PITCH + ((gg * G + h % G) & (RING - 1))] = hreg[e];
                else if (h < HROWS * G) {
                    const int hh = h - 33 * G;
                    HL[(hh / G) * PITCH + ((gg * G + hh % G) & (RING - 1))] = hreg[e];
                }
            }
        };
        stage(0);
        commit(0);
        if (lane == 0)  // corner r[i0-1, j0-1, 0] lives at step -1 of halo row jj = -1
            HU[RING - 1] = (A > 0 && B > 0) ? __ldcg(faceI + ((long long)(A - 1) * n1 + (j0 - 1)) * n2) : 0.f;
        __syncwarp();
        bar_arrive(2, NT + 32);                    // FULL(0)
        if (NGRP > 1) stage(1);
        for (int g = 0; g < NGRP; g++) {
            bar_sync(3, NT + 32);                  // DONE(g): faces of group g written
            if (lane == 0 && has_dep) st_release(progress + tile, (uint32_t)min((g + 1) * G, S));
            if (g + 1 < NGRP) {
                commit(g + 1);
                __syncwarp();
                bar_arrive(2, NT + 32);            // FULL(g+1)
            }
            if (g + 2 < NGRP) stage(g + 2);
        }
        return;
    }

    // ================================ compute ================================
    const int a = warp, b = lane;
    const int i = i0 + a, j = j0 + b;
    const bool row_ok = (i < n0) && (j < n1);
    const QParams P = make_qparams(*d_eb, radius);
    const double R_d = (double)radius;
    const bool wI = row_ok && (a == PI - 1) && (A < geo.nA - 1);
    const bool wJ = row_ok && (b == 31) && (B < nB - 1);
    float* fI = faceI + ((long long)A * n1 + j) * n2 - a - b;   // index by step s
    float* fJ = faceJ + ((long long)B * n0 + i) * n2 - a - b;
    const long long rowbase = tile_base + a * plane + (long long)b * n2 - a - b;  // + s
    const int src = (b + 31) & 31;
    uint32_t* INr = IN + tid * PITCH;
    float* ORr = OR + tid * PITCH;
    uint16_t* CRr = CR + tid * CPITCH;
    // warp-local staging / flush of this warp's 32 rows: lane -> (row q*4 + lane/8, offset lane%8)
    const int soff = lane & 7, sr = lane >> 3;
    const bool irow = (i < n0);
    const long long wbase = tile_base + a * plane - a;   // + rb*n2 - rb + s

    uint32_t creg[DEC ? 8 : 1];
    float vreg[DEC ? 8 : 1];
    auto stage_own = [&](int gg) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int rb = q * 4 + sr;
            const int k = gg * G + soff - a - rb;
            const bool ok = irow && (j0 + rb < n1) && (unsigned)k < (unsigned)n2;
            const long long t = wbase + (long long)rb * n2 - rb + gg * G + soff;
            const int slot = (gg * G + soff) & (RING - 1);
            if constexpr (DEC) {
                creg[q] = (uint32_t)radius;
                vreg[q] = 0.f;
                if (ok) {
                    if ((__ldg(bitmap + (t >> 5)) >> (t & 31)) & 1u) {
                        creg[q] = MARK;
                        vreg[q] = recon[t];
                    } else {
                        creg[q] = __ldg(codes_in + t);
                    }
                }
            } else {
                cp_async4_zfill(IN + (a * 32 + rb) * PITCH + slot, orig + (ok ? t : tile_base), ok);
            }
        }
    };
    auto commit_own = [&](int gg) {
        if constexpr (DEC) {
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int rb = q * 4 + sr;
                const int slot = (gg * G + soff) & (RING - 1);
                IN[(a * 32 + rb) * PITCH + slot] = creg[q];
                if (creg[q] == MARK) OR[(a * 32 + rb) * PITCH + slot] = vreg[q];
            }
        } else {
            cp_async_wait_all();
        }
        __syncwarp();
    };
    auto flush_own = [&](int gg) {
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int rb = q * 4 + sr;
            const int s = gg * G + soff;
            const int k = s - a - rb;
            if (irow && (j0 + rb < n1) && (unsigned)k < (unsigned)n2) {
                const long long t = wbase + (long long)rb * n2 - rb + s;
                if constexpr (DEC) recon[t] = OR[(a * 32 + rb) * PITCH + (s & (RING - 1))];
                else codes_out[t] = CR[(a * 32 + rb) * CPITCH + (s & (RING - 1))];
            }
        }
    };

    stage_own(0);
    commit_own(0);
    float recL = 0.f, upLf = 0.f;
    double selfL = 0.0, upL = 0.0, leftL = 0.0, diagL = 0.0;
    float fwdL = 0.f, fwdD = 0.f;   // lane 31: lane 0's left / diagonal for the next step

    for (int g = 0; g < NGRP; g++) {
        bar_sync(2, NT + 32);        // FULL(g): halos of group g in shared memory
        if (g + 1 < NGRP) stage_own(g + 1);
        const int s0 = g * G;
        const int sl0 = s0 & (RING - 1);
        if (b == 31) {
            fwdL = HL[(a + 1) * PITCH + sl0];
            fwdD = (a > 0) ? HL[a * PITCH + ((s0 - 1) & (RING - 1))] : HU[(s0 - 1) & (RING - 1)];
        }
#pragma unroll
        for (int st = 0; st < G; st++) {
            const int s = s0 + st;
            const int slot = sl0 + st;   // G divides RING: no wrap inside a group
            float upf;
            if constexpr (PI > 1) upf = (a > 0) ? RR[((s - 1) & 7) * NT + tid - 32] : HU[(b + 1) * PITCH + slot];
            else upf = HU[(b + 1) * PITCH + slot];
            const float leftf = __shfl_sync(FULL, b == 31 ? fwdL : recL, src);
            const float diagf = __shfl_sync(FULL, b == 31 ? fwdD : upLf, src);
            const double up = (double)(upf + 0.0f);   // the leading "0.0 + x" (normalises -0)
            const double left = (double)leftf, diag = (double)diagf;
            double pred = __dadd_rn(up, left);
            pred = __dadd_rn(pred, selfL);
            pred = __dsub_rn(pred, diag);
            pred = __dsub_rn(pred, upL);
            pred = __dsub_rn(pred, leftL);
            pred = __dadd_rn(pred, diagL);
            float rec;
            double recd;
            if constexpr (DEC) {
                const uint32_t c = INr[slot];
                if (c == MARK) {
                    rec = ORr[slot];
                } else {
                    rec = dequantize(pred, (int)c, P);
                    ORr[slot] = rec;
                }
                recd = (double)rec;
            } else {
                const float vf = __uint_as_float(INr[slot]);
                const double v = (double)vf;
                const double q = __dmul_rn(__dsub_rn(v, pred), P.inv2eb);
                const double sd = rint(q);
                const double fr = fabs(__dsub_rn(q, sd));
                int code;
                bool outl;
                if (!P.use_recip || fr >= 0.4999999990686774) {
                    code = quantize(v, pred, P, rec, outl);
                    recd = (double)rec;
                } else {
                    const float rc = __double2float_rn(__dadd_rn(pred, __dmul_rn(P.two_eb, sd)));
                    const double rcd = (double)rc;
                    const bool ok = fabs(sd) < R_d && fabs(__dsub_rn(rcd, v)) <= P.eb;
                    code = ok ? (int)sd + radius : radius;
                    rec = ok ? rc : vf;
                    recd = ok ? rcd : v;
                    outl = !ok;
                }
                CRr[slot] = (uint16_t)code;
                if (outl) {
                    const int k = s - a - b;
                    if (row_ok && (unsigned)k < (unsigned)n2) {
                        const long long t = rowbase + s;
                        atomicOr(bitmap + (t >> 5), 1u << (t & 31));
                    }
                }
            }
            {
                const int k = s - a - b;
                const bool act = (unsigned)k < (unsigned)n2;
                if (wI && act) fI[s] = rec;
                if (wJ && act) fJ[s] = rec;
            }
            if constexpr (PI > 1) RR[(s & 7) * NT + tid] = rec;
            recL = rec;
            upLf = upf;
            selfL = recd;
            upL = up;
            leftL = left;
            diagL = diag;
            if (st + 1 < G && b == 31) {
                fwdL = HL[(a + 1) * PITCH + slot + 1];
                fwdD = (a > 0) ? HL[a * PITCH + slot] : HU[slot];
            }
            if constexpr (PI > 1) bar_sync(1, NT);
            else __syncwarp();
        }
        bar_arrive(3, NT + 32);      // DONE(g)
        flush_own(g);
        if (g + 1 < NGRP) commit_own(g + 1);
    }
}

// Ticket order: tiles sorted by their expected start step lagI*A + lagJ*B
// (a topological order: both predecessors have strictly smaller keys), so
// resident CTAs are the ones closest to runnable.  Counting sort, one CTA.
__global__ void tile_order_kernel(int nA, int nB, int lagI, int lagJ, int* __restrict__ counts,
                                  int* __restrict__ order, int nf = 1) {
    // nf fields of nA x nB tiles: tile t of field f has id f*nA*nB + t and the
    // key of its field-local (A, B), so equal keys interleave the fields
    __shared__ uint32_t tmp[33];
    const int nt1 = nA * nB, ntile = nt1 * nf;
    const int K = lagI * (nA - 1) + lagJ * (nB - 1) + 1;
    auto key = [&](int t) { const int l = t % nt1; return lagI * (l / nB) + lagJ * (l % nB); };
    for (int q = threadIdx.x; q < K; q += blockDim.x) counts[q] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < ntile; t += blockDim.x) atomicAdd(&counts[key(t)], 1);
    __syncthreads();
    uint32_t carry = 0;
    for (int q0 = 0; q0 < K; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        const uint32_t x = q < K ? (uint32_t)counts[q] : 0u;
        uint32_t tot;
        const uint32_t p = block_exclusive_scan(x, tmp, &tot);
        if (q < K) counts[q] = (int)(carry + p);
        carry += tot;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntile; t += blockDim.x) {
        const int pos = atomicAdd(&counts[key(t)], 1);
        order[pos] = t;
    }
}

#include "lorenzo6.cuh"

// ------------------------------------------------------------------- 1D ---
// Encoder: one warp walks the chain.  At an event the exact quantizer runs;
// then the exact f32 interval [zlo, zhi] of inputs that keep a zero code
// (convex: the predicate is monotone in v on each side of the state) is
// pinned with 32-key windows around r -/+ eb, and the walk continues with
// plain float compares over 32K / 1K min-max summaries and coalesced
// element scans.
constexpr int BS1 = 1024;        // elements per summary block
constexpr int BS2 = 32 * BS1;    // elements per superblock
static_assert(BS1 == 1 << 10 && BS2 == 1 << 15, "the walker indexes blocks with shifts (t >= 0)");

__global__ void lz1d_super_kernel(const float* __restrict__ bmin, const float* __restrict__ bmax, long long nblk,
                                  float* __restrict__ smin, float* __restrict__ smax, long long nsb) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long sb = warp; sb < nsb; sb += nw) {
        const long long b = sb * 32 + lane;
        float lo = b < nblk ? bmin[b] : INFINITY, hi = b < nblk ? bmax[b] : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) { smin[sb] = lo; smax[sb] = hi; }
    }
}

FZB_DEV uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
FZB_DEV float kfloat(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k); }


// Superblock summaries live in shared memory (when they fit), and the
// element loads of the current block are issued before the zero-interval
// search so their latency overlaps it.
constexpr long long WALK_SMEM_SB = 24576;
#ifdef LZ7_TIMING
__device__ long long g_walk_stamp[8];
#endif   // superblocks cached in smem (196 KB)

constexpr int WIN1 = 4;                // window = 4 x 32 block summaries past the event's block
constexpr long long PF_AHEAD = 4096;   // blocks (16 MB) the prefetch CTA keeps ahead of the walker

FZB_DEV void walk_load_window(const float* __restrict__ bmin, const float* __restrict__ bmax, long long nblk,
                              long long b, float (&lo)[WIN1], float (&hi)[WIN1]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < WIN1; j++) {
        const long long bb = b + 1 + 32 * j + lane;
        lo[j] = bb < nblk ? __ldcg(bmin + bb) : INFINITY;
        hi[j] = bb < nblk ? __ldcg(bmax + bb) : -INFINITY;
    }
}

// First block >= b0 whose [min, max] leaves [zlo, zhi], or -1 (none).
FZB_DEV long long walk_far(long long b0, long long nblk, const float* __restrict__ bmin, const float* __restrict__ bmax,
                           const float* smin, const float* smax, long long nsb, float zlo, float zhi) {
    const int lane = threadIdx.x & 31;
    long long b = b0;
    while (b < nblk) {
        long long sb = b >> 5;
        const long long bb = sb * 32 + lane;
        const bool fail = bb >= b && bb < nblk && !(__ldcg(bmin + bb) >= zlo && __ldcg(bmax + bb) <= zhi);
        const unsigned fm = __ballot_sync(0xffffffffu, fail);
        if (fm) return sb * 32 + (__ffs(fm) - 1);
        // whole superblocks, 32 at a time
        for (;;) {
            const long long sq = sb + 1 + lane;
            const bool stop = sq < nsb && !(smin[sq] >= zlo && smax[sq] <= zhi);
            const unsigned sm = __ballot_sync(0xffffffffu, stop);
            if (sm) { b = (sb + __ffs(sm)) * 32; break; }
            sb += 32;
            if (sb + 1 >= nsb) return -1;
        }
    }
    return -1;
}

FZB_DEV void prefetch_line(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
FZB_DEV void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- 1D walker v3: group summaries + the exit block in shared memory -------
// Per event the chain is: quantize -> exact zero interval -> one ballot over
// the rest of the event's 32-element group (a register per lane) -> one
// ballot over the block's group summaries (a register per lane) -> one
// ballot over the window of block summaries (registers) -> ONE memory round
// trip for the exit block: its 32 group summaries (one word per lane) and its
// 1024 elements (cp.async into shared memory) arrive together; a ballot
// picks the group, one shared-memory load per lane and a ballot the element.
constexpr long long PF_CHUNK = 16;     // blocks per prefetch chunk (64 KB of x)

__global__ void lz1d_summary2_kernel(const float* __restrict__ x, long long n, uint16_t* __restrict__ codes,
                                     int radius, float* __restrict__ bmin, float* __restrict__ bmax,
                                     float* __restrict__ gmin, float* __restrict__ gmax, long long nblk,
                                     uint32_t* __restrict__ status) {
    // status (optional): FZB_ERR_NONFINITE for a NaN / inf element, as
    // fzb_minmax_f32 reports it (fzb_lorenzo1d_prepare_f32 replaces that pass)
    bool bad = false;
    // one warp per 1K block.  Row e = elements [128 e, 128 e + 128): lane l
    // loads float4 (128 e + 4 l) -- one coalesced 512-byte access per row --
    // so group g = 4 e + l / 8 is lanes 8(g & 3) .. +7 of row e (3 xor shuffles)
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const uint32_t rr = (uint32_t)radius | ((uint32_t)radius << 16);
    const bool vec = !((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(codes)) & 15);
    for (long long blk = warp; blk < nblk; blk += nw) {
        const long long b0 = blk * BS1;
        float4 q[8];
        if (vec && b0 + BS1 <= n) {
#pragma unroll
            for (int e = 0; e < 8; e++) q[e] = __ldg(reinterpret_cast<const float4*>(x + b0) + e * 32 + lane);
#pragma unroll
            for (int e = 0; e < 4; e++)   // 1024 codes = 128 x 16 bytes
                reinterpret_cast<uint4*>(codes + b0)[e * 32 + lane] = make_uint4(rr, rr, rr, rr);
            if (status) {
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const uint32_t m = 0x7f800000u;
                    bad |= ((__float_as_uint(q[e].x) & m) == m) | ((__float_as_uint(q[e].y) & m) == m) |
                           ((__float_as_uint(q[e].z) & m) == m) | ((__float_as_uint(q[e].w) & m) == m);
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; e++) {
                float v[4];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const long long t = b0 + 128 * e + 4 * lane + c;
                    v[c] = t < n ? x[t] : NAN;
                    if (t < n) {
                        codes[t] = (uint16_t)radius;
                        bad |= !isfinite(v[c]);
                    }
                }
                q[e] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
        float blo = INFINITY, bhi = -INFINITY;
#pragma unroll
        for (int e = 0; e < 8; e++) {
            // fminf/fmaxf drop the NaN padding of a partial block
            float lo = fminf(fminf(q[e].x, q[e].y), fminf(q[e].z, q[e].w));
            float hi = fmaxf(fmaxf(q[e].x, q[e].y), fmaxf(q[e].z, q[e].w));
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            }
            if ((lane & 7) == 0) {
                const long long g = blk * 32 + 4 * e + (lane >> 3);
                gmin[g] = isnan(lo) ? INFINITY : lo;   // an all-padding group stays empty
                gmax[g] = isnan(hi) ? -INFINITY : hi;
            }
            blo = fminf(blo, lo);
            bhi = fmaxf(bhi, hi);
        }
#pragma unroll
        for (int o = 8; o < 32; o <<= 1) {
            blo = fminf(blo, __shfl_xor_sync(0xffffffffu, blo, o));
            bhi = fmaxf(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        if (lane == 0) {
            bmin[blk] = isnan(blo) ? INFINITY : blo;
            bmax[blk] = isnan(bhi) ? -INFINITY : bhi;
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && lane == 0) set_err(status, FZB_ERR_NONFINITE);
}

// (min, max) of the field from its superblock summaries: the lohi of
// fzb_minmax_f32 (fminf / fmaxf, NaN-free once the status is clear)
__global__ void lz1d_lohi_kernel(const float* __restrict__ smin, const float* __restrict__ smax, long long nsb,
                                 float* __restrict__ lohi) {
    float lo = INFINITY, hi = -INFINITY;
    for (long long q = threadIdx.x; q < nsb; q += blockDim.x) {
        lo = fminf(lo, smin[q]);
        hi = fmaxf(hi, smax[q]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ float sl[32], sh[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sl[w] = lo; sh[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); q++) {
            lo = fminf(lo, sl[q]);
            hi = fmaxf(hi, sh[q]);
        }
        lohi[0] = lo;
        lohi[1] = hi;
    }
}

FZB_DEV void cp_async16(void* smem, const void* gmem, int nbytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(nbytes)
                 : "memory");
}

// The walker's quantizer: the lz7 step's exact shortcut (reciprocal multiply,
// rint via the 1.5*2^52 magic constant, which also yields the integer code);
// within 1e-9 of a .5 tie, or without a usable reciprocal, the IEEE-division
// quantizer decides (same argument as v6::lz7_kernel / common.cuh).
FZB_DEV int quantize_walk(double v, double pred, const QParams& P, float& rec, bool& outl) {
    const double q = __dmul_rn(__dsub_rn(v, pred), P.inv2eb);
    const double tq = __dadd_rn(q, 6755399441055744.0);
    const double sd = __dsub_rn(tq, 6755399441055744.0);   // rint(q); |q| >= 2^51 -> outlier anyway
    const double fr = fabs(__dsub_rn(q, sd));
    if (!P.use_recip || fr >= 0.4999999990686774) return quantize(v, pred, P, rec, outl);
    const float rc = __double2float_rn(__dadd_rn(pred, __dmul_rn(P.two_eb, sd)));
    const bool ok = (fabs(sd) < (double)P.radius) & (fabs(__dsub_rn((double)rc, v)) <= P.eb);
    outl = !ok;
    rec = ok ? rc : __double2float_rn(v);
    return ok ? (int)(uint32_t)__double_as_longlong(tq) + P.radius : P.radius;
}


// An INNER zero-code interval: [ilo, ihi] with |v - pred| <= eb - m/2 for
// every f32 v in it, m = eb 2^-20 + (|pred| + eb) 2^-44, which dominates the
// rounding of the few f64 ops below.  Such a v has |q| < 0.5 - 2^-22 (no tie
// re-division) and |RN32(pred) - v| <= eb, i.e. a zero code: the interval is
// a subset of the exact zero-code set, so a scan with it finds every event,
// plus -- when an element falls in the sliver between the two, width ~m --
// a false candidate, which the event step quantizes to code R with the state
// unchanged.  Six f64 ops instead of a ballot round over candidate keys.
FZB_DEV void zinner(double pred, const QParams& P, float& ilo, float& ihi) {
    const double m = __dadd_rn(__dmul_rn(P.eb, 9.5367431640625e-07), __dmul_rn(__dadd_rn(fabs(pred), P.eb), 5.684341886080802e-14));
    const double w = __dsub_rn(P.eb, m);
    const double hd = __dadd_rn(pred, w), ld = __dsub_rn(pred, w);
    float hf = __double2float_rn(hd), lf = __double2float_rn(ld);
    if ((double)hf > hd) hf = kfloat(fkey(hf) - 1u);   // largest f32 <= hd
    if ((double)lf < ld) lf = kfloat(fkey(lf) + 1u);   // smallest f32 >= ld
    ilo = lf;
    ihi = hf;
}

FZB_DEV void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// lane 0: arm the barrier for `bytes` and start one bulk copy global -> shared
FZB_DEV void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(bytes), "r"(b)
                 : "memory");
}
FZB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(b), "r"(parity)
                     : "memory");
}

template <bool VEC>
__global__ void __launch_bounds__(64) lz1d_walk3_kernel(const float* __restrict__ x, long long n,
                                                         uint16_t* __restrict__ codes, uint32_t* __restrict__ bitmap,
                                                         const float* __restrict__ bmin, const float* __restrict__ bmax,
                                                         long long nblk, const float* __restrict__ smin_g,
                                                         const float* __restrict__ smax_g, long long nsb,
                                                         const float* __restrict__ gmin, const float* __restrict__ gmax,
                                                         const double* __restrict__ d_eb, int radius,
                                                         long long pf_ahead, long long* pos_slot,
                                                         uint8_t* __restrict__ notr) {
    extern __shared__ float s_sum[];
    __shared__ __align__(128) float s_blk[2][BS1];   // double-buffered exit blocks
    __shared__ __align__(8) uint64_t s_bar[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    volatile long long* g_pos = reinterpret_cast<volatile long long*>(pos_slot);
    if (blockIdx.x == 1) {
        // ---- prefetch CTA (another SM: its bulk prefetches do not queue in
        //      front of the walker's own bulk copies)
        if (warp != 0 || pf_ahead <= 0 || !VEC) return;
        // ---- prefetch warp: keep x and the summaries of [walker, walker + pf_ahead) in L2
        long long done = 0;
        for (;;) {
            const long long cb = *g_pos;
            if (cb < 0) break;
            if (done < cb) done = cb & ~(PF_CHUNK - 1);
            const long long target = min(nblk, cb + pf_ahead);
            if (lane == 0) {
                while (done < target) {
                    const long long m = min(PF_CHUNK * BS1, n - (done << 10));
                    prefetch_l2(x + (done << 10), (uint32_t)(((m * 4) + 15) & ~15ll));
                    const long long gm = min(PF_CHUNK, nblk - done) * 32 * 4;
                    prefetch_l2(gmin + done * 32, (uint32_t)gm);
                    prefetch_l2(gmax + done * 32, (uint32_t)gm);
                    if ((done & 255) == 0) {
                        const uint32_t by = (uint32_t)(((min(256ll, nblk - done) * 4) + 15) & ~15ll);
                        prefetch_l2(bmin + done, by);
                        prefetch_l2(bmax + done, by);
                    }
                    done += PF_CHUNK;
                }
            }
            done = __shfl_sync(0xffffffffu, done, 0);
            __nanosleep(256);
        }
        return;
    }
    const bool cached = nsb <= WALK_SMEM_SB;
    const float* smin = smin_g;
    const float* smax = smax_g;
    if (cached) {
        for (long long q = threadIdx.x; q < nsb; q += blockDim.x) {
            s_sum[q] = smin_g[q];
            s_sum[nsb + q] = smax_g[q];
        }
        smin = s_sum;
        smax = s_sum + nsb;
    }
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0]);
        mbar_init(&s_bar[1]);
    }
    __syncthreads();
    if (warp == 1) return;
    // the bound goes through an opaque move: otherwise ptxas rematerialises
    // P's fields by re-loading *d_eb on the event chain (twice per event)
    double ebr;
    asm volatile("mov.f64 %0, %1;" : "=d"(ebr) : "d"(*d_eb));
    const QParams P = make_qparams(ebr, radius);
#ifdef LZ7_TIMING
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long c0 = clock64();
#define WSTAMP3(i) do { const long long c1 = clock64(); ph[i] += c1 - c0; c0 = c1; } while (0)
#else
#define WSTAMP3(i) do { } while (0)
#endif
    // current block cb (smem buffer `cur`): its group summaries, the window of
    // block summaries past it, and this lane's element of the event's group;
    // the *2 registers hold the block being loaded into buffer cur ^ 1
    float wlo[WIN1], whi[WIN1], wlo2[WIN1], whi2[WIN1];
    float glo, ghi, glo2, ghi2;
    float gv;
    long long cb = 0;
    int cg = 0, cur = 0;
    bool bulk[2] = {false, false}, pend[2] = {false, false};
    uint32_t par[2] = {0u, 0u};
    // start the loads of block b into buffer k (elements) and the *2 registers
    auto issue = [&](long long b, int k) {
        const long long base = b << 10;
        const bool bk = VEC && base + BS1 <= n;
        if (bk) {
            if (lane == 0) bulk_load(s_blk[k], x + base, BS1 * 4, &s_bar[k]);
        } else if (VEC) {
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const long long i = base + 128 * e + 4 * lane;
                const int nb = (int)max(0ll, min(16ll, (n - i) * 4));
                cp_async16(s_blk[k] + 128 * e + 4 * lane, x + (nb ? i : 0), nb);
            }
            v6::cp_async_commit();
        }
        if (k) { bulk[1] = bk; pend[1] = VEC; } else { bulk[0] = bk; pend[0] = VEC; }
        const long long gq = b * 32 + lane;
        glo2 = (base + 32 * lane < n) ? __ldcg(gmin + gq) : INFINITY;
        ghi2 = (base + 32 * lane < n) ? __ldcg(gmax + gq) : -INFINITY;
        walk_load_window(bmin, bmax, nblk, b, wlo2, whi2);
    };
    auto wait_buf = [&](int k) {
        const bool p = k ? pend[1] : pend[0];
        if (!p) return;
        const bool bk = k ? bulk[1] : bulk[0];
        if (bk) {
            mbar_wait(&s_bar[k], k ? par[1] : par[0]);
            if (k) par[1] ^= 1u; else par[0] ^= 1u;
        } else {
            v6::cp_async_wait_n<0>();
        }
        if (k) pend[1] = false; else pend[0] = false;
        __syncwarp();
    };
    auto commit = [&]() {   // the *2 registers become the current block's
        glo = glo2;
        ghi = ghi2;
#pragma unroll
        for (int j = 0; j < WIN1; j++) { wlo[j] = wlo2[j]; whi[j] = whi2[j]; }
    };
    auto group_val = [&](long long b, int g, int k) -> float {
        const long long i = (b << 10) + 32 * g + lane;
        if (VEC) return s_blk[k][32 * g + lane];
        return i < n ? __ldg(x + i) : 0.f;
    };
    auto window_first = [&](float lo, float hi) -> long long {
        long long fb = -1;
#pragma unroll
        for (int j = 0; j < WIN1; j++) {
            const unsigned fm = __ballot_sync(0xffffffffu, !(wlo[j] >= lo && whi[j] <= hi));
            if (fm && fb < 0) fb = cb + 1 + 32 * j + (__ffs(fm) - 1);
        }
        return fb;
    };
    issue(0, 0);
    commit();
    wait_buf(0);
    gv = group_val(0, 0, 0);
    long long t = 0;
    float xv = __shfl_sync(0xffffffffu, gv, 0);
    float r = 0.f;
    for (;;) {
        {   // event at t
            const double pred = (t == 0) ? 0.0 : __dadd_rn(0.0, (double)r);
            float rec;
            bool outl;
            const int c = quantize_walk((double)xv, pred, P, rec, outl);
            if (lane == 0) {
                if (c != radius) {
                    codes[t] = (uint16_t)c;
                    if (notr) notr[t >> 12] = 1;   // this 4096-code chunk holds a code != R
                }
                if (outl) atomicOr(bitmap + (t >> 5), 1u << (t & 31));
            }
            r = rec;
        }
        WSTAMP3(0);
        if (t + 1 >= n) break;
        const double pr = __dadd_rn(0.0, (double)r);
        const long long gbase = (cb << 10) + 32 * cg;
        // speculation: the window's exit block under the approximate bounds
        // RN32(pr -/+ eb) -- its loads go out now and overlap the exact inner
        // interval and the rest-of-block checks (they differ from the inner
        // interval's choice only when a block summary falls in the ~eb 2^-20
        // sliver, or when the exit is still in the current block)
        long long sb;
        {
            const float alo = __double2float_rn(__dsub_rn(pr, P.eb)), ahi = __double2float_rn(__dadd_rn(pr, P.eb));
            sb = window_first(alo, ahi);
            if (sb >= 0) {
                wait_buf(cur ^ 1);   // a stale speculative load may still write that buffer
                issue(sb, cur ^ 1);
            }
        }
        float zlo, zhi;
        zinner(pr, P, zlo, zhi);
        WSTAMP3(1);
        // (1) the rest of the event's group
        {
            const unsigned m = __ballot_sync(0xffffffffu, (gbase + lane > t) & (gbase + lane < n) &
                                                              !(gv >= zlo && gv <= zhi));
            if (m) {
                const int f = __ffs(m) - 1;
                t = gbase + f;
                xv = __shfl_sync(0xffffffffu, gv, f);
                WSTAMP3(2);
                continue;
            }
        }
        // (2) the rest of the block: its later groups
        {
            const unsigned m = __ballot_sync(0xffffffffu, (lane > cg) & !(glo >= zlo && ghi <= zhi));
            if (m) {
                cg = __ffs(m) - 1;
                gv = group_val(cb, cg, cur);
                const long long gb2 = (cb << 10) + 32 * cg;
                const unsigned m2 = __ballot_sync(0xffffffffu, (gb2 + lane < n) & !(gv >= zlo && gv <= zhi));
                const int f = __ffs(m2) - 1;
                t = gb2 + f;
                xv = __shfl_sync(0xffffffffu, gv, f);
                WSTAMP3(2);
                continue;
            }
        }
        // (3) the window of block summaries, else the superblocks
        long long fb = window_first(zlo, zhi);
        WSTAMP3(2);
        if (fb < 0) {
#ifdef LZ7_TIMING
            ph[4]++;
#endif
            fb = walk_far(cb + 1 + 32 * WIN1, nblk, bmin, bmax, smin, smax, nsb, zlo, zhi);
        }
        if (fb < 0) break;   // no further event: the rest keeps zero codes
        if (fb != sb) {   // speculation missed (or was not taken)
#ifdef LZ7_TIMING
            ph[5]++;
#endif
            wait_buf(cur ^ 1);
            issue(fb, cur ^ 1);
        }
        cur ^= 1;
        commit();
        cb = fb;
        if (lane == 0) *g_pos = cb;
        {
            const unsigned m = __ballot_sync(0xffffffffu, !(glo >= zlo && ghi <= zhi));   // the summary guarantees one
            cg = __ffs(m) - 1;
        }
        wait_buf(cur);
        gv = group_val(cb, cg, cur);
        {
            const long long gb2 = (cb << 10) + 32 * cg;
            const unsigned m2 = __ballot_sync(0xffffffffu, (gb2 + lane < n) & !(gv >= zlo && gv <= zhi));
            const int f = __ffs(m2) - 1;
            t = gb2 + f;
            xv = __shfl_sync(0xffffffffu, gv, f);
        }
#ifdef LZ7_TIMING
        ph[6]++;
#endif
        WSTAMP3(3);
    }
    // drain outstanding copies before the CTA exits
    wait_buf(0);
    wait_buf(1);
    if (lane == 0) *g_pos = -1;
#ifdef LZ7_TIMING
    if (lane == 0)
        for (int i = 0; i < 8; i++) g_walk_stamp[i] = ph[i];
#endif
}

// ---- 1D decode: events = nonzero code or outlier --------------------------
// Between events the recon value is bitwise constant: (1) per-1024-element
// warp chunks count events (code mask | outlier bitmap word), (2) scan,
// (3) compact event positions, (4) replay the chain per segment that starts
// at event 0 or at an outlier (outliers reset the state), writing each
// event's value into recon[pos], (5) fill the rest with the last event's
// value.
constexpr int EVC = 1024;  // elements per warp chunk (32 lanes x 32)

FZB_DEV uint32_t event_mask(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap, long long n,
                            long long base, int radius) {
    // base = first element of this lane's 32-element group (multiple of 32)
    uint32_t m = 0;
    if (base + 32 <= n) {
        const uint4* p = reinterpret_cast<const uint4*>(codes + base);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint4 q = __ldg(p + u);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
                m |= (uint32_t)((w[h] & 0xFFFFu) != (uint32_t)radius) << (u * 8 + h * 2);
                m |= (uint32_t)((w[h] >> 16) != (uint32_t)radius) << (u * 8 + h * 2 + 1);
            }
        }
        m |= __ldg(bitmap + (base >> 5));
    } else if (base < n) {
        for (int e = 0; e < 32 && base + e < n; e++) m |= (uint32_t)(codes[base + e] != radius) << e;
        m |= __ldg(bitmap + (base >> 5)) & (0xFFFFFFFFu >> (32 - (int)(n - base)));
    }
    return m;
}

__global__ void lz1d_event_count_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap,
                                        long long n, int radius, uint32_t* __restrict__ counts, long long nch) {
    const int lane = threadIdx.x & 31;
    const long long ch = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ch >= nch) return;
    uint32_t c = __popc(event_mask(codes, bitmap, n, ch * EVC + lane * 32, radius));
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[ch] = c;
}

__global__ void lz1d_event_compact_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap,
                                          long long n, int radius, const unsigned long long* __restrict__ offs,
                                          long long* __restrict__ evpos, long long nch) {
    const int lane = threadIdx.x & 31;
    const long long ch = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ch >= nch) return;
    if (offs[ch + 1] == offs[ch]) return;   // no event in this chunk (sparse data: most chunks): no reload
    const long long base = ch * EVC + lane * 32;
    uint32_t m = event_mask(codes, bitmap, n, base, radius);
    uint32_t c = __popc(m), inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    unsigned long long o = offs[ch] + inc - c;
    while (m) {
        const int e = __ffs(m) - 1;
        m &= m - 1;
        evpos[o++] = base + e;
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
        const bool o0 = (bitmap[p0 >> 5] >> (p0 & 31)) & 1u;
        if (!(e == 0 || o0)) continue;
        float r = 0.f;
        // the chain depends on r only: positions, flags and codes of the next
        // EV_AHEAD events are loaded together, so each event costs its
        // dequantization instead of three dependent global loads
        constexpr int EV_AHEAD = 8;
        bool done = false;
        for (unsigned long long q0 = e; q0 < nev && !done; q0 += EV_AHEAD) {
            long long pp[EV_AHEAD];
            uint32_t ww[EV_AHEAD];
            uint16_t cc[EV_AHEAD];
#pragma unroll
            for (int u = 0; u < EV_AHEAD; u++) pp[u] = q0 + u < nev ? evpos[q0 + u] : -1;
#pragma unroll
            for (int u = 0; u < EV_AHEAD; u++) {
                ww[u] = pp[u] >= 0 ? bitmap[pp[u] >> 5] : 0u;
                cc[u] = pp[u] >= 0 ? codes[pp[u]] : (uint16_t)radius;
            }
#pragma unroll
            for (int u = 0; u < EV_AHEAD; u++) {
                const long long p = pp[u];
                if (p < 0) { done = true; break; }
                const bool outl = (ww[u] >> (p & 31)) & 1u;
                if (q0 + u != e && outl) { done = true; break; }
                if (outl) {
                    r = recon[p];  // pre-scattered outlier value
                } else {
                    const double pred = (p == 0) ? 0.0 : __dadd_rn(0.0, (double)r);
                    r = dequantize(pred, (int)cc[u], P);
                    recon[p] = r;
                }
            }
        }
    }
}

// Chain v2: one warp per segment (event 0 or an outlier, up to the next
// outlier).  The warp gathers 32 events at a time (positions, flags, codes,
// pre-scattered outlier values) and precomputes every 2eb*(code - R) in
// parallel; only the reconstruction itself stays serial: per event
// rec = RN32(RN64(0.0 + r) + c) -- one f32->f64 convert, two adds, one
// convert back -- with the inputs broadcast by shuffles that do not depend
// on r.  (v1: one thread per segment, ~180 cycles per event on long segments.)
__global__ void __launch_bounds__(128) lz1d_chain2_kernel(const long long* __restrict__ evpos,
                                                          const unsigned long long* __restrict__ nev_p,
                                                          const uint16_t* __restrict__ codes,
                                                          const uint32_t* __restrict__ bitmap,
                                                          float* __restrict__ recon, const double* __restrict__ d_eb,
                                                          int radius) {
    const unsigned long long nev = *nev_p;
    const int lane = threadIdx.x & 31;
    const unsigned long long w0 = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const QParams P = make_qparams(*d_eb, radius);
    for (unsigned long long e = w0; e < nev; e += nw) {
        const long long p0 = evpos[e];
        const bool o0 = (__ldg(bitmap + (p0 >> 5)) >> (p0 & 31)) & 1u;
        if (!(e == 0 || o0)) continue;   // warp-uniform: not a segment head
        float r = 0.f;                   // state entering event 0 (every earlier element has code R)
        // one batch = 32 events, one per lane, software-pipelined: while batch
        // b runs its serial loop, batch b + 32's code / outlier loads (their
        // positions loaded one batch earlier) and batch b + 64's positions are
        // in flight
        struct Ev {
            long long pos;
            bool valid, isout;
            int code;
            float ov;
        };
        auto evp = [&](unsigned long long k) { return k < nev ? evpos[k] : 0ll; };
        auto load = [&](unsigned long long k, long long pos) {
            Ev v;
            v.valid = k < nev;
            v.pos = pos;
            v.isout = v.valid && ((__ldg(bitmap + (pos >> 5)) >> (pos & 31)) & 1u);
            v.code = v.valid ? (int)codes[pos] : radius;
            v.ov = v.isout ? recon[pos] : 0.f;
            return v;
        };
        Ev nx = load(e + lane, evp(e + lane));
        long long pnn = evp(e + 32 + lane);
        for (unsigned long long b = e;; b += 32) {
            const unsigned long long k = b + lane;
            const Ev cu = nx;
            nx = load(k + 32, pnn);
            pnn = evp(k + 64);
            const long long pos = cu.pos;
            const bool valid = cu.valid, isout = cu.isout;
            const double c = __dmul_rn(P.two_eb, (double)(cu.code - radius));
            const float ov = cu.ov;
            const unsigned stop = __ballot_sync(0xffffffffu, (isout && k != e) || !valid);
            const int lim = stop ? __ffs(stop) - 1 : 32;
            // RN64(0.0 + r) + c == RN64(r + c) for every c (the 0.0 + only turns -0 into +0,
            // which no sum can tell apart), so one add per event.  (RN32 as
            // x + 1.5 * 2^(e+29) - that constant, off the XU pipe, made this
            // chain slower: 148 -> 214 us on C4.)
            float mine = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const double cj = __shfl_sync(0xffffffffu, c, j);
                const bool oj = __shfl_sync(0xffffffffu, isout, j);
                const float ovj = __shfl_sync(0xffffffffu, ov, j);
                if (j < lim) {
                    r = oj ? ovj : __double2float_rn(__dadd_rn((double)r, cj));
                    if (lane == j) mine = r;
                }
            }
            if (lane < lim && !isout) recon[pos] = mine;
            if (lim < 32) break;
        }
    }
}

__global__ void lz1d_fill_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ bitmap, long long n,
                                 int radius, const unsigned long long* __restrict__ offs,
                                 const long long* __restrict__ evpos, float* __restrict__ recon, long long nch) {
    const int lane = threadIdx.x & 31;
    const long long ch = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ch >= nch) return;
    const long long base0 = ch * EVC;
    const long long base = base0 + lane * 32;
    const uint32_t m = event_mask(codes, bitmap, n, base, radius);
    // last event position at or before the end of each lane's group
    long long last = m ? base + 31 - __clz(m) : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, last, o);
        if (lane >= o) last = max(last, y);
    }
    long long carry = __shfl_up_sync(0xffffffffu, last, 1);
    if (lane == 0) carry = -1;
    if (carry < 0) {
        const unsigned long long o = offs[ch];
        carry = o > 0 ? evpos[o - 1] : -1;
    }
    // coalesced writes: row j is group j's 32 elements, one per lane; a
    // zero-code element reconstructs to f32(0.0 + r): the value of the last
    // event at or before it (or the carry), -0 -> +0; events keep their value
    for (int j = 0; j < 32; j++) {
        const long long gb = base0 + 32 * (long long)j;
        if (gb >= n) break;
        const uint32_t mj = __shfl_sync(0xffffffffu, m, j);
        const long long cj = __shfl_sync(0xffffffffu, carry, j);
        const uint32_t upto = mj & (0xFFFFFFFFu >> (31 - lane));   // events at positions <= lane
        const long long src = upto ? gb + 31 - __clz(upto) : cj;
        if (gb + lane < n && !((mj >> lane) & 1u)) recon[gb + lane] = src >= 0 ? recon[src] + 0.0f : 0.f;
    }
}

// Fill without re-reading the codes: a chunk's events are evpos[offs[ch] ..
// offs[ch+1]) (sorted); they set bits of a 1024-bit shared bitmap, and every
// other element takes f32(0.0 + r) of the last event at or before it (the
// chain pass wrote the event values into recon), -0 -> +0.  Traffic: the
// 4n-byte recon write plus the (few) event positions and values.
__global__ void __launch_bounds__(256) lz1d_fill2_kernel(const long long* __restrict__ evpos,
                                                          const unsigned long long* __restrict__ offs,
                                                          float* __restrict__ recon, long long n, long long nch) {
    __shared__ uint32_t s_bm[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long ch = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ch >= nch) return;
    const long long base0 = ch * EVC;
    const unsigned long long lo = offs[ch], hi = offs[ch + 1];
    if (lo == hi && base0 + EVC <= n && !(reinterpret_cast<uintptr_t>(recon) & 15)) {
        // no event in the chunk (most chunks of sparse data): one value, 16-byte stores
        const float v = lo > 0 ? recon[evpos[lo - 1]] + 0.0f : 0.f;
        const float4 q = make_float4(v, v, v, v);
#pragma unroll
        for (int e = 0; e < 8; e++) reinterpret_cast<float4*>(recon + base0)[e * 32 + lane] = q;
        return;
    }
    uint32_t* bm = s_bm[wib];
    bm[lane] = 0;
    __syncwarp();
    for (unsigned long long e = lo + lane; e < hi; e += 32) {
        const int o = (int)(evpos[e] - base0);
        atomicOr(bm + (o >> 5), 1u << (o & 31));
    }
    __syncwarp();
    const uint32_t mw = bm[lane];   // lane j: events of row j
    // last event strictly before row j: max over rows < j, else the previous chunk's last event
    long long last = mw ? base0 + 32 * lane + 31 - __clz(mw) : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, last, o);
        if (lane >= o) last = max(last, y);
    }
    long long carry = __shfl_up_sync(0xffffffffu, last, 1);
    if (lane == 0 || carry < 0) carry = (lane == 0 || carry < 0) ? (lo > 0 ? evpos[lo - 1] : -1) : carry;
    const float cval = carry >= 0 ? recon[carry] + 0.0f : 0.f;   // lane j: value entering row j
    for (int j = 0; j < 32; j++) {
        const long long gb = base0 + 32 * (long long)j;
        if (gb >= n) break;
        const uint32_t mj = __shfl_sync(0xffffffffu, mw, j);
        const float cj = __shfl_sync(0xffffffffu, cval, j);
        if (gb + lane < n && !((mj >> lane) & 1u)) {
            const uint32_t upto = mj & (0xFFFFFFFFu >> (31 - lane));   // events at positions <= lane
            recon[gb + lane] = upto ? recon[gb + 31 - __clz(upto)] + 0.0f : cj;
        }
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

template <int PI>
struct WaveWS {
    size_t ntile, fI, fJ, K, off_prog, off_order, off_counts, off_fI, total;
    WaveWS(int n0, int n1, int n2) {
        const size_t nA = (n0 + PI - 1) / PI, nB = (n1 + 31) / 32;
        ntile = nA * nB;
        fI = nA * (size_t)n1 * n2;
        fJ = nB * (size_t)n0 * n2;
        K = (size_t)(2 * G + PI) * (nA - 1) + (size_t)(2 * G + 32) * (nB - 1) + 1;
        auto al = [](size_t x) { return (x + 255) / 256 * 256; };
        off_prog = 256;
        off_order = off_prog + al(ntile * 4);
        off_counts = off_order + al(ntile * 4);
        off_fI = off_counts + al(K * 4);
        total = off_fI + al(fI * 4) + al(fJ * 4) + 256;
    }
};

template <int PI, bool DEC>
int launch_wave4(const float* orig, const uint16_t* codes_in, uint16_t* codes_out, uint32_t* bitmap, float* recon,
                 int n0, int n1, int n2, const double* d_eb, int radius, void* ws, size_t ws_bytes, cudaStream_t st) {
    Geo g;
    g.n0 = n0; g.n1 = n1; g.n2 = n2;
    g.nA = (n0 + PI - 1) / PI;
    g.nB = (n1 + 31) / 32;
    WaveWS<PI> L(n0, n1, n2);
    if (ws_bytes < L.total) return FZB_E_WORKSPACE;
    unsigned char* w = static_cast<unsigned char*>(ws);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(w + 128);
    uint32_t* progress = reinterpret_cast<uint32_t*>(w + L.off_prog);
    int* order = reinterpret_cast<int*>(w + L.off_order);
    int* counts = reinterpret_cast<int*>(w + L.off_counts);
    float* faceI = reinterpret_cast<float*>(w + L.off_fI);
    float* faceJ = reinterpret_cast<float*>(w + L.off_fI + (L.fI * 4 + 255) / 256 * 256);
    cudaMemsetAsync(w + 8, 0, L.off_order - 8, st);   // signature, ticket, progress (keeps the v7 epoch)
    tile_order_kernel<<<1, 1024, 0, st>>>(g.nA, g.nB, 2 * G + PI, 2 * G + 32, counts, order);
    const size_t smem = Smem4<PI, DEC>::bytes;
    auto kfn = lz_wave4_kernel<PI, DEC>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<(unsigned)L.ntile, (PI + 1) * 32, smem, st>>>(orig, codes_in, codes_out, bitmap, recon, faceI, faceJ,
                                                       progress, ticket, order, g, d_eb, radius);
    return fzb_check_launch();
}

template <int PI>
size_t wave_ws(int n0, int n1, int n2) {
    return WaveWS<PI>(n0, n1, n2).total;
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

// FZB_LORENZO=4 selects the previous (barrier-per-step) wavefront for A/B runs.
bool use_v4(uint32_t n2) {
    // v7 stages 16-byte row quads; rows that are not a multiple of 4 long use v4
    const char* e = getenv("FZB_LORENZO");
    return (e && e[0] == '4') || (n2 % 4 != 0);
}

// v7 wavefront configurations (W compute warps x R rows per thread); the
// tile height W*R must not exceed n0.  FZB_LZ_CFG=WxR overrides (tuning).
struct Cfg7 { int W, R; };
// Tile configuration: 4 warps x 2 rows is the throughput choice (3 CTAs/SM);
// when the whole launch has fewer 8x32 tiles than 3 per SM, the wavefront is
// latency-bound and 8 warps x 1 row (one chain per warp, lower step latency)
// is faster (C1 100x500x500: 208 tiles, -4%).
Cfg7 pick7(uint32_t n0, uint32_t n1 = 0, int nf = 1) {
    const char* e = getenv("FZB_LZ_CFG");
    if (e) {
        int W = 0, R = 0;
        if (sscanf(e, "%dx%d", &W, &R) == 2 && (uint32_t)(W * R) <= n0) return {W, R};
    }
    if (n0 >= 8) {
        const uint64_t tiles = (uint64_t)((n0 + 7) / 8) * ((n1 + 31) / 32) * (uint64_t)(nf > 0 ? nf : 1);
        return (n1 && tiles < (uint64_t)kNumSMs * 3) ? Cfg7{8, 1} : Cfg7{4, 2};
    }
    if (n0 >= 4) return {2, 2};
    if (n0 >= 2) return {1, 2};
    return {1, 1};
}

#define FZB_LZ7_CFGS(X) X(8, 2) X(4, 4) X(4, 2) X(4, 3) X(8, 1) X(2, 4) X(2, 2) X(1, 2) X(1, 1) X(16, 1) X(4, 1) X(2, 1)

template <bool DEC>
int launch_v7(const float* orig, const uint16_t* codes_in, uint16_t* codes_out, uint32_t* bitmap, float* recon,
              uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb, int radius, void* ws, size_t ws_bytes,
              cudaStream_t st) {
    const Cfg7 c = pick7(n0, n1);
#define FZB_LZ7_CASE(W_, R_)                                                                                   \
    if (c.W == W_ && c.R == R_)                                                                                 \
        return v6::launch7<W_, R_, DEC>(orig, codes_in, codes_out, bitmap, recon, n0, n1, n2, d_eb, radius, ws, \
                                        ws_bytes, st);
    FZB_LZ7_CFGS(FZB_LZ7_CASE)
#undef FZB_LZ7_CASE
    return FZB_E_ARG;
}

template <bool DEC>
int launch_v7_batch(const float* orig, const uint16_t* codes_in, uint16_t* codes_out, uint32_t* bitmap, float* recon,
                    uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb, int radius, void* ws, size_t ws_bytes,
                    cudaStream_t st, int nf, long long fstride, long long bstride) {
    const Cfg7 c = pick7(n0, n1, nf);
#define FZB_LZ7_BCASE(W_, R_)                                                                                      \
    if (c.W == W_ && c.R == R_)                                                                                     \
        return v6::launch7<W_, R_, DEC>(orig, codes_in, codes_out, bitmap, recon, n0, n1, n2, d_eb, radius, ws,     \
                                        ws_bytes, st, nf, fstride, bstride);
    FZB_LZ7_CFGS(FZB_LZ7_BCASE)
#undef FZB_LZ7_BCASE
    return FZB_E_ARG;
}

size_t v7_ws_batch(uint32_t nf, uint32_t n0, uint32_t n1, uint32_t n2) {
    const Cfg7 c = pick7(n0);
    switch (c.W * c.R) {
        case 1: return v6::WS7<1>(n0, n1, n2, nf).total;
        case 2: return v6::WS7<2>(n0, n1, n2, nf).total;
        case 4: return v6::WS7<4>(n0, n1, n2, nf).total;
        case 8: return v6::WS7<8>(n0, n1, n2, nf).total;
        case 12: return v6::WS7<12>(n0, n1, n2, nf).total;
        default: return v6::WS7<16>(n0, n1, n2, nf).total;
    }
}

size_t v7_ws(uint32_t n0, uint32_t n1, uint32_t n2) {
    // enough for every configuration pick7 may return (tuning overrides included)
    size_t m = 0;
    for (int pi : {1, 2, 4, 8, 12, 16}) {
        if ((uint32_t)pi > n0 && pi > 1) continue;
        size_t t = 0;
        switch (pi) {
            case 1: t = v6::WS7<1>(n0, n1, n2).total; break;
            case 2: t = v6::WS7<2>(n0, n1, n2).total; break;
            case 4: t = v6::WS7<4>(n0, n1, n2).total; break;
            case 8: t = v6::WS7<8>(n0, n1, n2).total; break;
            case 12: t = v6::WS7<12>(n0, n1, n2).total; break;
            default: t = v6::WS7<16>(n0, n1, n2).total; break;
        }
        m = t > m ? t : m;
    }
    return m;
}

// 1D encoder workspace: header, block / superblock / group summaries.
struct Walk1D {
    size_t o_bmin, o_bmax, o_smin, o_smax, o_gmin, o_gmax, total;
    explicit Walk1D(long long n) {
        const size_t nblk = (size_t)((n + BS1 - 1) / BS1), nsb = (nblk + 31) / 32;
        auto al = [](size_t x) { return (x + 255) / 256 * 256; };
        o_bmin = WS_HDR;
        o_bmax = o_bmin + al(nblk * 4);
        o_smin = o_bmax + al(nblk * 4);
        o_smax = o_smin + al(nsb * 4);
        o_gmin = o_smax + al(nsb * 4);
        o_gmax = o_gmin + al(nblk * 128);
        total = o_gmax + al(nblk * 128);
    }
};

}  // namespace

extern "C" {

FZB_API size_t fzb_lorenzo_workspace_bytes(uint32_t n0, uint32_t n1, uint32_t n2) {
    canon(n0, n1, n2);
    const long long n = (long long)n0 * n1 * n2;
    if (n0 == 1 && n1 == 1) {
        const long long nblk = (n + BS1 - 1) / BS1, nsb = (nblk + 31) / 32, nch = (n + EVC - 1) / EVC;
        const size_t enc = Walk1D(n).total;
        const size_t dec = WS_HDR + 2048 + (size_t)(nch + 1) * 12 + fzscan::ws_bytes(nch + 1) + (size_t)n * 8;
        return enc > dec ? enc : dec;
    }
    size_t w4;
    switch (pick_pi(n0)) {
        case 8: w4 = wave_ws<8>(n0, n1, n2); break;
        case 4: w4 = wave_ws<4>(n0, n1, n2); break;
        case 2: w4 = wave_ws<2>(n0, n1, n2); break;
        default: w4 = wave_ws<1>(n0, n1, n2); break;
    }
    const size_t w6 = v7_ws(n0, n1, n2);
    return w4 > w6 ? w4 : w6;
}

// 1D encode, step 1 (no error bound needed): the walker's group / block /
// superblock min-max summaries into d_ws, codes filled with radius; with
// d_lohi, also the field's (min, max) and FZB_ERR_NONFINITE exactly as
// fzb_minmax_f32 -- so a 1D field is read once before its bound is known.
FZB_API int fzb_lorenzo1d_prepare_f32(const float* d_in, uint64_t n, uint32_t radius, uint16_t* d_codes,
                                      float* d_lohi, void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (n == 0) return d_lohi ? FZB_E_ARG : 0;
    const long long nblk = ((long long)n + BS1 - 1) / BS1, nsb = (nblk + 31) / 32;
    // every summary array 256-byte aligned (the walker bulk-prefetches them)
    const Walk1D L((long long)n);
    if (ws_bytes < L.total) return FZB_E_WORKSPACE;
    invalidate_faces(d_ws, st);
    unsigned char* wb = static_cast<unsigned char*>(d_ws);
    float* bmin = reinterpret_cast<float*>(wb + L.o_bmin);
    float* bmax = reinterpret_cast<float*>(wb + L.o_bmax);
    float* smin = reinterpret_cast<float*>(wb + L.o_smin);
    float* smax = reinterpret_cast<float*>(wb + L.o_smax);
    lz1d_summary2_kernel<<<kNumSMs * 8, 256, 0, st>>>(d_in, (long long)n, d_codes, (int)radius, bmin, bmax,
                                                      reinterpret_cast<float*>(wb + L.o_gmin),
                                                      reinterpret_cast<float*>(wb + L.o_gmax), nblk,
                                                      d_lohi ? d_status : nullptr);
    lz1d_super_kernel<<<kNumSMs * 2, 256, 0, st>>>(bmin, bmax, nblk, smin, smax, nsb);
    if (d_lohi) lz1d_lohi_kernel<<<1, 1024, 0, st>>>(smin, smax, nsb, d_lohi);
    return fzb_check_launch();
}

// 1D encode, step 2: the event walker over the summaries of step 1 (same
// d_in, n, radius, d_codes and d_ws) with the resolved bound.
FZB_API int fzb_lorenzo1d_walk_f32(const float* d_in, uint64_t n, const double* d_eb, uint32_t radius,
                                   uint16_t* d_codes, uint32_t* d_bitmap, uint8_t* d_notr, void* d_ws,
                                   size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (n == 0) return 0;
    const long long nblk = ((long long)n + BS1 - 1) / BS1, nsb = (nblk + 31) / 32;
    const Walk1D L((long long)n);
    if (ws_bytes < L.total) return FZB_E_WORKSPACE;
    unsigned char* wb = static_cast<unsigned char*>(d_ws);
    float* bmin = reinterpret_cast<float*>(wb + L.o_bmin);
    float* bmax = reinterpret_cast<float*>(wb + L.o_bmax);
    float* smin = reinterpret_cast<float*>(wb + L.o_smin);
    float* smax = reinterpret_cast<float*>(wb + L.o_smax);
    float* gmin = reinterpret_cast<float*>(wb + L.o_gmin);
    float* gmax = reinterpret_cast<float*>(wb + L.o_gmax);
    const size_t wsm = nsb <= WALK_SMEM_SB ? (size_t)nsb * 8 : 0;
    const bool vec = !(reinterpret_cast<uintptr_t>(d_in) & 15);
    auto kfn = vec ? lz1d_walk3_kernel<true> : lz1d_walk3_kernel<false>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
    const char* pfe = getenv("FZB_WALK_PF");
    const long long pf = pfe ? atoll(pfe) : PF_AHEAD;
    long long* pos = reinterpret_cast<long long*>(wb + 24);   // header words 6-7: walker position
    cudaMemsetAsync(pos, 0, 8, st);
    if (d_notr) cudaMemsetAsync(d_notr, 0, (size_t)((n + FZB_HF_CHUNK - 1) / FZB_HF_CHUNK), st);
    kfn<<<2, 64, wsm, st>>>(d_in, (long long)n, d_codes, d_bitmap, bmin, bmax, nblk, smin, smax, nsb, gmin, gmax,
                            d_eb, (int)radius, pf, pos, d_notr);
#ifdef LZ7_TIMING
    if (getenv("FZB_WALK_TWICE")) {
        cudaMemsetAsync(pos, 0, 8, st);
        kfn<<<2, 64, wsm, st>>>(d_in, (long long)n, d_codes, d_bitmap, bmin, bmax, nblk, smin, smax, nsb, gmin, gmax,
                                d_eb, (int)radius, pf, pos, d_notr);
    }
#endif
    return fzb_check_launch();
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
        const int rc = fzb_lorenzo1d_prepare_f32(d_in, (uint64_t)n, radius, d_codes, nullptr, d_ws, ws_bytes, nullptr,
                                                 stream);
        if (rc) return rc;
        return fzb_lorenzo1d_walk_f32(d_in, (uint64_t)n, d_eb, radius, d_codes, d_bitmap, nullptr, d_ws, ws_bytes,
                                      stream);
    }
    if (!use_v4(n2))
        return launch_v7<false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, (int)radius, d_ws, ws_bytes, st);
    switch (pick_pi(n0)) {
        case 8: return launch_wave4<8, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 4: return launch_wave4<4, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 2: return launch_wave4<2, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        default: return launch_wave4<1, false>(d_in, nullptr, d_codes, d_bitmap, nullptr, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
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
        const long long nch = (n + EVC - 1) / EVC;
        if (ws_bytes < fzb_lorenzo_workspace_bytes(1, 1, (uint32_t)n)) return FZB_E_WORKSPACE;
        invalidate_faces(d_ws, st);
        unsigned char* w = static_cast<unsigned char*>(d_ws) + WS_HDR;
        auto al = [](size_t x) { return (x + 255) / 256 * 256; };
        // counts / offsets carry one extra entry (0 / the total) so offs[ch + 1] is always valid
        unsigned long long* nev = reinterpret_cast<unsigned long long*>(w);
        uint32_t* counts = reinterpret_cast<uint32_t*>(w + 256);
        unsigned long long* offs = reinterpret_cast<unsigned long long*>(w + 256 + al((nch + 1) * 4));
        void* sws = w + 256 + al((nch + 1) * 4) + al((nch + 1) * 8);
        long long* evpos = reinterpret_cast<long long*>(w + 256 + al((nch + 1) * 4) + al((nch + 1) * 8) +
                                                        al(fzscan::ws_bytes(nch + 1)));
        const unsigned blocks = (unsigned)((nch * 32 + 255) / 256);
        cudaMemsetAsync(counts + nch, 0, 4, st);
        lz1d_event_count_kernel<<<blocks, 256, 0, st>>>(d_codes, d_bitmap, n, (int)radius, counts, nch);
        fzscan::exclusive(counts, nch + 1, offs, nev, sws, st);
        lz1d_event_compact_kernel<<<blocks, 256, 0, st>>>(d_codes, d_bitmap, n, (int)radius, offs, evpos, nch);
        lz1d_chain2_kernel<<<kNumSMs * 8, 128, 0, st>>>(evpos, nev, d_codes, d_bitmap, d_recon, d_eb, (int)radius);
        lz1d_fill2_kernel<<<blocks, 256, 0, st>>>(evpos, offs, d_recon, n, nch);
        return fzb_check_launch();
    }
    if (!use_v4(n2))
        return launch_v7<true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, (int)radius, d_ws, ws_bytes, st);
    switch (pick_pi(n0)) {
        case 8: return launch_wave4<8, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 4: return launch_wave4<4, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        case 2: return launch_wave4<2, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
        default: return launch_wave4<1, true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, n0, n1, n2, d_eb, radius, d_ws, ws_bytes, st);
    }
}

#ifdef LZ7_TIMING
FZB_API int fzb_debug_lz_timing(long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, v6::g_lz_stamp, sizeof(v6::g_lz_stamp));
}
FZB_API int fzb_debug_tile_times(unsigned long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, v6::g_tile_t, sizeof(v6::g_tile_t));
}
FZB_API int fzb_debug_walk_timing(long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, g_walk_stamp, sizeof(g_walk_stamp));
}
#endif

// ---- batches of same-shaped fields (several fields in flight per
// GPU).  One wavefront launch interleaves the tiles of all fields in one
// ticket order, so the GPU idles less than with one field at a time.  Field
// f lives at d_in + f * field_stride (codes / recon likewise) with its
// bitmap at d_bitmap + f * bitmap_stride_words and its bound at d_eb[f].
// Shapes the v7 wavefront does not take (1D, n2 % 4 != 0) run field by field.
FZB_API size_t fzb_lorenzo_batch_workspace_bytes(uint32_t nf, uint32_t n0, uint32_t n1, uint32_t n2) {
    const size_t one = fzb_lorenzo_workspace_bytes(n0, n1, n2);
    canon(n0, n1, n2);
    if (nf <= 1 || (n0 == 1 && n1 == 1) || use_v4(n2)) return one;
    const size_t b = v7_ws_batch(nf, n0, n1, n2);
    return b > one ? b : one;
}

FZB_API int fzb_lorenzo_encode_batch_f32(const float* d_in, uint32_t nf, uint64_t field_stride, uint32_t n0,
                                         uint32_t n1, uint32_t n2, const double* d_eb, uint32_t radius,
                                         uint16_t* d_codes, uint32_t* d_bitmap, uint64_t bitmap_stride_words,
                                         void* d_ws, size_t ws_bytes, void* stream) {
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    uint32_t c0 = n0, c1 = n1, c2 = n2;
    canon(c0, c1, c2);
    if (nf == 0 || (long long)c0 * c1 * c2 == 0) return 0;
    if (nf == 1 || (c0 == 1 && c1 == 1) || use_v4(c2)) {
        for (uint32_t f = 0; f < nf; f++) {
            const int rc = fzb_lorenzo_encode_f32(d_in + f * field_stride, n0, n1, n2, d_eb + f, radius,
                                                  d_codes + f * field_stride, d_bitmap + f * bitmap_stride_words, d_ws,
                                                  ws_bytes, stream);
            if (rc) return rc;
        }
        return 0;
    }
    return launch_v7_batch<false>(d_in, nullptr, d_codes, d_bitmap, nullptr, c0, c1, c2, d_eb, (int)radius, d_ws,
                                  ws_bytes, (cudaStream_t)stream, (int)nf, (long long)field_stride,
                                  (long long)bitmap_stride_words);
}

FZB_API int fzb_lorenzo_decode_batch_f32(const uint16_t* d_codes, const uint32_t* d_bitmap,
                                         uint64_t bitmap_stride_words, float* d_recon, uint32_t nf,
                                         uint64_t field_stride, uint32_t n0, uint32_t n1, uint32_t n2,
                                         const double* d_eb, uint32_t radius, void* d_ws, size_t ws_bytes,
                                         void* stream) {
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    uint32_t c0 = n0, c1 = n1, c2 = n2;
    canon(c0, c1, c2);
    if (nf == 0 || (long long)c0 * c1 * c2 == 0) return 0;
    if (nf == 1 || (c0 == 1 && c1 == 1) || use_v4(c2)) {
        for (uint32_t f = 0; f < nf; f++) {
            const int rc = fzb_lorenzo_decode_f32(d_codes + f * field_stride, d_bitmap + f * bitmap_stride_words,
                                                  d_recon + f * field_stride, n0, n1, n2, d_eb + f, radius, d_ws,
                                                  ws_bytes, stream);
            if (rc) return rc;
        }
        return 0;
    }
    return launch_v7_batch<true>(nullptr, d_codes, nullptr, const_cast<uint32_t*>(d_bitmap), d_recon, c0, c1, c2, d_eb,
                                 (int)radius, d_ws, ws_bytes, (cudaStream_t)stream, (int)nf, (long long)field_stride,
                                 (long long)bitmap_stride_words);
}

}  // extern "C"
