// lorenzo6.cuh -- register-resident exact Lorenzo wavefront (v6), 2D/3D.
//
// Reference: fzpipe predict.py:93-144 (_lorenzo_encode / _lorenzo_decode).
// Same recurrence, same 7-term f64 order and quantizer as lz_wave4 (see the
// arithmetic notes in lorenzo.cu / common.cuh); what changes is how the
// dependency DAG is mapped onto the SM:
//
//  * Tile = R i-rows x 32 j-lanes, marching along k; ONE compute warp owns a
//    tile.  Lane b holds all R rows of column j0+b in registers and at step
//    s computes the R elements (i0+r, j0+b, k = s-r-b): they are independent
//    of each other within a step (ILP R), every intra-thread neighbour (up,
//    self, up-left, ...) is a register from the previous one or two steps,
//    and the only cross-lane value per row and step is `left`, one 64-bit
//    shuffle (lane 0's left halo rides the same shuffle from lane 31).  No
//    barrier, no shared-memory ring on the dependency chain.
//  * Halos move as LL pairs: a 64-bit word {f32 value, u32 tag} written with
//    one 64-bit store, so value and tag become visible together and the
//    consumer needs no fence -- it polls until the tag matches.  Producer
//    tiles publish their last row (faceI) and lane 31 (faceJ) to global
//    memory every step (tag = launch epoch); the consumer CTA's helper warp
//    polls L2 and re-tags them into shared-memory rings (tag = step + 1)
//    which the compute warp checks one step before it needs them.
//  * The helper warp also stages the inputs (16-byte cp.async into a
//    k-indexed ring, zero-filled outside the field so steps before a row's
//    k == 0 compute exact zeros) and flushes the outputs, which the compute
//    warp writes in place into the same ring; helper <-> compute group
//    handshakes are release/acquire counters in shared memory.
//  * Tiles are claimed by an atomic ticket in topological (expected start)
//    order, so every CTA only waits on tiles that are resident or finished.
//
// Signed zeros: the recon values kept for prediction are normalised (x+0.0f)
// so `up` is never -0.0; then `up + left` equals the reference's
// `(0.0 + up) + left` and no partial sum is ever -0.0 (x + y == -0.0 needs
// both -0.0), which also makes absent neighbours (+0.0) exact.  The f32
// values written to the recon output keep their sign.
#pragma once

namespace v6 {

constexpr int G = 8;        // steps per group (staging / flush / handshake granularity)
constexpr int KR = 32;      // k-indexed ring slots per row (4 chunks of 8)
constexpr int IP = 36;      // ring pitch in words: multiple of 4 (16 B cp.async) and
                            // IP-1 odd, so lane b's row at k = c-b hits bank (3b + c) % 32
constexpr int SD = 2;       // staging distance: group j+SD is put in flight when group j completes
                            // (needs KR/8 >= SD + 1 chunks: its slots must already be flushed)
constexpr int HR = 32;      // halo ring slots (steps)
constexpr int GRD = 16;     // ghost ring slots between compute warps (steps)
constexpr int HUW = 33;     // ghost-row entries per step: corner + 32 lanes
constexpr uint32_t CODE_TAG = 0x7FC00000u;  // decode ring: NaN-tagged code; finite outliers stay raw f32 bits
constexpr int OFF = 2;      // element k = s - OFF - r - b at step s: every halo a step needs is from step >= 0

struct Geo6 {
    int n0, n1, n2, nA, nB, S;
    int vec;             // n2 % 4 == 0: 16-byte staging / flush
    int nt1;             // tiles per field (batched launches: global tile id T = field * nt1 + tile)
    long long fstride;   // elements between consecutive fields
    long long bstride;   // bitmap words between consecutive fields
};


FZB_DEV uint64_t ll_pack(float v, uint32_t tag) {
    return ((uint64_t)tag << 32) | (uint64_t)__float_as_uint(v);
}
FZB_DEV uint64_t ld_ll_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
FZB_DEV void st_ll_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
FZB_DEV void st_ll_gpu_if(bool pred, uint64_t* p, uint64_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.relaxed.gpu.global.u64 [%0], %1; }" ::"l"(p), "l"(v),
                 "r"((int)pred)
                 : "memory");
}
FZB_DEV uint64_t ld_ll_cta(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
FZB_DEV void st_ll_cta(uint64_t* p, uint64_t v) {
    asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}
FZB_DEV uint32_t ld_cta_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
FZB_DEV uint32_t ld_acq_cta(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
FZB_DEV void st_rel_cta(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
FZB_DEV void cp_async16_zfill(void* smem, const void* gmem, int nbytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(nbytes)
                 : "memory");
}
FZB_DEV void cp_async4_z(void* smem, const void* gmem, int nbytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(nbytes)
                 : "memory");
}

// Spin until every one of the n per-warp counters reaches `target`.
FZB_DEV void wait_min(const uint32_t* cnt, int n, uint32_t target) {
    while (true) {
        uint32_t m = 0xFFFFFFFFu;
        for (int q = 0; q < n; q++) {
            const uint32_t v = ld_acq_cta(cnt + q);
            m = v < m ? v : m;
        }
        if (m >= target) return;
        __nanosleep(32);
    }
}

// Chunk (8 consecutive k) of row (r, b), d = r + b, that group j first needs:
// the one holding its last k of the group (floor division).
FZB_DEV int chunk_of(int j, int d) { return (j * G + G - 1 - OFF - d) >> 3; }

// ------------------------------------------------------------------ helper
// Staging runs SD groups ahead.  Encode: 16-byte cp.async straight into the
// ring (one commit group per iteration).  Decode: the stager loads a group's
// code quads and bitmap words into registers one iteration before it
// NaN-tags them (splicing in outlier values) and stores them to the ring.
// Rows are spread as (row = q*16 + lane/2, half = lane&1).  v7 requires
// n2 % 4 == 0 (the host routes other shapes to v4), so a half-chunk is
// either entirely inside the field or entirely outside.
FZB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FZB_DEV void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Lane b of compute warp w owns rows a = w*R + r (r < R) of column j0+b and
// stages / flushes only those rows' ring lines, so staging needs no
// cross-lane or cross-warp handshake: a lane only ever reads its own cells.
struct OwnRow {
    long long t;   // flat index of element (i0+a, j0+b, k) for k = 0 (row base)
    bool ok;       // row inside the field
};

template <int R>
FZB_DEV void enc_stage_own(int j, uint32_t* ringl, const float* __restrict__ orig, const OwnRow* rows, int d0,
                           int n2) {
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int k = chunk_of(j, d0 + r) * 8;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int kk = k + 4 * h;
            const bool ok = rows[r].ok && kk >= 0 && kk < n2;   // n2 % 4 == 0: a quad is all-in or all-out
            cp_async16_zfill(ringl + r * 32 * IP + (kk & (KR - 1)), orig + (ok ? rows[r].t + kk : 0), ok ? 16 : 0);
        }
    }
}

template <int R>
struct DecRegs {
    uint2 c[2 * R];
    uint32_t bm[2 * R];
};
template <int R>
FZB_DEV void dec_load_own(int j, DecRegs<R>& D, const uint16_t* __restrict__ codes,
                          const uint32_t* __restrict__ bitmap, const OwnRow* rows, int d0, int n2) {
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int k = chunk_of(j, d0 + r) * 8;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int kk = k + 4 * h;
            const bool ok = rows[r].ok && kk >= 0 && kk < n2;
            const long long t = rows[r].t + kk;
            D.c[2 * r + h] = ok ? __ldg(reinterpret_cast<const uint2*>(codes + t)) : make_uint2(0, 0);
            D.bm[2 * r + h] = ok ? (__ldg(bitmap + (t >> 5)) >> (t & 31)) & 0xFu : 0u;   // t % 4 == 0: one word
        }
    }
}
template <int R>
FZB_DEV void dec_write_own(int j, const DecRegs<R>& D, uint32_t* ringl, const float* recon, const OwnRow* rows,
                           int d0, int n2, uint32_t pad_code) {
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int k = chunk_of(j, d0 + r) * 8;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int kk = k + 4 * h;
            const bool ok = rows[r].ok && kk >= 0 && kk < n2;
            const long long t = rows[r].t + kk;
            const uint2 c = D.c[2 * r + h];
            uint4 w = make_uint4(pad_code, pad_code, pad_code, pad_code);   // code R: exact zeros before k == 0
            if (ok) {
                w = make_uint4(CODE_TAG | (c.x & 0xFFFFu), CODE_TAG | (c.x >> 16), CODE_TAG | (c.y & 0xFFFFu),
                               CODE_TAG | (c.y >> 16));
                const uint32_t bits = D.bm[2 * r + h];
                if (bits) {  // rare: outlier values verbatim (pre-scattered into recon)
                    if (bits & 1u) w.x = __float_as_uint(recon[t]);
                    if (bits & 2u) w.y = __float_as_uint(recon[t + 1]);
                    if (bits & 4u) w.z = __float_as_uint(recon[t + 2]);
                    if (bits & 8u) w.w = __float_as_uint(recon[t + 3]);
                }
            }
            *reinterpret_cast<uint4*>(ringl + r * 32 * IP + (kk & (KR - 1))) = w;
        }
    }
}

// Flush chunk (chunk_of(j, d) - 1) of the lane's rows: complete once group j is done.
template <int R, bool DEC>
FZB_DEV void flush_own(int j, const uint32_t* ringl, uint16_t* __restrict__ codes_out, uint32_t* __restrict__ bitmap,
                       float* recon, const OwnRow* rows, int d0, int n2) {
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int k = (chunk_of(j, d0 + r) - 1) * 8;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int kk = k + 4 * h;
            if (rows[r].ok && kk >= 0 && kk < n2) {
                const long long t = rows[r].t + kk;
                const uint4 w = *reinterpret_cast<const uint4*>(ringl + r * 32 * IP + (kk & (KR - 1)));
                if constexpr (DEC) {
                    *reinterpret_cast<uint4*>(recon + t) = w;
                } else {
                    uint2 c;
                    c.x = (w.x & 0xFFFFu) | (w.y << 16);
                    c.y = (w.z & 0xFFFFu) | (w.w << 16);
                    *reinterpret_cast<uint2*>(codes_out + t) = c;
                    // bit 16 = outlier; t % 4 == 0, so the 4 flags share one bitmap word
                    const uint32_t ob =
                        ((w.x >> 16) & 1u) | ((w.y >> 15) & 2u) | ((w.z >> 14) & 4u) | ((w.w >> 13) & 8u);
                    if (ob) atomicOr(bitmap + (t >> 5), ob << (t & 31));
                }
            }
        }
    }
}

// Poll the faces this tile needs for the steps of group j and re-tag them
// into the shared halo rings (tag = step + 1):
//   HU[t][b]     ghost row i0-1, lane b     <- faceI(A-1, B)  at producer step t + PI
//   HL[t][0]     corner (i0-1, j0-1)        <- faceJ(A-1, B-1) row PI-1, step t + PI + 32
//   HL[t][1 + a] left halo of tile row a    <- faceJ(A, B-1)  row a,     step t + 32
template <int PI>
FZB_DEV void helper_halo(int j, uint64_t* HU, uint64_t* HL, const uint64_t* faceI, const uint64_t* faceJ, int tile,
                         int A, int B, int nB, int S, uint32_t epoch, int lane) {
    constexpr int NE = 32 + PI + 1;
    constexpr int E = NE * G;
    constexpr int EPL = (E + 31) / 32;
    const uint64_t* srcI = A > 0 ? faceI + (size_t)(tile - nB) * S * 32 : nullptr;
    const uint64_t* srcJ = B > 0 ? faceJ + (size_t)(tile - 1) * S * PI : nullptr;
    const uint64_t* srcC = (A > 0 && B > 0) ? faceJ + (size_t)(tile - nB - 1) * S * PI : nullptr;
    uint64_t val[EPL];
    const uint64_t* src[EPL];
    uint64_t* dst[EPL];
    uint32_t pend = 0;
#pragma unroll
    for (int q = 0; q < EPL; q++) {
        const int e = q * 32 + lane;
        const int tt = j * G + e / NE, c = e % NE;
        src[q] = nullptr;
        dst[q] = nullptr;
        val[q] = 0;
        if (e < E && tt < S) {
            if (c < 32) {
                dst[q] = HU + (tt & (HR - 1)) * 32 + c;
                if (srcI && tt + PI < S) src[q] = srcI + (size_t)(tt + PI) * 32 + c;
            } else if (c == 32) {
                dst[q] = HL + (tt & (HR - 1)) * (PI + 1);
                if (srcC && tt + PI + 32 < S) src[q] = srcC + (size_t)(tt + PI + 32) * PI + (PI - 1);
            } else {
                dst[q] = HL + (tt & (HR - 1)) * (PI + 1) + (c - 32);
                if (srcJ && tt + 32 < S) src[q] = srcJ + (size_t)(tt + 32) * PI + (c - 33);
            }
            if (src[q]) {
                val[q] = ld_ll_gpu(src[q]);
                pend |= 1u << q;
            } else {
                st_ll_cta(dst[q], ll_pack(0.f, (uint32_t)(tt + 1)));
            }
        }
    }
    while (true) {
#pragma unroll
        for (int q = 0; q < EPL; q++) {
            if ((pend >> q) & 1u) {
                if ((uint32_t)(val[q] >> 32) == epoch) {
                    const int tt = j * G + (q * 32 + lane) / NE;
                    st_ll_cta(dst[q], (val[q] & 0xFFFFFFFFull) | ((uint64_t)(tt + 1) << 32));
                    pend &= ~(1u << q);
                }
            }
        }
        if (!__any_sync(FULL, pend)) break;
#pragma unroll
        for (int q = 0; q < EPL; q++)
            if ((pend >> q) & 1u) val[q] = ld_ll_gpu(src[q]);
    }
}

constexpr double RINT_MAGIC = 6755399441055744.0;

// Debug timing (build with -DLZ7_TIMING): clock64 stamps of tile 0's compute
// warps at 4 points of every step; read back with fzb_debug_lz_timing.
#ifdef LZ7_TIMING
__device__ long long g_lz_stamp[8][1024][4];
__device__ unsigned long long g_tile_t[1 << 16][4];   // per global tile: claim, first step, end (ns), smid
FZB_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define LZ_STAMP(i)                                                                                    \
    do {                                                                                               \
        const long long c_ = clock64();                                                                \
        if (tile == 0 && b == 0 && s < 1024 && w < 8) g_lz_stamp[w][s][i] = c_;                        \
    } while (0)
#else
#define LZ_STAMP(i) \
    do {            \
    } while (0)
#endif

#ifndef LZ7_UNROLL
#define LZ7_UNROLL 2   // steps unrolled per iteration: the 8-step unroll thrashed the i-cache
#endif
constexpr int kStepUnroll = LZ7_UNROLL;

// Out of line (rare, and keeps the unrolled step body small): the exact
// IEEE-division quantizer; returns the ring word (code | outlier << 16).
__device__ __noinline__ uint32_t quantize_word_slow(float vf, double pred, QParams P, float* rec) {
    bool outl;
    float r;
    const int code = quantize((double)vf, pred, P, r, outl);
    *rec = r;
    return (uint32_t)code | (outl ? 0x10000u : 0u);
}   // 1.5 * 2^52: x + M - M == rint(x) for |x| < 2^51

// The next step's inputs (ghost-row value + lane -1 halos) carry LL tags.
// Halo rings are released per group (hready); the ghost row of warps w > 0
// arrives every step from warp w-1 and is LL-checked.
FZB_DEV bool ghost_ready(bool polled, uint64_t gh, uint32_t want) { return !polled || (uint32_t)(gh >> 32) == want; }
FZB_DEV void wait_ghost(bool polled, uint64_t& gh, uint32_t want, const uint64_t* gsrc) {
    while (!__all_sync(FULL, ghost_ready(polled, gh, want))) gh = ld_ll_cta(gsrc);
}

template <int W, int R, bool DEC>
struct Smem7 {
    static constexpr int PI = W * R;
    static constexpr size_t ring = (size_t)PI * 32 * IP * 4;
    static constexpr size_t hu = (size_t)HR * 32 * 8;
    static constexpr size_t hl = (size_t)HR * (PI + 1) * 8;
    static constexpr size_t gr = (size_t)W * GRD * 32 * 8;   // W-1 ghost rings + warp W-1's scratch
    static constexpr size_t bytes = ring + hu + hl + gr + 128;
};

// ------------------------------------------------------------------ kernel
// CTA = W compute warps (warp w owns tile rows a = w*R + r) + 1 helper warp.
// Warp w's ghost row (a = w*R - 1) arrives as LL pairs every step: from the
// helper (w = 0, row i0-1 of the tile above) or from warp w-1 (GR ring).
template <int W, int R, bool DEC>
__global__ void __launch_bounds__((W + 1) * 32, (W <= 4 ? 3 : 1))
lz7_kernel(const float* __restrict__ orig, const uint16_t* __restrict__ codes_in, uint16_t* __restrict__ codes_out,
           uint32_t* __restrict__ bitmap, float* recon, uint64_t* __restrict__ faceI, uint64_t* __restrict__ faceJ,
           const uint32_t* __restrict__ hdr, uint32_t* __restrict__ ticket, const int* __restrict__ order, Geo6 geo,
           const double* __restrict__ d_eb, int radius) {
    using SM = Smem7<W, R, DEC>;
    constexpr int PI = W * R;
    constexpr int NT = (W + 1) * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(smem_raw);
    uint64_t* HU = reinterpret_cast<uint64_t*>(smem_raw + SM::ring);
    uint64_t* HL = HU + HR * 32;
    uint64_t* GR = HL + HR * (PI + 1);
    uint32_t* flags = reinterpret_cast<uint32_t*>(smem_raw + SM::ring + SM::hu + SM::hl + SM::gr);   // [0] tile, [1] staged
    uint32_t* done = flags + 2;                                      // [w] groups finished by warp w
    uint32_t* hready = done + W;                                     // halo groups published
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    {   // ring: exact zeros (decode: code R) wherever a step before k == 0 looks;
        // halo rings: tag 0 / value 0 == "step -1" (all k < 0)
        const uint32_t pad = DEC ? (CODE_TAG | (uint32_t)radius) : 0u;
        for (int q = tid; q < PI * 32 * IP; q += NT) ring[q] = pad;
        const int nh = (int)((SM::hu + SM::hl + SM::gr) / 8);
        for (int q = tid; q < nh; q += NT) HU[q] = 0;
    }
    if (tid == 0) flags[0] = (uint32_t)order[atomicAdd(ticket, 1u)];
#ifdef LZ7_TIMING
    if (tid == 0 && flags[0] < (1u << 16)) {
        g_tile_t[flags[0]][0] = gtimer();
        unsigned sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        g_tile_t[flags[0]][3] = sm;
    }
#endif
    if (tid < W + 2) flags[1 + tid] = 0;
    __syncthreads();
    // global tile id -> (field, tile): faces are indexed by the global id (the
    // neighbours a tile reads never cross a field), data by the field offset
    const int T = (int)flags[0];
    const int fld = T / geo.nt1, tile = T % geo.nt1;
    orig += (size_t)fld * geo.fstride;
    codes_in += (size_t)fld * geo.fstride;
    codes_out += (size_t)fld * geo.fstride;
    recon += (size_t)fld * geo.fstride;
    bitmap += (size_t)fld * geo.bstride;
    d_eb += fld;
    const int nB = geo.nB, S = geo.S;
    const int A = tile / nB, B = tile % nB;
    const int i0 = A * PI, j0 = B * 32;
    const int NGRP = S / G;
    const uint32_t epoch = hdr[0];

    if (warp == W) {
        // ================= halo warp: polls the faces a group at a time, up to 3 groups ahead =================
        // Group jg's ring slots (steps 8jg-32..) are free once every warp finished group jg-3.
        for (int jg = 0; jg < NGRP; jg++) {
            if (jg >= 3) wait_min(done, W, (uint32_t)(jg - 2));
            helper_halo<PI>(jg, HU, HL, faceI, faceJ, T, A, B, nB, S, epoch, lane);
            __syncwarp();
            if (lane == 0) st_rel_cta(hready, (uint32_t)(jg + 1));
        }
        return;
    }

    // ============================ compute warps ============================
    // One basic block per step and ONE warp-uniform branch: the ghost row of
    // warps w > 0 (written by warp w-1 every step) is loaded at the start of
    // the step that precedes its use and its LL tag is checked at the end,
    // together with the rare near-tie flag of the reciprocal quantizer; halo
    // rings (helper-written) are released per group by `hready`.  Outlier
    // flags ride in bit 16 of the ring word (the stager sets the bitmap).
    const int w = warp, b = lane;
    const QParams P = make_qparams(*d_eb, radius);
    const double R_d = (double)radius;
    // state per row x: 0 = ghost row (w*R - 1), 1..R = rows w*R .. w*R+R-1
    double C1[R + 1], C2[R + 1], L1[R + 1], L2[R + 1];
#pragma unroll
    for (int x = 0; x <= R; x++) C1[x] = C2[x] = L1[x] = L2[x] = 0.0;
    const bool polled = (w > 0);
    const uint64_t* ghost_src = polled ? GR + (size_t)(w - 1) * GRD * 32 + b : HU + b;   // + slot*32
    // warp W-1 has no consumer in the CTA: its ghost stores go to a scratch ring
    uint64_t* ghost_dst = GR + (size_t)(w < W - 1 ? w : W - 1) * GRD * 32 + b;
    const int gmask = polled ? GRD - 1 : HR - 1;   // ghost source ring depth
    const bool pubI = (w == W - 1) && (A < geo.nA - 1);
    uint64_t* fI = faceI + (size_t)T * S * 32 + b;
    const bool pubJ = (B < nB - 1) && (b == 31);
    uint64_t* fJ = faceJ + (size_t)T * S * PI + w * R;
    const bool l0 = (b == 0);
    const uint64_t* hlw = HL + w * R;   // + slot*(PI+1): entries x = 0..R (row w*R-1+x)
    uint32_t* ringl = ring + (w * R * 32 + b) * IP;
    // step s consumes step s-1's ghost value and lane -1 halos (step -1: zeros)
    uint64_t gh = 0;
    float hf[R + 1];
    float upn[R + 1];   // this step's left neighbours, shuffled at the end of the previous step
#pragma unroll
    for (int x = 0; x <= R; x++) hf[x] = upn[x] = 0.f;

    // ---- own-row staging: SD groups in flight (encode: cp.async groups;
    //      decode: one group of loads in registers, stored a group early)
    OwnRow rows[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int i = i0 + w * R + r, jj = j0 + b;
        rows[r].ok = (i < geo.n0) && (jj < geo.n1);
        rows[r].t = rows[r].ok ? ((long long)i * geo.n1 + jj) * geo.n2 : 0;
    }
    const int d0 = w * R + b;
    const uint32_t pad = CODE_TAG | (uint32_t)radius;
    DecRegs<R> D;
    if constexpr (!DEC) {
        for (int q = 0; q < SD; q++) {
            if (q < NGRP) enc_stage_own<R>(q, ringl, orig, rows, d0, geo.n2);
            cp_async_commit();
        }
    } else {
        dec_load_own<R>(0, D, codes_in, bitmap, rows, d0, geo.n2);
        dec_write_own<R>(0, D, ringl, recon, rows, d0, geo.n2, pad);
        if (NGRP > 1) dec_load_own<R>(1, D, codes_in, bitmap, rows, d0, geo.n2);
    }

    for (int g = 0; g < NGRP; g++) {
        if constexpr (!DEC) cp_async_wait_n<SD - 1>();   // this lane's copies of group g landed
        if (ld_acq_cta(hready) < (uint32_t)(g + 1))
            while (ld_acq_cta(hready) < (uint32_t)(g + 1)) __nanosleep(32);
#ifdef LZ7_TIMING
        if (g == 0 && w == 0 && b == 0 && T < (1 << 16)) g_tile_t[T][1] = gtimer();
#endif
        // stay within 15 steps of warp w+1 (the ghost ring holds GRD = 16)
        if (w + 1 < W && ld_acq_cta(done + w + 1) + 1 < (uint32_t)g)
            while (ld_acq_cta(done + w + 1) + 1 < (uint32_t)g) __nanosleep(32);
#pragma unroll kStepUnroll
        for (int st = 0; st < G; st++) {
            const int s = g * G + st;
            const int cs = s & (HR - 1);
            LZ_STAMP(0);
            // ---- next step's inputs: ghost (tag checked at the end) and halos
            const uint32_t want = (uint32_t)(s + 1);
            uint64_t ghn = ld_ll_cta(ghost_src + (s & gmask) * 32);
            float hfn[R + 1];
#pragma unroll
            for (int x = 0; x <= R; x++) hfn[x] = __uint_as_float((uint32_t)ld_ll_cta(hlw + cs * (PI + 1) + x));
            // this step's inputs (encode: v, decode: code word) are independent of the
            // prediction: read them now so their latency hides under the shuffles and
            // the 7-term sum (a pinned asm load: the compiler would sink a plain one)
            const int u = s - OFF - w * R - b;
            uint32_t* cell[R + 1];
            uint32_t raw[R + 1];
#pragma unroll
            for (int x = 1; x <= R; x++) {
                cell[x] = ringl + (x - 1) * 32 * IP + ((u - (x - 1)) & (KR - 1));
                raw[x] = ld_cta_u32(cell[x]);
            }
            LZ_STAMP(1);
            C1[0] = (double)__uint_as_float((uint32_t)gh);
            // ---- left neighbours: lane b-1's previous values (shuffled at the end of the
            //      previous step, off this step's chain); lane 0 <- lane -1 halo
            double Ln[R + 1];
#pragma unroll
            for (int x = 0; x <= R; x++) Ln[x] = (double)(l0 ? hf[x] : upn[x]);
            double pred[R + 1];
#pragma unroll
            for (int x = 1; x <= R; x++) {
                double p = __dadd_rn(C1[x - 1], Ln[x]);   // up + left (up never -0.0)
                p = __dadd_rn(p, C1[x]);                   // + self
                p = __dsub_rn(p, L1[x - 1]);               // - diag
                p = __dsub_rn(p, C2[x - 1]);               // - up(k-1)
                p = __dsub_rn(p, L1[x]);                   // - left(k-1)
                pred[x] = __dadd_rn(p, L2[x - 1]);         // + diag(k-1)
            }
            LZ_STAMP(2);
            double Cn[R + 1];
            float Fn[R + 1];
            uint32_t slow = 0;
            if constexpr (!DEC) {
                uint32_t word[R + 1];
#pragma unroll
                for (int x = 1; x <= R; x++) {
                    const float vf = __uint_as_float(raw[x]) + 0.0f;   // normalised -0 (same quantisation)
                    const double v = (double)vf;
                    const double q = __dmul_rn(__dsub_rn(v, pred[x]), P.inv2eb);
                    const double t = __dadd_rn(q, RINT_MAGIC);
                    const double sd = __dsub_rn(t, RINT_MAGIC);   // rint(q) (|q| >= 2^51 -> outlier anyway)
                    const double fr = fabs(__dsub_rn(q, sd));
                    slow |= (uint32_t)(fr >= 0.4999999990686774) << x;
                    const float rc = __double2float_rn(__dadd_rn(pred[x], __dmul_rn(P.two_eb, sd)));
                    const double rcd = (double)rc;
                    const bool okq = (fabs(sd) < R_d) & (fabs(__dsub_rn(rcd, v)) <= P.eb);
                    const int si = (int)(uint32_t)__double_as_longlong(t);
                    word[x] = okq ? (uint32_t)(si + radius) : ((uint32_t)radius | 0x10000u);
                    Fn[x] = okq ? rc : vf;
                    Cn[x] = okq ? rcd : v;
                }
                if (!P.use_recip) slow = ~1u;
                // ---- the step's one branch: ghost not yet published, or a near-tie
                if (!__all_sync(FULL, (slow == 0) & ghost_ready(polled, ghn, want))) {
#pragma unroll
                    for (int x = 1; x <= R; x++) {
                        if ((slow >> x) & 1u) {
                            // frac(|q|) within ~1e-9 of .5: the exact IEEE-division quantizer decides
                            float rec;
                            word[x] = quantize_word_slow(__uint_as_float(raw[x]) + 0.0f, pred[x], P, &rec);
                            Fn[x] = rec;
                            Cn[x] = (double)rec;
                        }
                    }
                    wait_ghost(polled, ghn, want, ghost_src + (s & gmask) * 32);
                }
#pragma unroll
                for (int x = 1; x <= R; x++) *cell[x] = word[x];
            } else {
#pragma unroll
                for (int x = 1; x <= R; x++) {
                    const uint32_t wv = raw[x];
                    const bool is_code = (wv & 0x7F800000u) == 0x7F800000u;
                    // (code - R) exactly via the 2^52 mantissa trick, no int->double convert
                    const double cm = __dsub_rn(__longlong_as_double(0x4330000000000000ll | (long long)(wv & 0xFFFFu)),
                                                4503599627370496.0 + R_d);
                    const float rc = __double2float_rn(__dadd_rn(pred[x], __dmul_rn(P.two_eb, cm)));   // never -0.0
                    const float ov = __uint_as_float(wv) + 0.0f;   // outlier (verbatim in the output)
                    *cell[x] = is_code ? __float_as_uint(rc) : wv;
                    Fn[x] = is_code ? rc : ov;
                    Cn[x] = (double)Fn[x];
                }
                if (!__all_sync(FULL, ghost_ready(polled, ghn, want))) wait_ghost(polled, ghn, want, ghost_src + (s & gmask) * 32);
            }
            LZ_STAMP(3);
            // ---- the ghost row for warp w+1 first (it waits on it), then the next
            //      step's left neighbours: the shuffles' latency hides under the
            //      face publishes and the history shift
            st_ll_cta(ghost_dst + (s & (GRD - 1)) * 32, ll_pack(Fn[R], (uint32_t)(s + 1)));
            upn[0] = __shfl_up_sync(FULL, __uint_as_float((uint32_t)ghn), 1);
#pragma unroll
            for (int x = 1; x <= R; x++) upn[x] = __shfl_up_sync(FULL, Fn[x], 1);
            // ---- publish the faces (predicated, no branches)
            st_ll_gpu_if(pubI, fI + (size_t)s * 32, ll_pack(Fn[R], epoch));
#pragma unroll
            for (int x = 1; x <= R; x++) st_ll_gpu_if(pubJ, fJ + (size_t)s * PI + (x - 1), ll_pack(Fn[x], epoch));
            // ---- shift the history
#pragma unroll
            for (int x = 0; x <= R; x++) {
                C2[x] = C1[x];
                L2[x] = L1[x];
                L1[x] = Ln[x];
                hf[x] = hfn[x];
            }
#pragma unroll
            for (int x = 1; x <= R; x++) C1[x] = Cn[x];
            gh = ghn;
        }
        // ---- own rows: flush what group g completed, stage group g+SD (decode: g+1 / load g+2)
        flush_own<R, DEC>(g, ringl, codes_out, bitmap, recon, rows, d0, geo.n2);
        if constexpr (!DEC) {
            if (g + SD < NGRP) enc_stage_own<R>(g + SD, ringl, orig, rows, d0, geo.n2);
            cp_async_commit();
        } else {
            if (g + 1 < NGRP) dec_write_own<R>(g + 1, D, ringl, recon, rows, d0, geo.n2, pad);
            if (g + 2 < NGRP) dec_load_own<R>(g + 2, D, codes_in, bitmap, rows, d0, geo.n2);
        }
        __syncwarp();
        if (b == 0) st_rel_cta(done + w, (uint32_t)(g + 1));
    }
    // the last chunk of every row completes with the last group
    flush_own<R, DEC>(NGRP, ringl, codes_out, bitmap, recon, rows, d0, geo.n2);
#ifdef LZ7_TIMING
    if (w == W - 1 && b == 0 && T < (1 << 16)) g_tile_t[T][2] = gtimer();
#endif
}

// Header words: see WS_HDR in lorenzo.cu.
__global__ void lz7_prep_kernel(uint32_t* hdr, unsigned long long sig) {
    hdr[0] += 1u;   // launch epoch: face tags of earlier launches never match
    hdr[1] = 0u;    // ticket
    unsigned long long* cur = reinterpret_cast<unsigned long long*>(hdr + 2);
    hdr[4] = (*cur != sig) ? 1u : 0u;
    *cur = sig;
}
// Zero the faces when the layout changed (then every tag is 0 < epoch).
__global__ void lz7_clear_kernel(const uint32_t* __restrict__ hdr, uint4* __restrict__ p, size_t n16) {
    if (!hdr[4]) return;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n16; q += (size_t)gridDim.x * blockDim.x)
        p[q] = make_uint4(0, 0, 0, 0);
}
inline unsigned long long layout_sig(int pi, int n0, int n1, int n2, int nf) {
    unsigned long long h = 1469598103934665603ull;
    const long long v[5] = {pi, n0, n1, n2, nf};
    for (int q = 0; q < 5; q++) h = (h ^ (unsigned long long)v[q]) * 1099511628211ull;
    return h | 1ull;
}

template <int PI>
struct WS7 {
    size_t ntile, S, K, off_order, off_counts, off_fI, off_fJ, total;
    WS7(int n0, int n1, int n2, int nf = 1) {
        const size_t nA = (n0 + PI - 1) / PI, nB = (n1 + 31) / 32;
        ntile = nA * nB * (size_t)nf;   // all fields of a batch
        // last element: k = n2-1 at a + b = PI + 30; whole groups (the compute warps run them)
        S = ((size_t)n2 + PI + 30 + OFF + G - 1) / G * G;
        K = (size_t)(PI + 8) * (nA - 1) + (size_t)(32 + 8) * (nB - 1) + 1;
        auto al = [](size_t x) { return (x + 255) / 256 * 256; };
        off_order = 256;
        off_counts = off_order + al(ntile * 4);
        off_fI = off_counts + al(K * 4);
        off_fJ = off_fI + al(ntile * S * 32 * 8);
        total = off_fJ + al(ntile * S * PI * 8);
    }
};

template <int W, int R, bool DEC>
int launch7(const float* orig, const uint16_t* codes_in, uint16_t* codes_out, uint32_t* bitmap, float* recon, int n0,
            int n1, int n2, const double* d_eb, int radius, void* ws, size_t ws_bytes, cudaStream_t st, int nf = 1,
            long long fstride = 0, long long bstride = 0) {
    constexpr int PI = W * R;
    WS7<PI> L(n0, n1, n2, nf);
    if (ws_bytes < L.total) return FZB_E_WORKSPACE;
    Geo6 g;
    g.n0 = n0; g.n1 = n1; g.n2 = n2;
    g.nA = (n0 + PI - 1) / PI;
    g.nB = (n1 + 31) / 32;
    g.S = (int)L.S;
    g.vec = (n2 % 4 == 0) ? 1 : 0;
    g.nt1 = g.nA * g.nB;
    g.fstride = fstride;
    g.bstride = bstride;
    unsigned char* w = static_cast<unsigned char*>(ws);
    uint32_t* hdr = reinterpret_cast<uint32_t*>(w);
    int* order = reinterpret_cast<int*>(w + L.off_order);
    int* counts = reinterpret_cast<int*>(w + L.off_counts);
    uint64_t* faceI = reinterpret_cast<uint64_t*>(w + L.off_fI);
    uint64_t* faceJ = reinterpret_cast<uint64_t*>(w + L.off_fJ);
    lz7_prep_kernel<<<1, 1, 0, st>>>(hdr, layout_sig(PI, n0, n1, n2, nf));
    lz7_clear_kernel<<<kNumSMs * 4, 256, 0, st>>>(hdr, reinterpret_cast<uint4*>(faceI), (L.total - L.off_fI) / 16);
    tile_order_kernel<<<1, 1024, 0, st>>>(g.nA, g.nB, PI + 8, 32 + 8, counts, order, nf);
    const size_t smem = Smem7<W, R, DEC>::bytes;
    auto kfn = lz7_kernel<W, R, DEC>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<(unsigned)L.ntile, (W + 1) * 32, smem, st>>>(orig, codes_in, codes_out, bitmap, recon, faceI, faceJ, hdr,
                                                      hdr + 1, order, g, d_eb, radius);
    return fzb_check_launch();
}

}  // namespace v6
