// bitshuffle.cu -- FZ-GPU bitshuffle + zero-word dictionary elision (sm_100a).
//
// Reference: fzpipe encode.py:324-391.  Codes are u16, zero-padded to
// 256-code blocks; each block is 16 bit planes of 8 LE u32 words, word
// blk*128 + p*8 + w holding bit p of codes[blk*256 + 32w + j] at bit j.  The
// bitmap has one bit per word (LSB-first == LE u32 word blk*4 + i/32, bit
// i%32), the payload keeps the nonzero words in index order.
//
// One warp owns a block at a time; lane l = 4w + i holds codes 8l..8l+7
// (one 16-byte load) and ends up owning the four words with index
// 32i + 8c + w (c = 0..3), i.e. planes p = 4i + c of the 32-code group w.
// The bit matrix is moved with register arithmetic instead of 128 ballots:
//   (1) two 8x8 bit transposes (64-bit masked-XOR network) turn the lane's
//       8 codes into 16 plane bytes e_p;
//   (2) word (p, w) is byte e_p of the four lanes of group w: a 4-lane
//       exchange (3 xor-shuffles) plus a 4x4 byte transpose (PRMT).
// A word is nonzero iff bit p of the OR of its 32 codes is set, so block
// word counts, the bitmap and every word's payload rank come from 16-bit
// OR reductions -- cheap enough to publish a CTA's aggregate for the
// decoupled look-back *before* the transposes, which then hide the
// look-back latency.  The decoder runs the same network backwards.
#include "common.cuh"
#include "scan.cuh"
#include "lookback.cuh"

namespace {

constexpr int BS_THREADS = 256;
constexpr int BS_WARPS = BS_THREADS / 32;
constexpr int BS_BPW = 4;                         // blocks per warp
constexpr int BS_BPC = BS_WARPS * BS_BPW;         // blocks per CTA (32 -> 8192 codes)

using fzlb::LB_AGG;
using fzlb::LB_PRE;
using fzlb::lookback;

FZB_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// 8x8 bit transpose of the 64-bit word (hi:lo): bit 8j+k <-> bit 8k+j.
FZB_DEV void t8x8(uint32_t& lo, uint32_t& hi) {
    uint32_t t;
    t = (lo ^ (lo >> 7)) & 0x00AA00AAu; lo ^= t ^ (t << 7);
    t = (hi ^ (hi >> 7)) & 0x00AA00AAu; hi ^= t ^ (t << 7);
    t = (lo ^ (lo >> 14)) & 0x0000CCCCu; lo ^= t ^ (t << 14);
    t = (hi ^ (hi >> 14)) & 0x0000CCCCu; hi ^= t ^ (t << 14);
    t = (lo ^ (hi << 4)) & 0xF0F0F0F0u; lo ^= t; hi ^= t >> 4;
}

// 8 codes (LE u16 pairs in r.x..r.w) -> plane bytes: E[k] holds e_{4k..4k+3},
// e_p bit j = bit p of code j.  Self-inverse up to the packing (see below).
FZB_DEV void codes_to_planes(const uint4 r, uint32_t E[4]) {
    uint32_t lo0 = prmt(r.x, r.y, 0x6420), lo1 = prmt(r.z, r.w, 0x6420);   // low bytes of codes 0..7
    uint32_t hi0 = prmt(r.x, r.y, 0x7531), hi1 = prmt(r.z, r.w, 0x7531);   // high bytes
    t8x8(lo0, lo1);
    t8x8(hi0, hi1);
    E[0] = lo0; E[1] = lo1; E[2] = hi0; E[3] = hi1;
}
FZB_DEV uint4 planes_to_codes(const uint32_t E[4]) {
    uint32_t lo0 = E[0], lo1 = E[1], hi0 = E[2], hi1 = E[3];
    t8x8(lo0, lo1);
    t8x8(hi0, hi1);
    uint4 r;
    r.x = prmt(lo0, hi0, 0x5140);
    r.y = prmt(lo0, hi0, 0x7362);
    r.z = prmt(lo1, hi1, 0x5140);
    r.w = prmt(lo1, hi1, 0x7362);
    return r;
}

FZB_DEV uint32_t sel4(const uint32_t E[4], int k) {
    const uint32_t a = (k & 1) ? E[1] : E[0], b = (k & 1) ? E[3] : E[2];
    return (k & 2) ? b : a;
}

// Lane (w, i): plane bytes E (own codes) -> its 4 words W[c] = word (4i+c, w).
// A[x] = E_i of lane i^x; V_c = byte c of A[0..3]; word_c = V_c with byte
// position x moved to x^i.
FZB_DEV void planes_to_words(const uint32_t E[4], int i, uint32_t xsel, uint32_t W[4]) {
    uint32_t A[4];
    A[0] = sel4(E, i);
#pragma unroll
    for (int x = 1; x < 4; x++) A[x] = __shfl_xor_sync(0xffffffffu, sel4(E, i ^ x), x);
    const uint32_t t0 = prmt(A[0], A[1], 0x5140), t1 = prmt(A[2], A[3], 0x5140);   // bytes 0,1 interleaved
    const uint32_t t2 = prmt(A[0], A[1], 0x7362), t3 = prmt(A[2], A[3], 0x7362);   // bytes 2,3
    W[0] = prmt(prmt(t0, t1, 0x5410), 0, xsel);
    W[1] = prmt(prmt(t0, t1, 0x7632), 0, xsel);
    W[2] = prmt(prmt(t2, t3, 0x5410), 0, xsel);
    W[3] = prmt(prmt(t2, t3, 0x7632), 0, xsel);
}
FZB_DEV void words_to_planes(const uint32_t W[4], int i, uint32_t xsel, uint32_t E[4]) {
    // undo the x^i byte move, then the 4x4 byte transpose gives A[x]
    const uint32_t v0 = prmt(W[0], 0, xsel), v1 = prmt(W[1], 0, xsel);
    const uint32_t v2 = prmt(W[2], 0, xsel), v3 = prmt(W[3], 0, xsel);
    const uint32_t u0 = prmt(v0, v1, 0x5140), u1 = prmt(v2, v3, 0x5140);
    const uint32_t u2 = prmt(v0, v1, 0x7362), u3 = prmt(v2, v3, 0x7362);
    uint32_t A[4];
    A[0] = prmt(u0, u1, 0x5410);
    A[1] = prmt(u0, u1, 0x7632);
    A[2] = prmt(u2, u3, 0x5410);
    A[3] = prmt(u2, u3, 0x7632);
    // A[x] = E_i of lane i^x  ->  E_k of this lane comes back from lane i^k's A[i^k]
    uint32_t R[4];
    R[0] = A[0];
#pragma unroll
    for (int x = 1; x < 4; x++) R[x] = __shfl_xor_sync(0xffffffffu, A[x], x);   // R[x] = E_{i^x} (own)
#pragma unroll
    for (int k = 0; k < 4; k++) E[k] = sel4(R, k ^ i);
}

// 16-bit OR of the 32 codes of this lane's group w (bit p set <=> word (p, w) nonzero)
FZB_DEV uint32_t group_or(const uint4 r) {
    uint32_t o = r.x | r.y | r.z | r.w;
    o = (o | (o >> 16)) & 0xFFFFu;
    o |= __shfl_xor_sync(0xffffffffu, o, 1);
    o |= __shfl_xor_sync(0xffffffffu, o, 2);
    return o;
}

// Bitmap word i of the block (bits 8c + w <-> plane 4i + c of group w), for the
// calling lane's i; every lane of the warp gets all four in BM[0..3].
FZB_DEV void block_bitmap(uint32_t gor, int w, int i, uint32_t BM[4]) {
    uint32_t mine = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) mine |= ((gor >> (4 * i + c)) & 1u) << (8 * c + w);
    mine |= __shfl_xor_sync(0xffffffffu, mine, 4);
    mine |= __shfl_xor_sync(0xffffffffu, mine, 8);
    mine |= __shfl_xor_sync(0xffffffffu, mine, 16);
#pragma unroll
    for (int k = 0; k < 4; k++) BM[k] = __shfl_sync(0xffffffffu, mine, k);
}

// Predicated read-only load (no branch around it): 0 when !p.
FZB_DEV uint32_t ldg_if(bool p, const uint32_t* ptr) {
    uint32_t v;
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.global.nc.u32 %0, [%1]; }"
                 : "=r"(v)
                 : "l"(ptr), "r"((int)p));
    return v;
}

FZB_DEV uint4 load_codes(const uint16_t* __restrict__ codes, uint64_t n, uint64_t blk, int lane) {
    const uint64_t t0 = blk * 256 + 8 * lane;
    if (t0 + 8 <= n) return __ldg(reinterpret_cast<const uint4*>(codes + t0));
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; j++) c[j] = (t0 + j < n) ? (uint32_t)__ldg(codes + t0 + j) : 0u;
    return make_uint4(c[0] | (c[1] << 16), c[2] | (c[3] << 16), c[4] | (c[5] << 16), c[6] | (c[7] << 16));
}


// Persistent variant: each CTA claims chunks of BS_BPC blocks by ticket (so
// look-back predecessors are always claimed earlier) and issues the next
// chunk's loads before the current chunk's transposes, look-back and payload
// stores, keeping HBM reads in flight across the whole CTA lifetime.
__global__ void __launch_bounds__(BS_THREADS) bs_enc4_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                             uint64_t nblocks, uint32_t nchunks,
                                                             uint32_t* __restrict__ bitmap,
                                                             uint32_t* __restrict__ payload,
                                                             unsigned long long* __restrict__ state,
                                                             uint32_t* __restrict__ ticket,
                                                             unsigned long long* __restrict__ nwords) {
    __shared__ uint32_t s_off[BS_BPC];
    __shared__ unsigned long long s_agg, s_excl;
    __shared__ uint32_t s_cta[2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = lane >> 2, gi = lane & 3;
    const uint32_t xsel = (uint32_t)(gi | ((1 ^ gi) << 4) | ((2 ^ gi) << 8) | ((3 ^ gi) << 12));
    if (threadIdx.x == 0) s_cta[0] = atomicAdd(ticket, 1u);
    __syncthreads();
    uint32_t cta = s_cta[0];
    uint4 r[BS_BPW];
    if (cta < nchunks) {
        const uint64_t blk0 = (uint64_t)cta * BS_BPC + warp * BS_BPW;
#pragma unroll
        for (int q = 0; q < BS_BPW; q++)
            r[q] = (blk0 + q < nblocks) ? load_codes(codes, n, blk0 + q, lane) : make_uint4(0, 0, 0, 0);
    }
    for (int it = 0; cta < nchunks; it++) {
        const uint64_t blk0 = (uint64_t)cta * BS_BPC + warp * BS_BPW;
        uint32_t gor[BS_BPW];
#pragma unroll
        for (int q = 0; q < BS_BPW; q++) {
            gor[q] = group_or(r[q]);
            uint32_t c = __popc(gor[q]);
#pragma unroll
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0) s_off[warp * BS_BPW + q] = c >> 2;
        }
        __syncthreads();   // (A) s_off complete; previous iteration fully done with s_excl / s_cta
        if (warp == 0) {
            const uint32_t a = s_off[lane];
            uint32_t incl = a;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            s_off[lane] = incl - a;
            if (lane == 31) {
                s_agg = incl;
                if (cta != 0) {
                    __threadfence();
                    atomicExch(state + cta, LB_AGG | (unsigned long long)incl);
                }
                s_cta[(it + 1) & 1] = atomicAdd(ticket, 1u);   // next chunk
            }
        }
        uint32_t Wd[BS_BPW][4];
#pragma unroll
        for (int q = 0; q < BS_BPW; q++) {
            uint32_t E[4];
            codes_to_planes(r[q], E);
            planes_to_words(E, gi, xsel, Wd[q]);
        }
        __syncthreads();   // (B) s_off prefix, s_agg, next ticket visible
        const uint32_t nxt = s_cta[(it + 1) & 1];
        if (nxt < nchunks) {   // next chunk's loads go out before the look-back and the stores
            const uint64_t nb0 = (uint64_t)nxt * BS_BPC + warp * BS_BPW;
#pragma unroll
            for (int q = 0; q < BS_BPW; q++)
                r[q] = (nb0 + q < nblocks) ? load_codes(codes, n, nb0 + q, lane) : make_uint4(0, 0, 0, 0);
        }
        if (warp == 0) {
            const unsigned long long agg = s_agg;
            const unsigned long long excl = lookback(cta, agg, state);
            if (lane == 0) {
                s_excl = excl;
                if (cta == nchunks - 1) *nwords = excl + agg;
            }
        }
        __syncthreads();   // (C) s_excl visible
#pragma unroll
        for (int q = 0; q < BS_BPW; q++) {
            const uint64_t blk = blk0 + q;
            if (blk >= nblocks) break;
            uint32_t BM[4];
            block_bitmap(gor[q], gw, gi, BM);
            if (lane < 4) bitmap[blk * 4 + lane] = sel4(BM, lane);
            const unsigned long long base = s_excl + s_off[warp * BS_BPW + q];
            uint32_t before = 0;
#pragma unroll
            for (int k = 0; k < 4; k++) before += (k < gi) ? __popc(BM[k]) : 0u;
            const uint32_t bmi = sel4(BM, gi);
#pragma unroll
            for (int c = 0; c < 4; c++) {
                if ((gor[q] >> (4 * gi + c)) & 1u) {
                    const uint32_t rank = before + __popc(bmi & ((1u << (8 * c + gw)) - 1u));
                    payload[base + rank] = Wd[q][c];
                }
            }
        }
        cta = nxt;
    }
}

// Per-chunk word counts of the decoder (bitmap popcounts): one warp per
// chunk of BS_BPC blocks (128 bitmap words, one uint4 per lane).
__global__ void __launch_bounds__(256) bs_dec_count2_kernel(const uint32_t* __restrict__ bitmap, uint64_t nblocks,
                                                            uint64_t nchunks, uint32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const uint64_t c = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (c >= nchunks) return;
    const uint64_t blk = c * BS_BPC + lane;   // BS_BPC == 32: one block (4 words) per lane
    uint32_t v = 0;
    if (blk < nblocks) {
        const uint4 bm = __ldg(reinterpret_cast<const uint4*>(bitmap) + blk);
        v = __popc(bm.x) + __popc(bm.y) + __popc(bm.z) + __popc(bm.w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) counts[c] = v;
}

__global__ void bs_check_kernel(const unsigned long long* __restrict__ tot, uint64_t payload_words,
                                uint32_t* __restrict__ status) {
    if (*tot != payload_words) set_err(status, FZB_ERR_BS_MISMATCH);   // encode.py:372-375
}

__global__ void __launch_bounds__(BS_THREADS) bs_dec3_kernel(const uint32_t* __restrict__ bitmap,
                                                             const uint32_t* __restrict__ payload,
                                                             uint64_t payload_words, uint64_t n, uint64_t nblocks,
                                                             uint32_t radius, const unsigned long long* __restrict__ offs,
                                                             uint16_t* __restrict__ codes, uint32_t* __restrict__ status) {
    __shared__ uint32_t s_off[BS_BPC];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = lane >> 2, gi = lane & 3;
    const uint32_t xsel = (uint32_t)(gi | ((1 ^ gi) << 4) | ((2 ^ gi) << 8) | ((3 ^ gi) << 12));
    const uint64_t cblk = (uint64_t)blockIdx.x * BS_BPC;
    if (warp == 0) {
        uint32_t a = 0;
        if (cblk + lane < nblocks) {
            const uint4 bm = __ldg(reinterpret_cast<const uint4*>(bitmap) + cblk + lane);
            a = __popc(bm.x) + __popc(bm.y) + __popc(bm.z) + __popc(bm.w);
        }
        uint32_t incl = a;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        s_off[lane] = incl - a;
    }
    __syncthreads();
    const unsigned long long cbase = offs[blockIdx.x];
    const uint32_t two_r = 2u * radius;
    bool pad_bad = false, range_bad = false;
    // phase 1: every block's payload loads in flight at once (branch-free:
    // predicated loads at 32-bit offsets from the block's payload base)
    const int lg = 31 - __clz(two_r);   // planes >= lg nonzero <=> some code may be >= 2^lg
    uint32_t W[BS_BPW][4];
    uint32_t high = 0;   // bitmap bits of planes >= lg (range check needed)
#pragma unroll
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = cblk + warp * BS_BPW + q;
        const bool inb = blk < nblocks;
        const uint4 bmv = inb ? __ldg(reinterpret_cast<const uint4*>(bitmap) + blk) : make_uint4(0, 0, 0, 0);
        const uint32_t BM[4] = {bmv.x, bmv.y, bmv.z, bmv.w};
        const unsigned long long base = cbase + s_off[warp * BS_BPW + q];
        const uint32_t* pb = payload + base;
        const long long room = (long long)payload_words - (long long)base;   // words left from base
        uint32_t before = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) before += (k < gi) ? __popc(BM[k]) : 0u;
        const uint32_t bmi = sel4(BM, gi);
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t bit = 8 * c + gw;
            const uint32_t rank = before + __popc(bmi & ((1u << bit) - 1u));
            W[q][c] = ldg_if(((bmi >> bit) & 1u) && (long long)rank < room, pb + rank);
            high |= (4 * gi + c >= lg) ? ((bmi >> bit) & 1u) : 0u;
        }
    }
    // no nonzero word in planes >= lg: every code < 2^lg <= 2R, no range check
    const bool check_range = __any_sync(0xffffffffu, high != 0);
    // phase 2: transposes and 16-byte code stores
#pragma unroll
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = cblk + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        uint32_t E[4];
        words_to_planes(W[q], gi, xsel, E);
        const uint4 rc = planes_to_codes(E);
        const uint64_t t0 = blk * 256 + 8 * lane;
        const uint32_t c8[8] = {rc.x & 0xFFFFu, rc.x >> 16, rc.y & 0xFFFFu, rc.y >> 16,
                                rc.z & 0xFFFFu, rc.z >> 16, rc.w & 0xFFFFu, rc.w >> 16};
        if (t0 + 8 <= n) {
            *reinterpret_cast<uint4*>(codes + t0) = rc;
            if (check_range) {
#pragma unroll
                for (int j = 0; j < 8; j++) range_bad |= c8[j] >= two_r;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (t0 + j < n) {
                    codes[t0 + j] = (uint16_t)c8[j];
                    range_bad |= c8[j] >= two_r;
                } else {
                    pad_bad |= c8[j] != 0;   // encode.py:386-387
                }
            }
        }
    }
    if (pad_bad) set_err(status, FZB_ERR_BS_PAD);
    if (range_bad) set_err(status, FZB_ERR_BS_RANGE);   // encode.py:389-390
}

uint64_t nblk_of(uint64_t n) { return (n + 255) / 256; }
uint64_t ncta_of(uint64_t n) { return (nblk_of(n) + BS_BPC - 1) / BS_BPC; }

}  // namespace

extern "C" {

FZB_API size_t fzb_bitshuffle_workspace_bytes(uint64_t n) {
    const uint64_t c = ncta_of(n);
    return 512 + ((c * 4 + 255) / 256) * 256 + ((c * 8 + 255) / 256) * 256 + fzscan::ws_bytes(c) + 512;
}

// Reference: encode.py:324-353.  d_codes needs 16-byte alignment.
FZB_API int fzb_bitshuffle_encode(const uint16_t* d_codes, uint64_t n, uint8_t* d_bitmap, uint32_t* d_payload,
                                  uint64_t* d_nwords, void* d_ws, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ws_bytes < fzb_bitshuffle_workspace_bytes(n)) return FZB_E_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(d_codes) % 16 || reinterpret_cast<uintptr_t>(d_bitmap) % 16) return FZB_E_ARG;
    const uint64_t nb = nblk_of(n), nc = ncta_of(n);
    if (nb == 0) {
        cudaMemsetAsync(d_nwords, 0, 8, st);
        return fzb_check_launch();
    }
    unsigned char* w = static_cast<unsigned char*>(d_ws);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(w);
    unsigned long long* state = reinterpret_cast<unsigned long long*>(w + 256);
    cudaMemsetAsync(w, 0, 256 + nc * 8, st);
    static int grid_cap_dev[64] = {0};   // resident CTAs of the persistent encoder, per device
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid_cap = grid_cap_dev[dev & 63];
    if (!grid_cap) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bs_enc4_kernel, BS_THREADS, 0);
        grid_cap = sms * (per > 0 ? per : 1);
    }
    {
        const unsigned grid = (unsigned)(nc < (uint64_t)grid_cap ? nc : (uint64_t)grid_cap);
        bs_enc4_kernel<<<grid, BS_THREADS, 0, st>>>(d_codes, n, nb, (uint32_t)nc, reinterpret_cast<uint32_t*>(d_bitmap),
                                                    d_payload, state, ticket,
                                                    reinterpret_cast<unsigned long long*>(d_nwords));
    }
    return fzb_check_launch();
}

// Reference: encode.py:356-391.  The host side has already checked bitmap
// length and payload % 4 (encode.py:362-371).
FZB_API int fzb_bitshuffle_decode(const uint8_t* d_bitmap, const uint32_t* d_payload, uint64_t payload_words,
                                  uint64_t n, uint32_t radius, uint16_t* d_codes, void* d_ws, size_t ws_bytes,
                                  uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (ws_bytes < fzb_bitshuffle_workspace_bytes(n)) return FZB_E_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(d_codes) % 16 || reinterpret_cast<uintptr_t>(d_bitmap) % 16) return FZB_E_ARG;
    const uint64_t nb = nblk_of(n), nc = ncta_of(n);
    if (nb == 0) return 0;
    unsigned char* w = static_cast<unsigned char*>(d_ws);
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(w);
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + 256);
    unsigned long long* offs = reinterpret_cast<unsigned long long*>(w + 256 + ((nc * 4 + 255) / 256) * 256);
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(d_bitmap);
    void* scan_ws = w + 256 + ((nc * 4 + 255) / 256) * 256 + ((nc * 8 + 255) / 256) * 256;
    bs_dec_count2_kernel<<<(unsigned)((nc + 7) / 8), 256, 0, st>>>(bm, nb, nc, counts);
    fzscan::exclusive(counts, nc, offs, tot, scan_ws, st);
    bs_check_kernel<<<1, 1, 0, st>>>(tot, payload_words, d_status);
    bs_dec3_kernel<<<(unsigned)nc, BS_THREADS, 0, st>>>(bm, d_payload, payload_words, n, nb, radius, offs, d_codes,
                                                       d_status);
    return fzb_check_launch();
}

}  // extern "C"
