// bitshuffle.cu -- FZ-GPU bitshuffle + zero-word dictionary elision (sm_100a).
//
// Reference: fzpipe encode.py:324-391.  Codes are u16, zero-padded to
// 256-code blocks; each block is 16 bit planes of 8 LE u32 words, word
// blk*128 + p*8 + w holding bit p of codes[blk*256 + 32w + j] at bit j --
// which is exactly __ballot_sync over a warp holding those 32 codes.  The
// bitmap has one bit per word (LSB-first == LE u32 word blk*4 + i/32, bit
// i%32), the payload keeps the nonzero words in index order.
//
// Encode: pass 1 = one warp per block, 128 ballots, bitmap words via 4 more
// ballots, per-CTA nonzero counts; scan; pass 2 = recompute the ballots and
// scatter the nonzero words at compacted offsets (coalesced).
// Decode: per-CTA popcounts, scan, then one warp per block gathers its
// nonzero words and inverts the transpose with 128 shuffles.
#include "common.cuh"

namespace {

constexpr int BS_THREADS = 256;
constexpr int BS_WARPS = BS_THREADS / 32;
constexpr int BS_BPW = 8;                         // blocks per warp
constexpr int BS_BPC = BS_WARPS * BS_BPW;         // blocks per CTA (64 -> 16384 codes)

// all 128 words of block `blk`; lane l keeps words l, l+32, l+64, l+96
FZB_DEV void block_words(const uint16_t* __restrict__ codes, uint64_t n, uint64_t blk, uint32_t mine[4]) {
    const int lane = threadIdx.x & 31;
    uint32_t c[8];
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const uint64_t t = blk * 256 + 32 * w + lane;
        c[w] = t < n ? (uint32_t)__ldg(codes + t) : 0u;
    }
#pragma unroll
    for (int s = 0; s < 4; s++) mine[s] = 0;
#pragma unroll
    for (int p = 0; p < 16; p++)
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const int i = p * 8 + w;
            const uint32_t x = __ballot_sync(0xffffffffu, (c[w] >> p) & 1u);
            if (lane == (i & 31)) mine[i >> 5] = x;
        }
}

__global__ void __launch_bounds__(BS_THREADS) bs_enc_count_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                                  uint64_t nblocks, uint32_t* __restrict__ bitmap,
                                                                  uint32_t* __restrict__ counts) {
    __shared__ uint32_t wc[BS_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cnt = 0;
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        uint32_t mine[4];
        block_words(codes, n, blk, mine);
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const uint32_t bm = __ballot_sync(0xffffffffu, mine[s] != 0u);
            if (lane == s) bitmap[blk * 4 + s] = bm;
            cnt += __popc(bm);
        }
    }
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < BS_WARPS; w++) t += wc[w];
        counts[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(BS_THREADS) bs_enc_write_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                                  uint64_t nblocks, const uint32_t* __restrict__ bitmap,
                                                                  const unsigned long long* __restrict__ offs,
                                                                  uint32_t* __restrict__ payload) {
    __shared__ uint32_t wc[BS_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp counts from the stored bitmap
    uint32_t cnt = 0;
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        if (lane < 4) cnt += __popc(bitmap[blk * 4 + lane]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    unsigned long long o = offs[blockIdx.x];
    for (int w = 0; w < warp; w++) o += wc[w];
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        uint32_t mine[4];
        block_words(codes, n, blk, mine);
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const uint32_t bm = __ballot_sync(0xffffffffu, mine[s] != 0u);
            if (mine[s]) payload[o + __popc(bm & lanemask_lt())] = mine[s];
            o += __popc(bm);
        }
    }
}

// Single-pass encoder: ballots once, per-CTA nonzero-word count published
// through decoupled look-back (CTA order from an atomic ticket, so every
// predecessor is resident or done), then compacted payload writes.
// State word per CTA: bits 62-63 = flag (1 aggregate, 2 inclusive prefix),
// bits 0-61 = value.
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 62) - 1;

FZB_DEV unsigned long long ld_volatile64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(BS_THREADS) bs_enc_fused_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                                  uint64_t nblocks, uint32_t* __restrict__ bitmap,
                                                                  uint32_t* __restrict__ payload,
                                                                  unsigned long long* __restrict__ state,
                                                                  uint32_t* __restrict__ ticket,
                                                                  unsigned long long* __restrict__ nwords) {
    __shared__ uint32_t wc[BS_WARPS];
    __shared__ unsigned long long s_excl;
    __shared__ uint32_t s_cta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_cta = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t cta = s_cta;
    uint32_t mine[BS_BPW][4];
    uint32_t bms[BS_BPW][4];
    uint32_t cnt = 0;
#pragma unroll
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)cta * BS_BPC + warp * BS_BPW + q;
        if (blk < nblocks) {
            block_words(codes, n, blk, mine[q]);
        } else {
#pragma unroll
            for (int s = 0; s < 4; s++) mine[q][s] = 0;
        }
#pragma unroll
        for (int s = 0; s < 4; s++) {
            bms[q][s] = __ballot_sync(0xffffffffu, mine[q][s] != 0u);
            cnt += __popc(bms[q][s]);
        }
        if (blk < nblocks && lane < 4) bitmap[blk * 4 + lane] = bms[q][0] * (lane == 0) + bms[q][1] * (lane == 1) +
                                                                 bms[q][2] * (lane == 2) + bms[q][3] * (lane == 3);
    }
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
        uint32_t agg = 0;
        for (int w = 0; w < BS_WARPS; w++) agg += wc[w];
        unsigned long long excl = 0;
        if (cta == 0) {
            if (lane == 0) {
                __threadfence();
                atomicExch(state, LB_PRE | agg);
            }
        } else {
            if (lane == 0) {
                __threadfence();
                atomicExch(state + cta, LB_AGG | agg);
            }
            // parallel look-back over 32 predecessors at a time
            long long base = (long long)cta - 1;
            while (true) {
                const long long p = base - lane;
                unsigned long long v = LB_PRE;  // lanes before CTA 0 act as prefix 0
                if (p >= 0) {
                    do { v = ld_volatile64(state + p); } while ((v >> 62) == 0);
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                const int stop = pre ? __ffs(pre) - 1 : 32;
                unsigned long long add = (lane <= stop && p >= 0) ? (v & LB_VAL) : 0ull;
#pragma unroll
                for (int o = 16; o; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
                excl += add;
                if (pre) break;
                base -= 32;
            }
            if (lane == 0) {
                __threadfence();
                atomicExch(state + cta, LB_PRE | (excl + agg));
            }
        }
        if (lane == 0) {
            s_excl = excl;
            if ((uint64_t)(cta + 1) * BS_BPC >= nblocks) *nwords = excl + agg;
        }
    }
    __syncthreads();
    unsigned long long o = s_excl;
    for (int w = 0; w < warp; w++) o += wc[w];
#pragma unroll
    for (int q = 0; q < BS_BPW; q++) {
#pragma unroll
        for (int s = 0; s < 4; s++) {
            if (mine[q][s]) payload[o + __popc(bms[q][s] & lanemask_lt())] = mine[q][s];
            o += __popc(bms[q][s]);
        }
    }
}

// Decoder: each warp stages its block's 128 words in shared memory, every
// lane then extracts its own bit from each word (broadcast reads).
__global__ void __launch_bounds__(BS_THREADS) bs_dec2_kernel(const uint32_t* __restrict__ bitmap,
                                                             const uint32_t* __restrict__ payload, uint64_t payload_words,
                                                             uint64_t n, uint64_t nblocks, uint32_t radius,
                                                             const unsigned long long* __restrict__ offs,
                                                             uint16_t* __restrict__ codes, uint32_t* __restrict__ status) {
    __shared__ uint32_t wc[BS_WARPS];
    __shared__ __align__(16) uint32_t sw[BS_WARPS][128];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cnt = 0;
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        if (lane < 4) cnt += __popc(bitmap[blk * 4 + lane]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    unsigned long long o = offs[blockIdx.x];
    for (int w = 0; w < warp; w++) o += wc[w];
    bool pad_bad = false, range_bad = false;
    uint32_t* W = sw[warp];
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const uint32_t bm = bitmap[blk * 4 + s];
            uint32_t x = 0u;
            if ((bm >> lane) & 1u) {
                const unsigned long long pos = o + __popc(bm & lanemask_lt());
                if (pos < payload_words) x = payload[pos];
            }
            W[s * 32 + lane] = x;
            o += __popc(bm);
        }
        __syncwarp();
        uint32_t c[8];
#pragma unroll
        for (int w = 0; w < 8; w++) c[w] = 0;
#pragma unroll
        for (int p = 0; p < 16; p++) {
            const uint4 lo = *reinterpret_cast<const uint4*>(W + p * 8);
            const uint4 hi = *reinterpret_cast<const uint4*>(W + p * 8 + 4);
            const uint32_t x[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int w = 0; w < 8; w++) c[w] |= ((x[w] >> lane) & 1u) << p;
        }
        __syncwarp();
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const uint64_t t = blk * 256 + 32 * w + lane;
            if (t < n) {
                codes[t] = (uint16_t)c[w];
                range_bad |= c[w] >= 2 * radius;
            } else {
                pad_bad |= c[w] != 0;
            }
        }
    }
    if (pad_bad) set_err(status, FZB_ERR_BS_PAD);
    if (range_bad) set_err(status, FZB_ERR_BS_RANGE);
}

__global__ void scan_counts_u64_kernel(const uint32_t* __restrict__ cnt, uint64_t m,
                                       unsigned long long* __restrict__ offs, unsigned long long* __restrict__ tot) {
    __shared__ unsigned long long tmp[33];
    unsigned long long carry = 0;
    for (uint64_t b0 = 0; b0 < m; b0 += blockDim.x) {
        const uint64_t q = b0 + threadIdx.x;
        const unsigned long long x = q < m ? cnt[q] : 0ull;
        unsigned long long t;
        const unsigned long long p = block_exclusive_scan64(x, tmp, &t);
        if (q < m) offs[q] = carry + p;
        carry += t;
    }
    if (threadIdx.x == 0) *tot = carry;
}

__global__ void __launch_bounds__(BS_THREADS) bs_dec_count_kernel(const uint32_t* __restrict__ bitmap, uint64_t nblocks,
                                                                  uint32_t* __restrict__ counts) {
    __shared__ uint32_t tmp[33];
    uint32_t c = 0;
    const uint64_t w0 = (uint64_t)blockIdx.x * BS_BPC * 4;
    for (int e = threadIdx.x; e < BS_BPC * 4; e += blockDim.x)
        if (w0 + e < nblocks * 4) c += __popc(bitmap[w0 + e]);
    uint32_t tot;
    block_exclusive_scan(c, tmp, &tot);
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void bs_check_total_kernel(const unsigned long long* __restrict__ tot, uint64_t payload_words,
                                      uint32_t* __restrict__ status) {
    if (*tot != payload_words) set_err(status, FZB_ERR_BS_MISMATCH);
}

__global__ void __launch_bounds__(BS_THREADS) bs_dec_kernel(const uint32_t* __restrict__ bitmap,
                                                            const uint32_t* __restrict__ payload, uint64_t payload_words,
                                                            uint64_t n, uint64_t nblocks, uint32_t radius,
                                                            const unsigned long long* __restrict__ offs,
                                                            uint16_t* __restrict__ codes, uint32_t* __restrict__ status) {
    __shared__ uint32_t wc[BS_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cnt = 0;
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        if (lane < 4) cnt += __popc(bitmap[blk * 4 + lane]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    unsigned long long o = offs[blockIdx.x];
    for (int w = 0; w < warp; w++) o += wc[w];
    bool pad_bad = false, range_bad = false;
    for (int q = 0; q < BS_BPW; q++) {
        const uint64_t blk = (uint64_t)blockIdx.x * BS_BPC + warp * BS_BPW + q;
        if (blk >= nblocks) break;
        uint32_t mine[4];
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const uint32_t bm = bitmap[blk * 4 + s];
            mine[s] = 0u;
            if ((bm >> lane) & 1u) {
                const unsigned long long pos = o + __popc(bm & lanemask_lt());
                if (pos < payload_words) mine[s] = payload[pos];
            }
            o += __popc(bm);
        }
        uint32_t c[8];
#pragma unroll
        for (int w = 0; w < 8; w++) c[w] = 0;
#pragma unroll
        for (int p = 0; p < 16; p++)
#pragma unroll
            for (int w = 0; w < 8; w++) {
                const int i = p * 8 + w;
                const uint32_t x = __shfl_sync(0xffffffffu, mine[i >> 5], i & 31);
                c[w] |= ((x >> lane) & 1u) << p;
            }
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const uint64_t t = blk * 256 + 32 * w + lane;
            if (t < n) {
                codes[t] = (uint16_t)c[w];
                range_bad |= c[w] >= 2 * radius;
            } else {
                pad_bad |= c[w] != 0;
            }
        }
    }
    if (pad_bad) set_err(status, FZB_ERR_BS_PAD);
    if (range_bad) set_err(status, FZB_ERR_BS_RANGE);
}

uint64_t nblk_of(uint64_t n) { return (n + 255) / 256; }
uint64_t ncta_of(uint64_t n) { return (nblk_of(n) + BS_BPC - 1) / BS_BPC; }

}  // namespace

extern "C" {

FZB_API size_t fzb_bitshuffle_workspace_bytes(uint64_t n) {
    const uint64_t c = ncta_of(n);
    return 512 + ((c * 4 + 255) / 256) * 256 + c * 8 + 256;
}

FZB_API int fzb_bitshuffle_encode(const uint16_t* d_codes, uint64_t n, uint8_t* d_bitmap, uint32_t* d_payload,
                                  uint64_t* d_nwords, void* d_ws, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ws_bytes < fzb_bitshuffle_workspace_bytes(n)) return FZB_E_WORKSPACE;
    const uint64_t nb = nblk_of(n), nc = ncta_of(n);
    if (nb == 0) {
        cudaMemsetAsync(d_nwords, 0, 8, st);
        return fzb_check_launch();
    }
    unsigned char* w = static_cast<unsigned char*>(d_ws);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(w);
    unsigned long long* state = reinterpret_cast<unsigned long long*>(w + 256);
    cudaMemsetAsync(w, 0, 256 + nc * 8, st);
    bs_enc_fused_kernel<<<(unsigned)nc, BS_THREADS, 0, st>>>(d_codes, n, nb, reinterpret_cast<uint32_t*>(d_bitmap),
                                                            d_payload, state, ticket,
                                                            reinterpret_cast<unsigned long long*>(d_nwords));
    return fzb_check_launch();
}

// Host side has already checked bitmap length and payload % 4 (encode.py:362-371).
FZB_API int fzb_bitshuffle_decode(const uint8_t* d_bitmap, const uint32_t* d_payload, uint64_t payload_words,
                                  uint64_t n, uint32_t radius, uint16_t* d_codes, void* d_ws, size_t ws_bytes,
                                  uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (ws_bytes < fzb_bitshuffle_workspace_bytes(n)) return FZB_E_WORKSPACE;
    const uint64_t nb = nblk_of(n), nc = ncta_of(n);
    if (nb == 0) return 0;
    unsigned char* w = static_cast<unsigned char*>(d_ws);
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(w);
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + 256);
    unsigned long long* offs = reinterpret_cast<unsigned long long*>(w + 256 + ((nc * 4 + 255) / 256) * 256);
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(d_bitmap);
    bs_dec_count_kernel<<<(unsigned)nc, BS_THREADS, 0, st>>>(bm, nb, counts);
    scan_counts_u64_kernel<<<1, 1024, 0, st>>>(counts, nc, offs, tot);
    bs_check_total_kernel<<<1, 1, 0, st>>>(tot, payload_words, d_status);
    bs_dec2_kernel<<<(unsigned)nc, BS_THREADS, 0, st>>>(bm, d_payload, payload_words, n, nb, radius, offs, d_codes,
                                                        d_status);
    return fzb_check_launch();
}

}  // extern "C"
