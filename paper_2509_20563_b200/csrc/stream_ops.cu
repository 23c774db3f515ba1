// stream_ops.cu -- HBM-streaming kernels: min/max + bound, fill, histogram,
// outlier compaction/scatter.
//
//  * min/max (pipeline.py:360-361, core.py:162-163): one pass of 128-bit
//    loads instead of the reference's four numpy scans; partials per CTA,
//    then a one-CTA final reduce.  eb_abs is computed on the device.
//  * histogram (encode.py:79-111): privatised shared-memory bins with
//    __match_any_sync warp aggregation (quant codes are sharply peaked);
//    top-k is bitwise identical to exact by contract, so one kernel serves
//    both methods.
//  * outliers (predict.py:212-214): the predictor kernels set one bit per
//    outlier; compaction is a popcount/scan pass in index order, so the
//    list comes out sorted exactly like np.nonzero.
#include "common.cuh"

namespace {

constexpr int MM_THREADS = 256;
constexpr int MM_BLOCKS = kNumSMs * 4;

__global__ void __launch_bounds__(MM_THREADS) minmax_partial_kernel(const float* __restrict__ x, uint64_t n,
                                                                    float* __restrict__ part, uint32_t* __restrict__ status) {
    float lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    const uint64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + 3 * stride < n4; q += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldcs(x4 + q + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            lo = fminf(lo, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
            hi = fmaxf(hi, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            bad |= !(isfinite(v[u].x) && isfinite(v[u].y) && isfinite(v[u].z) && isfinite(v[u].w));
        }
    }
    for (; q < n4; q += stride) {
        const float4 v = __ldcs(x4 + q);
        lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
        hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    if (blockIdx.x == 0) {
        for (uint64_t t = n4 * 4 + threadIdx.x; t < n; t += blockDim.x) {
            const float v = x[t];
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
            bad |= !isfinite(v);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ float sl[32], sh[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sl[w] = lo; sh[w] = hi; }
    if (__syncthreads_or(bad) && threadIdx.x == 0) set_err(status, FZB_ERR_NONFINITE);
    if (w == 0) {
        lo = lane < (int)(blockDim.x >> 5) ? sl[lane] : INFINITY;
        hi = lane < (int)(blockDim.x >> 5) ? sh[lane] : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            part[2 * blockIdx.x] = lo;
            part[2 * blockIdx.x + 1] = hi;
        }
    }
}

__global__ void minmax_final_kernel(const float* __restrict__ part, int np, float* __restrict__ lohi) {
    float lo = INFINITY, hi = -INFINITY;
    for (int q = threadIdx.x; q < np; q += blockDim.x) {
        lo = fminf(lo, part[2 * q]);
        hi = fmaxf(hi, part[2 * q + 1]);
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

__global__ void resolve_kernel(const float* __restrict__ lohi, int mode, double mag, double* __restrict__ eb) {
    // core.py:167: float(spec.magnitude) * (hi - lo), Python floats (f64)
    *eb = mode ? __dmul_rn(mag, __dsub_rn((double)lohi[1], (double)lohi[0])) : mag;
}

__global__ void fill_u16_kernel(uint16_t* __restrict__ d, uint64_t n, uint16_t v) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n8 = n / 8;
    uint4 pat;
    const uint32_t w = (uint32_t)v | ((uint32_t)v << 16);
    pat.x = pat.y = pat.z = pat.w = w;
    uint4* d8 = reinterpret_cast<uint4*>(d);
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n8; q += stride) d8[q] = pat;
    for (uint64_t t = n8 * 8 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) d[t] = v;
}

// ----------------------------------------------------------------- histogram
constexpr int HIST_THREADS = 256;
constexpr uint32_t HIST_SMEM_BINS = 16384;

// Privatised histogram (encode.py:79-84): each warp owns a sub-histogram in
// shared memory and every thread merges runs of equal codes before it
// touches a bin, so the heavily skewed code distribution of smooth fields
// (most codes are R) costs a handful of atomics instead of one per code.
constexpr int HIST_UNROLL = 4;
__global__ void __launch_bounds__(HIST_THREADS) hist_smem_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                                 uint32_t nbins, int nsub,
                                                                 unsigned long long* __restrict__ out,
                                                                 uint32_t* __restrict__ status,
                                                                 uint8_t* __restrict__ notr) {
    extern __shared__ uint32_t sb[];
    // notr (optional): notr[c] = 1 iff 4096-code chunk c holds a code != R = nbins / 2
    const uint32_t rr = (nbins / 2) * 0x00010001u;
    // (a warp-aggregated store -- one ballot per uint4 -- was slower: 131 ->
    // 148 us on C4; the flag costs ~15 us there and saves the ~100 us count read)
    auto flag = [&](const uint4& v, uint64_t q8) {
        if (((v.x ^ rr) | (v.y ^ rr) | (v.z ^ rr) | (v.w ^ rr)) != 0u && notr) notr[q8 >> 9] = 1;
    };
    for (uint32_t q = threadIdx.x; q < nbins * (uint32_t)nsub; q += blockDim.x) sb[q] = 0;
    __syncthreads();
    uint32_t* mine = sb + (size_t)((threadIdx.x >> 5) % nsub) * nbins;
    uint32_t cur = 0xFFFFFFFFu, cnt = 0;
    bool bad = false;
    auto put = [&](uint32_t c) {
        if (c == cur) {
            cnt++;
        } else {
            if (cnt) {
                if (cur < nbins) atomicAdd(mine + cur, cnt);
                else bad = true;
            }
            cur = c;
            cnt = 1;
        }
    };
    const uint64_t n8 = n / 8;
    const uint4* c8 = reinterpret_cast<const uint4*>(codes);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // HIST_UNROLL independent 16-byte loads in flight per thread (the run
    // merging below is a serial chain; the loads must not wait on it)
    uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + (HIST_UNROLL - 1) * stride < n8; q += HIST_UNROLL * stride) {
        uint4 v[HIST_UNROLL];
#pragma unroll
        for (int u = 0; u < HIST_UNROLL; u++) v[u] = __ldcs(c8 + q + u * stride);
#pragma unroll
        for (int u = 0; u < HIST_UNROLL; u++) {
            flag(v[u], q + u * stride);
            put(v[u].x & 0xFFFFu); put(v[u].x >> 16);
            put(v[u].y & 0xFFFFu); put(v[u].y >> 16);
            put(v[u].z & 0xFFFFu); put(v[u].z >> 16);
            put(v[u].w & 0xFFFFu); put(v[u].w >> 16);
        }
    }
    for (; q < n8; q += stride) {
        const uint4 v = __ldcs(c8 + q);
        flag(v, q);
        put(v.x & 0xFFFFu); put(v.x >> 16);
        put(v.y & 0xFFFFu); put(v.y >> 16);
        put(v.z & 0xFFFFu); put(v.z >> 16);
        put(v.w & 0xFFFFu); put(v.w >> 16);
    }
    if (blockIdx.x == 0)
        for (uint64_t t = n8 * 8 + threadIdx.x; t < n; t += blockDim.x) {
            const uint32_t c = codes[t];
            if (notr && c != nbins / 2) notr[t >> 12] = 1;
            put(c);
        }
    if (cnt) {
        if (cur < nbins) atomicAdd(mine + cur, cnt);
        else bad = true;
    }
    if (bad) set_err(status, FZB_ERR_CODE_RANGE);
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nbins; q += blockDim.x) {
        uint32_t t = 0;
        for (int w = 0; w < nsub; w++) t += sb[(size_t)w * nbins + q];
        if (t) atomicAdd(out + q, (unsigned long long)t);
    }
}

// Histogram with the chunk flags as INPUT (fzb_histogram_flagged): a full
// 4096-code chunk whose flag is clear holds only R = nbins / 2 and is
// counted without being read; one warp per flagged chunk, 16 coalesced
// 16-byte loads per lane, run-merged into per-warp shared sub-histograms.
__global__ void __launch_bounds__(HIST_THREADS) hist_flagged_kernel(const uint16_t* __restrict__ codes, uint64_t n,
                                                                    uint32_t nbins, int nsub,
                                                                    const uint8_t* __restrict__ notr,
                                                                    unsigned long long* __restrict__ out,
                                                                    uint32_t* __restrict__ status) {
    extern __shared__ uint32_t sb[];
    for (uint32_t q = threadIdx.x; q < nbins * (uint32_t)nsub; q += blockDim.x) sb[q] = 0;
    __syncthreads();
    uint32_t* mine = sb + (size_t)((threadIdx.x >> 5) % nsub) * nbins;
    const uint32_t R = nbins / 2;
    const int lane = threadIdx.x & 31;
    uint32_t cur = 0xFFFFFFFFu, cnt = 0;
    unsigned long long nr = 0;   // codes of unread (all-R) chunks
    bool bad = false;
    auto put = [&](uint32_t c) {
        if (c == cur) {
            cnt++;
        } else {
            if (cnt) {
                if (cur < nbins) atomicAdd(mine + cur, cnt);
                else bad = true;
            }
            cur = c;
            cnt = 1;
        }
    };
    const uint64_t nc = (n + 4095) / 4096, nfull = n / 4096;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    // the warp reads the flags of its next 32 chunks at once (one per lane)
    // and visits only the flagged ones
    for (uint64_t c0 = warp; c0 < nc; c0 += 32 * nw) {
        const uint64_t mc = c0 + (uint64_t)lane * nw;
        const bool skip = mc < nfull && !notr[mc];
        if (skip) nr += 4096;
        unsigned todo = __ballot_sync(0xffffffffu, mc < nc && !skip);
        while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint64_t c = c0 + (uint64_t)j * nw;
        const uint64_t b0 = c * 4096;
        if (c < nfull) {
            const uint4* c8 = reinterpret_cast<const uint4*>(codes + b0);
            uint4 v[16];
#pragma unroll
            for (int u = 0; u < 16; u++) v[u] = __ldcs(c8 + u * 32 + lane);
#pragma unroll
            for (int u = 0; u < 16; u++) {
                put(v[u].x & 0xFFFFu); put(v[u].x >> 16);
                put(v[u].y & 0xFFFFu); put(v[u].y >> 16);
                put(v[u].z & 0xFFFFu); put(v[u].z >> 16);
                put(v[u].w & 0xFFFFu); put(v[u].w >> 16);
            }
        } else {
            for (uint64_t t = b0 + lane; t < n; t += 32) put(codes[t]);
        }
        }
    }
    if (cnt) {
        if (cur < nbins) atomicAdd(mine + cur, cnt);
        else bad = true;
    }
    if (bad) set_err(status, FZB_ERR_CODE_RANGE);
#pragma unroll
    for (int o = 16; o; o >>= 1) nr += __shfl_xor_sync(0xffffffffu, nr, o);   // one atomic per warp
    if (lane == 0 && nr) atomicAdd(out + R, nr);
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nbins; q += blockDim.x) {
        uint32_t t = 0;
        for (int w = 0; w < nsub; w++) t += sb[(size_t)w * nbins + q];
        if (t) atomicAdd(out + q, (unsigned long long)t);
    }
}

__global__ void hist_global_kernel(const uint16_t* __restrict__ codes, uint64_t n, uint32_t nbins,
                                   unsigned long long* __restrict__ out, uint32_t* __restrict__ status,
                                   uint8_t* __restrict__ notr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint32_t c = codes[t];
        if (notr && c != nbins / 2) notr[t >> 12] = 1;
        if (c >= nbins) set_err(status, FZB_ERR_CODE_RANGE);
        else atomicAdd(out + c, 1ull);
    }
}

// ------------------------------------------------------------------ outliers
constexpr int OC_WORDS = 2048;  // bitmap words per CTA (65536 elements)
constexpr int OC_THREADS = 256;

__global__ void __launch_bounds__(OC_THREADS) outlier_count_kernel(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                                   uint32_t* __restrict__ counts) {
    __shared__ uint32_t tmp[33];
    const uint64_t base = (uint64_t)blockIdx.x * OC_WORDS;
    uint32_t c = 0;
    if (base + OC_WORDS <= nwords && !(reinterpret_cast<uintptr_t>(bm) & 15)) {
        const uint4* b4 = reinterpret_cast<const uint4*>(bm + base);
        for (int e = threadIdx.x; e < OC_WORDS / 4; e += blockDim.x) {
            const uint4 v = __ldg(b4 + e);
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
    } else {
        for (int e = threadIdx.x; e < OC_WORDS; e += blockDim.x)
            if (base + e < nwords) c += __popc(bm[base + e]);
    }
    uint32_t tot;
    block_exclusive_scan(c, tmp, &tot);
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void scan_u32_to_u64_kernel(const uint32_t* __restrict__ cnt, uint64_t m,
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

__global__ void __launch_bounds__(OC_THREADS) outlier_write_kernel(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                                   const float* __restrict__ x,
                                                                   const uint32_t* __restrict__ counts,
                                                                   const unsigned long long* __restrict__ offs,
                                                                   unsigned long long* __restrict__ idx,
                                                                   float* __restrict__ vals) {
    __shared__ uint32_t tmp[33];
    if (counts[blockIdx.x] == 0) return;   // outliers are rare: most CTAs have none
    const uint64_t base = (uint64_t)blockIdx.x * OC_WORDS;
    unsigned long long o = offs[blockIdx.x];
    for (int e0 = 0; e0 < OC_WORDS; e0 += blockDim.x) {
        const uint64_t wq = base + e0 + threadIdx.x;
        uint32_t w = wq < nwords ? bm[wq] : 0u;
        uint32_t tot;
        uint32_t p = block_exclusive_scan(__popc(w), tmp, &tot);
        while (w) {
            const int bit = __ffs(w) - 1;
            w &= w - 1;
            const unsigned long long t = wq * 32ull + bit;
            idx[o + p] = t;
            vals[o + p] = x[t];
            p++;
        }
        o += tot;
    }
}

__global__ void outlier_scatter_kernel(const unsigned long long* __restrict__ idx, const float* __restrict__ vals,
                                       uint64_t k, uint64_t n, const uint16_t* __restrict__ codes, int radius,
                                       float* __restrict__ recon, uint32_t* __restrict__ bm,
                                       uint32_t* __restrict__ status) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += stride) {
        const unsigned long long t = idx[q];
        if (t >= n) {  // pipeline.py:410-411 (u64, so "< 0" cannot happen)
            set_err(status, FZB_ERR_OUTLIER_RANGE);
            continue;
        }
        if (q > 0 && idx[q - 1] >= t) set_err(status, FZB_ERR_OUTLIER_ORDER);  // core.py:212-213
        if (codes != nullptr && codes[t] != radius) set_err(status, FZB_ERR_OUTLIER_CODE);  // core.py:214-215
        recon[t] = vals[q];
        atomicOr(bm + (t >> 5), 1u << (t & 31));
    }
}

// core.py:214-215 on its own: the sentinel check of the outlier list against
// decoded codes, for DAGs where the scatter runs beside the codec decode.
__global__ void outlier_check_kernel(const unsigned long long* __restrict__ idx, uint64_t k, uint64_t n,
                                     const uint16_t* __restrict__ codes, int radius, uint32_t* __restrict__ status) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += stride) {
        const unsigned long long t = idx[q];
        if (t < n && codes[t] != radius) set_err(status, FZB_ERR_OUTLIER_CODE);
    }
}

}  // namespace

// ---------------------------------------------------------------- quality
// fzpipe metrics.quality (metrics.py:49-75) on device, bit-identical: the
// MSE is np.mean(d * d) with d = f64(orig) - f64(recon), and numpy sums a
// contiguous f64 array pairwise (halve at multiples of 8 down to blocks of
// <= 128, each block summed by 8 strided accumulators then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail in order).  The host
// builds that split tree (it depends on n only); this kernel sums its
// leaves, one warp per leaf, and reduces max|d|, min/max(orig) exactly.
constexpr int QL_WARPS = 8;

FZB_DEV unsigned long long f32_key(float v) {   // order-preserving f32 -> u32
    const uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(QL_WARPS * 32) quality_leaf_kernel(const float* __restrict__ orig,
                                                                     const float* __restrict__ recon,
                                                                     const uint64_t* __restrict__ leaf_off,
                                                                     const uint16_t* __restrict__ leaf_len,
                                                                     uint64_t nleaves, double* __restrict__ leaf_sum,
                                                                     unsigned long long* __restrict__ red) {
    __shared__ double sq[QL_WARPS][128];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint64_t leaf = (uint64_t)blockIdx.x * QL_WARPS + wl;
    double maxe = 0.0;
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    if (leaf < nleaves) {
        const uint64_t off = leaf_off[leaf];
        const int m = leaf_len[leaf];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = q * 32 + lane;
            if (i < m) {
                const float o = orig[off + i];
                const double d = __dsub_rn((double)o, (double)recon[off + i]);
                sq[wl][i] = __dmul_rn(d, d);
                maxe = fmax(maxe, fabs(d));
                const uint32_t k = (uint32_t)f32_key(o);
                kmin = min(kmin, k);
                kmax = max(kmax, k);
            }
        }
        __syncwarp();
        double res = 0.0;
        if (m < 8) {
            if (lane == 0)
                for (int i = 0; i < m; i++) res = __dadd_rn(res, sq[wl][i]);
        } else {
            double r = 0.0;
            const int full = m - (m & 7);
            if (lane < 8) {
                r = sq[wl][lane];
                for (int i = 8 + lane; i < full; i += 8) r = __dadd_rn(r, sq[wl][i]);
            }
            const double r1 = __shfl_down_sync(0xffffffffu, r, 1);
            const double p01 = __dadd_rn(r, r1);                              // lanes 0,2,4,6: r_j + r_j+1
            const double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
            const double q03 = __dadd_rn(p01, p23);                           // lanes 0,4
            const double q47 = __shfl_down_sync(0xffffffffu, q03, 4);
            if (lane == 0) {
                res = __dadd_rn(q03, q47);
                for (int i = full; i < m; i++) res = __dadd_rn(res, sq[wl][i]);
            }
        }
        if (lane == 0) leaf_sum[leaf] = res;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        maxe = fmax(maxe, __shfl_xor_sync(0xffffffffu, maxe, o));
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0 && leaf < nleaves) {
        atomicMax(red + 0, (unsigned long long)__double_as_longlong(maxe));   // >= 0: bit order == value order
        atomicMin(red + 1, (unsigned long long)kmin);
        atomicMax(red + 2, (unsigned long long)kmax);
    }
}

extern "C" {

FZB_API int fzb_abi_version(void) { return 1; }

// Timing inside CUDA graphs: an event recorded during stream capture with
// cudaEventRecordExternal becomes an event-record node, so a replayed graph
// still reports per-kernel times (cudaEventElapsedTime after the replay).
FZB_API int fzb_event_create(void** event) { return (int)cudaEventCreate(reinterpret_cast<cudaEvent_t*>(event)); }
FZB_API int fzb_event_destroy(void* event) { return (int)cudaEventDestroy((cudaEvent_t)event); }
FZB_API int fzb_event_record(void* event, void* stream, int external) {
    return (int)cudaEventRecordWithFlags((cudaEvent_t)event, (cudaStream_t)stream,
                                         external ? cudaEventRecordExternal : cudaEventRecordDefault);
}
FZB_API int fzb_event_elapsed_ms(void* start, void* stop, float* ms) {
    return (int)cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop);
}

FZB_API size_t fzb_minmax_workspace_bytes(uint64_t) { return (size_t)MM_BLOCKS * 2 * sizeof(float); }

FZB_API int fzb_minmax_f32(const float* d_in, uint64_t n, float* d_lohi, void* d_ws, size_t ws_bytes,
                           uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return FZB_E_ARG;
    if (ws_bytes < fzb_minmax_workspace_bytes(n)) return FZB_E_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(d_in) & 15) return FZB_E_ARG;
    float* part = static_cast<float*>(d_ws);
    minmax_partial_kernel<<<MM_BLOCKS, MM_THREADS, 0, st>>>(d_in, n, part, d_status);
    minmax_final_kernel<<<1, 1024, 0, st>>>(part, MM_BLOCKS, d_lohi);
    return fzb_check_launch();
}

FZB_API int fzb_resolve_bound(const float* d_lohi, int eb_mode, double magnitude, double* d_eb, void* stream) {
    resolve_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_lohi, eb_mode, magnitude, d_eb);
    return fzb_check_launch();
}

FZB_API int fzb_fill_u16(uint16_t* d_dst, uint64_t n, uint16_t value, void* stream) {
    if (n == 0) return 0;
    if (reinterpret_cast<uintptr_t>(d_dst) & 15) return FZB_E_ARG;
    fill_u16_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(d_dst, n, value);
    return fzb_check_launch();
}

FZB_API int fzb_histogram(const uint16_t* d_codes, uint64_t n, uint32_t nbins, uint64_t* d_bins, uint32_t* d_status,
                          void* stream) {
    return fzb_histogram_chunks(d_codes, n, nbins, d_bins, nullptr, d_status, stream);
}

FZB_API int fzb_histogram_flagged(const uint16_t* d_codes, uint64_t n, uint32_t nbins, uint64_t* d_bins,
                                  const uint8_t* d_notr, uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (nbins == 0 || !d_notr) return FZB_E_ARG;
    if (nbins > HIST_SMEM_BINS || (reinterpret_cast<uintptr_t>(d_codes) & 15))   // read everything
        return fzb_histogram(d_codes, n, nbins, d_bins, d_status, stream);
    cudaMemsetAsync(d_bins, 0, (size_t)nbins * 8, st);
    if (n == 0) return fzb_check_launch();
    int nsub = HIST_THREADS / 32;
    while (nsub > 1 && (size_t)nsub * nbins * 4 > 64 * 1024) nsub >>= 1;
    const size_t smem = (size_t)nbins * 4 * nsub;
    cudaFuncSetAttribute(hist_flagged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    hist_flagged_kernel<<<kNumSMs * 4, HIST_THREADS, smem, st>>>(d_codes, n, nbins, nsub, d_notr,
                                                                reinterpret_cast<unsigned long long*>(d_bins),
                                                                d_status);
    return fzb_check_launch();
}

FZB_API int fzb_histogram_chunks(const uint16_t* d_codes, uint64_t n, uint32_t nbins, uint64_t* d_bins,
                                 uint8_t* d_notr, uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (nbins == 0) return FZB_E_ARG;
    cudaMemsetAsync(d_bins, 0, (size_t)nbins * 8, st);
    if (d_notr) cudaMemsetAsync(d_notr, 0, (size_t)((n + FZB_HF_CHUNK - 1) / FZB_HF_CHUNK), st);
    if (n == 0) return fzb_check_launch();
    unsigned long long* out = reinterpret_cast<unsigned long long*>(d_bins);
    if (nbins <= HIST_SMEM_BINS && !(reinterpret_cast<uintptr_t>(d_codes) & 15)) {
        // one sub-histogram per warp while they fit in 64 KB
        int nsub = HIST_THREADS / 32;
        while (nsub > 1 && (size_t)nsub * nbins * 4 > 64 * 1024) nsub >>= 1;
        const size_t smem = (size_t)nbins * 4 * nsub;
        cudaFuncSetAttribute(hist_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        uint64_t blocks = (n / 8 + HIST_THREADS - 1) / HIST_THREADS;
        const uint64_t cap = (uint64_t)kNumSMs * 4;
        if (blocks > cap) blocks = cap;
        if (blocks == 0) blocks = 1;
        hist_smem_kernel<<<(unsigned)blocks, HIST_THREADS, smem, st>>>(d_codes, n, nbins, nsub, out, d_status, d_notr);
    } else {
        hist_global_kernel<<<kNumSMs * 8, 256, 0, st>>>(d_codes, n, nbins, out, d_status, d_notr);
    }
    return fzb_check_launch();
}

FZB_API size_t fzb_outlier_workspace_bytes(uint64_t n) {
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t nblk = (nwords + OC_WORDS - 1) / OC_WORDS;
    return 256 + ((nblk * 4 + 255) / 256) * 256 + nblk * 8 + 256;
}

FZB_API int fzb_outlier_compact(const uint32_t* d_bitmap, uint64_t n, const float* d_in, uint64_t* d_idx,
                                float* d_vals, uint64_t* d_count, void* d_ws, size_t ws_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (ws_bytes < fzb_outlier_workspace_bytes(n)) return FZB_E_WORKSPACE;
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t nblk = (nwords + OC_WORDS - 1) / OC_WORDS;
    if (nblk == 0) {
        cudaMemsetAsync(d_count, 0, 8, st);
        return fzb_check_launch();
    }
    unsigned char* w = static_cast<unsigned char*>(d_ws);
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + 256);
    unsigned long long* offs = reinterpret_cast<unsigned long long*>(w + 256 + ((nblk * 4 + 255) / 256) * 256);
    outlier_count_kernel<<<(unsigned)nblk, OC_THREADS, 0, st>>>(d_bitmap, nwords, counts);
    scan_u32_to_u64_kernel<<<1, 1024, 0, st>>>(counts, nblk, offs, reinterpret_cast<unsigned long long*>(d_count));
    outlier_write_kernel<<<(unsigned)nblk, OC_THREADS, 0, st>>>(d_bitmap, nwords, d_in, counts, offs,
                                                               reinterpret_cast<unsigned long long*>(d_idx), d_vals);
    return fzb_check_launch();
}

FZB_API int fzb_outlier_scatter(const uint64_t* d_idx, const float* d_vals, uint64_t k, uint64_t n,
                                const uint16_t* d_codes, uint32_t radius, float* d_recon, uint32_t* d_bitmap,
                                uint32_t* d_status, void* stream) {
    if (k == 0) return 0;
    unsigned blocks = (unsigned)((k + 255) / 256);
    if (blocks > (unsigned)kNumSMs * 8) blocks = kNumSMs * 8;
    outlier_scatter_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const unsigned long long*>(d_idx), d_vals, k, n, d_codes, (int)radius, d_recon, d_bitmap,
        d_status);
    return fzb_check_launch();
}

FZB_API int fzb_outlier_check(const uint64_t* d_idx, uint64_t k, uint64_t n, const uint16_t* d_codes,
                              uint32_t radius, uint32_t* d_status, void* stream) {
    if (k == 0) return 0;
    unsigned blocks = (unsigned)((k + 255) / 256);
    if (blocks > (unsigned)kNumSMs * 8) blocks = kNumSMs * 8;
    outlier_check_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const unsigned long long*>(d_idx), k, n, d_codes, (int)radius, d_status);
    return fzb_check_launch();
}

// Leaves of numpy's pairwise-sum tree (offsets, lengths <= 128, in order) of
// d*d, plus red[0] = max|d| (f64 bits), red[1] / red[2] = ordered keys of
// min / max(orig).  red must be initialised to {0, ~0, 0} by the caller.
FZB_API int fzb_quality_leaves(const float* d_orig, const float* d_recon, const uint64_t* d_leaf_off,
                               const uint16_t* d_leaf_len, uint64_t nleaves, double* d_leaf_sum,
                               unsigned long long* d_red, void* stream) {
    if (nleaves == 0) return 0;
    const uint64_t blocks = (nleaves + QL_WARPS - 1) / QL_WARPS;
    quality_leaf_kernel<<<(unsigned)blocks, QL_WARPS * 32, 0, (cudaStream_t)stream>>>(
        d_orig, d_recon, d_leaf_off, d_leaf_len, nleaves, d_leaf_sum, d_red);
    return fzb_check_launch();
}

}  // extern "C"
