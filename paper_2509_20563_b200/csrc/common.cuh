// common.cuh -- shared device helpers for the FZModules B200 kernels.
//
// Arithmetic contract (reference predict.py:70-90):
// every predictor operation is an IEEE f64 op with round-to-nearest and NO
// fused multiply-add, so results are bit-identical to the numba reference.
// We build with -fmad=false and also spell the ops with _rn intrinsics.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fzb200.h"

#define FZB_DEV __device__ __forceinline__

// Device-side error bits (OR-ed into a status word; mapped to FZError
// classes by the Python shim, see paper_2509_20563_b200/_lib.py).
enum : uint32_t {
    FZB_ERR_CODE_RANGE = 1u << 0,      // CodeOutOfRange (encode.py:72-76)
    FZB_ERR_MALFORMED = 1u << 1,       // MalformedCodes (core.py:200-215, predict.py:245-246)
    FZB_ERR_HF_TRUNCATED = 1u << 2,    // Truncated (encode.py:307-308)
    FZB_ERR_HF_CORRUPT = 1u << 3,      // CorruptStream: no codeword (encode.py:309-310)
    FZB_ERR_HF_LONG = 1u << 4,         // CorruptStream: stream longer (encode.py:311-312)
    FZB_ERR_HF_PAD = 1u << 5,          // CorruptStream: nonzero padding (encode.py:313-316)
    FZB_ERR_BS_PAD = 1u << 6,          // CorruptPayload: block padding (encode.py:386-387)
    FZB_ERR_BS_RANGE = 1u << 7,        // CorruptPayload: code >= 2R (encode.py:389-390)
    FZB_ERR_NONFINITE = 1u << 8,       // non-finite input (core.py:98-100)
    FZB_ERR_OUTLIER_RANGE = 1u << 9,   // CorruptPayload: outlier index out of range (pipeline.py:410-411)
    FZB_ERR_OUTLIER_ORDER = 1u << 10,  // MalformedCodes: indices not increasing (core.py:212-213)
    FZB_ERR_OUTLIER_CODE = 1u << 11,   // MalformedCodes: no sentinel at outlier (core.py:214-215)
    FZB_ERR_HF_MISMATCH = 1u << 12,    // CorruptStream: histogram inconsistent (encode.py:289-290)
    FZB_ERR_HF_SYNC = 1u << 13,        // internal: decoder did not synchronise (retry)
    FZB_ERR_BS_MISMATCH = 1u << 14,    // BitmapPayloadMismatch: popcount != words (encode.py:372-375)
    FZB_ERR_DQ_RANGE = 1u << 15,       // dual-quant (opt-in): |x / 2eb| >= 2^27
};

FZB_DEV void set_err(uint32_t* status, uint32_t bit) { atomicOr(status, bit); }

// ---------------------------------------------------------------- quantizer
// Reference _quant_store (predict.py:70-90), restated bit-exactly:
//   q = RN(RN(v - pred) / two_eb); aq = |q|; f = floor(aq);
//   r = (aq - f >= 0.5) ? f + 1 : f;
//   if r < R: s = ±r; rec = RN32(RN(pred + RN(two_eb * s))); accept iff
//             RN(|rec - v|) <= eb
//   else / on reject: code R, recon = f32(v), outlier.
// The division is replaced by a multiply with the f64 reciprocal; the
// product differs from the quotient by at most ~3 ulp, which can only
// change the rounding decision when frac(|q|) is within a few ulp of 0.5,
// so that band (8 ulp-equivalents, relative) recomputes with IEEE division.
struct QParams {
    double eb, two_eb, inv2eb;
    int radius;
    int use_recip;
};

FZB_DEV QParams make_qparams(double eb, int radius) {
    QParams p;
    p.eb = eb;
    p.two_eb = __dmul_rn(2.0, eb);
    p.inv2eb = __drcp_rn(p.two_eb);
    p.radius = radius;
    // reciprocal path only for normal, finite reciprocals
    p.use_recip = (isfinite(p.inv2eb) && p.two_eb >= 2.2250738585072014e-308) ? 1 : 0;
    return p;
}

// Returns the stored code (s + R, or R for an outlier) and writes rec.
// `outlier` is set when the element must be stored verbatim.
FZB_DEV int quantize(double v, double pred, const QParams& P, float& rec, bool& outlier) {
    double d = __dsub_rn(v, pred);
    double q, aq, f, fr;
    if (P.use_recip) {
        q = __dmul_rn(d, P.inv2eb);
        aq = fabs(q);
        f = floor(aq);
        fr = __dsub_rn(aq, f);
        double tol = __dmul_rn(aq, 1.7763568394002505e-15) + 1e-300;  // 8 * 2^-52 * aq
        if (fabs(__dsub_rn(fr, 0.5)) <= tol) {
            q = __ddiv_rn(d, P.two_eb);
            aq = fabs(q);
            f = floor(aq);
            fr = __dsub_rn(aq, f);
        }
    } else {
        q = __ddiv_rn(d, P.two_eb);
        aq = fabs(q);
        f = floor(aq);
        fr = __dsub_rn(aq, f);
    }
    double r = (fr >= 0.5) ? __dadd_rn(f, 1.0) : f;
    if (r < (double)P.radius) {
        int s = (int)r;
        if (q < 0.0) s = -s;
        float rc = __double2float_rn(__dadd_rn(pred, __dmul_rn(P.two_eb, (double)s)));
        if (fabs(__dsub_rn((double)rc, v)) <= P.eb) {
            rec = rc;
            outlier = false;
            return s + P.radius;
        }
    }
    rec = __double2float_rn(v);
    outlier = true;
    return P.radius;
}

// Reference decode step (predict.py:143-144 / 178-179).
FZB_DEV float dequantize(double pred, int code, const QParams& P) {
    return __double2float_rn(__dadd_rn(pred, __dmul_rn(P.two_eb, (double)(code - P.radius))));
}

// ------------------------------------------------------------ memory model
FZB_DEV uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
FZB_DEV void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

FZB_DEV uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Block-wide exclusive scan of one u32 per thread (blockDim multiple of 32,
// <= 1024).  `tmp` needs 32 words of shared memory.  Returns the exclusive
// prefix; *total receives the block sum.
FZB_DEV uint32_t block_exclusive_scan(uint32_t x, uint32_t* tmp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) tmp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? tmp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        tmp[lane] = wi - w;
        if (lane == 31) tmp[32] = wi;
    }
    __syncthreads();
    uint32_t r = tmp[warp] + inc - x;
    if (total) *total = tmp[32];
    __syncthreads();
    return r;
}

FZB_DEV unsigned long long block_exclusive_scan64(unsigned long long x, unsigned long long* tmp,
                                                  unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) tmp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < nw ? tmp[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        tmp[lane] = wi - w;
        if (lane == 31) tmp[32] = wi;
    }
    __syncthreads();
    unsigned long long r = tmp[warp] + inc - x;
    if (total) *total = tmp[32];
    __syncthreads();
    return r;
}

// 148 SMs on B200; grids for streaming kernels are sized as multiples.
static constexpr int kNumSMs = 148;

static inline int fzb_check_launch() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -(int)e;
}
