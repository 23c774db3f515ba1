// dualquant.cu -- dual-quantization Lorenzo predictor (opt-in pipelines 3/4).
//
// north_star items (1) and (4): the FZ-GPU / cuSZ
// "dual-quant" formulation of Lorenzo.  Every value is prequantized first,
//     p = rint(x / 2eb)                     (f64, |x / 2eb| < 2^27)
// and the Lorenzo difference runs on the INTEGERS p (no reconstruction
// feedback), so every element is independent:
//     delta = p - sum_{nonempty S of the axes} (-1)^(|S|+1) p[shifted by S]
// (absent neighbours are 0).  code = delta + R when |delta| < R and the
// reconstruction RN32(2eb p) is within eb of x; otherwise the element is an
// outlier: code R, and the archive keeps its index, its original value and
// its delta.  The inverse of the Lorenzo difference is the inclusive prefix
// sum along every axis, so decompression is k-, j- and i-scans of the deltas
// followed by x' = RN32(2eb p) and the outlier values scattered on top.
//
// This predictor does NOT reproduce the reference's feedback Lorenzo (whose
// codes it changes on 0.9-60% of elements); it is a
// separate pipeline id, never one of presets 0-2.  Its own bit-exact oracle
// is oracle/fzoracle.py dq_* (numpy).
#include <stdint.h>

#include "common.cuh"
#include "scan.cuh"

namespace {

constexpr double DQ_PMAX = 134217728.0;              // |x / 2eb| < 2^27: deltas (8 terms) and partial sums fit int32

struct DQ {
    double eb, two_eb, inv2eb;
    float lo_thr, hi_thr;   // |rec - x| below lo_thr: within eb; above hi_thr: not (f32 compares)
    int radius;
};
FZB_DEV DQ make_dq(double eb, int radius) {
    DQ d;
    d.eb = eb;
    d.two_eb = __dmul_rn(2.0, eb);
    d.inv2eb = __drcp_rn(d.two_eb);
    d.lo_thr = __double2float_rd(__dmul_rn(eb, 1.0 - 9.5367431640625e-07));
    d.hi_thr = __double2float_ru(__dmul_rn(eb, 1.0 + 9.5367431640625e-07));
    d.radius = radius;
    return d;
}
// prequantization p = rint(x / 2eb): the f64 product rounded half-even by the
// 1.5*2^52 magic add (exact for |q| < 2^51), which also yields p as the low
// word and (double)p as t - M -- no f64<->int conversions (they run on the
// narrow XU pipe); out-of-range values flag the status word (the host raises)
constexpr double DQ_MAGIC = 6755399441055744.0;
struct PQ {
    int p;
    double pd;   // (double)p
};
FZB_DEV PQ dq_pq(float x, const DQ& d, uint32_t* status) {
    const double q = __dmul_rn((double)x, d.inv2eb);
    PQ r;
    if (!(fabs(q) < DQ_PMAX)) {
        set_err(status, FZB_ERR_DQ_RANGE);
        r.p = 0;
        r.pd = 0.0;
        return r;
    }
    const double t = __dadd_rn(q, DQ_MAGIC);
    r.p = (int)__double2loint(t);
    r.pd = __dsub_rn(t, DQ_MAGIC);
    return r;
}
FZB_DEV int dq_p(float x, const DQ& d, uint32_t* status) { return dq_pq(x, d, status).p; }

// code / outlier of one element.  |RN32(2eb p) - x| <= eb: the f32 difference
// is exact when the two are within a factor 2 (Sterbenz) and otherwise off
// by at most 2^-24 relative, so outside a 2^-20 band around eb the f32
// compare decides; inside it the f64 difference does (exactly the spec).
FZB_DEV void dq_emit(long long t, float x, double pd, long long delta, const DQ& d, uint16_t* codes,
                     uint32_t* bitmap) {
    const float rec = __double2float_rn(__dmul_rn(d.two_eb, pd));
    const float df = fabsf(rec - x);
    bool near = df <= d.eb ? true : false;
    if (df < d.lo_thr) near = true;
    else if (df > d.hi_thr) near = false;
    else near = fabs(__dsub_rn((double)rec, (double)x)) <= d.eb;
    const bool ok = (delta > -(long long)d.radius) & (delta < (long long)d.radius) & near;
    codes[t] = (uint16_t)(ok ? (int)delta + d.radius : d.radius);
    if (!ok) atomicOr(bitmap + (t >> 5), 1u << (t & 31));
}

// ---- encode, 2D/3D: delta = D_i D_j D_k p (backward differences).  CTA =
// 8 warps; warp w owns rows j0 + 4w .. 4w+3 of a 32 (k) x 32 (j) tile and the
// CTA marches along i through DQ_ICH planes.  D_k is one shuffle (lane 0
// takes the k0-1 halo), D_j is register-to-register within a warp's rows and
// one shared-memory word from the warp above (warp 0: the j0-1 halo row),
// D_i subtracts the previous plane's D_j D_k p kept in registers.  The next
// plane's inputs are loaded before the current plane is processed.
constexpr int DQ_R = 4, DQ_ICH = 16;

__global__ void __launch_bounds__(256) dq_encode3_kernel(const float* __restrict__ x, int n0, int n1, int n2,
                                                          const double* __restrict__ d_eb, int radius,
                                                          uint16_t* __restrict__ codes, uint32_t* __restrict__ bitmap,
                                                          uint32_t* __restrict__ status) {
    __shared__ int s_q1[9][32];   // [w + 1]: D_k p of warp w's last row; [0]: the j0-1 halo row
    const DQ d = make_dq(*d_eb, radius);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int k0 = blockIdx.x * 32, j0 = blockIdx.y * (8 * DQ_R), i0 = blockIdx.z * DQ_ICH;
    const int k = k0 + lane;
    const int i1 = min(i0 + DQ_ICH, n0);
    const bool kin = k < n2;
    auto ld = [&](int i, int j, int kk) -> float {
        return (i >= 0 && j >= 0 && kk >= 0 && j < n1 && kk < n2) ? __ldg(x + ((long long)i * n1 + j) * n2 + kk) : 0.f;
    };
    // D_k p of one row at plane i from (own element, k0-1 halo); absent elements are p = 0
    auto dk = [&](float xv, float xh, int i, int j, double& pd) -> int {
        const bool in = i >= 0 && j >= 0 && j < n1;
        PQ a;
        a.p = 0;
        a.pd = 0.0;
        if (in && kin) a = dq_pq(xv, d, status);
        pd = a.pd;
        const int ph = (in && lane == 0 && k0 > 0) ? dq_p(xh, d, status) : 0;
        const int left = __shfl_up_sync(0xffffffffu, a.p, 1);
        return a.p - (lane == 0 ? ph : left);
    };
    float xr[DQ_R], xk[DQ_R], xhr = 0.f, xhk = 0.f;   // next plane's inputs (rows, k0-1 halos, j0-1 row)
    auto load = [&](int i) {
#pragma unroll
        for (int r = 0; r < DQ_R; r++) {
            const int j = j0 + DQ_R * w + r;
            xr[r] = ld(i, j, k);
            xk[r] = lane == 0 ? ld(i, j, k0 - 1) : 0.f;
        }
        if (w == 0) {
            xhr = ld(i, j0 - 1, k);
            xhk = lane == 0 ? ld(i, j0 - 1, k0 - 1) : 0.f;
        }
    };
    int q2p[DQ_R];
#pragma unroll
    for (int r = 0; r < DQ_R; r++) q2p[r] = 0;
    load(i0 - 1);
    for (int i = i0 - 1; i < i1; i++) {
        float cr[DQ_R], ck[DQ_R];
#pragma unroll
        for (int r = 0; r < DQ_R; r++) { cr[r] = xr[r]; ck[r] = xk[r]; }
        const float chr = xhr, chk = xhk;
        if (i + 1 < i1) load(i + 1);
        int q1[DQ_R];
        double pds[DQ_R];
#pragma unroll
        for (int r = 0; r < DQ_R; r++) q1[r] = dk(cr[r], ck[r], i, j0 + DQ_R * w + r, pds[r]);
        s_q1[w + 1][lane] = q1[DQ_R - 1];
        if (w == 0) {
            double unused;
            s_q1[0][lane] = dk(chr, chk, i, j0 - 1, unused);
        }
        __syncthreads();
        const int up = s_q1[w][lane];   // D_k p of row j0 + 4w - 1
#pragma unroll
        for (int r = 0; r < DQ_R; r++) {
            const int q2 = q1[r] - (r == 0 ? up : q1[r - 1]);
            const int j = j0 + DQ_R * w + r;
            if (i >= i0 && kin && j < n1) {
                const long long t = ((long long)i * n1 + j) * n2 + k;
                dq_emit(t, cr[r], pds[r], (long long)q2 - q2p[r], d, codes, bitmap);
            }
            q2p[r] = q2;
        }
        __syncthreads();   // s_q1 is rewritten by the next plane
    }
}

// ---- encode, 1D: delta = p[t] - p[t-1]
__global__ void dq_encode1_kernel(const float* __restrict__ x, long long n, const double* __restrict__ d_eb,
                                  int radius, uint16_t* __restrict__ codes, uint32_t* __restrict__ bitmap,
                                  uint32_t* __restrict__ status) {
    const DQ d = make_dq(*d_eb, radius);
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const float xv = __ldg(x + t);
        const PQ a = dq_pq(xv, d, status);
        const int pp = t > 0 ? dq_p(__ldg(x + t - 1), d, status) : 0;
        dq_emit(t, xv, a.pd, (long long)a.p - pp, d, codes, bitmap);
    }
}

// deltas of the (compacted, sorted) outliers, recomputed from the field
__global__ void dq_outlier_delta_kernel(const float* __restrict__ x, int n0, int n1, int n2,
                                        const unsigned long long* __restrict__ idx,
                                        const unsigned long long* __restrict__ kp, const double* __restrict__ d_eb,
                                        int radius, int* __restrict__ deltas, uint32_t* __restrict__ status) {
    const DQ d = make_dq(*d_eb, radius);
    const unsigned long long k = *kp;
    for (unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; q < k;
         q += (unsigned long long)gridDim.x * blockDim.x) {
        const long long t = (long long)idx[q];
        const int kk = (int)(t % n2), jj = (int)((t / n2) % n1), ii = (int)(t / ((long long)n1 * n2));
        auto P = [&](int a, int b, int c) -> long long {
            if (a < 0 || b < 0 || c < 0) return 0;
            return dq_p(__ldg(x + ((long long)a * n1 + b) * n2 + c), d, status);
        };
        const long long s = P(ii, jj, kk) - P(ii, jj - 1, kk) - P(ii, jj, kk - 1) + P(ii, jj - 1, kk - 1) -
                            P(ii - 1, jj, kk) + P(ii - 1, jj - 1, kk) + P(ii - 1, jj, kk - 1) - P(ii - 1, jj - 1, kk - 1);
        deltas[q] = (int)s;   // |s| < 8 * 2^27: fits
    }
}

// ---- decode -------------------------------------------------------------
// outlier deltas into the work buffer (int view of the output) + flags
__global__ void dq_delta_scatter_kernel(const unsigned long long* __restrict__ idx, const int* __restrict__ deltas,
                                        uint64_t k, uint64_t n, int* __restrict__ work, uint32_t* __restrict__ bm,
                                        uint32_t* __restrict__ status) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long t = idx[q];
        if (t >= n) {
            set_err(status, FZB_ERR_OUTLIER_RANGE);
            continue;
        }
        if (q > 0 && idx[q - 1] >= t) set_err(status, FZB_ERR_OUTLIER_ORDER);
        work[t] = deltas[q];
        atomicOr(bm + (t >> 5), 1u << (t & 31));
    }
}

FZB_DEV int dq_delta_at(const uint16_t* codes, const uint32_t* bm, const int* work, long long t, int radius) {
    return ((bm[t >> 5] >> (t & 31)) & 1u) ? work[t] : (int)codes[t] - radius;
}

// k axis: one warp per segment of a row (a whole row when n2 <= KSEG, else
// KSEG-long pieces).  Passes of 128 elements: lane l owns 4 consecutive
// ones, lane-local sums + one warp shuffle scan + the running carry.  Long
// rows add each piece's carry from the biased chunk-sum scan (fzscan on
// u32 sums + 2^29 each, then the bias removed).
constexpr int KSEG = 8192;
constexpr uint32_t KBIAS = 1u << 29;   // |piece sum| = |p[end] - p[start - 1]| < 2^28

FZB_DEV long long warp_excl_scan(long long v, long long& total) {
    const int lane = threadIdx.x & 31;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - v;
}

template <bool SUM_ONLY>
__global__ void __launch_bounds__(256) dq_kscan_kernel(const uint16_t* __restrict__ codes,
                                                        const uint32_t* __restrict__ bm, int* __restrict__ work,
                                                        long long rows, int n2, int spr, int radius,
                                                        uint32_t* __restrict__ seg_sums,
                                                        const unsigned long long* __restrict__ seg_off,
                                                        const double* __restrict__ d_eb, int final_axis) {
    const int lane = threadIdx.x & 31;
    const long long seg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (seg >= rows * spr) return;
    const long long row = seg / spr;
    const int sc = (int)(seg % spr);
    const long long base = row * n2 + (long long)sc * KSEG;
    const int len = min(KSEG, n2 - sc * KSEG);
    long long carry = 0;
    if (!SUM_ONLY && spr > 1) {   // exclusive prefix of this piece within its row (bias removed)
        const unsigned long long o = seg_off[seg], o0 = seg_off[row * spr];
        carry = (long long)(o - o0) - (long long)(seg - row * spr) * (long long)KBIAS;
    }
    const double two_eb = __dmul_rn(2.0, *d_eb);
    float* out = reinterpret_cast<float*>(work);
    for (int p0 = 0; p0 < len; p0 += 128) {
        const int o = p0 + 4 * lane;
        int v[4];
        long long s = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            v[e] = (o + e < len) ? dq_delta_at(codes, bm, work, base + o + e, radius) : 0;
            s += v[e];
        }
        long long tot;
        const long long ex = warp_excl_scan(s, tot);
        if (!SUM_ONLY) {
            long long acc = carry + ex;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                acc += v[e];
                if (o + e < len) {
                    if (final_axis) out[base + o + e] = __double2float_rn(__dmul_rn(two_eb, (double)acc));
                    else work[base + o + e] = (int)acc;
                }
            }
        }
        carry += tot;
    }
    if (SUM_ONLY && lane == 0) seg_sums[seg] = (uint32_t)((long long)KBIAS + carry);
}

// Scan along a strided axis in AX_CH-long pieces (enough parallelism even for
// a 2D field's few columns): piece sums, per-column carries, then each piece
// re-scanned from its carry.  Column (o, q) of axis length `len`, stride
// `inner`; the last axis writes x' = RN32(2eb p) as f32 in place.
constexpr int AX_CH = 64;

__global__ void dq_axsum_kernel(const int* __restrict__ work, long long outer, int len, long long inner, int nch,
                                long long* __restrict__ sums) {
    const long long tot = outer * nch * inner;
    for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < tot;
         id += (long long)gridDim.x * blockDim.x) {
        const long long q = id % inner, oc = id / inner;
        const int c = (int)(oc % nch);
        const long long o = oc / nch;
        const int* p = work + o * (long long)len * inner + q;
        const int a1 = min(len, (c + 1) * AX_CH);
        long long s = 0;
#pragma unroll 8
        for (int a = c * AX_CH; a < a1; a++) s += p[(long long)a * inner];
        sums[id] = s;
    }
}

__global__ void dq_axcarry_kernel(long long* __restrict__ sums, long long outer, int nch, long long inner) {
    const long long cols = outer * inner;
    for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < cols;
         id += (long long)gridDim.x * blockDim.x) {
        const long long q = id % inner, o = id / inner;
        long long acc = 0;
        for (int c = 0; c < nch; c++) {
            long long* s = sums + (o * nch + c) * inner + q;
            const long long v = *s;
            *s = acc;
            acc += v;
        }
    }
}

__global__ void dq_axapply_kernel(int* __restrict__ work, long long outer, int len, long long inner, int nch,
                                  const long long* __restrict__ sums, const double* __restrict__ d_eb, int final_axis) {
    const double two_eb = __dmul_rn(2.0, *d_eb);
    float* out = reinterpret_cast<float*>(work);
    const long long tot = outer * nch * inner;
    for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < tot;
         id += (long long)gridDim.x * blockDim.x) {
        const long long q = id % inner, oc = id / inner;
        const int c = (int)(oc % nch);
        const long long o = oc / nch;
        const long long b = o * (long long)len * inner + q;
        const int a1 = min(len, (c + 1) * AX_CH);
        long long acc = sums[id];
#pragma unroll 8
        for (int a = c * AX_CH; a < a1; a++) {
            const long long t = b + (long long)a * inner;
            acc += work[t];
            if (final_axis) out[t] = __double2float_rn(__dmul_rn(two_eb, (double)acc));
            else work[t] = (int)acc;
        }
    }
}

__global__ void dq_value_scatter_kernel(const unsigned long long* __restrict__ idx, const float* __restrict__ vals,
                                        uint64_t k, uint64_t n, float* __restrict__ out) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long t = idx[q];
        if (t < n) out[t] = vals[q];
    }
}

// direct pass: thread per column, enough columns to fill the GPU
__global__ void dq_axdirect_kernel(int* __restrict__ work, long long outer, int len, long long inner,
                                   const double* __restrict__ d_eb, int final_axis) {
    const double two_eb = __dmul_rn(2.0, *d_eb);
    float* out = reinterpret_cast<float*>(work);
    const long long cols = outer * inner;
    for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < cols;
         id += (long long)gridDim.x * blockDim.x) {
        const long long q = id % inner, o = id / inner;
        const long long b = o * (long long)len * inner + q;
        long long acc = 0;
#pragma unroll 8
        for (int a = 0; a < len; a++) {
            const long long t = b + (long long)a * inner;
            acc += work[t];
            if (final_axis) out[t] = __double2float_rn(__dmul_rn(two_eb, (double)acc));
            else work[t] = (int)acc;
        }
    }
}

void axis_scan(int* work, long long outer, int len, long long inner, long long* sums, const double* d_eb, bool final_axis,
               cudaStream_t st) {
    if (outer * inner >= (1ll << 17)) {
        const unsigned g = (unsigned)min((outer * inner + 255) / 256, (long long)kNumSMs * 32);
        dq_axdirect_kernel<<<g, 256, 0, st>>>(work, outer, len, inner, d_eb, final_axis ? 1 : 0);
        return;
    }
    const int nch = (len + AX_CH - 1) / AX_CH;
    const long long tot = outer * nch * inner;
    const unsigned g = (unsigned)min((tot + 255) / 256, (long long)kNumSMs * 32);
    dq_axsum_kernel<<<g, 256, 0, st>>>(work, outer, len, inner, nch, sums);
    const unsigned gc = (unsigned)min((outer * inner + 255) / 256, (long long)kNumSMs * 32);
    dq_axcarry_kernel<<<gc, 256, 0, st>>>(sums, outer, nch, inner);
    dq_axapply_kernel<<<g, 256, 0, st>>>(work, outer, len, inner, nch, sums, d_eb, final_axis ? 1 : 0);
}

}  // namespace

extern "C" {

// Encode: d_codes u16[n], d_bitmap (zeroed) receives the outlier flags.
FZB_API int fzb_dualquant_encode_f32(const float* d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb,
                                     uint32_t radius, uint16_t* d_codes, uint32_t* d_bitmap, uint32_t* d_status,
                                     void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    const long long n = (long long)n0 * n1 * n2;
    if (n == 0) return 0;
    if (n0 == 1 && n1 == 1) {
        dq_encode1_kernel<<<kNumSMs * 16, 256, 0, st>>>(d_in, n, d_eb, (int)radius, d_codes, d_bitmap, d_status);
    } else {
        const dim3 grid((n2 + 31) / 32, (n1 + 8 * DQ_R - 1) / (8 * DQ_R), (n0 + DQ_ICH - 1) / DQ_ICH);
        dq_encode3_kernel<<<grid, 256, 0, st>>>(d_in, (int)n0, (int)n1, (int)n2, d_eb, (int)radius, d_codes,
                                               d_bitmap, d_status);
    }
    return fzb_check_launch();
}

// The deltas of the k compacted outliers (*d_k of them, indices sorted).
FZB_API int fzb_dualquant_outlier_deltas(const float* d_in, uint32_t n0, uint32_t n1, uint32_t n2,
                                         const uint64_t* d_idx, const uint64_t* d_k, const double* d_eb,
                                         uint32_t radius, int32_t* d_deltas, uint32_t* d_status, void* stream) {
    dq_outlier_delta_kernel<<<kNumSMs * 2, 256, 0, (cudaStream_t)stream>>>(
        d_in, (int)n0, (int)n1, (int)n2, reinterpret_cast<const unsigned long long*>(d_idx),
        reinterpret_cast<const unsigned long long*>(d_k), d_eb, (int)radius, d_deltas, d_status);
    return fzb_check_launch();
}

FZB_API size_t fzb_dualquant_decode_workspace_bytes(uint32_t n0, uint32_t n1, uint32_t n2) {
    const long long rows = (long long)n0 * n1;
    const long long spr = ((long long)n2 + KSEG - 1) / KSEG;
    const long long nseg = rows * spr;
    const size_t kb = (size_t)nseg * 4 + 256 + (size_t)(nseg + 1) * 8 + 256 + fzscan::ws_bytes(nseg + 1) + 256;
    const long long aj = (long long)n0 * ((n1 + AX_CH - 1) / AX_CH) * n2;   // j-axis piece sums
    const long long ai = (long long)((n0 + AX_CH - 1) / AX_CH) * n1 * n2;   // i-axis piece sums
    const size_t ab = (size_t)(aj > ai ? aj : ai) * 8 + 256;
    return kb > ab ? kb : ab;
}

// Decode: codes + outlier deltas/values -> d_out f32[n].  d_bitmap zeroed.
FZB_API int fzb_dualquant_decode_f32(const uint16_t* d_codes, const uint64_t* d_idx, const int32_t* d_deltas,
                                     const float* d_vals, uint64_t k, uint32_t n0, uint32_t n1, uint32_t n2,
                                     const double* d_eb, uint32_t radius, uint32_t* d_bitmap, float* d_out,
                                     void* d_ws, size_t ws_bytes, uint32_t* d_status, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    const long long n = (long long)n0 * n1 * n2;
    if (n == 0) return 0;
    if (ws_bytes < fzb_dualquant_decode_workspace_bytes(n0, n1, n2)) return FZB_E_WORKSPACE;
    int* work = reinterpret_cast<int*>(d_out);
    const unsigned kb = (unsigned)(k ? (k + 255) / 256 : 1);
    if (k)
        dq_delta_scatter_kernel<<<kb < (unsigned)kNumSMs * 8 ? kb : kNumSMs * 8, 256, 0, st>>>(
            reinterpret_cast<const unsigned long long*>(d_idx), d_deltas, k, (uint64_t)n, work, d_bitmap, d_status);
    // k axis
    const long long rows = (long long)n0 * n1;
    const int spr = (int)(((long long)n2 + KSEG - 1) / KSEG);
    const long long nseg = rows * spr;
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    unsigned char* wsb = static_cast<unsigned char*>(d_ws);
    uint32_t* seg_sums = reinterpret_cast<uint32_t*>(wsb);
    unsigned long long* seg_off = reinterpret_cast<unsigned long long*>(wsb + al((size_t)nseg * 4 + 4));
    void* scan_ws = wsb + al((size_t)nseg * 4 + 4) + al((size_t)(nseg + 1) * 8);
    long long* sums = static_cast<long long*>(d_ws);   // the axis scans reuse the workspace afterwards
    const bool one_d = (n0 == 1 && n1 == 1);
    const unsigned kblocks = (unsigned)((nseg * 32 + 255) / 256);
    if (spr > 1) {
        dq_kscan_kernel<true><<<kblocks, 256, 0, st>>>(d_codes, d_bitmap, work, rows, (int)n2, spr, (int)radius,
                                                       seg_sums, nullptr, d_eb, 0);
        fzscan::exclusive(seg_sums, (uint64_t)nseg, seg_off, nullptr, scan_ws, st);
    }
    dq_kscan_kernel<false><<<kblocks, 256, 0, st>>>(d_codes, d_bitmap, work, rows, (int)n2, spr, (int)radius,
                                                    seg_sums, seg_off, d_eb, one_d ? 1 : 0);
    if (!one_d) {
        // j axis (per plane i, column k), then i (column (j, k))
        const bool three_d = n0 > 1;
        axis_scan(work, n0, (int)n1, n2, sums, d_eb, !three_d, st);
        if (three_d) axis_scan(work, 1, (int)n0, (long long)n1 * n2, sums, d_eb, true, st);
    }
    // the outliers' original values on top
    if (k)
        dq_value_scatter_kernel<<<kb < (unsigned)kNumSMs * 8 ? kb : kNumSMs * 8, 256, 0, st>>>(
            reinterpret_cast<const unsigned long long*>(d_idx), d_vals, k, (uint64_t)n, d_out);
    return fzb_check_launch();
}

}  // extern "C"
