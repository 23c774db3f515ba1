// interp.cu -- G-Interp (multi-level spline interpolation) predictor for sm_100a.
//
// Reference: fzpipe predict.py:147-201 (_interp_predict / _interp_pass),
// 270-344 (interp_quantize / interp_reconstruct).  The field keeps a coarse
// anchor lattice (stride 16) verbatim; levels h = 8, 4, 2, 1 then fill the
// odd multiples of h along axis 0, 1, 2 in turn.  Every pass reads only
// points finished by earlier passes, so all targets of one pass are
// independent (SURVEY.md finding 5): one grid-stride kernel per non-empty
// pass, threads mapped to the innermost lattice axis for coalescing.  The
// cubic/linear/copy stencils and the quantizer keep the reference's exact
// f64 operation order (no FMA).
#include <stdlib.h>

#include "common.cuh"

namespace {

// q / d for 32-bit q by a multiply-high (round-up method, exact for every
// 32-bit q): the lattice index decomposition ran two 64-bit divisions per
// target, the bulk of the passes' instructions.
struct FastDiv {
    uint32_t d, m;
    int l;
};
FastDiv fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.l = 0;
    while ((1ull << f.l) < d) f.l++;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << f.l) - d)) / d) + 1);
    return f;
}
FZB_DEV uint32_t fdiv(uint32_t q, const FastDiv& f) {
    return (uint32_t)(((unsigned long long)__umulhi(f.m, q) + q) >> f.l);
}
FZB_DEV FastDiv fastdiv_dev(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.l = d > 1 ? 32 - __clz(d - 1) : 0;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << f.l) - d)) / d) + 1);
    return f;
}

struct Pass {
    long long n0, n1, n2;
    long long h;
    // target lattice: start/step/count per axis
    long long s0, d0, c0, s1, d1, c1, s2, d2, c2;
    long long total;
    FastDiv f1, f2;   // by c1, c2 (valid when total < 2^32)
};

FZB_DEV double interp_pred(const float* __restrict__ r, long long t, long long c, long long n, long long sh,
                           long long h, const double* w) {
    // predict.py:151-160
    if (c - 3 * h >= 0 && c + 3 * h < n) {
        double acc = __dmul_rn(w[0], (double)r[t - 3 * sh]);
        acc = __dadd_rn(acc, __dmul_rn(w[1], (double)r[t - sh]));
        acc = __dadd_rn(acc, __dmul_rn(w[2], (double)r[t + sh]));
        acc = __dadd_rn(acc, __dmul_rn(w[3], (double)r[t + 3 * sh]));
        return acc;
    }
    if (c + h < n) return __dadd_rn(__dmul_rn(0.5, (double)r[t - sh]), __dmul_rn(0.5, (double)r[t + sh]));
    return (double)r[t - sh];
}

// interp_pred on a pointer to the target, 32-bit coordinates (shared-memory tiles)
FZB_DEV double interp_pred_s(const float* r, int c, int n, int sh, int h, const double* w) {
    if (c - 3 * h >= 0 && c + 3 * h < n) {
        double acc = __dmul_rn(w[0], (double)r[-3 * sh]);
        acc = __dadd_rn(acc, __dmul_rn(w[1], (double)r[-sh]));
        acc = __dadd_rn(acc, __dmul_rn(w[2], (double)r[sh]));
        acc = __dadd_rn(acc, __dmul_rn(w[3], (double)r[3 * sh]));
        return acc;
    }
    if (c + h < n) return __dadd_rn(__dmul_rn(0.5, (double)r[-sh]), __dmul_rn(0.5, (double)r[sh]));
    return (double)r[-sh];
}


template <int AXIS, bool DEC>
__global__ void __launch_bounds__(256) interp_pass_kernel(const float* __restrict__ orig, uint16_t* __restrict__ codes,
                                                          float* __restrict__ recon, uint32_t* __restrict__ bitmap,
                                                          Pass p, const double* __restrict__ d_eb, int radius,
                                                          double w0, double w1, double w2, double w3) {
    const QParams P = make_qparams(*d_eb, radius);
    const double w[4] = {w0, w1, w2, w3};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < p.total; q += stride) {
        long long q0, q1, q2;
        if (p.total <= 0xFFFFFFFFll) {
            const uint32_t u = (uint32_t)q;
            const uint32_t r1 = fdiv(u, p.f2);
            q2 = (long long)(u - r1 * p.f2.d);
            const uint32_t z0 = fdiv(r1, p.f1);
            q1 = (long long)(r1 - z0 * p.f1.d);
            q0 = z0;
        } else {
            q2 = q % p.c2;
            const long long r1 = q / p.c2;
            q1 = r1 % p.c1;
            q0 = r1 / p.c1;
        }
        const long long i = p.s0 + q0 * p.d0, j = p.s1 + q1 * p.d1, k = p.s2 + q2 * p.d2;
        const long long t = (i * p.n1 + j) * p.n2 + k;
        double pred;
        if (AXIS == 0) pred = interp_pred(recon, t, i, p.n0, p.h * p.n1 * p.n2, p.h, w);
        else if (AXIS == 1) pred = interp_pred(recon, t, j, p.n1, p.h * p.n2, p.h, w);
        else pred = interp_pred(recon, t, k, p.n2, p.h, p.h, w);
        if constexpr (DEC) {
            if ((bitmap[t >> 5] >> (t & 31)) & 1u) continue;
            recon[t] = dequantize(pred, (int)codes[t], P);
        } else {
            float rec;
            bool outl;
            const int c = quantize((double)__ldg(orig + t), pred, P, rec, outl);
            codes[t] = (uint16_t)c;
            recon[t] = rec;
            if (outl) atomicOr(bitmap + (t >> 5), 1u << (t & 31));
        }
    }
}

// anchors: orig[::a, ::a, ::a] -> anchor buffer and recon (encode), or
// anchor buffer -> recon (decode); predict.py:301-302, 341-342.
template <bool DEC>
__global__ void anchor_kernel(const float* __restrict__ orig, float* __restrict__ anchors, float* __restrict__ recon,
                              long long n1, long long n2, long long a, long long A0, long long A1, long long A2) {
    const long long total = A0 * A1 * A2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
        const long long z = q % A2, r = q / A2, y = r % A1, x = r / A1;
        const long long t = ((x * a) * n1 + y * a) * n2 + z * a;
        if constexpr (DEC) {
            recon[t] = anchors[q];
        } else {
            const float v = orig[t];
            anchors[q] = v;
            recon[t] = v;
        }
    }
}

Pass make_pass(long long n0, long long n1, long long n2, long long h, int axis) {
    Pass p;
    p.n0 = n0; p.n1 = n1; p.n2 = n2; p.h = h;
    const long long h2 = 2 * h;
    auto cnt = [](long long s, long long d, long long n) { return s < n ? (n - s + d - 1) / d : 0; };
    // predict.py:169-201 loop bounds
    if (axis == 0) { p.s0 = h; p.d0 = h2; p.s1 = 0; p.d1 = h2; p.s2 = 0; p.d2 = h2; }
    else if (axis == 1) { p.s0 = 0; p.d0 = h; p.s1 = h; p.d1 = h2; p.s2 = 0; p.d2 = h2; }
    else { p.s0 = 0; p.d0 = h; p.s1 = 0; p.d1 = h; p.s2 = h; p.d2 = h2; }
    p.c0 = cnt(p.s0, p.d0, n0);
    p.c1 = cnt(p.s1, p.d1, n1);
    p.c2 = cnt(p.s2, p.d2, n2);
    p.total = p.c0 * p.c1 * p.c2;
    if (p.total > 0 && p.total <= 0xFFFFFFFFll) {
        p.f1 = fastdiv((uint32_t)p.c1);
        p.f2 = fastdiv((uint32_t)p.c2);
    }
    return p;
}

template <bool DEC>
int run_passes(const float* orig, uint16_t* codes, float* recon, uint32_t* bitmap, uint32_t n0, uint32_t n1,
               uint32_t n2, const double* d_eb, uint32_t radius, uint32_t stride, const double* w, cudaStream_t st,
               long long hmin = 1) {
    for (long long h = stride / 2; h >= hmin; h /= 2) {
        for (int axis = 0; axis < 3; axis++) {
            const Pass p = make_pass(n0, n1, n2, h, axis);
            if (p.total == 0) continue;
            long long blocks = (p.total + 255) / 256;
            if (blocks > (long long)kNumSMs * 16) blocks = (long long)kNumSMs * 16;
            if (axis == 0)
                interp_pass_kernel<0, DEC><<<(unsigned)blocks, 256, 0, st>>>(orig, codes, recon, bitmap, p, d_eb, (int)radius, w[0], w[1], w[2], w[3]);
            else if (axis == 1)
                interp_pass_kernel<1, DEC><<<(unsigned)blocks, 256, 0, st>>>(orig, codes, recon, bitmap, p, d_eb, (int)radius, w[0], w[1], w[2], w[3]);
            else
                interp_pass_kernel<2, DEC><<<(unsigned)blocks, 256, 0, st>>>(orig, codes, recon, bitmap, p, d_eb, (int)radius, w[0], w[1], w[2], w[3]);
        }
    }
    return fzb_check_launch();
}

// ---- 2D fields: all levels of a 128 x 128 tile in shared memory ----------
// A target of pass (h, axis) reads points at +-h and +-3h along its axis, all
// finished by earlier passes, so the values a tile needs form a region that
// grows by 3h per axis going back through the passes:
//   (1,k): tile   (1,j): +3 in k   (2,k): +3,+3   (2,j): +3,+9   (4,k): +9,+9
//   (4,j): +9,+21 (8,k): +21,+21   (8,j): +21,+45 -> anchors within +-45.
// One CTA loads the anchors of its tile +-45 (a 218 x 218 f32 region, 190 KB
// of shared memory) and runs the eight passes over those shrinking regions
// with the reference's exact stencil and quantizer: the halo is recomputed
// (~20% extra work, nearly all of it at the coarse levels, which hold few
// points) instead of eight grid-wide passes through HBM.  Only the tile's
// own codes / outlier flags (encode) or reconstructions (decode) are written.

struct Pass2 {
    int h, axis, xj, xk;
};
struct Plan2 {
    Pass2 p[8];
    int np, halo;
};
Plan2 plan2(int htop) {
    // passes in the reference order (levels h = htop .. 1, axis j then k);
    // regions back from the last pass
    Plan2 pl;
    pl.np = 0;
    for (int h = htop; h >= 1; h /= 2) {
        pl.p[pl.np++] = {h, 1, 0, 0};
        pl.p[pl.np++] = {h, 2, 0, 0};
    }
    int xj = 0, xk = 0;
    for (int q = pl.np - 1; q >= 0; q--) {
        pl.p[q].xj = xj;
        pl.p[q].xk = xk;
        if (pl.p[q].axis == 1) xj += 3 * pl.p[q].h; else xk += 3 * pl.p[q].h;
    }
    pl.halo = xj > xk ? xj : xk;
    return pl;
}

// The kernel runs on the sub-lattice of every g-th point (n1 x n2 = its
// extents, gn2 = the field's row pitch): g = 1 runs levels 2, 1 of the field;
// g = 4 runs the field's levels 8, 4 as levels 2, 1 of the 4-lattice -- the
// boundary rules only compare c +- 3h with the extent, which scales exactly.
// Targets of one pass are independent (they read only earlier passes), so a
// thread gathers IB of them at once -- their global operands (orig value,
// or code + outlier bit) loaded back to back -- before computing any: one
// memory latency per IB targets instead of per target.

template <int T, int NT, int IB, int MINB, bool DEC>
__global__ void __launch_bounds__(NT, MINB) interp2d_tile_kernel(const float* __restrict__ orig,
                                                           const uint16_t* __restrict__ codes_in,
                                                           uint16_t* __restrict__ codes, float* __restrict__ recon,
                                                           uint32_t* __restrict__ bitmap, long long n1, long long n2,
                                                           int g, long long gn2, Plan2 pl, const double* __restrict__ d_eb,
                                                           int radius, double w0, double w1, double w2, double w3) {
    extern __shared__ float Rs[];
    const QParams P = make_qparams(*d_eb, radius);
    const double w[4] = {w0, w1, w2, w3};
    const int H = pl.halo, PW = T + 2 * H;   // region pitch
    const long long j0 = (long long)blockIdx.y * T, k0 = (long long)blockIdx.x * T;
    const long long rj0 = j0 - H, rk0 = k0 - H;   // region origin (global)
    const int J0 = (int)j0, K0 = (int)k0, RJ0 = (int)rj0, RK0 = (int)rk0, N1 = (int)n1, N2 = (int)n2;
    // the region's points of the levels above the tile's (lattice 2 * htop):
    // anchors and coarse-level reconstructions, both already in `recon`
    {
        const int stride = 2 * pl.p[0].h;
        const long long aj = ((max(rj0, 0ll) + stride - 1) / stride) * stride;
        const long long ak = ((max(rk0, 0ll) + stride - 1) / stride) * stride;
        const long long ej = min(rj0 + PW, n1), ek = min(rk0 + PW, n2);
        const int cj = aj < ej ? (int)((ej - aj + stride - 1) / stride) : 0;
        const int ck = ak < ek ? (int)((ek - ak + stride - 1) / stride) : 0;
        for (int q = threadIdx.x; q < cj * ck; q += NT) {
            const int qj = q / ck, qk = q - qj * ck;
            const long long j = aj + (long long)qj * stride, k = ak + (long long)qk * stride;
            Rs[(j - rj0) * PW + (k - rk0)] = recon[g * j * gn2 + g * k];
        }
    }
    __syncthreads();
    for (int pi = 0; pi < pl.np; pi++) {
        const Pass2 ps = pl.p[pi];
        const int h = ps.h;
        // target lattice: axis j: j = h (mod 2h), k = 0 (mod 2h); axis k: j = 0 (mod h), k = h (mod 2h)
        // all index math in 32 bits (run_tiles2d: n1, n2 < 2^30)
        const int sj = ps.axis == 1 ? h : 0, dj = ps.axis == 1 ? 2 * h : h;
        const int sk = ps.axis == 1 ? 0 : h, dk = 2 * h;
        const int lj = max(J0 - ps.xj, 0), hj = min(J0 + T + ps.xj, N1);
        const int lk = max(K0 - ps.xk, 0), hk = min(K0 + T + ps.xk, N2);
        auto first = [](int lo, int st, int d) { return lo <= st ? st : st + ((lo - st + d - 1) / d) * d; };
        const int fj = first(lj, sj, dj), fk = first(lk, sk, dk);
        const int cj = fj < hj ? (hj - fj + dj - 1) / dj : 0;
        const int ck = fk < hk ? (hk - fk + dk - 1) / dk : 0;
        const int tot = cj * ck;
        if (tot == 0) continue;   // uniform across the CTA
        const FastDiv fck = fastdiv_dev((uint32_t)ck);
        const int sh = ps.axis == 1 ? h * PW : h;
        const int cn = ps.axis == 1 ? N1 : N2;
        // local index of (fj, fk) and per-step deltas
        const int l0 = (fj - RJ0) * PW + (fk - RK0), ldj = dj * PW;
        for (int base = threadIdx.x; base < tot; base += NT * IB) {
            int li[IB], cc[IB];
            long long tt[IB];
            float ov[IB];
            int cv[IB];
            bool ob[IB], own[IB];
#pragma unroll
            for (int u = 0; u < IB; u++) {
                const int q = base + u * NT;
                li[u] = -1;
                if (q < tot) {
                    const int qj = (int)fdiv((uint32_t)q, fck), qk = q - qj * ck;
                    const int j = fj + qj * dj, k = fk + qk * dk;
                    li[u] = l0 + qj * ldj + qk * dk;
                    cc[u] = ps.axis == 1 ? j : k;
                    own[u] = (unsigned)(j - J0) < (unsigned)T && (unsigned)(k - K0) < (unsigned)T;
                    tt[u] = (long long)(g * j) * gn2 + (long long)g * k;
                    if constexpr (DEC) {
                        cv[u] = (int)codes_in[tt[u]];
                        ob[u] = (bitmap[tt[u] >> 5] >> (tt[u] & 31)) & 1u;
                        if (ob[u]) ov[u] = recon[tt[u]];   // pre-scattered outlier value
                    } else {
                        ov[u] = __ldg(orig + tt[u]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < IB; u++) {
                if (li[u] < 0) continue;
                const double pred = interp_pred_s(Rs + li[u], cc[u], cn, sh, h, w);
                float rec;
                const long long t = tt[u];
                if constexpr (DEC) {
                    rec = ob[u] ? ov[u] : dequantize(pred, cv[u], P);
                    if (own[u] && !ob[u]) recon[t] = rec;
                } else {
                    bool outl;
                    const int c = quantize((double)ov[u], pred, P, rec, outl);
                    if (own[u]) {
                        if (g > 1) recon[t] = rec;   // the field-level kernel reads the 4-lattice
                        codes[t] = (uint16_t)c;
                        if (outl) atomicOr(bitmap + (t >> 5), 1u << (t & 31));
                    }
                }
                Rs[li[u]] = rec;
            }
        }
        __syncthreads();
    }
}

template <int T, int NT, int IB, int MINB, bool DEC>
int launch_tiles2d(const float* orig, uint16_t* codes, float* recon, uint32_t* bitmap, uint32_t n1, uint32_t n2,
                   int g, const double* d_eb, uint32_t radius, int htop, const double* w, cudaStream_t st) {
    const Plan2 pl = plan2(htop);
    const int PW = T + 2 * pl.halo;
    const size_t smem = (size_t)PW * PW * 4;
    if (smem > 227 * 1024) return FZB_E_ARG;
    auto kfn = interp2d_tile_kernel<T, NT, IB, MINB, DEC>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t m1 = (n1 - 1) / g + 1, m2 = (n2 - 1) / g + 1;   // sub-lattice extents
    const dim3 grid((m2 + T - 1) / T, (m1 + T - 1) / T);
    kfn<<<grid, NT, smem, st>>>(orig, codes, codes, recon, bitmap, m1, m2, g, n2, pl, d_eb, (int)radius, w[0], w[1],
                                w[2], w[3]);
    return fzb_check_launch();
}

// 2D fields (anchor stride 4..64): levels stride/2 .. 4 as one tile kernel on
// the 4-lattice, levels 2, 1 as one on the field -- two launches instead of
// 2 log2(stride) grid-wide passes through HBM.
template <bool DEC>
int run_tiles2d(const float* orig, uint16_t* codes, float* recon, uint32_t* bitmap, uint32_t n1, uint32_t n2,
                const double* d_eb, uint32_t radius, uint32_t stride, const double* w, cudaStream_t st) {
    if (stride >= 8) {
        const int rc = launch_tiles2d<32, 128, 2, 1, DEC>(orig, codes, recon, bitmap, n1, n2, 4, d_eb, radius,
                                                          (int)stride / 8, w, st);
        if (rc) return rc;
    }
    // (A/B on C3: 32-tiles 88/71 us, 48-tiles 63/55 us, 64-tiles 57/54 us enc/dec)
    return launch_tiles2d<64, 128, 2, 7, DEC>(orig, codes, recon, bitmap, n1, n2, 1, d_eb, radius, 2, w, st);
}

// ---- sampled profiling (opt-in pipeline 5, cuSZ-i / QoZ style) ----------
// Candidates c = 3 s + w: anchor stride 16 (s = 0) or 8 (s = 1) x weights
// cubic (-1, 9, 9, -1)/16, linear (0, 1, 1, 0)/2, natural cubic
// (-3, 23, 23, -3)/40.  Sample = every point of the 16-cells whose cell
// coordinates are multiples of 4 (1/64 of a 3D field); each is an anchor of
// the candidate's lattice (32 bits) or the target of exactly one pass (level
// h = lowest set bit of its coordinates, axis = the last axis with that bit)
// and costs bitlen(rint(|pred - x| / 2eb)) with pred from ORIGINAL values
// and the reference's cubic / linear / copy boundary rules.  Integer sums:
// order-independent, so the CPU spec (oracle) reproduces the choice exactly.
__constant__ double kProfW[3][4] = {{-0.0625, 0.5625, 0.5625, -0.0625},
                                    {0.0, 0.5, 0.5, 0.0},
                                    {-0.075, 0.575, 0.575, -0.075}};

FZB_DEV int lowbit_of(long long c) { return c == 0 ? 62 : __ffsll(c) - 1; }

__global__ void __launch_bounds__(256) interp_profile_kernel(const float* __restrict__ x, long long n0, long long n1,
                                                              long long n2, const double* __restrict__ d_eb,
                                                              unsigned long long* __restrict__ scores) {
    const double inv2eb = __drcp_rn(__dmul_rn(2.0, *d_eb));
    const long long C0 = (n0 + 15) / 16, C1 = (n1 + 15) / 16, C2 = (n2 + 15) / 16;
    const long long S0 = (C0 + 3) / 4, S1 = (C1 + 3) / 4, S2 = (C2 + 3) / 4;
    const long long total = S0 * S1 * S2 * 4096;
    unsigned long long acc[6] = {0, 0, 0, 0, 0, 0};
    const long long ext[3] = {n0, n1, n2};
    const long long str[3] = {n1 * n2, n2, 1};
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const int u = (int)(q & 15), v = (int)((q >> 4) & 15), ww = (int)((q >> 8) & 15);
        const long long cell = q >> 12;
        const long long c2 = cell % S2, c1 = (cell / S2) % S1, c0 = cell / (S1 * S2);
        const long long co[3] = {64 * c0 + ww, 64 * c1 + v, 64 * c2 + u};
        if (co[0] >= n0 || co[1] >= n1 || co[2] >= n2) continue;
        const long long t = (co[0] * n1 + co[1]) * n2 + co[2];
        const double xv = (double)__ldg(x + t);
        const int lb[3] = {lowbit_of(co[0]), lowbit_of(co[1]), lowbit_of(co[2])};
        const int m = min(lb[0], min(lb[1], lb[2]));
#pragma unroll
        for (int s = 0; s < 2; s++) {
            if (m >= (s == 0 ? 4 : 3)) {   // an anchor of this lattice
#pragma unroll
                for (int wi = 0; wi < 3; wi++) acc[3 * s + wi] += 32;
                continue;
            }
            const long long h = 1ll << m;
            const int ax = lb[2] == m ? 2 : (lb[1] == m ? 1 : 0);
            const long long c = co[ax], n = ext[ax], sh = h * str[ax];
#pragma unroll
            for (int wi = 0; wi < 3; wi++) {
                double pred;
                if (c - 3 * h >= 0 && c + 3 * h < n) {
                    pred = __dmul_rn(kProfW[wi][0], (double)__ldg(x + t - 3 * sh));
                    pred = __dadd_rn(pred, __dmul_rn(kProfW[wi][1], (double)__ldg(x + t - sh)));
                    pred = __dadd_rn(pred, __dmul_rn(kProfW[wi][2], (double)__ldg(x + t + sh)));
                    pred = __dadd_rn(pred, __dmul_rn(kProfW[wi][3], (double)__ldg(x + t + 3 * sh)));
                } else if (c + h < n) {
                    pred = __dadd_rn(__dmul_rn(0.5, (double)__ldg(x + t - sh)), __dmul_rn(0.5, (double)__ldg(x + t + sh)));
                } else {
                    pred = (double)__ldg(x + t - sh);
                }
                double e = __dmul_rn(fabs(__dsub_rn(pred, xv)), inv2eb);
                e = e < 1073741824.0 ? e : 1073741824.0;
                const unsigned int iv = (unsigned int)rint(e);
                acc[3 * s + wi] += iv ? (unsigned long long)(32 - __clz(iv)) : 0ull;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 6; c++) {
        unsigned long long v = acc[c];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(scores + c, v);
    }
}

}  // namespace

extern "C" {

// Caller: d_codes pre-filled with `radius` (predict.py:297), d_bitmap zeroed.
// Dims are the reference's padded (n0, n1, n2) (predict.py:204-205).
FZB_API int fzb_interp_encode_f32(const float* d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb,
                                  uint32_t radius, uint32_t anchor_stride, const double* h_weights4,
                                  uint16_t* d_codes, float* d_recon, uint32_t* d_bitmap, float* d_anchors,
                                  void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (anchor_stride < 4 || (anchor_stride & (anchor_stride - 1))) return FZB_E_ARG;
    const long long a = anchor_stride;
    const long long A0 = (n0 - 1) / a + 1, A1 = (n1 - 1) / a + 1, A2 = (n2 - 1) / a + 1;
    anchor_kernel<false><<<kNumSMs * 2, 256, 0, st>>>(d_in, d_anchors, d_recon, n1, n2, a, A0, A1, A2);
    if (n0 == 1 && n1 > 1 && n1 < (1u << 30) && n2 < (1u << 30) && anchor_stride <= 64 && !getenv("FZB_INTERP_PASSES"))   // 2D: every level of a tile in shared memory
        return run_tiles2d<false>(d_in, d_codes, d_recon, d_bitmap, n1, n2, d_eb, radius, anchor_stride, h_weights4, st);
    return run_passes<false>(d_in, d_codes, d_recon, d_bitmap, n0, n1, n2, d_eb, radius, anchor_stride, h_weights4, st);
}

// Caller: d_recon holds the outlier values and d_bitmap their flags
// (fzb_outlier_scatter); anchors are scattered here.
FZB_API int fzb_interp_decode_f32(const uint16_t* d_codes, const uint32_t* d_bitmap, const float* d_anchors,
                                  float* d_recon, uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb,
                                  uint32_t radius, uint32_t anchor_stride, const double* h_weights4, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (radius == 0 || radius > 32768) return FZB_E_RADIUS;
    if (anchor_stride < 4 || (anchor_stride & (anchor_stride - 1))) return FZB_E_ARG;
    const long long a = anchor_stride;
    const long long A0 = (n0 - 1) / a + 1, A1 = (n1 - 1) / a + 1, A2 = (n2 - 1) / a + 1;
    anchor_kernel<true><<<kNumSMs * 2, 256, 0, st>>>(nullptr, const_cast<float*>(d_anchors), d_recon, n1, n2, a, A0, A1, A2);
    if (n0 == 1 && n1 > 1 && n1 < (1u << 30) && n2 < (1u << 30) && anchor_stride <= 64 && !getenv("FZB_INTERP_PASSES"))
        return run_tiles2d<true>(nullptr, const_cast<uint16_t*>(d_codes), d_recon, const_cast<uint32_t*>(d_bitmap), n1,
                                 n2, d_eb, radius, anchor_stride, h_weights4, st);
    return run_passes<true>(nullptr, const_cast<uint16_t*>(d_codes), d_recon, const_cast<uint32_t*>(d_bitmap), n0, n1,
                            n2, d_eb, radius, anchor_stride, h_weights4, st);
}

// Sampled profiling scores of the 6 (anchor stride, weights) candidates of
// pipeline 5 into d_scores (u64[6], zeroed here).
FZB_API int fzb_interp_profile(const float* d_in, uint32_t n0, uint32_t n1, uint32_t n2, const double* d_eb,
                               uint64_t* d_scores, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(d_scores, 0, 6 * 8, st);
    interp_profile_kernel<<<kNumSMs * 4, 256, 0, st>>>(d_in, n0, n1, n2, d_eb,
                                                      reinterpret_cast<unsigned long long*>(d_scores));
    return fzb_check_launch();
}

}  // extern "C"
