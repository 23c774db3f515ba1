// scan.cuh -- multi-level exclusive scan of u32 counts into u64 offsets.
// Level 1: per-1024-chunk sums; level 2: one CTA scans the (<= 1M) chunk
// sums in 1024-wide passes; level 3: per-chunk local scan + chunk offset.
#pragma once
#include "common.cuh"

namespace fzscan {

constexpr int CH = 1024;

static __global__ void chunk_sum_kernel(const uint32_t* __restrict__ in, uint64_t m, unsigned long long* __restrict__ part) {
    __shared__ unsigned long long tmp[33];
    const uint64_t q = (uint64_t)blockIdx.x * CH + threadIdx.x;
    const unsigned long long x = q < m ? in[q] : 0ull;
    unsigned long long t;
    block_exclusive_scan64(x, tmp, &t);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

static __global__ void part_scan_kernel(unsigned long long* __restrict__ part, uint64_t np, unsigned long long* __restrict__ tot) {
    __shared__ unsigned long long tmp[33];
    unsigned long long carry = 0;
    for (uint64_t b0 = 0; b0 < np; b0 += blockDim.x) {
        const uint64_t q = b0 + threadIdx.x;
        const unsigned long long x = q < np ? part[q] : 0ull;
        unsigned long long t;
        const unsigned long long p = block_exclusive_scan64(x, tmp, &t);
        if (q < np) part[q] = carry + p;
        carry += t;
    }
    if (threadIdx.x == 0 && tot) *tot = carry;
}

static __global__ void chunk_apply_kernel(const uint32_t* __restrict__ in, uint64_t m, const unsigned long long* __restrict__ part,
                                   unsigned long long* __restrict__ out) {
    __shared__ unsigned long long tmp[33];
    const uint64_t q = (uint64_t)blockIdx.x * CH + threadIdx.x;
    const unsigned long long x = q < m ? in[q] : 0ull;
    const unsigned long long p = block_exclusive_scan64(x, tmp, nullptr);
    if (q < m) out[q] = part[blockIdx.x] + p;
}

inline size_t ws_bytes(uint64_t m) { return ((m + CH - 1) / CH) * 8 + 256; }

// out[q] = sum(in[0..q)), *tot = sum(in)  (tot may be null)
inline void exclusive(const uint32_t* in, uint64_t m, unsigned long long* out, unsigned long long* tot, void* ws,
                      cudaStream_t st) {
    const uint64_t np = (m + CH - 1) / CH;
    unsigned long long* part = static_cast<unsigned long long*>(ws);
    if (np == 0) {
        if (tot) cudaMemsetAsync(tot, 0, 8, st);
        return;
    }
    chunk_sum_kernel<<<(unsigned)np, CH, 0, st>>>(in, m, part);
    part_scan_kernel<<<1, 1024, 0, st>>>(part, np, tot);
    chunk_apply_kernel<<<(unsigned)np, CH, 0, st>>>(in, m, part, out);
}

}  // namespace fzscan
