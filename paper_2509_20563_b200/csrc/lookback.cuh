// lookback.cuh -- decoupled look-back prefix (single-pass scan) for persistent
// kernels whose CTAs claim chunks by an atomic ticket, so every predecessor
// chunk is claimed (resident or finished) before its successor waits on it.
#pragma once
#include "common.cuh"

namespace fzlb {

// per-chunk state word: bits 62-63 flag (1 aggregate, 2 inclusive prefix), 0-61 value
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 62) - 1;

FZB_DEV unsigned long long ld_volatile64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// CTA-wide exclusive prefix of `agg` by decoupled look-back (CTA ids from a
// ticket, so every predecessor is resident or done).  Called by warp 0.
FZB_DEV unsigned long long lookback(uint32_t cta, unsigned long long agg, unsigned long long* state) {
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    if (cta == 0) {
        if (lane == 0) {
            __threadfence();
            atomicExch(state, LB_PRE | agg);
        }
        return 0;
    }
    long long base = (long long)cta - 1;
    while (true) {
        const long long p = base - lane;
        unsigned long long v = LB_PRE;   // lanes before CTA 0 act as prefix 0
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
    return excl;
}

}  // namespace fzlb
