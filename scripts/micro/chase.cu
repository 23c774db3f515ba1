// Dependent-load latency for the 1D walker's access pattern: one warp jumps
// ~180 KB per step through a 1.1 GB array and loads a 4 KB block (8 x 16 B
// per lane), the next address depending on the loaded data.  Variants: cold
// (DRAM), after an L2 prefetch of the whole path, and a 2 MB L2-resident ring.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chase(const float* __restrict__ x, long long n, long long stride, int steps, int mode,
                      long long* out) {
    const int lane = threadIdx.x;
    long long pos = 0;
    float acc = 0.f;
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) {
        const float4* p = reinterpret_cast<const float4*>(x + pos);
        float s = 0.f;
        if (mode == 0) {
#pragma unroll
            for (int e = 0; e < 8; e++) { float4 q = __ldg(p + e * 32 + lane); s += q.x + q.w; }
        } else {
            float4 q = __ldcg(p + lane); s = q.x;
        }
        // data-dependent next position (s is ~0 for the zero-filled array)
        acc += s;
        pos += stride + (long long)(s * 0.f);
        if (pos + 1024 > n) pos = 0;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = (t1 - t0) / steps; out[1] = (long long)acc; }
}
__global__ void prefetch_all(const float* x, long long n) {
    for (long long q = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 32; q < n; q += (long long)gridDim.x * blockDim.x * 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + q));
}
int main() {
    long long n = 280953867ll;
    float* x; cudaMalloc(&x, n * 4); cudaMemset(x, 0, n * 4);
    long long* o; cudaMalloc(&o, 16); long long h[2];
    const long long strides[3] = {45056, 1024, 256};
    for (int si = 0; si < 3; si++) {
        long long stride = strides[si];
        int steps = 4000;
        // cold: flush L2 by touching another 512 MB
        float* junk; cudaMalloc(&junk, 512ll << 20); cudaMemset(junk, 1, 512ll << 20);
        chase<<<1, 32>>>(x, n, stride, steps, 0, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("stride %lld floats: 4KB block load, cold  : %lld cycles/step\n", stride, h[0]);
        chase<<<1, 32>>>(x, n, stride, steps, 0, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("stride %lld floats: 4KB block load, rerun : %lld cycles/step (footprint %lld MB)\n", stride, h[0], steps * stride * 4 >> 20);
        cudaMemset(junk, 1, 512ll << 20);
        chase<<<1, 32>>>(x, n, stride, steps, 1, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("stride %lld floats: 512B ldcg, cold       : %lld cycles/step\n", stride, h[0]);
        chase<<<1, 32>>>(x, n, stride, steps, 1, o); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("stride %lld floats: 512B ldcg, rerun      : %lld cycles/step\n", stride, h[0]);
        cudaFree(junk);
    }
    return 0;
}
