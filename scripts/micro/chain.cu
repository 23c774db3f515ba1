// Dependent-chain latencies of the Lorenzo step's building blocks (cycles per iteration).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N 2048
__device__ __forceinline__ double rnd24(double x) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    const uint64_t r = (b + (0x0FFFFFFFull + (((uint32_t)b >> 29) & 1u))) & ~0x1FFFFFFFull;
    return __longlong_as_double((long long)r);
}
__global__ void k_int(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = rnd24(__dadd_rn(a, 1.2345e-3));
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_f2f(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = (double)__double2float_rn(__dadd_rn(a, 1.2345e-3));
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_dadd(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = __dadd_rn(a, 1.2345e-3);
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_shfl_d(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = __dadd_rn(__shfl_up_sync(0xffffffffu, a, 1), 1.0);
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_shfl_f(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = __dadd_rn((double)__shfl_up_sync(0xffffffffu, (float)a, 1), 1.0);
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_int_only(double* o, double x, long long* cyc) {
    uint64_t a = (uint64_t)threadIdx.x * 12345;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) a = (a + (0x0FFFFFFFull + (((uint32_t)a >> 29) & 1u))) & ~0x1FFFFFFFull ^ 0x1234567ull;
    long long t1 = clock64();
    o[threadIdx.x] = (double)a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_vote(double* o, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
        a = __dadd_rn(a, 1.0);
        if (!__all_sync(0xffffffffu, a < 1e300)) a = 0.0;
    }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
int main() {
    double* od; long long* c; long long h;
    cudaMalloc(&od, 8192 * 8); cudaMalloc(&c, 8);
    auto run = [&](const char* name, auto launch) { launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-36s %lld cycles\n", name, h); };
    run("DADD", [&] { k_dadd<<<1, 32>>>(od, 1.0, c); });
    run("DADD + int rnd24", [&] { k_int<<<1, 32>>>(od, 1.0, c); });
    run("DADD + F2F pair", [&] { k_f2f<<<1, 32>>>(od, 1.0, c); });
    run("int rnd24 only (+xor)", [&] { k_int_only<<<1, 32>>>(od, 1.0, c); });
    run("SHFL f64 + DADD", [&] { k_shfl_d<<<1, 32>>>(od, 1.0, c); });
    run("F2F + SHFL f32 + F2F + DADD", [&] { k_shfl_f<<<1, 32>>>(od, 1.0, c); });
    run("DADD + vote + branch", [&] { k_vote<<<1, 32>>>(od, 1.0, c); });
    run("DADD + int rnd24, 12 warps", [&] { k_int<<<1, 384>>>(od, 1.0, c); });
    run("DADD + F2F pair, 12 warps", [&] { k_f2f<<<1, 384>>>(od, 1.0, c); });
    return 0;
}
