// Dependent-chain latency microbenchmarks (cycles per op) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define N 4096
__global__ void k_dadd(double* o, double x, long long* cyc) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __dadd_rn(a, b); b = __dadd_rn(b, a); }
    long long t1 = clock64();
    o[threadIdx.x] = a + b; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (2 * N);
}
__global__ void k_dmul(double* o, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __dmul_rn(a, 1.0000001); }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_f2f(double* o, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { float f = __double2float_rn(a); a = (double)f + 1e-9; }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_frnd(double* o, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = rint(a) + 0.25; }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_fadd(float* o, float x, long long* cyc) {
    float a = x, b = x * 0.5f;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __fadd_rn(a, b); b = __fadd_rn(b, a); }
    long long t1 = clock64();
    o[threadIdx.x] = a + b; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (2 * N);
}
__global__ void k_shfl(float* o, float x, long long* cyc) {
    float a = x + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __shfl_up_sync(0xffffffffu, a, 1) + 1.0f; }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_bar(float* o, float x, long long* cyc) {
    __shared__ float s[1024];
    float a = x;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { s[threadIdx.x] = a; __syncthreads(); a = s[(threadIdx.x + 32) & (blockDim.x - 1)] + 1.f; }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
__global__ void k_ddiv(double* o, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; i++) { a = __ddiv_rn(a, 1.0000001) + 1e-300; }
    long long t1 = clock64();
    o[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (N / 16);
}
__global__ void k_dadd_tp(double* o, double x, long long* cyc) {
    double a = x, b = x * 0.5, c2 = x * 0.25, d = x * 0.125;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __dadd_rn(a, 1e-7); b = __dadd_rn(b, 1e-7); c2 = __dadd_rn(c2, 1e-7); d = __dadd_rn(d, 1e-7); }
    long long t1 = clock64();
    o[threadIdx.x] = a + b + c2 + d; if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 100 / (4 * N);
}
__global__ void k_fadd_tp(float* o, float x, long long* cyc) {
    float a = x, b = x * 0.5f, c2 = x * 0.25f, d = x * 0.125f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { a = __fadd_rn(a, 1e-7f); b = __fadd_rn(b, 1e-7f); c2 = __fadd_rn(c2, 1e-7f); d = __fadd_rn(d, 1e-7f); }
    long long t1 = clock64();
    o[threadIdx.x] = a + b + c2 + d; if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 100 / (4 * N);
}
__global__ void k_f2f_tp(double* o, double x, long long* cyc) {
    double a = x, b = x * 0.5;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; i++) { float f = __double2float_rn(a); float g = __double2float_rn(b); a = (double)f; b = (double)g; }
    long long t1 = clock64();
    o[threadIdx.x] = a + b; if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 100 / (2 * N);
}
int main() {
    double* od; float* of; long long* c; long long h;
    cudaMalloc(&od, 8192); cudaMalloc(&of, 8192); cudaMalloc(&c, 8);
    auto run = [&](const char* name, auto launch) { launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-28s %lld cycles\n", name, h); };
    run("DADD dep chain", [&] { k_dadd<<<1, 32>>>(od, 1.0, c); });
    run("DMUL dep chain", [&] { k_dmul<<<1, 32>>>(od, 1.0, c); });
    run("F2F f64->f32->f64 + DADD", [&] { k_f2f<<<1, 32>>>(od, 1.0, c); });
    run("FRND + DADD", [&] { k_frnd<<<1, 32>>>(od, 1.0, c); });
    run("DDIV (IEEE) + DADD", [&] { k_ddiv<<<1, 32>>>(od, 1.0, c); });
    run("FADD dep chain", [&] { k_fadd<<<1, 32>>>(of, 1.0f, c); });
    run("SHFL.UP + FADD", [&] { k_shfl<<<1, 32>>>(of, 1.0f, c); });
    run("STS+BAR(256)+LDS+FADD", [&] { k_bar<<<1, 256>>>(of, 1.0f, c); });
    run("STS+BAR(64)+LDS+FADD", [&] { k_bar<<<1, 64>>>(of, 1.0f, c); });
    run("DADD chain, 8 warps/SMSP", [&] { k_dadd<<<1, 1024>>>(od, 1.0, c); });
    run("DADD x4 indep, 1 warp (x100)", [&] { k_dadd_tp<<<1, 32>>>(od, 1.0, c); });
    run("DADD x4 indep, 4 warps (x100)", [&] { k_dadd_tp<<<1, 128>>>(od, 1.0, c); });
    run("DADD x4 indep, 16 warps (x100)", [&] { k_dadd_tp<<<1, 512>>>(od, 1.0, c); });
    run("DADD x4 indep, 32 warps (x100)", [&] { k_dadd_tp<<<1, 1024>>>(od, 1.0, c); });
    run("FADD x4 indep, 32 warps (x100)", [&] { k_fadd_tp<<<1, 1024>>>(of, 1.0f, c); });
    run("F2F pair, 1 warp (x100)", [&] { k_f2f_tp<<<1, 32>>>(od, 1.0, c); });
    run("F2F pair, 16 warps (x100)", [&] { k_f2f_tp<<<1, 512>>>(od, 1.0, c); });
    return 0;
}
