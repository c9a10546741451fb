// Microbenchmark (not product code): FP64 DFMA and F2F.F64.F32 issue rates on this GPU,
// against FP32 FFMA -- decides whether FP64 belongs in the key / staging kernels.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void __launch_bounds__(256) k(float* out, int reps, float seed) {
    double a[8]; float f[8];
    for (int i = 0; i < 8; ++i) { a[i] = seed * (i + threadIdx.x); f[i] = seed * (i + threadIdx.x); }
    const double b = 1.0000001, c = 1e-9;
    const float bf = 1.0000001f, cf = 1e-9f;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (V == 0) a[i] = fma(a[i], b, c);
            else if (V == 1) f[i] = fmaf(f[i], bf, cf);
            else if (V == 2) a[i] += (double)f[i];           // F2F + DADD
            else a[i] = fma((double)f[i], (double)f[(i + 1) & 7], a[i]);  // 2 F2F + DFMA
        }
        if (V >= 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = f[i] * bf;
        }
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i] + f[i];
    out[blockIdx.x * 256 + threadIdx.x] = (float)s;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* nm[] = {"DFMA", "FFMA", "F2F.F64.F32 + DADD (+FMUL)", "2 F2F + DFMA (+FMUL)"};
    for (int v = 0; v < 4; ++v) {
        auto kern = v == 0 ? k<0> : v == 1 ? k<1> : v == 2 ? k<2> : k<3>;
        const int reps = 4096;
        kern<<<148 * 8, 256>>>(o, reps, 1e-3f); cudaDeviceSynchronize();
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); kern<<<148 * 8, 256>>>(o, reps, 1e-3f); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = 148.0 * 8 * 256 * reps * 8;
        printf("%-28s %.3f ms  %.2f Gop/s  %.1f per clk per SM\n", nm[v], ms, ops / ms / 1e6, ops / (ms * 1e-3) / (clk * 1e3) / 148);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
