// Dependent-chain latencies of the f64 / conversion ops the march uses (clock64, one warp).
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__global__ void k(double* out, long long* cyc, double x0) {
    double x = x0 + threadIdx.x * 1e-9;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = __dadd_rn(x, 1e-3);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = __dmul_rn(x, 1.0000001);
    t1 = clock64(); cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = __fma_rn(x, 1.0000001, 1e-7);
    t1 = clock64(); cyc[2] = t1 - t0;
    // DDIV chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = __ddiv_rn(x, 1.0000001);
    t1 = clock64(); cyc[3] = t1 - t0;
    // F2I + I2F chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) { int v = __double2int_rz(x * 1e6); x = (double)v * 1e-6 + 0.5; }
    t1 = clock64(); cyc[4] = t1 - t0;
    // floor chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = floor(x * 3.7) * 0.27 + 0.1;
    t1 = clock64(); cyc[5] = t1 - t0;
    // FADD f32 chain
    float f = (float)x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) f = __fadd_rn(f, 1e-3f);
    t1 = clock64(); cyc[6] = t1 - t0;
    // F2F f64->f32->f64
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; i++) x = (double)__double2float_rn(x) + 1e-3;
    t1 = clock64(); cyc[7] = t1 - t0;
    out[threadIdx.x] = x + f;
}
int main() {
    double* o; long long* c;
    cudaMallocManaged(&o, 32 * 8); cudaMallocManaged(&c, 16 * 8);
    k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
    const char* nm[] = {"DADD", "DMUL", "DFMA", "DDIV(__ddiv_rn)", "F2I+DMUL+I2F+DFMA", "DMUL+FLOOR+DMUL+DADD", "FADD", "F2F.F32.F64+F2F+DADD"};
    for (int i = 0; i < 8; i++) printf("%-24s %6.1f cycles/iter (loop incl.)\n", nm[i], (double)c[i] / N);
    return 0;
}
