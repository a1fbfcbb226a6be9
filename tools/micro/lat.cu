#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
template <int T>
__global__ void k(double *out, long long *cyc, int n) {
    __shared__ double sm[1024];
    const int lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < 1024; e += 32) sm[e] = 1.0 / (e + 1);
    __syncwarp();
    double a0 = 1 + lane, a1 = 2, a2 = 3, a3 = 4, a4 = 5, a5 = 6, a6 = 7, a7 = 8;
    int idx = lane;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (T == 0) { a0 = fma(a0, 0.999, 1e-9); }
        if (T == 1) { a0 = fma(a0, 0.999, 1e-9); a1 = fma(a1, 0.999, 1e-9); a2 = fma(a2, 0.999, 1e-9); a3 = fma(a3, 0.999, 1e-9); }
        if (T == 2) { a0 = fma(a0, 0.999, 1e-9); a1 = fma(a1, 0.999, 1e-9); a2 = fma(a2, 0.999, 1e-9); a3 = fma(a3, 0.999, 1e-9);
                      a4 = fma(a4, 0.999, 1e-9); a5 = fma(a5, 0.999, 1e-9); a6 = fma(a6, 0.999, 1e-9); a7 = fma(a7, 0.999, 1e-9); }
        if (T == 3) { a0 = __shfl_sync(FULL, a0, (lane + 1) & 31); }
        if (T == 4) { a0 = __shfl_sync(FULL, a0, (lane + 1) & 31); a1 = __shfl_sync(FULL, a1, (lane + 1) & 31);
                      a2 = __shfl_sync(FULL, a2, (lane + 1) & 31); a3 = __shfl_sync(FULL, a3, (lane + 1) & 31); }
        if (T == 5) { idx = (int)sm[idx & 1023] + ((lane + i) & 511); }
        if (T == 6) { a0 = a0 * 1.0000001; }
        if (T == 7) { float f = __int_as_float(idx); f = __shfl_sync(FULL, f, (lane + 1) & 31); idx = __float_as_int(f) + 1; }
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
    out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + idx;
}
template <int T> void run(const char *name) {
    double *out; long long *cyc; cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 8);
    const int n = 100000;
    k<T><<<1, 32>>>(out, cyc, n); k<T><<<1, 32>>>(out, cyc, n);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s: %.2f cycles per iteration\n", name, (double)h / n);
}
int main() {
    run<0>("1 dependent DFMA");
    run<1>("4 independent DFMA chains");
    run<2>("8 independent DFMA chains");
    run<3>("1 dependent SHFL (64-bit)");
    run<4>("4 independent SHFL (64-bit) chains");
    run<5>("dependent LDS.64 (+cvt)");
    run<6>("1 dependent DMUL");
    run<7>("1 dependent SHFL (32-bit)");
    return 0;
}
