// probe.cu -- measurement probes for the B200 (sm_100a), not part of the method:
//   mhdp_probe_fp64_peak  : FP64 FMA throughput (flop/s) of the whole GPU, SIMT DFMA pipes
//                           ("FP64 peak is not in MP. Measure it")
//   mhdp_probe_latencies  : cycles of the dependency steps the coarse triangular solve
//                           (K8) is built from: dependent DFMA, the Markstein division,
//                           a warp shuffle broadcast, a shared-memory flag round trip
//                           between two warps of one CTA and a global-memory flag round
//                           trip between two CTAs on different SMs.
//   mhdp_probe_pivot_div  : PivotDiv (k2_common.cuh: the multipliers of K6 / K7) applied to
//                           caller-supplied numerators and pivots, for the test that pins it
//                           to the IEEE quotient (tests/test_gpu_edge.py)
// Built by paper_2104_14855_b200/build_lib.py into tools/libprobe.so; bench.py reports
// the FP64 peak next to the K6 / K7 flop rates.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2104_14855_b200/csrc/k2_common.cuh"   // PivotDiv (header-only use)

namespace {

__global__ void __launch_bounds__(256) k_fma_peak(double *out, int iters, double seed) {
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = seed + threadIdx.x * 1e-9 + q;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = fma(a[q], m, c);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += a[q];
    if (s == 12345.678) out[0] = s;   // never true; keeps the chains alive
}

__global__ void k_lat(long long *cyc, double *sink, int n, double y) {
    // 0: dependent DFMA   1: Markstein division step (3 dependent ops)
    // 2: shfl broadcast chain (+ DFMA)   3: IEEE division (operator /)
    const int lane = threadIdx.x & 31;
    double z = 1.0 + lane * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) z = fma(z, 0.9999999, 1e-9);
    long long t1 = clock64();
    const double u = 1.0 / y;
    for (int i = 0; i < n; ++i) {
        const double q = z * y;
        const double r = fma(-q, u, z);
        z = fma(r, y, q) + 1e-300;
    }
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) z = fma(__shfl_sync(0xffffffffu, z, i & 31), 0.9999999, 1e-9);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) z = z / u + 1e-300;
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
    }
    sink[threadIdx.x] = z;
}

// two warps of one CTA ping-pong through a shared-memory word
__global__ void k_smem_pingpong(long long *cyc, int n) {
    __shared__ volatile int flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    if (lane == 0) {
        for (int i = 0; i < n; ++i) {
            if (w == 0) { while (flag != 2 * i) {} flag = 2 * i + 1; }
            else        { while (flag != 2 * i + 1) {} flag = 2 * i + 2; }
        }
    }
    __syncwarp();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
}

// two CTAs ping-pong through a global word (acquire / release at gpu scope)
__global__ void k_gmem_pingpong(long long *cyc, int *flag, int n) {
    if (threadIdx.x != 0) return;
    const int b = blockIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const int want = 2 * i + b;
        int v;
        do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        } while (v != want);
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(want + 1) : "memory");
    }
    long long t1 = clock64();
    if (b == 0) cyc[5] = t1 - t0;
}

}  // namespace

namespace {
__global__ void __launch_bounds__(256) k_pivot_div(const double *__restrict__ x, int n, const double *__restrict__ piv,
                                                   double *__restrict__ out) {
    const mhdp::PivotDiv dv(piv[blockIdx.x]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[(size_t)blockIdx.x * n + i] = dv(x[i]);
}
}  // namespace

extern "C" {

// FP64 FMA throughput in flop/s (2 per FMA); returns < 0 on a CUDA error
double mhdp_probe_fp64_peak(int device) {
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return -1;
    const int iters = 4096, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma_peak<<<blocks, 256>>>(out, 64, 1.0);   // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_fma_peak<<<blocks, 256>>>(out, iters, 1.0 + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return -1;
    const double flops = 2.0 * 8.0 * iters * 256.0 * blocks;
    return flops / (best * 1e-3);
}

// cycles per step: out[0] dependent DFMA, [1] Markstein division step, [2] shfl + DFMA,
// [3] IEEE division, [4] smem flag round trip (two warps), [5] global flag round trip
// (two CTAs).  Returns 0 on success.
int mhdp_probe_latencies(int device, double *out) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    long long *cyc = nullptr;
    double *sink = nullptr;
    int *flag = nullptr;
    if (cudaMalloc(&cyc, 8 * sizeof(long long)) || cudaMalloc(&sink, 64 * sizeof(double)) ||
        cudaMalloc(&flag, sizeof(int)))
        return 2;
    const int n = 4096, np = 2048;
    k_lat<<<1, 32>>>(cyc, sink, n, 1.2345);
    k_lat<<<1, 32>>>(cyc, sink, n, 1.2345);
    k_smem_pingpong<<<1, 64>>>(cyc, np);
    cudaMemset(flag, 0, sizeof(int));
    k_gmem_pingpong<<<2, 32>>>(cyc, flag, np);
    long long h[6];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const int err = cudaGetLastError() != cudaSuccess;
    cudaFree(cyc); cudaFree(sink); cudaFree(flag);
    if (err) return 3;
    for (int i = 0; i < 4; ++i) out[i] = (double)h[i] / n;
    out[4] = (double)h[4] / np;   // one round trip = two flag handoffs
    out[5] = (double)h[5] / np;
    return 0;
}

// out[j * n + i] = PivotDiv(piv[j])(x[i]) for n numerators and m pivots (host arrays)
int mhdp_probe_pivot_div(int device, const double *x, int n, const double *piv, int m, double *out) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    double *dx = nullptr, *dp = nullptr, *dout = nullptr;
    if (cudaMalloc(&dx, sizeof(double) * n) != cudaSuccess || cudaMalloc(&dp, sizeof(double) * m) != cudaSuccess ||
        cudaMalloc(&dout, sizeof(double) * (size_t)n * m) != cudaSuccess)
        return 2;
    cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, piv, sizeof(double) * m, cudaMemcpyHostToDevice);
    k_pivot_div<<<(unsigned)m, 256>>>(dx, n, dp, dout);
    cudaMemcpy(out, dout, sizeof(double) * (size_t)n * m, cudaMemcpyDeviceToHost);
    const int err = cudaGetLastError() != cudaSuccess;
    cudaFree(dx); cudaFree(dp); cudaFree(dout);
    return err ? 3 : 0;
}

}  // extern "C"
