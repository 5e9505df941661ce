// FP64 pipe microbenchmark (context for the roofline; not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fp64_peak scripts/fp64_peak.cu
// Measures: DADD throughput (independent chains), DMUL throughput, and the per-split
// sequence of the DP (T1, T3a, DSETP, selects, coefficient adds, DMUL, 2 DADD, DSETP,
// min/argmin selects) with TE independent splits per step.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dadd(double *out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
            x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dmul(double *out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a);
            x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, a); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, a);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// Dependent-chain latency of DADD (one thread).
__global__ void k_dadd_lat(double *out, int iters, double a) {
    double x = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) x = __dadd_rn(x, a);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int TE>
__global__ void k_split(double *out, int iters, const double *src) {
    double LT1[TE], LT3[TE], LTS[TE], LC1[TE], best[TE];
    int widx[TE];
#pragma unroll
    for (int t = 0; t < TE; ++t) {
        LT1[t] = src[t] + threadIdx.x; LT3[t] = src[t + 8]; LTS[t] = src[t + 16] + 0.001 * threadIdx.x; LC1[t] = 3 + t;
        best[t] = 1e300; widx[t] = 0;
    }
    double xT1 = src[24], xT3 = src[25], xTS = src[26], xr = src[27], c3 = 6.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < TE; ++t) {
            const double T1 = __dadd_rn(LT1[t], xT1);
            const double T3a = __dadd_rn(LT3[t], xT1);
            const bool left = LTS[t] >= xTS;
            const double cL = __dadd_rn(c3, LC1[t]);
            const double cR = t == 0 ? xr : __dadd_rn(xr, (double)(4 * t));
            const double ts = left ? LTS[t] : xTS;
            const double T3 = left ? T3a : xT3;
            const double c = __hiloint2double(left ? __double2hiint(cL) : __double2hiint(cR), 0);
            const double tot = __dadd_rn(__dadd_rn(T1, __dmul_rn(c, ts)), T3);
            const bool upd = tot <= best[t];
            best[t] = upd ? tot : best[t];
            widx[t] = upd ? i : widx[t];
        }
        c3 = __dadd_rn(c3, 3.0);
        xTS = __dadd_rn(xTS, 1e-9);
    }
    double s = 0;
    int w = 0;
#pragma unroll
    for (int t = 0; t < TE; ++t) { s += best[t]; w += widx[t]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + w;
}

int main() {
    double *out, *src;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
    cudaMalloc(&src, 64 * sizeof(double));
    double h[64];
    for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 0.25;
    cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int blocks = 148 * 4, threads = warps * 32 / 4;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_dadd<<<blocks, threads>>>(out, iters, 1e-9);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters * 64;
        printf("DADD warps/SM=%d: %.3f ms, %.2f T inst/s\n", warps, ms, ops / ms / 1e9);
        cudaEventRecord(a);
        k_dmul<<<blocks, threads>>>(out, iters, 1.0000001);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("DMUL warps/SM=%d: %.3f ms, %.2f T inst/s\n", warps, ms, ops / ms / 1e9);
    }
    {
        cudaEventRecord(a);
        k_dadd_lat<<<1, 32>>>(out, iters, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("DADD latency ~ %.2f ns per dependent op (%.1f cycles at max clock %d kHz)\n",
               ms * 1e6 / (iters * 16.0), ms * 1e6 / (iters * 16.0) * clk * 1e-6, clk);
    }
    for (int warps = 8; warps <= 32; warps *= 2) {
        const int blocks = 148 * 4, threads = warps * 32 / 4;
        float ms;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_split<4><<<blocks, threads>>>(out, iters, src);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        double splits = (double)blocks * threads * iters * 4;
        printf("split TE=4 warps/SM=%d: %.2f G splits/s = %.1f%% of 7-instr FP64 roofline (18.61 T)\n", warps,
               splits / ms / 1e6, 100.0 * splits * 7 / (ms * 1e-3) / 18.61248e12);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_split<8><<<blocks, threads>>>(out, iters, src);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        splits = (double)blocks * threads * iters * 8;
        printf("split TE=8 warps/SM=%d: %.2f G splits/s = %.1f%% of 7-instr FP64 roofline (18.61 T)\n", warps,
               splits / ms / 1e6, 100.0 * splits * 7 / (ms * 1e-3) / 18.61248e12);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
