// Microbenchmark of the W-kernel inner step (TE = 4 register tile, ring min, flush test)
// with alternative instruction mixes for the same exact arithmetic.  Context tool only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o build/split_variants scripts/mb/split_variants.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double4 ldg4(const double4 *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p)), b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

constexpr int TE = 4;

__device__ __forceinline__ double hi_c(double cL, double cR, bool left) {
    return __hiloint2double(left ? __double2hiint(cL) : __double2hiint(cR), 0);
}

// V0: as oob_wave_w.cuh (coefficients in binary64, hi-word select)
__device__ __forceinline__ double tot_v0(double LT1, double LT3, double LTS, double cL, double RT1, double RT3,
                                         double RTS, double cR) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double ts = left ? LTS : RTS;
    const double T3 = left ? T3a : RT3;
    const double c = hi_c(cL, cR, left);
    return __dadd_rn(__dadd_rn(T1, __dmul_rn(c, ts)), T3);
}
// V2: both products, select T2 and T3
__device__ __forceinline__ double tot_v2(double LT1, double LT3, double LTS, double cL, double RT1, double RT3,
                                         double RTS, double cR) {
    const double T1 = __dadd_rn(LT1, RT1);
    const double T3a = __dadd_rn(LT3, RT1);
    const bool left = LTS >= RTS;
    const double T2 = left ? __dmul_rn(cL, LTS) : __dmul_rn(cR, RTS);
    const double T3 = left ? T3a : RT3;
    return __dadd_rn(__dadd_rn(T1, T2), T3);
}
// float coefficient -> binary64 high word (exact for integers < 2^21)
__device__ __forceinline__ double f2d_int(float f) {
    return __hiloint2double((int)((__float_as_uint(f) >> 3) + 0x38000000u), 0);
}

template <int V, bool GX = false, int FSTR = 5, int PASS = 0>
__global__ void __launch_bounds__(256, 2) k_step(const double4 *stream, int nsteps, double *out) {
    __shared__ double4 sx[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sx[i] = stream[i];
    __shared__ unsigned filt[1024];
    __shared__ ulonglong2 cas_arr[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cas_arr[i] = make_ulonglong2(~0ull, ~0ull);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) filt[i] = 0u;   // nothing passes
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double RT1[TE], RT3[TE], RTS[TE], RC1[TE];
    float RC1f[TE];
#pragma unroll
    for (int t = 0; t < TE; ++t) {
        RT1[t] = 10.0 + lane + t; RT3[t] = 5.0 + t; RTS[t] = 3.0 + 0.01 * lane + 0.1 * t; RC1[t] = 2.0 + t;
        RC1f[t] = 2.0f + t;
    }
    double best[TE];
    int widx[TE];
#pragma unroll
    for (int t = 0; t < TE; ++t) { best[t] = 1e300; widx[t] = 0; }
    double cst = 3.0;
    float cstf = 3.0f;
    const double xadd = 4.0 * lane;
    const float xaddf = 4.0f * lane;
    int acc = 0;
    double4 x = GX ? ldg4(stream) : sx[0];
    for (int blk = 0; blk < nsteps; blk += TE) {
#pragma unroll
        for (int I = 0; I < TE; ++I) {
            const double4 nx = GX ? ldg4(stream + ((blk + I + 1) & 255)) : sx[(blk + I + 1) & 255];
            const double xc = __dadd_rn(x.w, xadd);
            const float xcf = (float)(blk + I) + xaddf;
#pragma unroll
            for (int t = 0; t < TE; ++t) {
                const int sl = (I + t) % TE;
                double tot;
                if (V == 0) {
                    const double cs = t == 0 ? xc : __dadd_rn(xc, (double)(4 * t));
                    const double ct = __dadd_rn(RC1[t], cst);
                    tot = tot_v0(RT1[t], RT3[t], RTS[t], ct, x.x, x.y, x.z, cs);
                } else if (V == 1) {   // float coefficients
                    const float csf = t == 0 ? xcf : xcf + (float)(4 * t);
                    const float ctf = RC1f[t] + cstf;
                    const double T1 = __dadd_rn(RT1[t], x.x);
                    const double T3a = __dadd_rn(RT3[t], x.x);
                    const bool left = RTS[t] >= x.z;
                    const double ts = left ? RTS[t] : x.z;
                    const double T3 = left ? T3a : x.y;
                    const double c = f2d_int(left ? ctf : csf);
                    tot = __dadd_rn(__dadd_rn(T1, __dmul_rn(c, ts)), T3);
                } else {
                    const double cs = t == 0 ? xc : __dadd_rn(xc, (double)(4 * t));
                    const double ct = __dadd_rn(RC1[t], cst);
                    tot = tot_v2(RT1[t], RT3[t], RTS[t], ct, x.x, x.y, x.z, cs);
                }
                if (t == TE - 1) { best[sl] = tot; widx[sl] = t; }
                else {
                    const bool upd = tot <= best[sl];
                    best[sl] = upd ? tot : best[sl];
                    widx[sl] = upd ? t : widx[sl];
                }
            }
            cst = __dadd_rn(cst, 3.0);
            cstf += 3.0f;
            const unsigned bh = (unsigned)__double2hiint(best[I]);
            const int fi = (lane * FSTR + blk + I) & 1023;
            if (PASS == 0) {
                if (bh <= filt[fi]) acc += widx[I];   // never taken
            } else {
                // pass with probability PASS/1024 per lane (hash of the step), then a 128-bit
                // shared CAS loop as in the real flush
                const unsigned hsh = (unsigned)(blk + I) * 2654435761u ^ (unsigned)lane * 40503u;
                if (((hsh >> 7) & 1023u) < (unsigned)PASS || bh <= filt[fi]) {
                    const unsigned addr = (unsigned)__cvta_generic_to_shared(cas_arr + (fi & 255));
                    unsigned long long cx, cy;
                    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(cx), "=l"(cy) : "r"(addr) : "memory");
                    const unsigned long long bb = (unsigned long long)__double_as_longlong(best[I]);
                    const unsigned key = (unsigned)widx[I];
                    while (bb < cx || (bb == cx && key < (unsigned)cy)) {
                        unsigned long long ox, oy;
                        asm volatile("{\n\t.reg .b128 d, c, v;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
                                     "atom.shared.cas.b128 d, [%6], c, v;\n\tmov.b128 {%0, %1}, d;\n\t}"
                                     : "=l"(ox), "=l"(oy) : "l"(cx), "l"(cy), "l"(bb), "l"((unsigned long long)key), "r"(addr) : "memory");
                        if (ox == cx && oy == cy) break;
                        cx = ox; cy = oy;
                    }
                }
            }
            x = nx;
        }
    }
    double s = acc;
#pragma unroll
    for (int t = 0; t < TE; ++t) s += best[t];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double4 *st; double *out;
    cudaMalloc(&st, 256 * sizeof(double4)); cudaMalloc(&out, 148 * 2 * 256 * sizeof(double));
    double4 h[256];
    for (int i = 0; i < 256; ++i) h[i] = make_double4(7.0 + i * 0.01, 2.0 + i * 0.02, 2.9 + (i % 7) * 0.05, 3.0 + i % 5);
    cudaMemcpy(st, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int nsteps = 4096;
    const double splits = 148.0 * 2 * 256 * nsteps * TE;
    float ms;
#define RUN(V, GX, FS, PS)                                                                               \
    for (int rep = 0; rep < 2; ++rep) {                                                              \
        cudaEventRecord(a); k_step<V, GX, FS, PS><<<148 * 2, 256>>>(st, nsteps, out); cudaEventRecord(b); \
        cudaEventSynchronize(b);                                                                     \
    }                                                                                                \
    cudaEventElapsedTime(&ms, a, b);                                                                 \
    printf("V%d GX=%d FSTR=%d PASS=%d/1024: %.3f ms  %.1f G splits/s  frac = %.1f%%  cycles/warp-split = %.2f\n", V, GX, FS, PS, ms, \
           splits / ms / 1e6, 100.0 * splits * 7 / (ms * 1e-3) / 18.61248e12, 592 * 1.965e9 / (splits / 32 / (ms * 1e-3)));
    RUN(0, false, 5, 0) RUN(0, true, 4, 0) RUN(0, true, 4, 4) RUN(0, true, 4, 14) RUN(0, true, 4, 40)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
