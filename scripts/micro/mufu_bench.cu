// Dev microbenchmark: per-SM throughput of ex2 variants and an FMA-pipe 2^x polynomial (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters, float seed) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-3f - 1.0f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {  // ex2.approx.ftz.f32
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            } else if (MODE == 1) {  // f16x2
                unsigned u = __float_as_uint(a[i]);
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u));
                a[i] = __uint_as_float(u);
            } else if (MODE == 2) {  // bf16x2
                unsigned u = __float_as_uint(a[i]);
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u));
                a[i] = __uint_as_float(u);
            } else if (MODE == 3) {  // FFMA 3-reg chain
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(seed), "f"(a[(i + 1) & 7]));
            } else if (MODE == 4) {  // polynomial 2^x, x in [-30, 0]: 3 FADD + 3 FFMA + shift-add
                float x = a[i];
                float t = x + 12582912.0f;
                float nf = t - 12582912.0f;
                float f = x - nf;
                float p = fmaf(f, 0.0555041f, 0.2402265f);
                p = fmaf(p, f, 0.6931472f);
                p = fmaf(p, f, 1.0f);
                a[i] = __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23)) - 1.5f;
            } else if (MODE == 5) {  // mixed: 6 MUFU + 2 poly per 8
                if (i < 6) {
                    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                    a[i] -= 1.5f;
                } else {
                    float x = a[i];
                    float t = x + 12582912.0f;
                    float nf = t - 12582912.0f;
                    float f = x - nf;
                    float p = fmaf(f, 0.0555041f, 0.2402265f);
                    p = fmaf(p, f, 0.6931472f);
                    p = fmaf(p, f, 1.0f);
                    a[i] = __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23)) - 1.5f;
                }
            } else if (MODE == 6) {  // MUFU + FFMA + F2FP realistic per-elem mix (ex2, fma, cvt pack every 2)
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                a[i] = fmaf(a[i], seed, -1.5f);
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int per_elem) {
    float* out;
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        k<MODE><<<148, warps * 32>>>(out, iters, 0.5f);
        cudaEventRecord(e0);
        k<MODE><<<148, warps * 32>>>(out, iters, 0.5f);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)iters * 8 * warps * 32 * per_elem;  // per SM
        double clk = ms * 1e-3 * 1.965e9;
        printf("%-28s warps/SM=%2d  %.2f results/clk/SM (assuming 1965 MHz)  %.3f ms\n", name, warps, ops / clk, ms);
    }
    cudaFree(out);
}

int main() {
    run<0>("ex2.approx.ftz.f32", 1);
    run<1>("ex2.approx.f16x2 (2/op)", 2);
    run<2>("ex2.approx.ftz.bf16x2 (2/op)", 2);
    run<3>("fma.rn.f32 3-reg", 1);
    run<4>("poly 2^x (FMA pipe)", 1);
    run<5>("mixed 6 MUFU + 2 poly", 1);
    run<6>("ex2 + ffma", 1);
    return 0;
}
