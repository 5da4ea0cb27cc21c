// Dev microbenchmark (sm_100a): per-SM throughput of the instructions the softmax warps of K2 issue -- MUFU ex2 in its
// f32 / f16x2 / bf16x2 forms, the packed f32->bf16/f16 conversions, packed FMA, 3-input max -- alone and in the mixes a
// tile body uses, at 1, 2 and 4 warps per scheduler.  Results are "elements per clock per SM" from clock64 on one SM
// (independent of the DVFS state).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define R 16  // independent registers per thread

template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, long long* clk, int iters, float seed) {
    float a[R];
    unsigned u[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        a[i] = seed * (threadIdx.x + i) * 1e-3f - 1.0f;
        u[i] = __float_as_uint(a[i]);
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // ex2.f32
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        } else if (MODE == 1) {  // ex2.f16x2
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
        } else if (MODE == 2) {  // ex2.bf16x2
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
        } else if (MODE == 3) {  // cvt.rn.bf16x2.f32 (F2FP)
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) % R]));
#pragma unroll
            for (int i = 0; i < R; ++i) a[i] = __uint_as_float(u[i] ^ 0x3f000000u);
        } else if (MODE == 4) {  // cvt.rn.f16x2.f32
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) % R]));
#pragma unroll
            for (int i = 0; i < R; ++i) a[i] = __uint_as_float(u[i] ^ 0x3f000000u);
        } else if (MODE == 5) {  // fma.rn.f32x2
#pragma unroll
            for (int i = 0; i < R; i += 2)
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %2}; mov.b64 z, {%3, %3};\n\t"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "+f"(a[i]), "+f"(a[i + 1]) : "f"(seed), "f"(0.25f));
        } else if (MODE == 6) {  // 3-input max
#pragma unroll
            for (int i = 0; i < R; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) % R]), "f"(a[(i + 2) % R]));
        } else if (MODE == 7) {  // tile body, no bias: per 2 elems FFMA2 + 2 MUFU + F2FP (+ result feeds back)
#pragma unroll
            for (int i = 0; i < R; i += 2) {
                float x0, x1;
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "=f"(x0), "=f"(x1) : "f"(a[i]), "f"(a[i + 1]), "f"(seed), "f"(-0.25f));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(x0), "f"(x1));
            }
#pragma unroll
            for (int i = 0; i < R; i += 2) a[i] = __uint_as_float(u[i] & 0x3fffffffu);
        } else if (MODE == 8) {  // tile body with f16x2 exp: per 2 elems FFMA2 + F2FP(f16x2) + 1 MUFU.f16x2
#pragma unroll
            for (int i = 0; i < R; i += 2) {
                float x0, x1;
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "=f"(x0), "=f"(x1) : "f"(a[i]), "f"(a[i + 1]), "f"(seed), "f"(-0.25f));
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(x0), "f"(x1));
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
            }
#pragma unroll
            for (int i = 0; i < R; i += 2) a[i] = __uint_as_float(u[i] & 0x3fffffffu);
        } else if (MODE == 9) {  // tile body, bf16x2 exp
#pragma unroll
            for (int i = 0; i < R; i += 2) {
                float x0, x1;
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "=f"(x0), "=f"(x1) : "f"(a[i]), "f"(a[i + 1]), "f"(seed), "f"(-0.25f));
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(x0), "f"(x1));
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
            }
#pragma unroll
            for (int i = 0; i < R; i += 2) a[i] = __uint_as_float(u[i] & 0x3fffffffu);
        } else if (MODE == 10) {  // MUFU f32 with integer-pipe bf16 rounding (PRMT) instead of F2FP
#pragma unroll
            for (int i = 0; i < R; i += 2) {
                float x0, x1;
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "=f"(x0), "=f"(x1) : "f"(a[i]), "f"(a[i + 1]), "f"(seed), "f"(-0.25f));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                u[i] = __byte_perm(__float_as_uint(x0) + 0x8000u, __float_as_uint(x1) + 0x8000u, 0x7632);
            }
#pragma unroll
            for (int i = 0; i < R; i += 2) a[i] = __uint_as_float(u[i] & 0x3fffffffu);
        } else if (MODE == 11) {  // packed polynomial 2^x on the FMA pipe (f32x2): 3 add/sub + 3 fma per pair + 2 LEA-ish
#pragma unroll
            for (int i = 0; i < R; i += 2) {
                asm volatile(
                    "{.reg .b64 x, t, n, f, p, c, m; .reg .b32 t0, t1, p0, p1;\n\t"
                    "mov.b64 x, {%0, %1}; mov.b64 m, {%2, %2};\n\t"
                    "add.rn.f32x2 t, x, m;\n\t"
                    "sub.rn.f32x2 n, t, m;\n\t"
                    "sub.rn.f32x2 f, x, n;\n\t"
                    "mov.b64 c, {%3, %3}; mov.b64 p, {%4, %4};\n\t"
                    "fma.rn.f32x2 p, p, f, c;\n\t"
                    "mov.b64 c, {%5, %5};\n\t"
                    "fma.rn.f32x2 p, p, f, c;\n\t"
                    "mov.b64 c, {%6, %6};\n\t"
                    "fma.rn.f32x2 p, p, f, c;\n\t"
                    "mov.b64 {t0, t1}, t; mov.b64 {p0, p1}, p;\n\t"
                    "shl.b32 t0, t0, 23; shl.b32 t1, t1, 23; add.u32 p0, p0, t0; add.u32 p1, p1, t1;\n\t"
                    "mov.b32 %0, p0; mov.b32 %1, p1;}"
                    : "+f"(a[i]), "+f"(a[i + 1])
                    : "f"(12582912.0f), "f"(0.242611319f), "f"(0.0551717501f), "f"(0.693260968f), "f"(0.999928057f));
                a[i] -= 1.5f;
                a[i + 1] -= 1.5f;
            }
        }
    }
    const long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) s += a[i] + __uint_as_float(u[i] & 0x3fffffffu);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MODE>
void run(const char* name, double elems_per_iter_per_thread) {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 8);
    const int iters = 2048;
    printf("%-44s", name);
    for (int warps = 4; warps <= 16; warps *= 2) {
        k<MODE><<<148, warps * 32>>>(out, clk, iters, 0.5f);
        k<MODE><<<148, warps * 32>>>(out, clk, iters, 0.5f);
        long long c = 0;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double el = (double)iters * elems_per_iter_per_thread * warps * 32;
        printf("  w/SMSP=%d: %6.2f el/clk/SM", warps / 4, el / (double)c);
    }
    printf("\n");
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    run<0>("ex2.approx.ftz.f32", R);
    run<1>("ex2.approx.f16x2 (2 el/op)", 2 * R);
    run<2>("ex2.approx.ftz.bf16x2 (2 el/op)", 2 * R);
    run<3>("cvt.rn.bf16x2.f32 (2 el/op, + 1 LOP)", 2 * R);
    run<4>("cvt.rn.f16x2.f32 (2 el/op, + 1 LOP)", 2 * R);
    run<5>("fma.rn.f32x2 (2 el/op)", R);
    run<6>("max.f32 3-input (2 el/op)", 2 * R);
    run<7>("body: FFMA2 + 2 ex2.f32 + cvt.bf16x2", R);
    run<8>("body: FFMA2 + cvt.f16x2 + ex2.f16x2", R);
    run<9>("body: FFMA2 + cvt.bf16x2 + ex2.bf16x2", R);
    run<10>("body: FFMA2 + 2 ex2.f32 + PRMT rounding", R);
    run<11>("poly 2^x f32x2 (FMA pipe)", R);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
