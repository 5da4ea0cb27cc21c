// ba_common.cuh -- shared declarations for the sm_100a BinaryAttention kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "binattn_cuda.h"

namespace ba {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Device-side view of one forward call (all pointers device pointers).
struct FwdArgs {
    const void* V;            // [BH, N, d] in_dtype
    const uint64_t* q_words;  // [BH, N, W64]
    const uint64_t* k_words;  // [BH, N, W64]
    const float* mu_q;        // [BH]
    const float* mu_k;        // [BH]
    const unsigned char* k_exp;  // [BH, ceil(N/64), KPAD/16, 64, 16] e4m3 +-1.0 bytes of K in UMMA tile order (second-generation
                                 // tcgen05 kernel only; nullptr when the workspace has no room for it)
    const unsigned char* q_exp;  // [BH, ceil(N/256), 2, KPAD/16, 128, 16] the same for Q in 128-row tiles, two per unit
    const void* bias;         // dense: [bias_heads, N, bias_ld]; rel1d: [bias_heads, 2N-1]; or nullptr
    int bias_kind;            // BA_BIAS_NONE / BA_BIAS_DENSE / BA_BIAS_REL1D / BA_BIAS_REL2D ([bias_heads, 2, 2g-1]; tc2 kernel only)
    float* O;                 // [BH, N, d] fp32 -- or bf16 storage when out_bf16 (see store_out)
    int out_bf16;             // ba_params.out_bf16
    float* row_max;           // [BH, N] or nullptr
    float* row_sum;           // [BH, N] or nullptr
    int64_t bias_ld;
    int BH, H, N, d, W64;
    int bias_heads;
    int unit0, unit1;         // 256-query-row units [unit0, unit1) of THIS call's heads to compute (unit1 == 0: all of them)
    int head0;                // index of this call's first head in the caller's [B*H] grid (bias table = (head0+head) % H % bias_heads)
    int bias_dtype;
    int in_dtype;
    float inv_tau;
};

// Launchers implemented in the .cu files; each returns the number of kernels it launched (>0) or a
// negative cudaError_t.
int launch_pack_signs(const void* X, int in_dtype, int64_t heads, int N, int d, uint64_t* words, float* mu,
                      float* partials, unsigned int* tickets, cudaStream_t stream);
int pack_partials_per_head(int N, int d, int in_dtype);
int launch_binary_logits(const uint64_t* qw, const uint64_t* kw, int N, int d, int32_t* S, cudaStream_t stream);
int launch_attn_simt(const FwdArgs& a, cudaStream_t stream);
int launch_quantize_values(const void* V, int in_dtype, int64_t heads, int N, int d, int8_t* vq, int ldq, double* scales,
                           cudaStream_t stream);
int launch_attn_int8(const FwdArgs& a, const int8_t* vq, int ldq, const double* scales, int block_cols, cudaStream_t stream);
inline int i8_level_ld(int d) { return (d + 15) / 16 * 16; }  // row stride of the workspace's s8 level plane: 16-byte multiples for TMA
int launch_attn_tcgen05(const FwdArgs& a, cudaStream_t stream);
int launch_attn_tc2_i8(const FwdArgs& a, const int8_t* vq, int ldq, const double* scales, int block_cols, cudaStream_t stream);  // 0: shape not taken
// Shapes the second-generation tcgen05 kernel (attn_tc2.cuh) takes; decides whether the workspace carries the expanded K plane.
inline bool tc2_shape_ok(int in_dtype, int N, int d) {
    const char* e = getenv("BA_TC2_MIN_N");  // dev knob; default: below ~512 keys the first-generation kernel is faster (measured)
    const int min_n = e ? atoi(e) : 512;
    return in_dtype == BA_BF16 && d % 8 == 0 && d <= 128 && N >= (min_n < 128 ? 128 : min_n);
}
// Shapes the I8 mode of that kernel takes (quantize_pv = true on the tensor cores): the s32 accumulator and the fp32 O share the
// 256 TMEM columns of a query tile with the two S stages, and the s8 value rows must be 16-byte multiples for TMA.
// Heads wider than 64 run one pass per 64-column slice of V (the logits and weights are recomputed: they are the cheap half).
inline bool tc2_i8_shape_ok(int in_dtype, int N, int d) { return in_dtype == BA_BF16 && d % 8 == 0 && d <= 128 && N >= 128; }
inline size_t tc2_kexp_bytes(int64_t heads, int N, int d) {  // whole 64-key tiles per head
    return (size_t)heads * ((N + 63) / 64 * 64) * ((d + 31) / 32 * 32);
}
inline size_t tc2_qexp_bytes(int64_t heads, int N, int d) {  // whole 256-row units per head
    return (size_t)heads * ((N + 255) / 256 * 256) * ((d + 31) / 32 * 32);
}
// diagnostics (fidelity.cu)
int launch_head_mean_abs(const void* Q, const void* K, int dtype, int64_t count, double* mu, cudaStream_t stream);
int launch_probs_rows(const void* Q, const void* K, const void* bias, const int32_t* rows, int nrows, const double* mu, double* P,
                      double tau, int64_t bias_ld, int N, int d, int in_dtype, int bias_dtype, int bias_kind, int mode,
                      cudaStream_t stream);
int fidelity_topk_max();
int launch_fidelity_rows(const double* A, const double* B, int64_t rows, int cols, int keff, double* partial, cudaStream_t stream);
bool tcgen05_supported(const ba_params* p, const char** why);

__device__ __forceinline__ float to_float(float x) { return x; }
__device__ __forceinline__ float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_float(__half x) { return __half2float(x); }

__device__ __forceinline__ float load_as_float(const void* base, int dtype, int64_t idx) {
    if (dtype == BA_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
    if (dtype == BA_F16) return __half2float(static_cast<const __half*>(base)[idx]);
    return static_cast<const float*>(base)[idx];
}

__host__ __device__ inline int dtype_size(int dtype) { return dtype == BA_F32 ? 4 : 2; }

// One element of O (flat index over [BH, N, d]): float32, or bfloat16 rounded to nearest-even when the call asked for it.
__device__ __forceinline__ void store_out(const FwdArgs& a, int64_t idx, float v) {
    if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.O)[idx] = __float2bfloat16_rn(v);
    else a.O[idx] = v;
}

// Shard units (BA_UNIT_ROWS = 256 query rows) of a call: count per head, and "does the call compute row `row` of head `head`".
__host__ __device__ inline int units_per_head(int N) { return (N + 255) / 256; }
__host__ __device__ inline bool row_in_units(const FwdArgs& a, int head, int row) {
    if (a.unit1 == 0) return true;
    const int u = head * units_per_head(a.N) + row / 256;
    return u >= a.unit0 && u < a.unit1;
}

}  // namespace ba
