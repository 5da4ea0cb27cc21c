// attn_simt.cu -- K2 (CUDA-core variant): fused BinaryAttention forward on the SIMT pipes.
//
// Follows binattn::binary_attention_fused with quantize_pv = false (proj/src/attention.cpp:250-382):
//   score  = mu_q*mu_k * dot / tau + bias           (attention.cpp:34-36; dot = d - 2*popc(q^k), bitops.cpp:59-67)
//   online softmax with running max / sum           (attention.cpp:306-324)
//   O += P * V, final O / l                          (attention.cpp:326-331, 354-364)
// in fp32, base-2 exponent domain.  This is the "CUDA-core popc" candidate of BASELINE.json's north star
// and the fallback for shapes the tcgen05 kernel does not take (any N, any d <= 256, any input dtype,
// any bias stride).  One thread owns one query row and a 32-column slice of O; key tiles of 32 rows are
// staged in shared memory (packed K words + V widened to fp32) and read as warp-wide broadcasts.
#include "ba_common.cuh"

namespace ba {

constexpr int kSimtRows = 64;   // query rows per CTA
constexpr int kSimtKeys = 32;   // keys per shared-memory tile
constexpr int kSimtSlice = 32;  // O columns per thread
constexpr int kSimtMaxW64 = 4;  // d <= 256

__global__ void __launch_bounds__(kSimtRows * 8, 1) attn_simt_kernel(const __grid_constant__ FwdArgs a, int row_blocks) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ns = blockDim.y;            // number of 32-column slices = ceil(d/32)
    const int dp = ns * kSimtSlice;       // padded head dim in shared memory
    float* sv = reinterpret_cast<float*>(smem_raw);                                 // [kSimtKeys][dp]
    uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw + sizeof(float) * kSimtKeys * dp);  // [kSimtKeys][W64]

    const int head = blockIdx.x / row_blocks;
    const int rb = blockIdx.x - head * row_blocks;
    if (!row_in_units(a, head, rb * kSimtRows)) return;  // unit-sharded call (kSimtRows divides 256: a block lies in one unit)
    const int tx = threadIdx.x, sl = threadIdx.y;
    const int tid = sl * kSimtRows + tx, nthreads = kSimtRows * ns;
    const int row = rb * kSimtRows + tx;
    const bool row_ok = row < a.N;
    const int N = a.N, d = a.d, w64 = a.W64;

    uint64_t qb[kSimtMaxW64];
#pragma unroll
    for (int w = 0; w < kSimtMaxW64; ++w)
        qb[w] = (row_ok && w < w64) ? a.q_words[((int64_t)head * N + row) * w64 + w] : 0ull;

    // scale in the base-2 domain: x2 = dot * (mu_q*mu_k/tau*log2e) + bias*log2e
    const float sc2 = a.mu_q[head] * a.mu_k[head] * a.inv_tau * kLog2e;
    // dense: pointer to this row of the N x N table, element j; relative-1d (attention.cpp:65-76): pointer to the head's
    // 2N-1 offsets, element row - j + N - 1
    const char* bias_row = nullptr;
    const bool rel1d = a.bias_kind == BA_BIAS_REL1D;
    if (a.bias && row_ok) {
        const int64_t table = (a.head0 + head) % a.H % a.bias_heads;
        bias_row = static_cast<const char*>(a.bias) +
                   (rel1d ? table * (2 * (int64_t)N - 1) : (table * N + row) * a.bias_ld) * dtype_size(a.bias_dtype);
    }

    float o[kSimtSlice];
#pragma unroll
    for (int c = 0; c < kSimtSlice; ++c) o[c] = 0.f;
    float m = -INFINITY, l = 0.f;

    for (int j0 = 0; j0 < N; j0 += kSimtKeys) {
        const int nk = min(kSimtKeys, N - j0);
        __syncthreads();
        for (int t = tid; t < kSimtKeys * w64; t += nthreads) {
            const int jj = t / w64, w = t - jj * w64;
            sk[t] = jj < nk ? a.k_words[((int64_t)head * N + j0 + jj) * w64 + w] : 0ull;
        }
        for (int t = tid; t < kSimtKeys * dp; t += nthreads) {
            const int jj = t / dp, c = t - jj * dp;
            sv[t] = (jj < nk && c < d) ? load_as_float(a.V, a.in_dtype, ((int64_t)head * N + j0 + jj) * d + c) : 0.f;
        }
        __syncthreads();
        if (!row_ok) continue;
        for (int jj = 0; jj < nk; ++jj) {
            int diff = 0;
#pragma unroll
            for (int w = 0; w < kSimtMaxW64; ++w)
                if (w < w64) diff += __popcll(qb[w] ^ sk[jj * w64 + w]);
            float x2 = (float)(d - 2 * diff) * sc2;
            if (bias_row) x2 = fmaf(load_as_float(bias_row, a.bias_dtype, rel1d ? row - (j0 + jj) + N - 1 : j0 + jj), kLog2e, x2);
            if (x2 == -INFINITY) continue;  // masked key (bias = -inf): weight 0, and never exp2(-inf - -inf) while m is still -inf
            if (x2 > m) {  // running-max update (attention.cpp:308-324); first key: alpha = exp2(-inf) = 0
                const float alpha = exp2f(m - x2);
                l *= alpha;
#pragma unroll
                for (int c = 0; c < kSimtSlice; ++c) o[c] *= alpha;
                m = x2;
            }
            const float p = exp2f(x2 - m);
            l += p;
            const float4* v4 = reinterpret_cast<const float4*>(sv + jj * dp + sl * kSimtSlice);
#pragma unroll
            for (int c = 0; c < kSimtSlice / 4; ++c) {
                const float4 v = v4[c];
                o[4 * c + 0] = fmaf(p, v.x, o[4 * c + 0]);
                o[4 * c + 1] = fmaf(p, v.y, o[4 * c + 1]);
                o[4 * c + 2] = fmaf(p, v.z, o[4 * c + 2]);
                o[4 * c + 3] = fmaf(p, v.w, o[4 * c + 3]);
            }
        }
    }
    if (!row_ok) return;
    const float inv_l = 1.0f / l;
    const int64_t obase = ((int64_t)head * N + row) * d + sl * kSimtSlice;
#pragma unroll
    for (int c = 0; c < kSimtSlice; ++c)
        if (sl * kSimtSlice + c < d) store_out(a, obase + c, o[c] * inv_l);
    if (sl == 0) {
        if (a.row_max) a.row_max[(int64_t)head * N + row] = m * kLn2;  // back to natural units
        if (a.row_sum) a.row_sum[(int64_t)head * N + row] = l;
    }
}

int launch_attn_simt(const FwdArgs& a, cudaStream_t stream) {
    const int ns = (a.d + kSimtSlice - 1) / kSimtSlice;
    if (ns > 8 || a.W64 > kSimtMaxW64) return -(int)cudaErrorInvalidValue;
    const int row_blocks = (a.N + kSimtRows - 1) / kSimtRows;
    const dim3 block(kSimtRows, ns);
    const size_t smem = sizeof(float) * kSimtKeys * ns * kSimtSlice + sizeof(uint64_t) * kSimtKeys * a.W64;
    attn_simt_kernel<<<(unsigned)(a.BH * row_blocks), block, smem, stream>>>(a, row_blocks);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ba
