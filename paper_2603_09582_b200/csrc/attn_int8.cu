// attn_int8.cu -- the reference's DEFAULT mode, quantize_pv = true (Algorithm 1 of the paper):
//   K1v  quantize_values   per-channel s8 levels of V (proj/src/quantize.cpp:57-74): delta[c] = max_i|V[i,c]| / 127
//                          (1 for an all-zero column), Vq[i,c] = round_half_away(V[i,c] / delta[c])
//   K2q  fused attention   per key block of block_cols columns (attention.cpp:284-343): block max, m_new, rescale,
//                          P^ = exp(S - m_new), l = rescale*l + sum P^, O *= rescale, acc(int32) = sum_j round(255 P^_j) * Vq[j,:],
//                          O += acc; epilogue Y = O / l / 255 * delta[c] (attention.cpp:354-364)
// CUDA-core, correctness-first implementation: the integer products run on the SIMT pipes, one
// thread per (query row, 32-column slice of d) like attn_simt.cu.  The result depends on block_cols exactly as the
// reference's does (the u8 grid of P^ is relative to the running max after each key block), so the same block size must
// be used on both sides; blocks of up to 64 keys are staged in shared memory.  K1v works in fp64 so that the s8 levels
// and the scales are bit-identical to the reference's; K2q works in fp32 (a weight that lands within ~1e-5 of a .5
// rounding boundary may round the other way than in fp64 -- parity is by tolerance, as SURVEY.md 8f says).
#include "ba_common.cuh"

namespace ba {

constexpr int kQvThreads = 256;
constexpr int kI8Rows = 64;     // query rows per CTA
constexpr int kI8Slice = 32;    // O columns per thread
constexpr int kI8MaxBc = 64;    // keys per block staged in shared memory
constexpr int kI8MaxW64 = 4;    // d <= 256

// K1v, quantize_values (quantize.cpp:57-74) in three small launches over a (head, 256-row chunk) grid:
//   A  column abs-max: per-thread running max over its rows, then one atomicMax per column and CTA on the LOW WORD of the
//      head's scales[] slot (zeroed first; non-negative floats order like their bit patterns, and max is order independent,
//      so the result is exact);
//   B  levels: delta = amax / 127 (1 for an all-zero column) and round_half_away(v / delta), both in fp64 like the reference
//      => bit-identical s8 levels;
//   C  the slots become the fp64 scales.
// Thread (ty, tx): tx = group of 8 consecutive columns, ty = row lane.  (The first build ran one CTA per head with a
// shared-memory atomicMax per ELEMENT: ~0.4 ms at 16 heads x 4096 keys, more than the attention kernel it feeds.)
constexpr int kQvChunk = 256;  // rows per CTA

__device__ __forceinline__ void qv_load8(const void* V, int in_dtype, int64_t off, int c0, int d, float (&v)[8]) {
    if (in_dtype != BA_F32 && c0 + 8 <= d && (off & 7) == 0) {  // 16 aligned bytes of bf16 / fp16
        const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(V) + off);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (in_dtype == BA_BF16) {
                v[2 * i] = __uint_as_float(ww[i] << 16);
                v[2 * i + 1] = __uint_as_float(ww[i] & 0xFFFF0000u);
            } else {
                const __half2 hh = *reinterpret_cast<const __half2*>(&ww[i]);
                v[2 * i] = __low2float(hh);
                v[2 * i + 1] = __high2float(hh);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = c0 + i < d ? load_as_float(V, in_dtype, off + i) : 0.f;
    }
}

__global__ void __launch_bounds__(kQvThreads) qv_amax_kernel(const void* V, int in_dtype, int N, int d, int chunks, double* scales) {
    __shared__ unsigned int amax_bits[256];
    const int head = blockIdx.x / chunks, chunk = blockIdx.x - head * chunks;
    const int cg = (d + 7) / 8, tx = threadIdx.x % cg, ty = threadIdx.x / cg, rows_per_pass = kQvThreads / cg;
    for (int c = threadIdx.x; c < 256; c += kQvThreads) amax_bits[c] = 0u;
    __syncthreads();
    const int r1 = min(N, (chunk + 1) * kQvChunk);
    if (ty < rows_per_pass) {
        float m[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int row = chunk * kQvChunk + ty; row < r1; row += rows_per_pass) {
            float v[8];
            qv_load8(V, in_dtype, ((int64_t)head * N + row) * d + tx * 8, tx * 8, d, v);
#pragma unroll
            for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], fabsf(v[i]));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (tx * 8 + i < d) atomicMax(&amax_bits[tx * 8 + i], __float_as_uint(m[i]));
    }
    __syncthreads();
    unsigned int* slots = reinterpret_cast<unsigned int*>(scales + (int64_t)head * d);  // low word of each fp64 slot (little endian)
    for (int c = threadIdx.x; c < d; c += kQvThreads) atomicMax(slots + 2 * c, amax_bits[c]);
}

__global__ void __launch_bounds__(kQvThreads) qv_levels_kernel(const void* V, int in_dtype, int N, int d, int chunks, const double* scales,
                                                               int8_t* vq, int ldq) {
    const int head = blockIdx.x / chunks, chunk = blockIdx.x - head * chunks;
    const int cg = (d + 7) / 8, tx = threadIdx.x % cg, ty = threadIdx.x / cg, rows_per_pass = kQvThreads / cg;
    __shared__ double sdelta[256];
    __shared__ float srdelta[256];
    const unsigned int* slots = reinterpret_cast<const unsigned int*>(scales + (int64_t)head * d);
    for (int c = threadIdx.x; c < 256; c += kQvThreads) {  // one pair of fp64 divisions per column and CTA, not per thread
        const double amax = c < d ? (double)__uint_as_float(slots[2 * c]) : 0.0;
        const double dl = amax > 0.0 ? amax / 127.0 : 1.0;  // quantize.cpp:61-66
        sdelta[c] = dl;
        srdelta[c] = (float)(1.0 / dl);
    }
    __syncthreads();
    if (ty >= rows_per_pass) return;
    double delta[8];
    float rdelta[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        delta[i] = sdelta[(tx * 8 + i) & 255];
        rdelta[i] = srdelta[(tx * 8 + i) & 255];
    }
    const int r1 = min(N, (chunk + 1) * kQvChunk);
    for (int row = chunk * kQvChunk + ty; row < r1; row += rows_per_pass) {
        float v[8];
        const int64_t off = ((int64_t)head * N + row) * d + tx * 8;
        qv_load8(V, in_dtype, off, tx * 8, d, v);
        int8_t q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            // round_half_away(v / delta) in fp64 decides (quantize.cpp:68-72).  An fp32 estimate of the quotient is within
            // 2e-5 of it (|v / delta| <= 127), so away from the rounding boundaries -- more than 1e-4 from a half-integer --
            // both round to the same level and the fp64 division is skipped (it is ~20 instructions on a narrow pipe).
            const float xe = v[i] * rdelta[i];
            const float fr = fabsf(xe) - floorf(fabsf(xe));
            q[i] = fabsf(fr - 0.5f) > 1e-4f ? (int8_t)__float2int_rn(xe) : (int8_t)round((double)v[i] / delta[i]);
        }
        const int64_t qoff = ((int64_t)head * N + row) * ldq + tx * 8;  // level rows may be padded (ldq >= d)
        if (tx * 8 + 8 <= d && (qoff & 7) == 0) {
            *reinterpret_cast<uint2*>(vq + qoff) = *reinterpret_cast<const uint2*>(q);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (tx * 8 + i < d) vq[qoff + i] = q[i];
        }
    }
}

// Heads of at most one chunk (N <= 256: the ViT shapes): the three steps in ONE launch, one CTA per head -- the second pass
// over the head's 25-50 KB comes out of L1 / L2, and nothing goes through global atomics.
__global__ void __launch_bounds__(kQvThreads) qv_head_kernel(const void* V, int in_dtype, int N, int d, double* scales, int8_t* vq, int ldq) {
    __shared__ unsigned int amax_bits[256];
    __shared__ double sdelta[256];
    __shared__ float srdelta[256];
    const int head = blockIdx.x;
    const int cg = (d + 7) / 8, tx = threadIdx.x % cg, ty = threadIdx.x / cg, rows_per_pass = kQvThreads / cg;
    for (int c = threadIdx.x; c < 256; c += kQvThreads) amax_bits[c] = 0u;
    __syncthreads();
    if (ty < rows_per_pass) {
        float m[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int row = ty; row < N; row += rows_per_pass) {
            float v[8];
            qv_load8(V, in_dtype, ((int64_t)head * N + row) * d + tx * 8, tx * 8, d, v);
#pragma unroll
            for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], fabsf(v[i]));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (tx * 8 + i < d) atomicMax(&amax_bits[tx * 8 + i], __float_as_uint(m[i]));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 256; c += kQvThreads) {
        const double amax = c < d ? (double)__uint_as_float(amax_bits[c]) : 0.0;
        const double dl = amax > 0.0 ? amax / 127.0 : 1.0;  // quantize.cpp:61-66
        sdelta[c] = dl;
        srdelta[c] = (float)(1.0 / dl);
        if (c < d) scales[(int64_t)head * d + c] = dl;
    }
    __syncthreads();
    if (ty >= rows_per_pass) return;
    double delta[8];
    float rdelta[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        delta[i] = sdelta[(tx * 8 + i) & 255];
        rdelta[i] = srdelta[(tx * 8 + i) & 255];
    }
    for (int row = ty; row < N; row += rows_per_pass) {
        float v[8];
        qv_load8(V, in_dtype, ((int64_t)head * N + row) * d + tx * 8, tx * 8, d, v);
        int8_t q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // as in qv_levels_kernel
            const float xe = v[i] * rdelta[i];
            const float fr = fabsf(xe) - floorf(fabsf(xe));
            q[i] = fabsf(fr - 0.5f) > 1e-4f ? (int8_t)__float2int_rn(xe) : (int8_t)round((double)v[i] / delta[i]);
        }
        const int64_t qoff = ((int64_t)head * N + row) * ldq + tx * 8;
        if (tx * 8 + 8 <= d && (qoff & 7) == 0) {
            *reinterpret_cast<uint2*>(vq + qoff) = *reinterpret_cast<const uint2*>(q);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (tx * 8 + i < d) vq[qoff + i] = q[i];
        }
    }
}

__global__ void qv_scales_kernel(double* scales, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double amax = (double)__uint_as_float(reinterpret_cast<const unsigned int*>(scales + i)[0]);
    scales[i] = amax > 0.0 ? amax / 127.0 : 1.0;
}

__global__ void __launch_bounds__(kI8Rows * 8, 1) attn_int8_kernel(const __grid_constant__ FwdArgs a, const int8_t* __restrict__ vq, int ldq,
                                                                   const double* __restrict__ scales, int row_blocks, int bc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ns = blockDim.y;           // 32-column slices = ceil(d/32)
    const int dp = ns * kI8Slice;        // padded head dim in shared memory
    // s8 V levels of the key block, four consecutive keys of one column per 32-bit word ([kI8MaxBc/4][dp] words), so one
    // dp4a.u32.s32 multiplies four u8 weights with four s8 levels of a column (exact in int32, like the reference's loop)
    uint32_t* sv4 = reinterpret_cast<uint32_t*>(smem_raw);
    uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kI8MaxBc * dp);       // [kI8MaxBc][W64]
    int8_t* sv = reinterpret_cast<int8_t*>(smem_raw);
    const int head = blockIdx.x / row_blocks, rb = blockIdx.x - head * row_blocks;
    if (!row_in_units(a, head, rb * kI8Rows)) return;  // unit-sharded call (kI8Rows divides 256)
    const int tx = threadIdx.x, sl = threadIdx.y;
    const int tid = sl * kI8Rows + tx, nthreads = kI8Rows * ns;
    const int row = rb * kI8Rows + tx;
    const bool row_ok = row < a.N;
    const int N = a.N, d = a.d, w64 = a.W64;

    uint64_t qb[kI8MaxW64];
#pragma unroll
    for (int w = 0; w < kI8MaxW64; ++w) qb[w] = (row_ok && w < w64) ? a.q_words[((int64_t)head * N + row) * w64 + w] : 0ull;
    const float sc = a.mu_q[head] * a.mu_k[head] * a.inv_tau;  // score = mu_q*mu_k*dot/tau + bias (attention.cpp:34-36)
    const char* bias_row = nullptr;
    const bool rel1d = a.bias_kind == BA_BIAS_REL1D;
    if (a.bias && row_ok) {
        const int64_t table = (a.head0 + head) % a.H % a.bias_heads;
        bias_row = static_cast<const char*>(a.bias) +
                   (rel1d ? table * (2 * (int64_t)N - 1) : (table * N + row) * a.bias_ld) * dtype_size(a.bias_dtype);
    }
    auto score = [&](int jj, int j) {  // natural-log units, like the reference
        int diff = 0;
#pragma unroll
        for (int w = 0; w < kI8MaxW64; ++w)
            if (w < w64) diff += __popcll(qb[w] ^ sk[jj * w64 + w]);
        float x = (float)(d - 2 * diff) * sc;
        if (bias_row) x += load_as_float(bias_row, a.bias_dtype, rel1d ? row - j + N - 1 : j);
        return x;
    };

    float o[kI8Slice];
#pragma unroll
    for (int c = 0; c < kI8Slice; ++c) o[c] = 0.f;
    float m = -INFINITY, l = 0.f;

    for (int j0 = 0; j0 < N; j0 += bc) {
        const int nk = min(bc, N - j0);
        __syncthreads();
        for (int t = tid; t < nk * w64; t += nthreads) sk[t] = a.k_words[((int64_t)head * N + j0) * w64 + t];
        for (int t = tid; t < ((nk + 3) / 4 * 4) * dp; t += nthreads) {  // byte (jj, c) lives at ((jj/4)*dp + c)*4 + jj%4
            const int jj = t / dp, c = t - jj * dp;
            sv[((jj >> 2) * dp + c) * 4 + (jj & 3)] = (jj < nk && c < d) ? vq[((int64_t)head * N + j0 + jj) * ldq + c] : (int8_t)0;
        }
        __syncthreads();
        if (!row_ok) continue;
        float bm = -INFINITY;  // block max (attention.cpp:308-309)
        for (int jj = 0; jj < nk; ++jj) bm = fmaxf(bm, score(jj, j0 + jj));
        const float m_new = fmaxf(m, bm);
        const float rescale = expf(m - m_new);  // exp(-inf) = 0 on the first block
        int acc[kI8Slice];
#pragma unroll
        for (int c = 0; c < kI8Slice; ++c) acc[c] = 0;
        float rs = 0.f;
        for (int j4 = 0; j4 < nk; j4 += 4) {
            uint32_t p4 = 0;  // four u8 weights, key j4 in the low byte (zero past the block)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (j4 + e < nk) {
                    const float p = expf(score(j4 + e, j0 + j4 + e) - m_new);
                    rs += p;
                    p4 |= (uint32_t)floorf(fmaf(p, 255.0f, 0.5f)) << (8 * e);  // round_half_away of a non-negative value
                }
            }
            const uint32_t* v4 = sv4 + (j4 >> 2) * dp + sl * kI8Slice;
#pragma unroll
            for (int c = 0; c < kI8Slice; ++c)
                asm("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(p4), "r"(v4[c]));
        }
        l = rescale * l + rs;
        m = m_new;
#pragma unroll
        for (int c = 0; c < kI8Slice; ++c) o[c] = o[c] * rescale + (float)acc[c];
    }
    if (!row_ok) return;
    const int64_t obase = ((int64_t)head * N + row) * d + sl * kI8Slice;
#pragma unroll
    for (int c = 0; c < kI8Slice; ++c)
        if (sl * kI8Slice + c < d) store_out(a, obase + c, o[c] / l / 255.0f * (float)scales[(int64_t)head * d + sl * kI8Slice + c]);
    if (sl == 0) {
        if (a.row_max) a.row_max[(int64_t)head * N + row] = m;
        if (a.row_sum) a.row_sum[(int64_t)head * N + row] = l;
    }
}

int launch_quantize_values(const void* V, int in_dtype, int64_t heads, int N, int d, int8_t* vq, int ldq, double* scales,
                           cudaStream_t stream) {
    if (d > 256) return -(int)cudaErrorInvalidValue;
    if (heads == 0 || N == 0) return 0;
    const int chunks = (N + kQvChunk - 1) / kQvChunk;
    if (chunks == 1) {
        qv_head_kernel<<<(unsigned)heads, kQvThreads, 0, stream>>>(V, in_dtype, N, d, scales, vq, ldq);
        const cudaError_t e1 = cudaGetLastError();
        return e1 == cudaSuccess ? 1 : -(int)e1;
    }
    cudaError_t e = cudaMemsetAsync(scales, 0, (size_t)heads * d * sizeof(double), stream);
    if (e != cudaSuccess) return -(int)e;
    qv_amax_kernel<<<(unsigned)(heads * chunks), kQvThreads, 0, stream>>>(V, in_dtype, N, d, chunks, scales);
    qv_levels_kernel<<<(unsigned)(heads * chunks), kQvThreads, 0, stream>>>(V, in_dtype, N, d, chunks, scales, vq, ldq);
    qv_scales_kernel<<<(unsigned)((heads * d + 255) / 256), 256, 0, stream>>>(scales, heads * d);
    e = cudaGetLastError();
    return e == cudaSuccess ? 3 : -(int)e;
}

int launch_attn_int8(const FwdArgs& a, const int8_t* vq, int ldq, const double* scales, int block_cols, cudaStream_t stream) {
    const int ns = (a.d + kI8Slice - 1) / kI8Slice;
    if (ns > 8 || a.W64 > kI8MaxW64 || block_cols < 1 || block_cols > kI8MaxBc) return -(int)cudaErrorInvalidValue;
    const int row_blocks = (a.N + kI8Rows - 1) / kI8Rows;
    const dim3 block(kI8Rows, ns);
    const size_t smem = (size_t)kI8MaxBc * ns * kI8Slice + sizeof(uint64_t) * kI8MaxBc * a.W64;  // s8 tile + packed K words
    attn_int8_kernel<<<(unsigned)(a.BH * row_blocks), block, smem, stream>>>(a, vq, ldq, scales, row_blocks, block_cols);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ba
