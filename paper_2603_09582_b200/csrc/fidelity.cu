// fidelity.cu -- caller-side diagnostics of the BinaryAttention path: attention-map rows
// for sampled query rows and the reference's attention-map fidelity metrics.  Not on the hot path: plain fp64 CUDA-core
// kernels whose arithmetic follows the reference line by line, so the parity bar is ~1e-12, not the 2e-3 of the
// bf16 product path.
//
//   probs_rows_kernel     P[r, :] = softmax_j(score(rows[r], j)) for one head
//                           mode 0  score = q_i.k_j / tau + bias                       attention.cpp:99-147  (reference_attention, with_probs)
//                           mode 1  score = mu_q*mu_k*(d - 2 popc(q^k)) / tau + bias   attention.cpp:149-248 (binary_attention_unfused, with_probs)
//   head_mean_abs_kernel  mu = mean |x| of one head (quantize.cpp:16-23), fp64
//   fidelity_rows_kernel  per-row partial sums of attention_fidelity (fidelity.cpp:40-85) + per-row top-k overlap
//                         (topk_indices, fidelity.cpp:26-36: ties toward the lower column) + the row-stochastic check
//                         (fidelity.cpp:12-24); the host adds the rows in order, so the result is deterministic.
#include "ba_common.cuh"

namespace ba {

constexpr int kDiagThreads = 256;
constexpr int kTopKMax = 128;  // k' = min(k, cols) the per-row selection supports

// Fixed-order block reductions (thread t's value lives in smem[t]; tree over powers of two).
__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int s = kDiagThreads / 2; s > 0; s >>= 1) {
        if (t < s) sh[t] += sh[t + s];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}
__device__ __forceinline__ double block_max(double v, double* sh) {
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int s = kDiagThreads / 2; s > 0; s >>= 1) {
        if (t < s) sh[t] = fmax(sh[t], sh[t + s]);
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kDiagThreads) head_mean_abs_kernel(const void* Q, const void* K, int dtype, int64_t count, double* mu) {
    __shared__ double sh[kDiagThreads];
    const void* X = blockIdx.x == 0 ? Q : K;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += kDiagThreads) acc += fabs((double)load_as_float(X, dtype, i));
    const double tot = block_sum(acc, sh);
    if (threadIdx.x == 0) mu[blockIdx.x] = tot / (double)count;
}

struct ProbsArgs {
    const void* Q;     // this head's [N, d]
    const void* K;
    const void* bias;  // table of this head (dense: [N, bias_ld]; rel1d: [2N-1]) or nullptr
    const int32_t* rows;
    const double* mu;  // {mu_q, mu_k} (mode 1)
    double* P;         // [nrows, N]
    double tau;
    int64_t bias_ld;
    int N, d, in_dtype, bias_dtype, bias_kind, mode;
};

__global__ void __launch_bounds__(kDiagThreads) probs_rows_kernel(const __grid_constant__ ProbsArgs a) {
    __shared__ double sh[kDiagThreads];
    __shared__ double qrow[256];     // d <= 256
    __shared__ uint64_t qbits[4];
    const int r = blockIdx.x, i = a.rows[r], N = a.N, d = a.d;
    double* prow = a.P + (int64_t)r * N;
    for (int c = threadIdx.x; c < d; c += kDiagThreads) qrow[c] = (double)load_as_float(a.Q, a.in_dtype, (int64_t)i * d + c);
    __syncthreads();
    if (threadIdx.x < 4) {
        uint64_t w = 0;
        for (int c = threadIdx.x * 64; c < min(d, threadIdx.x * 64 + 64); ++c)
            if (qrow[c] >= 0.0) w |= 1ull << (c & 63);  // bitops.cpp:45: +0 and -0 map to +1
        qbits[threadIdx.x] = w;
    }
    __syncthreads();
    const double mu_prod = a.mode == 1 ? a.mu[0] * a.mu[1] : 0.0;
    double mx = -INFINITY;
    for (int j = threadIdx.x; j < N; j += kDiagThreads) {
        double s;
        if (a.mode == 1) {
            int ham = 0;
            for (int w = 0; w * 64 < d; ++w) {
                uint64_t kw = 0;
                for (int c = w * 64; c < min(d, w * 64 + 64); ++c)
                    if (load_as_float(a.K, a.in_dtype, (int64_t)j * d + c) >= 0.0f) kw |= 1ull << (c & 63);
                ham += __popcll(qbits[w] ^ kw);
            }
            s = mu_prod * (double)(d - 2 * ham) / a.tau;  // attention.cpp:34-36 (binary_score), same order
        } else {
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot = __dadd_rn(dot, __dmul_rn(qrow[c], (double)load_as_float(a.K, a.in_dtype, (int64_t)j * d + c)));
            s = dot / a.tau;  // attention.cpp:119-121 (no FMA: the reference is built with -ffp-contract=off)
        }
        if (a.bias) {
            const int64_t idx = a.bias_kind == BA_BIAS_REL1D ? (int64_t)i - j + N - 1 : (int64_t)i * a.bias_ld + j;
            s += (double)load_as_float(a.bias, a.bias_dtype, idx);
        }
        prow[j] = s;
        mx = fmax(mx, s);
    }
    mx = block_max(mx, sh);
    double acc = 0.0;
    for (int j = threadIdx.x; j < N; j += kDiagThreads) {
        const double e = exp(prow[j] - mx);
        prow[j] = e;
        acc += e;
    }
    const double l = block_sum(acc, sh);
    for (int j = threadIdx.x; j < N; j += kDiagThreads) prow[j] /= l;
}

// Per-row top-k of one matrix row into `out` (shared memory): selection of the maximum k times, ties toward the lower
// column; `picked` entries of earlier rounds are skipped.
__device__ void row_topk(const double* row, int cols, int keff, int* out, double* shv, int* shi) {
    const int t = threadIdx.x;
    for (int round = 0; round < keff; ++round) {
        double bv = -INFINITY;
        int bi = cols;  // "none"
        for (int j = t; j < cols; j += kDiagThreads) {
            bool used = false;
            for (int q = 0; q < round; ++q) used |= (out[q] == j);
            if (used) continue;
            const double v = row[j];
            if (bi == cols || v > bv) {  // strided scan visits columns in increasing order: strict > keeps the lower one
                bv = v;
                bi = j;
            }
        }
        shv[t] = bv;
        shi[t] = bi;
        __syncthreads();
        for (int s = kDiagThreads / 2; s > 0; s >>= 1) {
            if (t < s) {
                const int oi = shi[t + s];
                const double ov = shv[t + s];
                if (oi != cols && (shi[t] == cols || ov > shv[t] || (ov == shv[t] && oi < shi[t]))) {
                    shv[t] = ov;
                    shi[t] = oi;
                }
            }
            __syncthreads();
        }
        if (t == 0) out[round] = shi[0];
        __syncthreads();
    }
}

// partial[row][8] = {dot, |a|^2, |b|^2, sum|a-b|, sum|a|, sum (a-b)^2, hits / k', flag}; flag != 0: not row-stochastic
__global__ void __launch_bounds__(kDiagThreads) fidelity_rows_kernel(const double* __restrict__ A, const double* __restrict__ B, int cols,
                                                                     int keff, double* __restrict__ partial) {
    __shared__ double sh[kDiagThreads];
    __shared__ int shi[kDiagThreads];
    __shared__ int ta[kTopKMax], tb[kTopKMax];
    __shared__ int hits;
    const int row = blockIdx.x, t = threadIdx.x;
    const double* a = A + (int64_t)row * cols;
    const double* b = B + (int64_t)row * cols;
    double dot = 0, na = 0, nb = 0, l1d = 0, l1r = 0, sq = 0, sa = 0, sb = 0;
    int bad = 0;
    for (int j = t; j < cols; j += kDiagThreads) {
        const double x = a[j], y = b[j];
        dot += x * y;
        na += x * x;
        nb += y * y;
        l1d += fabs(x - y);
        l1r += fabs(x);
        sq += (x - y) * (x - y);
        sa += x;
        sb += y;
        bad |= (x < -1e-6) || (y < -1e-6);
    }
    dot = block_sum(dot, sh);
    na = block_sum(na, sh);
    nb = block_sum(nb, sh);
    l1d = block_sum(l1d, sh);
    l1r = block_sum(l1r, sh);
    sq = block_sum(sq, sh);
    sa = block_sum(sa, sh);
    sb = block_sum(sb, sh);
    const double nbad = block_sum((double)bad, sh);
    row_topk(a, cols, keff, ta, sh, shi);
    row_topk(b, cols, keff, tb, sh, shi);
    if (t == 0) hits = 0;
    __syncthreads();
    if (t < keff) {
        int h = 0;
        for (int q = 0; q < keff; ++q) h |= (ta[q] == tb[t]);
        if (h) atomicAdd(&hits, 1);
    }
    __syncthreads();
    if (t == 0) {
        double* p = partial + (int64_t)row * 8;
        p[0] = dot;
        p[1] = na;
        p[2] = nb;
        p[3] = l1d;
        p[4] = l1r;
        p[5] = sq;
        p[6] = (double)hits / (double)keff;
        p[7] = (nbad > 0.0 || fabs(sa - 1.0) > 1e-6 || fabs(sb - 1.0) > 1e-6) ? 1.0 : 0.0;
    }
}

int launch_head_mean_abs(const void* Q, const void* K, int dtype, int64_t count, double* mu, cudaStream_t stream) {
    head_mean_abs_kernel<<<2, kDiagThreads, 0, stream>>>(Q, K, dtype, count, mu);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

int launch_probs_rows(const void* Q, const void* K, const void* bias, const int32_t* rows, int nrows, const double* mu, double* P,
                      double tau, int64_t bias_ld, int N, int d, int in_dtype, int bias_dtype, int bias_kind, int mode,
                      cudaStream_t stream) {
    if (d > 256) return -(int)cudaErrorInvalidValue;
    ProbsArgs a{Q, K, bias, rows, mu, P, tau, bias_ld, N, d, in_dtype, bias_dtype, bias_kind, mode};
    probs_rows_kernel<<<(unsigned)nrows, kDiagThreads, 0, stream>>>(a);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

int fidelity_topk_max() { return kTopKMax; }

int launch_fidelity_rows(const double* A, const double* B, int64_t rows, int cols, int keff, double* partial, cudaStream_t stream) {
    fidelity_rows_kernel<<<(unsigned)rows, kDiagThreads, 0, stream>>>(A, B, cols, keff, partial);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ba
