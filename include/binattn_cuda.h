/*
 * binattn_cuda.h -- C ABI of the B200-native BinaryAttention forward path.
 *
 * This is the drop-in boundary around the reference's one hot path
 *     binattn::binary_attention_fused(q, k, v, cfg)        proj/include/binattn/attention.hpp:69-71
 * and the L1 functions it calls
 *     binattn::binary_quantize / pack_signs                proj/src/quantize.cpp:16-23, bitops.cpp:37-49
 *     binattn::binary_gemm                                 proj/src/bitops.cpp:96-131   (verification only)
 * mapped to BASELINE.json's operator shape  binary_attention(Q, K, V, bias, scale) -> O:
 *     Q,K,V  <-> q,k,v  (batched here as [B,H,N,d]; the reference is one call per head)
 *     bias   <-> cfg.bias after materialize_bias (dense N x N, attention.cpp:55-97), shared over the batch
 *     scale  <-> 1 / cfg.temperature (default 1/sqrt(d), attention.cpp:49); the data-dependent factor
 *                mu_q * mu_k (attention.cpp:262-264) is computed INSIDE the call, as in the reference.
 *     O      <-> AttentionOutput::output;  row_max / row_sum <-> AttentionOutput::row_max / row_sum.
 *
 * Conventions: plain C, no exceptions cross the boundary.  Every entry point returns a ba_status;
 * ba_last_error() gives the thread-local message.  Status codes mirror the reference's exception
 * types (proj/include/binattn/errors.hpp:10-55): BA_ERR_SHAPE <-> ShapeError, BA_ERR_VALIDATION <->
 * ValidationError.  All tensor pointers are DEVICE pointers owned by the caller unless the function
 * name ends in _host.  `stream` is a cudaStream_t passed as void*; calls are asynchronous on it.
 * One ba_handle per device, used from one host thread AND ONE STREAM at a time: the handle owns scratch that every call
 * reuses (the default workspace, K1's ticket counters, the expanded relative-2d table), so two calls in flight on different
 * streams would race on it -- serialise them, or create one handle per stream.  Entry points bind to the handle's device
 * for their duration and restore the caller's current device.  There is no CPU fallback: without a CUDA device ba_create
 * fails with BA_ERR_CUDA.
 *
 * Accuracy of O (tensor-core path, quantize_pv = 0): the softmax weights are rounded to bf16 before the P.V contraction, each
 * within 2^-9 relative of exp(S - m), so for ANY input |O - O_fp64| <= 2^-9 * max_j |v_j - O| <= 2^-8 * max|V|.  When a row
 * spreads its weight over many keys the roundings average out: <= 1e-3 max-abs on every BASELINE.json configuration
 * (N(0,1) inputs), the 2e-3 bar of the parity tests.  Peaked rows (a few dominant keys, e.g. inputs scaled by 2..8) approach
 * the bound; INTEGRATION.md has the measured error-vs-peakedness table.  The CUDA-core kernel keeps fp32 weights.
 */
#ifndef BINATTN_CUDA_H
#define BINATTN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BA_OK = 0,
    BA_ERR_SHAPE = 1,       /* binattn::ShapeError       (errors.hpp:16-19; attention.cpp:21-23, 60-61) */
    BA_ERR_VALIDATION = 2,  /* binattn::ValidationError  (errors.hpp:22-25; attention.cpp:24-28)        */
    BA_ERR_CUDA = 3,        /* CUDA runtime / driver failure, or no device                               */
    BA_ERR_UNSUPPORTED = 4  /* requested kernel cannot run this shape / dtype                            */
} ba_status;

typedef enum { BA_BF16 = 0, BA_F16 = 1, BA_F32 = 2 } ba_dtype;

typedef enum {
    BA_KERNEL_AUTO = 0,    /* tcgen05 path when the shape allows it, else the CUDA-core path */
    BA_KERNEL_SIMT = 1,    /* CUDA-core xor+popc logits, fp32 FMA P.V (any N, d <= 256, any dtype) */
    BA_KERNEL_TCGEN05 = 2  /* +-1 e4m3 QK^T and bf16 P.V on tcgen05/TMEM, V by TMA (bf16, d % 8 == 0, d <= 128) */
} ba_kernel;

typedef enum {
    BA_BIAS_NONE = 0,
    BA_BIAS_DENSE = 1,  /* DenseBias: N x N table (attention.hpp:15-17, attention.cpp:59-63) */
    BA_BIAS_REL1D = 2,  /* Relative1dBias: b_ij = offsets[i - j + N - 1], 2N-1 entries per table (attention.hpp:18-21,
                           attention.cpp:65-76); generated inside the kernel, no N x N table ever exists */
    BA_BIAS_REL2D = 3   /* Relative2dBias: tokens on a g x g grid, g = sqrt(N) (N must be a perfect square, else BA_ERR_SHAPE
                           like attention.cpp:79-81), b_ij = row_offsets[ri - rj + g - 1] + col_offsets[ci - cj + g - 1]
                           (attention.hpp:22-26, attention.cpp:78-96).  Generated inside the kernel from the two tables
                           held in shared memory when the second-generation tcgen05 kernel takes the shape (N >= 512,
                           g % 32 == 0: N = 1024, 4096, 16384); otherwise expanded ONCE on the device into a handle-owned
                           fp32 table and fed to the dense path */
} ba_bias_mode;

/* Q, K, V: [B, H, N, d] row-major contiguous, dtype in_dtype.  O: [B, H, N, d] float32.
 * bias (bias_mode == BA_BIAS_DENSE): [bias_heads, N, bias_ld] with bias_heads in {1, H}; head (b,h)
 * reads table h % bias_heads; bias_ld >= N is the row stride in elements (0 means N).
 * bias (bias_mode == BA_BIAS_REL1D): [bias_heads, 2N-1] contiguous offsets (bias_ld is ignored).
 * bias (bias_mode == BA_BIAS_REL2D): [bias_heads, 2, 2g-1] contiguous: row_offsets then col_offsets of each table (bias_ld ignored). */
typedef struct {
    int32_t B, H, N, d;
    int32_t in_dtype;    /* ba_dtype of Q, K, V */
    int32_t bias_mode;   /* ba_bias_mode */
    int32_t bias_heads;  /* 1 or H */
    int32_t bias_dtype;  /* BA_BF16 or BA_F32 (bf16 tables take the TMA path of the tensor-core kernels; rows that are not
                            16-byte multiples are re-laid once per call into a padded copy owned by the handle) */
    int64_t bias_ld;     /* elements; 0 -> N */
    float inv_tau;       /* 1 / temperature; must be > 0 (attention.cpp:24-25); use 1/sqrt(d) for AttentionConfig::make */
    int32_t kernel;      /* ba_kernel */
    int32_t quantize_pv; /* AttentionConfig::quantize_pv (attention.hpp:35): 0 = fp P.V (tensor-core product path),
                            1 = the reference's default u8 x s8 integer P.V: on the tensor cores
                            (tcgen05.mma.kind::i8, s32 accumulation per key block) for bf16 inputs with d % 8 == 0, d <= 128,
                            N >= 128, block_cols = 64 and no bias or a dense bf16 table with 16-byte rows; on the CUDA cores
                            (dp4a) for every other shape.  kernel = BA_KERNEL_TCGEN05 insists on the former. */
    int32_t block_cols;  /* key-block size of the quantize_pv=1 path (AttentionConfig::block_cols, attention.cpp:50-51):
                            the u8 weight grid is relative to the running max after each block, so the result depends
                            on it exactly as the reference's does.  0 -> min(64, N); at most 64.  Ignored otherwise. */
    int64_t unit_begin;  /* Launcher partition finer than heads: when unit_end > unit_begin,              */
    int64_t unit_end;    /* ba_binary_attention_fwd computes ONLY the query rows of units [unit_begin, unit_end) of the flattened
                            (b, h, BA_UNIT_ROWS-row block) grid -- B*H*ceil(N/BA_UNIT_ROWS) units, see ba_shard_units -- and leaves
                            every other row of O / row_max / row_sum untouched.  A range may split a head: K, V and the
                            per-head scales of every head it touches are still processed whole.  0, 0 = all units. */
    int32_t out_bf16;    /* 0: O is float32 (AttentionOutput::output, attention.hpp:44).  1: O is written as bfloat16
                            [B,H,N,d] -- the fp32 result rounded to nearest-even in the kernel's epilogue, i.e. exactly
                            what converting the fp32 output afterwards gives, without the fp32 round trip through HBM.
                            The O argument then points to bf16 storage.  row_max / row_sum stay float32. */
    int32_t bias_on_device; /* ba_binary_attention_host only: 1 = `bias` is already a DEVICE pointer (the table is a model
                            parameter uploaded once, not an input of every call); Q, K, V and O stay host buffers.  0 = the
                            table is copied from host memory in every call like the other inputs. */
} ba_params;

#define BA_UNIT_ROWS 256 /* query rows of one shard unit (one unit of the second-generation kernel, two of the first's) */

typedef struct ba_handle ba_handle;

/* Handle lifetime.  ba_create binds to `device` (cudaSetDevice) and allocates small per-device state. */
int ba_create(int device, ba_handle** out);
int ba_destroy(ba_handle* h);

/* Bytes of scratch ba_binary_attention_fwd needs for these params: the packed sign planes of Q and K
 * ([B,H,N,ceil(d/64)] u64 each, byte-identical to BitMatrix::words(), tensor.hpp:57-94) plus the
 * per-head mean-abs scales.  Pass workspace = NULL to let the handle own (and cache) it. */
size_t ba_workspace_bytes(const ba_params* p);

/* binary_quantize (quantize.cpp:16-23) for every head of X [B,H,N,d]:
 *   words[b,h,i,w]  bit c%64 of word c/64 = 1 iff X[b,h,i,c] >= 0  (pad bits zero; bitops.cpp:37-49)
 *   mu[b,h]         mean |X[b,h,:,:]| (float32; nullable) */
int ba_pack_signs(ba_handle* h, const ba_params* p, const void* X, uint64_t* words, float* mu, void* stream);

/* quantize_values (quantize.cpp:57-74) for every head of V [B,H,N,d]: vq[b,h,i,c] = round_half_away(V / scales[b,h,c]),
 * scales[b,h,c] = max_i |V[b,h,i,c]| / 127 (1 for an all-zero column), computed in fp64 like the reference. */
int ba_quantize_values(ba_handle* h, const ba_params* p, const void* V, int8_t* vq, double* scales, void* stream);

/* binary_gemm (bitops.cpp:96-131) for ONE head: S[i,j] = d - 2*popc(q_i xor k_j), int32 [N,N].
 * Verification only (the fused kernel never materialises S). */
int ba_binary_logits(ba_handle* h, const ba_params* p, const uint64_t* q_words, const uint64_t* k_words,
                     int64_t head_index, int32_t* S, void* stream);

/* Attention-map rows of ONE head for the fidelity diagnostics (the reference's `with_probs` outputs):
 *   P[r, :] = softmax_j(score(rows[r], j)), fp64 [nrows, N] (device), rows = device int32 [nrows] query-row indices.
 *   mode BA_PROBS_FULL    score = q_i.k_j / tau + bias                        reference_attention      (attention.cpp:99-147)
 *   mode BA_PROBS_BINARY  score = mu_q*mu_k*(d - 2 popc(q^k)) / tau + bias    binary_attention_unfused (attention.cpp:149-248)
 * Q, K: [B,H,N,d] in_dtype; bias as in ba_binary_attention_fwd.  mu and the sign bits are computed in the call (fp64). */
enum { BA_PROBS_FULL = 0, BA_PROBS_BINARY = 1 };
int ba_attention_probs(ba_handle* h, const ba_params* p, int mode, const void* Q, const void* K, const void* bias,
                       int64_t head_index, const int32_t* rows, int nrows, double* P, void* stream);

/* attention_fidelity (fidelity.hpp:12-18, fidelity.cpp:40-85) of two row-stochastic fp64 [rows, cols] device matrices:
 * flattened cosine, ||ref-other||_1 / ||ref||_1, RMSE, mean per-row top-k overlap / k' (k' = min(k, cols), ties toward the
 * lower column).  Rows must be probability vectors to 1e-6 (BA_ERR_VALIDATION otherwise, fidelity.cpp:12-24), k >= 1.
 * Synchronises `stream`; the result is written to host memory. */
typedef struct ba_fidelity {
    double cos_sim, relative_l1, rmse, precision_at_k;
} ba_fidelity;
int ba_attention_fidelity(ba_handle* h, const double* p_ref, const double* p_other, int64_t rows, int64_t cols, int64_t k,
                          ba_fidelity* out, void* stream);
/* Same with HOST matrices (what a reference caller holds: DenseMatrix::data()); staged through device memory. */
int ba_attention_fidelity_host(ba_handle* h, const double* p_ref, const double* p_other, int64_t rows, int64_t cols, int64_t k,
                               ba_fidelity* out);

/* binary_attention_fused (attention.cpp:250-382), quantize_pv = false semantics, for all B*H heads.
 * row_max / row_sum: optional [B,H,N] float32 (AttentionOutput::row_max / row_sum, attention.hpp:45-46).
 * quantize_pv = 1 selects the reference's integer P.V mode (attention.cpp:332-343, 361-363). */
int ba_binary_attention_fwd(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                            const void* bias, void* O, float* row_max, float* row_sum, void* workspace,
                            void* stream);

/* Same call with HOST buffers (what a reference-side binding uses): copies Q,K,V(,bias) to the device,
 * runs ba_binary_attention_fwd, copies O (and row_max/row_sum when non-NULL) back, and synchronises.
 * Device staging buffers are owned and cached by the handle.  Pinned host memory makes the copies async. */
int ba_binary_attention_host(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                             const void* bias, void* O, float* row_max, float* row_sum);

/* Launcher partition: contiguous range of the flattened B*H head grid owned by
 * `rank` of `world` single-GPU processes.  No collective is needed on the hot path. */
int ba_shard_range(int64_t total_heads, int world, int rank, int64_t* begin, int64_t* end);

/* The same partition over (head, row-block) units for grids with few heads per GPU (BASELINE.json configs[4]: 16 heads over
 * 8 GPUs): contiguous range of the B*H*ceil(N/BA_UNIT_ROWS) units owned by `rank`; pass it as ba_params.unit_begin/unit_end.
 * Ranks that share a head each process that head's K and V; inputs are resident per GPU, so nothing is exchanged. */
int ba_shard_units(const ba_params* p, int world, int rank, int64_t* unit_begin, int64_t* unit_end);

/* Which kernel ba_binary_attention_fwd would run for these params (resolves BA_KERNEL_AUTO). */
int ba_select_kernel(const ba_params* p);

/* Number of CUDA kernels launched through this handle so far (bench.py's gpu_launches). */
int64_t ba_launch_count(const ba_handle* h);

/* Per-kernel timing for the roofline report.  After ba_profile_begin(h, max_calls) every
 * ba_binary_attention_fwd call records three CUDA events on ITS launching stream (before K1, between K1
 * and K2, after K2) until max_calls calls were seen.  ba_profile_end synchronises those events, returns
 * the number of profiled calls and the summed durations in milliseconds, and switches profiling off. */
int ba_profile_begin(ba_handle* h, int max_calls);
int ba_profile_end(ba_handle* h, int* calls, double* pack_ms, double* attn_ms);

const char* ba_last_error(void);
int ba_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BINATTN_CUDA_H */
