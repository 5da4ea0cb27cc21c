// binattn_cuda.cu -- host side of the C ABI declared in include/binattn_cuda.h.
//
// Thin by design: validates the call the way binattn::check_shapes does (proj/src/attention.cpp:17-29),
// lays the workspace out, and launches K1 (pack_signs.cu) followed by one fused K2 kernel
// (attn_tcgen05.cu or attn_simt.cu).  No CPU fallback exists: every compute entry point ends in a
// CUDA kernel launch or an error code.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>

#include "ba_common.cuh"

namespace ba {
int launch_expand_rel2d(const void* tables, int dtype, int heads, int N, int g, float* out, cudaStream_t stream);  // bias_expand.cu
int launch_pad_bias_rows(const void* in, int64_t ld_in, int heads, int N, int64_t ld_out, void* out, cudaStream_t stream);  // bias_expand.cu
int launch_pack_signs_qk(const void* Q, const void* K, int in_dtype, int64_t heads, int N, int d, uint64_t* q_words,
                         uint64_t* k_words, float* mu_q, float* mu_k, float* partials, unsigned int* tickets,
                         cudaStream_t stream);
}

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define BA_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(BA_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int grid_side(int n) {  // g with g*g == n, or 0
    int g = (int)std::lround(std::sqrt((double)n));
    return (g > 0 && (long long)g * g == n) ? g : 0;
}

struct Layout {
    size_t q_words, k_words, mu_q, mu_k, partials, vq, vscales, kexp, qexp, total;
    int64_t BH;
    int W64, chunks;
};

Layout make_layout(const ba_params* p, int64_t heads = -1) {
    Layout L{};
    L.BH = heads >= 0 ? heads : (int64_t)p->B * p->H;
    L.W64 = (p->d + 63) / 64;
    L.chunks = ba::pack_partials_per_head(p->N, p->d, p->in_dtype);
    const size_t plane = align_up((size_t)L.BH * p->N * L.W64 * sizeof(uint64_t), 256);
    size_t off = 0;
    L.q_words = off; off += plane;
    L.k_words = off; off += plane;
    L.mu_q = off; off += align_up((size_t)L.BH * sizeof(float), 256);
    L.mu_k = off; off += align_up((size_t)L.BH * sizeof(float), 256);
    L.partials = off; off += align_up(2 * (size_t)L.BH * L.chunks * sizeof(float), 256);
    L.vq = L.vscales = off;
    if (p->quantize_pv) {  // s8 levels of V and their per-channel fp64 scales (quantize_values)
        L.vq = off; off += align_up((size_t)L.BH * p->N * ba::i8_level_ld(p->d), 256);  // rows padded to 16 bytes (TMA)
        L.vscales = off; off += align_up((size_t)L.BH * p->d * sizeof(double), 256);
    }
    L.kexp = off;  // expanded K plane of the second-generation tcgen05 kernel (e4m3 +-1.0 bytes, UMMA tile order)
    L.qexp = off;
    if (p->kernel != BA_KERNEL_SIMT &&
        (p->quantize_pv ? ba::tc2_i8_shape_ok(p->in_dtype, p->N, p->d) : ba::tc2_shape_ok(p->in_dtype, p->N, p->d))) {
        off += align_up(ba::tc2_kexp_bytes(L.BH, p->N, p->d), 256);
        L.qexp = off;
        off += align_up(ba::tc2_qexp_bytes(L.BH, p->N, p->d), 256);
    }
    L.total = off;
    return L;
}

int check_params(const ba_params* p, bool need_attention) {
    if (!p) return fail(BA_ERR_SHAPE, "params is NULL");
    if (p->B < 1 || p->H < 1 || p->N < 1 || p->d < 1)  // quantize.cpp:17 (empty matrix), attention.cpp:21-23
        return fail(BA_ERR_SHAPE, "attention: Q, K, V must be [B,H,N,d] with all extents >= 1 (got %d,%d,%d,%d)", p->B,
                    p->H, p->N, p->d);
    if (p->in_dtype != BA_BF16 && p->in_dtype != BA_F16 && p->in_dtype != BA_F32)
        return fail(BA_ERR_VALIDATION, "in_dtype must be BA_BF16, BA_F16 or BA_F32");
    if (!need_attention) return BA_OK;
    if (!(p->inv_tau > 0.0f) || !(p->inv_tau < INFINITY))  // attention.cpp:24-25
        return fail(BA_ERR_VALIDATION, "attention: temperature must be positive");
    if (p->bias_mode != BA_BIAS_NONE && p->bias_mode != BA_BIAS_DENSE && p->bias_mode != BA_BIAS_REL1D &&
        p->bias_mode != BA_BIAS_REL2D)
        return fail(BA_ERR_VALIDATION, "bias_mode must be BA_BIAS_NONE, BA_BIAS_DENSE, BA_BIAS_REL1D or BA_BIAS_REL2D");
    if (p->bias_mode == BA_BIAS_REL2D) {
        if (grid_side(p->N) == 0)  // attention.cpp:79-81
            return fail(BA_ERR_SHAPE, "bias: relative-2d requires N to be a perfect square");
        if (p->bias_heads != 1 && p->bias_heads != p->H)  // attention.cpp:82-83 (tables must match the head)
            return fail(BA_ERR_SHAPE, "bias: relative-2d tables must be [1 or H, 2, 2*sqrt(N)-1]");
        if (p->bias_dtype != BA_BF16 && p->bias_dtype != BA_F32)
            return fail(BA_ERR_VALIDATION, "bias_dtype must be BA_BF16 or BA_F32");
    }
    if (p->bias_mode == BA_BIAS_REL1D) {
        if (p->bias_heads != 1 && p->bias_heads != p->H)  // attention.cpp:66-67 (offsets must match the head)
            return fail(BA_ERR_SHAPE, "bias: relative-1d offsets must be [1 or H, 2N-1]");
        if (p->bias_dtype != BA_BF16 && p->bias_dtype != BA_F32)
            return fail(BA_ERR_VALIDATION, "bias_dtype must be BA_BF16 or BA_F32");
    }
    if (p->bias_mode == BA_BIAS_DENSE) {
        if (p->bias_heads != 1 && p->bias_heads != p->H)  // attention.cpp:60-61 (table must match the head)
            return fail(BA_ERR_SHAPE, "bias: dense table must be [1 or H, N, N]");
        if (p->bias_ld != 0 && p->bias_ld < p->N) return fail(BA_ERR_SHAPE, "bias: bias_ld must be >= N");
        if (p->bias_dtype != BA_BF16 && p->bias_dtype != BA_F32)
            return fail(BA_ERR_VALIDATION, "bias_dtype must be BA_BF16 or BA_F32");
    }
    if (p->d > 256) return fail(BA_ERR_UNSUPPORTED, "head dim %d > 256 is not supported", p->d);
    if (p->unit_begin != 0 || p->unit_end != 0) {
        const int64_t total = (int64_t)p->B * p->H * ba::units_per_head(p->N);
        if (p->unit_begin < 0 || p->unit_end < p->unit_begin || p->unit_end > total)
            return fail(BA_ERR_VALIDATION, "unit range [%lld, %lld) outside [0, %lld]", (long long)p->unit_begin,
                        (long long)p->unit_end, (long long)total);
    }
    if (p->out_bf16 != 0 && p->out_bf16 != 1) return fail(BA_ERR_VALIDATION, "out_bf16 must be 0 (float32 O) or 1 (bfloat16 O)");
    if (p->bias_on_device != 0 && p->bias_on_device != 1) return fail(BA_ERR_VALIDATION, "bias_on_device must be 0 or 1");
    if (p->quantize_pv) {
        const int bc = p->block_cols ? p->block_cols : (p->N < 64 ? p->N : 64);
        if (bc < 1 || bc > p->N)  // attention.cpp:26-28
            return fail(BA_ERR_VALIDATION, "attention: block sizes must be in [1, N]");
        if (bc > 64) return fail(BA_ERR_UNSUPPORTED, "quantize_pv: block_cols %d > 64 is not supported", bc);
    }
    return BA_OK;
}

}  // namespace

constexpr int kHostChunksMax = 32;

struct ba_handle {
    int device = 0;
    int64_t launches = 0;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    unsigned int* tickets = nullptr;
    size_t tickets_n = 0;
    float* partials = nullptr;  // for standalone ba_pack_signs
    size_t partials_n = 0;
    double* diag = nullptr;     // {mu_q, mu_k} of ba_attention_probs
    size_t diag_bytes = 0;
    void* rel2d = nullptr;      // Relative2dBias expanded to a dense fp32 [bias_heads, N, N] table (shapes the in-kernel path does not take)
    size_t rel2d_bytes = 0;
    void* bias_pad = nullptr;   // dense bf16 bias re-laid with 16-byte rows for the TMA tile loads (tables whose rows are not)
    size_t bias_pad_bytes = 0;
    // host-buffer path: copy-in stream, compute stream, copy-out stream + per-chunk events
    cudaStream_t stream = nullptr, stream_in = nullptr, stream_out = nullptr;
    cudaEvent_t ev_in[kHostChunksMax] = {}, ev_done[kHostChunksMax] = {};
    void* stage[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t stage_bytes[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // per-kernel profiling (ba_profile_begin/end)
    cudaEvent_t* prof_ev = nullptr;
    int prof_cap = 0, prof_n = 0;
};

namespace {

// Entry points bind to the handle's device for their duration and put the caller's current device back (a process
// holding handles on several GPUs must not have its current device changed behind its back).
struct DeviceGuard {
    int prev = -1;
    cudaError_t err;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
#define BA_BIND_DEVICE(h)                                                                                         \
    DeviceGuard guard_((h)->device);                                                                              \
    if (guard_.err != cudaSuccess) return fail(BA_ERR_CUDA, "cudaSetDevice(%d): %s", (h)->device, cudaGetErrorString(guard_.err))

int ensure(void** ptr, size_t* have, size_t need, bool zero) {
    if (*have >= need && *ptr) return BA_OK;
    if (*ptr) BA_CUDA(cudaFree(*ptr));
    *ptr = nullptr;
    *have = 0;
    BA_CUDA(cudaMalloc(ptr, need));
    if (zero) {
        // The zero fill runs on the legacy default stream; the kernels that count on it run on streams that do not order
        // against that stream (cudaStreamNonBlocking), so it must have landed before this returns.
        BA_CUDA(cudaMemset(*ptr, 0, need));
        BA_CUDA(cudaDeviceSynchronize());
    }
    *have = need;
    return BA_OK;
}

int ensure_tickets(ba_handle* h, size_t n) {
    size_t have = h->tickets_n * sizeof(unsigned int);
    void* p = h->tickets;
    const int rc = ensure(&p, &have, align_up(n * sizeof(unsigned int), 256), true);
    h->tickets = static_cast<unsigned int*>(p);
    h->tickets_n = have / sizeof(unsigned int);
    return rc;
}

}  // namespace

extern "C" {

const char* ba_last_error(void) { return g_err; }
int ba_version(void) { return 1; }

int ba_create(int device, ba_handle** out) {
    if (!out) return fail(BA_ERR_VALIDATION, "out is NULL");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(BA_ERR_CUDA, "no CUDA device (%s); this library has no CPU fallback",
                    e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(BA_ERR_VALIDATION, "device %d out of range [0,%d)", device, count);
    DeviceGuard guard_(device);
    if (guard_.err != cudaSuccess) return fail(BA_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(guard_.err));
    cudaDeviceProp prop{};
    BA_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(BA_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device,
                    prop.major, prop.minor);
    ba_handle* h = new ba_handle();
    h->device = device;
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream_out, cudaStreamNonBlocking);
    for (int i = 0; i < kHostChunksMax && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        ba_destroy(h);
        return fail(BA_ERR_CUDA, "cudaStreamCreate/cudaEventCreate: %s", cudaGetErrorString(e));
    }
    *out = h;
    return BA_OK;
}

int ba_destroy(ba_handle* h) {
    if (!h) return BA_OK;
    DeviceGuard guard_(h->device);
    if (h->prof_ev) {  // ba_profile_begin without ba_profile_end
        for (int i = 0; i < 3 * h->prof_cap; ++i) cudaEventDestroy(h->prof_ev[i]);
        delete[] h->prof_ev;
    }
    if (h->ws) cudaFree(h->ws);
    if (h->tickets) cudaFree(h->tickets);
    if (h->partials) cudaFree(h->partials);
    if (h->diag) cudaFree(h->diag);
    if (h->rel2d) cudaFree(h->rel2d);
    if (h->bias_pad) cudaFree(h->bias_pad);
    for (void* s : h->stage)
        if (s) cudaFree(s);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->stream_in) cudaStreamDestroy(h->stream_in);
    if (h->stream_out) cudaStreamDestroy(h->stream_out);
    for (int i = 0; i < kHostChunksMax; ++i) {
        if (h->ev_in[i]) cudaEventDestroy(h->ev_in[i]);
        if (h->ev_done[i]) cudaEventDestroy(h->ev_done[i]);
    }
    delete h;
    return BA_OK;
}

size_t ba_workspace_bytes(const ba_params* p) {
    if (check_params(p, false) != BA_OK) return 0;
    return make_layout(p).total;
}

int64_t ba_launch_count(const ba_handle* h) { return h ? h->launches : 0; }

int ba_profile_begin(ba_handle* h, int max_calls) {
    if (!h || max_calls < 1) return fail(BA_ERR_VALIDATION, "profile_begin: need a handle and max_calls >= 1");
    BA_BIND_DEVICE(h);
    if (h->prof_ev) {
        for (int i = 0; i < 3 * h->prof_cap; ++i) cudaEventDestroy(h->prof_ev[i]);
        delete[] h->prof_ev;
        h->prof_ev = nullptr;
    }
    h->prof_ev = new cudaEvent_t[3 * (size_t)max_calls];
    for (int i = 0; i < 3 * max_calls; ++i) BA_CUDA(cudaEventCreate(&h->prof_ev[i]));
    h->prof_cap = max_calls;
    h->prof_n = 0;
    return BA_OK;
}

int ba_profile_end(ba_handle* h, int* calls, double* pack_ms, double* attn_ms) {
    if (!h || !h->prof_ev) return fail(BA_ERR_VALIDATION, "profile_end without profile_begin");
    double k1 = 0.0, k2 = 0.0;
    for (int i = 0; i < h->prof_n; ++i) {
        float a = 0.f, b = 0.f;
        BA_CUDA(cudaEventSynchronize(h->prof_ev[3 * i + 2]));
        BA_CUDA(cudaEventElapsedTime(&a, h->prof_ev[3 * i], h->prof_ev[3 * i + 1]));
        BA_CUDA(cudaEventElapsedTime(&b, h->prof_ev[3 * i + 1], h->prof_ev[3 * i + 2]));
        k1 += a;
        k2 += b;
    }
    if (calls) *calls = h->prof_n;
    if (pack_ms) *pack_ms = k1;
    if (attn_ms) *attn_ms = k2;
    for (int i = 0; i < 3 * h->prof_cap; ++i) cudaEventDestroy(h->prof_ev[i]);
    delete[] h->prof_ev;
    h->prof_ev = nullptr;
    h->prof_cap = h->prof_n = 0;
    return BA_OK;
}

int ba_shard_range(int64_t total, int world, int rank, int64_t* begin, int64_t* end) {
    if (total < 0 || world < 1 || rank < 0 || rank >= world || !begin || !end)
        return fail(BA_ERR_VALIDATION, "shard_range: need total >= 0 and 0 <= rank < world");
    const int64_t base = total / world, rem = total % world;  // first `rem` ranks own one extra head
    *begin = rank * base + (rank < rem ? rank : rem);
    *end = *begin + base + (rank < rem ? 1 : 0);
    return BA_OK;
}

int ba_shard_units(const ba_params* p, int world, int rank, int64_t* begin, int64_t* end) {
    if (!p || p->B < 1 || p->H < 1 || p->N < 1) return fail(BA_ERR_SHAPE, "shard_units: params must carry B, H, N >= 1");
    return ba_shard_range((int64_t)p->B * p->H * ba::units_per_head(p->N), world, rank, begin, end);
}

// Heads with fewer keys than this run the CUDA-core kernel under BA_KERNEL_AUTO: a 64-key tensor-core tile has nothing to win
// there, and with a handful of keys every row is peaked, which is where the bf16 weights of the tensor-core path cost accuracy
// (2.1e-3 ... 2.5e-3 at N = 2 and 7 in scripts/fuzz_auto.py; the CUDA-core kernel keeps fp32 weights).  BA_KERNEL_TCGEN05 still
// takes them.
static const int kAutoMinKeysTc = 32;

int ba_select_kernel(const ba_params* p) {
    if (check_params(p, true) != BA_OK) return -1;
    const char* why = nullptr;
    if (p->kernel == BA_KERNEL_SIMT) return BA_KERNEL_SIMT;
    if (p->quantize_pv) {  // the tensor-core kernel of the integer mode where the launch will take it (see ba_params.quantize_pv)
        const int bc = p->block_cols ? p->block_cols : (p->N < 64 ? p->N : 64);
        const int64_t ld = p->bias_ld ? p->bias_ld : p->N;
        const bool bias_ok = p->bias_mode == BA_BIAS_NONE || (p->bias_mode == BA_BIAS_DENSE && p->bias_dtype == BA_BF16 && ld >= p->N);
        const bool tc = ba::tcgen05_supported(p, &why) && ba::tc2_i8_shape_ok(p->in_dtype, p->N, p->d) && bc == 64 && bias_ok;
        return tc ? BA_KERNEL_TCGEN05 : (p->kernel == BA_KERNEL_TCGEN05 ? -1 : BA_KERNEL_SIMT);
    }
    if (!ba::tcgen05_supported(p, &why)) return p->kernel == BA_KERNEL_TCGEN05 ? -1 : BA_KERNEL_SIMT;
    return (p->kernel == BA_KERNEL_AUTO && p->N < kAutoMinKeysTc) ? BA_KERNEL_SIMT : BA_KERNEL_TCGEN05;
}

int ba_pack_signs(ba_handle* h, const ba_params* p, const void* X, uint64_t* words, float* mu, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, false);
    if (rc) return rc;
    if (!X || !words) return fail(BA_ERR_SHAPE, "pack_signs: X and words must be non-NULL");
    BA_BIND_DEVICE(h);
    const Layout L = make_layout(p);
    if ((rc = ensure_tickets(h, 2 * (size_t)L.BH))) return rc;
    size_t have = h->partials_n;
    void* pp = h->partials;
    if ((rc = ensure(&pp, &have, align_up((size_t)L.BH * L.chunks * sizeof(float), 256), false))) return rc;
    h->partials = static_cast<float*>(pp);
    h->partials_n = have;
    const int n = ba::launch_pack_signs(X, p->in_dtype, L.BH, p->N, p->d, words, mu, h->partials, h->tickets,
                                        static_cast<cudaStream_t>(stream));
    if (n < 0) return fail(BA_ERR_CUDA, "pack_signs launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    return BA_OK;
}

int ba_quantize_values(ba_handle* h, const ba_params* p, const void* V, int8_t* vq, double* scales, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, false);
    if (rc) return rc;
    if (!V || !vq || !scales) return fail(BA_ERR_SHAPE, "quantize_values: V, vq and scales must be non-NULL");
    if (p->d > 256) return fail(BA_ERR_UNSUPPORTED, "head dim %d > 256 is not supported", p->d);
    BA_BIND_DEVICE(h);
    const int n = ba::launch_quantize_values(V, p->in_dtype, (int64_t)p->B * p->H, p->N, p->d, vq, p->d, scales,
                                             static_cast<cudaStream_t>(stream));
    if (n < 0) return fail(BA_ERR_CUDA, "quantize_values launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    return BA_OK;
}

int ba_binary_logits(ba_handle* h, const ba_params* p, const uint64_t* q_words, const uint64_t* k_words,
                     int64_t head_index, int32_t* S, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, false);
    if (rc) return rc;
    if (!q_words || !k_words || !S) return fail(BA_ERR_SHAPE, "binary_logits: NULL pointer");
    const int64_t BH = (int64_t)p->B * p->H;
    if (head_index < 0 || head_index >= BH) return fail(BA_ERR_SHAPE, "binary_logits: head %lld outside [0,%lld)",
                                                        (long long)head_index, (long long)BH);
    BA_BIND_DEVICE(h);
    const int W64 = (p->d + 63) / 64;
    const int64_t off = head_index * p->N * W64;
    const int n = ba::launch_binary_logits(q_words + off, k_words + off, p->N, p->d, S, static_cast<cudaStream_t>(stream));
    if (n < 0) return fail(BA_ERR_CUDA, "binary_logits launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    return BA_OK;
}

int ba_attention_probs(ba_handle* h, const ba_params* p, int mode, const void* Q, const void* K, const void* bias,
                       int64_t head_index, const int32_t* rows, int nrows, double* P, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, true);
    if (rc) return rc;
    if (mode != BA_PROBS_FULL && mode != BA_PROBS_BINARY) return fail(BA_ERR_VALIDATION, "attention_probs: unknown mode %d", mode);
    if (p->bias_mode == BA_BIAS_REL2D) return fail(BA_ERR_UNSUPPORTED, "attention_probs: pass the relative-2d bias as a dense table");
    if (!Q || !K || !rows || !P) return fail(BA_ERR_SHAPE, "attention_probs: NULL pointer");
    if (p->bias_mode != BA_BIAS_NONE && !bias) return fail(BA_ERR_SHAPE, "attention_probs: bias_mode set but bias is NULL");
    if (nrows < 1) return fail(BA_ERR_SHAPE, "attention_probs: nrows must be >= 1");
    const int64_t BH = (int64_t)p->B * p->H;
    if (head_index < 0 || head_index >= BH)
        return fail(BA_ERR_SHAPE, "attention_probs: head %lld outside [0,%lld)", (long long)head_index, (long long)BH);
    BA_BIND_DEVICE(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    rc = ensure(reinterpret_cast<void**>(&h->diag), &h->diag_bytes, 2 * sizeof(double), false);
    if (rc) return rc;
    const int64_t head_elems = (int64_t)p->N * p->d;
    const char* q = static_cast<const char*>(Q) + head_index * head_elems * ba::dtype_size(p->in_dtype);
    const char* k = static_cast<const char*>(K) + head_index * head_elems * ba::dtype_size(p->in_dtype);
    const int64_t bias_ld = p->bias_ld ? p->bias_ld : p->N;
    const char* b = nullptr;
    if (p->bias_mode != BA_BIAS_NONE) {
        const int64_t tab = (head_index % p->H) % p->bias_heads;
        const int64_t per = p->bias_mode == BA_BIAS_REL1D ? 2 * (int64_t)p->N - 1 : (int64_t)p->N * bias_ld;
        b = static_cast<const char*>(bias) + tab * per * ba::dtype_size(p->bias_dtype);
    }
    int n = 0;
    if (mode == BA_PROBS_BINARY) {
        n = ba::launch_head_mean_abs(q, k, p->in_dtype, head_elems, h->diag, st);
        if (n < 0) return fail(BA_ERR_CUDA, "attention_probs (mean abs) launch: %s", cudaGetErrorString((cudaError_t)(-n)));
        h->launches += n;
    }
    n = ba::launch_probs_rows(q, k, b, rows, nrows, h->diag, P, 1.0 / (double)p->inv_tau, bias_ld, p->N, p->d, p->in_dtype,
                              p->bias_dtype, p->bias_mode, mode, st);
    if (n < 0) return fail(BA_ERR_CUDA, "attention_probs launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    return BA_OK;
}

int ba_attention_fidelity(ba_handle* h, const double* p_ref, const double* p_other, int64_t rows, int64_t cols, int64_t k,
                          ba_fidelity* out, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    if (!p_ref || !p_other || !out) return fail(BA_ERR_SHAPE, "attention_fidelity: NULL pointer");
    if (rows < 1 || cols < 1 || cols > INT32_MAX) return fail(BA_ERR_SHAPE, "attention_fidelity: shape mismatch");  // fidelity.cpp:42-43
    if (k < 1) return fail(BA_ERR_VALIDATION, "attention_fidelity: k must be >= 1");                                // fidelity.cpp:44
    const int64_t keff = k < cols ? k : cols;
    if (keff > ba::fidelity_topk_max())
        return fail(BA_ERR_UNSUPPORTED, "attention_fidelity: min(k, cols) = %lld > %d is not supported", (long long)keff,
                    ba::fidelity_topk_max());
    BA_BIND_DEVICE(h);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* partial = nullptr;
    BA_CUDA(cudaMalloc(&partial, (size_t)rows * 8 * sizeof(double)));
    const int n = ba::launch_fidelity_rows(p_ref, p_other, rows, (int)cols, (int)keff, partial, st);
    if (n < 0) {
        cudaFree(partial);
        return fail(BA_ERR_CUDA, "attention_fidelity launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    }
    h->launches += n;
    std::vector<double> host((size_t)rows * 8);
    cudaError_t e = cudaMemcpyAsync(host.data(), partial, host.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(partial);
    if (e != cudaSuccess) return fail(BA_ERR_CUDA, "attention_fidelity: %s", cudaGetErrorString(e));
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int64_t r = 0; r < rows; ++r) {  // rows added in order: deterministic
        if (host[r * 8 + 7] != 0.0)
            return fail(BA_ERR_VALIDATION, "attention_fidelity: row %lld is not a probability vector (1e-6)", (long long)r);
        for (int c = 0; c < 7; ++c) acc[c] += host[r * 8 + c];
    }
    out->cos_sim = acc[0] / (std::sqrt(acc[1]) * std::sqrt(acc[2]));
    out->relative_l1 = acc[3] / acc[4];
    out->rmse = std::sqrt(acc[5] / ((double)rows * (double)cols));
    out->precision_at_k = acc[6] / (double)rows;
    return BA_OK;
}

int ba_attention_fidelity_host(ba_handle* h, const double* p_ref, const double* p_other, int64_t rows, int64_t cols, int64_t k,
                               ba_fidelity* out) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    if (!p_ref || !p_other || !out) return fail(BA_ERR_SHAPE, "attention_fidelity: NULL pointer");
    if (rows < 1 || cols < 1) return fail(BA_ERR_SHAPE, "attention_fidelity: shape mismatch");
    BA_BIND_DEVICE(h);
    const size_t bytes = (size_t)rows * (size_t)cols * sizeof(double);
    double* dev = nullptr;
    BA_CUDA(cudaMalloc(&dev, 2 * bytes));
    cudaError_t e = cudaMemcpy(dev, p_ref, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dev + (size_t)rows * cols, p_other, bytes, cudaMemcpyHostToDevice);
    int rc = BA_OK;
    if (e != cudaSuccess) rc = fail(BA_ERR_CUDA, "attention_fidelity: %s", cudaGetErrorString(e));
    else rc = ba_attention_fidelity(h, dev, dev + (size_t)rows * cols, rows, cols, k, out, nullptr);
    cudaFree(dev);
    return rc;
}

// A dense bf16 bias table the tensor-core kernels cannot tile by TMA (rows or base not 16-byte aligned: e.g. a contiguous
// [H,197,197] table) is copied once per call into a row-padded table owned by the handle; *bias and *pp (a copy of the
// caller's params with the new row stride) then describe that table.  Tables above 2 GiB are left alone (they take the
// direct-load path of the first-generation kernel / the CUDA-core kernel of the integer mode).
static int maybe_pad_bias(ba_handle* h, const ba_params* p, int kernel, const void** bias, ba_params* pp, cudaStream_t stream) {
    *pp = *p;
    if (p->bias_mode != BA_BIAS_DENSE || !*bias || p->bias_dtype != BA_BF16 || p->in_dtype != BA_BF16 || kernel != BA_KERNEL_TCGEN05)
        return BA_OK;
    const int64_t ld = p->bias_ld ? p->bias_ld : p->N;
    if ((ld * 2) % 16 == 0 && reinterpret_cast<uintptr_t>(*bias) % 16 == 0) return BA_OK;
    const int64_t ld_out = ((int64_t)p->N + 7) / 8 * 8;
    const size_t need = (size_t)p->bias_heads * p->N * ld_out * 2;
    if (need > ((size_t)2 << 30) || getenv("BA_NO_BIAS_PAD")) return BA_OK;
    int rc = ensure(&h->bias_pad, &h->bias_pad_bytes, need, false);
    if (rc) return rc;
    const int n = ba::launch_pad_bias_rows(*bias, ld, p->bias_heads, p->N, ld_out, h->bias_pad, stream);
    if (n < 0) return fail(BA_ERR_CUDA, "bias row padding launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    *bias = h->bias_pad;
    pp->bias_ld = ld_out;
    return BA_OK;
}

// One K1 + K2 pass over `heads` consecutive heads starting at grid index head0; every tensor pointer already points at
// that first head.  `ws` holds make_layout(p, heads).total bytes, `tickets` 2*heads zeroed counters.
static int fwd_range(ba_handle* h, const ba_params* p, int kernel, int64_t head0, int64_t heads, const void* Q, const void* K,
                     const void* V, const void* bias, void* O, float* row_max, float* row_sum, char* ws,
                     unsigned int* tickets, cudaStream_t stream, bool prof, int unit0 = 0, int unit1 = 0) {
    const Layout L = make_layout(p, heads);
    ba::FwdArgs a{};
    a.V = V;
    a.q_words = reinterpret_cast<uint64_t*>(ws + L.q_words);
    a.k_words = reinterpret_cast<uint64_t*>(ws + L.k_words);
    a.mu_q = reinterpret_cast<float*>(ws + L.mu_q);
    a.mu_k = reinterpret_cast<float*>(ws + L.mu_k);
    a.k_exp = L.total > L.kexp ? reinterpret_cast<const unsigned char*>(ws + L.kexp) : nullptr;
    a.q_exp = L.total > L.kexp ? reinterpret_cast<const unsigned char*>(ws + L.qexp) : nullptr;
    a.bias = p->bias_mode != BA_BIAS_NONE ? bias : nullptr;
    a.bias_kind = p->bias_mode;
    a.bias_dtype = p->bias_dtype;
    a.bias_ld = p->bias_ld ? p->bias_ld : p->N;
    if (p->bias_mode == BA_BIAS_REL2D) {
        const int g = grid_side(p->N);
        const bool in_kernel = kernel == BA_KERNEL_TCGEN05 && !p->quantize_pv && ba::tc2_shape_ok(p->in_dtype, p->N, p->d) &&
                               g % 32 == 0 && g <= 128 && !(getenv("BA_TC2") && atol(getenv("BA_TC2")) == 0) && a.k_exp &&
                               reinterpret_cast<uintptr_t>(V) % 16 == 0 && reinterpret_cast<uintptr_t>(O) % (p->out_bf16 ? 16 : 32) == 0;
        if (!in_kernel) {  // expand once into the handle's fp32 table and run the dense path (attention.cpp:78-96)
            const size_t need = (size_t)p->bias_heads * p->N * p->N * sizeof(float);
            int rc = ensure(&h->rel2d, &h->rel2d_bytes, need, false);
            if (rc) return rc;
            const int ne = ba::launch_expand_rel2d(bias, p->bias_dtype, p->bias_heads, p->N, g, static_cast<float*>(h->rel2d), stream);
            if (ne < 0) return fail(BA_ERR_CUDA, "relative-2d expansion launch: %s", cudaGetErrorString((cudaError_t)(-ne)));
            h->launches += ne;
            a.bias = h->rel2d;
            a.bias_kind = BA_BIAS_DENSE;
            a.bias_dtype = BA_F32;
            a.bias_ld = p->N;
        }
    }
    a.O = static_cast<float*>(O);
    a.out_bf16 = p->out_bf16 ? 1 : 0;
    a.row_max = row_max;
    a.row_sum = row_sum;
    a.BH = (int)heads;
    a.H = p->H;
    a.N = p->N;
    a.d = p->d;
    a.W64 = L.W64;
    a.bias_heads = p->bias_mode != BA_BIAS_NONE ? p->bias_heads : 1;
    a.head0 = (int)(head0 % p->H);
    a.unit0 = unit0;
    a.unit1 = unit1;
    a.in_dtype = p->in_dtype;
    a.inv_tau = p->inv_tau;

    cudaEvent_t* ev = prof ? h->prof_ev + 3 * h->prof_n : nullptr;
    if (prof) BA_CUDA(cudaEventRecord(ev[0], stream));
    int n = ba::launch_pack_signs_qk(Q, K, p->in_dtype, heads, p->N, p->d, const_cast<uint64_t*>(a.q_words),
                                     const_cast<uint64_t*>(a.k_words), const_cast<float*>(a.mu_q),
                                     const_cast<float*>(a.mu_k), reinterpret_cast<float*>(ws + L.partials), tickets, stream);
    if (n < 0) return fail(BA_ERR_CUDA, "pack_signs launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    if (prof) BA_CUDA(cudaEventRecord(ev[1], stream));
    if (p->quantize_pv) {  // the reference's default mode: s8 V levels (K1v), then the integer P.V kernel
        int8_t* vq = reinterpret_cast<int8_t*>(ws + L.vq);
        double* vs = reinterpret_cast<double*>(ws + L.vscales);
        const int ldq = ba::i8_level_ld(p->d);
        n = ba::launch_quantize_values(V, p->in_dtype, heads, p->N, p->d, vq, ldq, vs, stream);
        if (n < 0) return fail(BA_ERR_CUDA, "quantize_values launch: %s", cudaGetErrorString((cudaError_t)(-n)));
        h->launches += n;
        const int bc = p->block_cols ? p->block_cols : (p->N < 64 ? p->N : 64);
        // tensor-core path (u8 x s8 tcgen05.mma.kind::i8, the I8 mode of the second-generation kernel) where it takes the
        // shape; the CUDA-core kernel otherwise -- unless the caller insisted on the tensor cores
        n = kernel == BA_KERNEL_TCGEN05 ? ba::launch_attn_tc2_i8(a, vq, ldq, vs, bc, stream) : 0;
        if (n == 0 && p->kernel == BA_KERNEL_TCGEN05)
            return fail(BA_ERR_UNSUPPORTED, "quantize_pv=1 on the tensor cores needs bf16 inputs, d %% 8 == 0, d <= 128, N >= 128, "
                                            "block_cols = 64 and no bias or a dense bf16 table with 16-byte rows");
        if (n == 0) n = ba::launch_attn_int8(a, vq, ldq, vs, bc, stream);
    } else {
        n = kernel == BA_KERNEL_TCGEN05 ? ba::launch_attn_tcgen05(a, stream) : ba::launch_attn_simt(a, stream);
    }
    if (n < 0) return fail(BA_ERR_CUDA, "attention launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    if (prof) {
        BA_CUDA(cudaEventRecord(ev[2], stream));
        h->prof_n++;
    }
    return BA_OK;
}

static int resolve_kernel(const ba_params* p, int* kernel) {
    const char* why = "";
    const bool tc_ok = ba::tcgen05_supported(p, &why);
    int k = p->kernel;
    if (p->quantize_pv) {  // integer P.V: the tensor-core kernel where it takes the shape (decided at launch), else the CUDA cores
        if (k != BA_KERNEL_AUTO && k != BA_KERNEL_TCGEN05 && k != BA_KERNEL_SIMT) return fail(BA_ERR_VALIDATION, "unknown kernel id");
        *kernel = (k != BA_KERNEL_SIMT && ba::tc2_i8_shape_ok(p->in_dtype, p->N, p->d) && tc_ok) ? BA_KERNEL_TCGEN05 : BA_KERNEL_SIMT;
        if (k == BA_KERNEL_TCGEN05 && *kernel != BA_KERNEL_TCGEN05)
            return fail(BA_ERR_UNSUPPORTED, "quantize_pv=1 on the tensor cores needs bf16 inputs, d %% 8 == 0, d <= 128 and N >= 128");
        return BA_OK;
    }
    if (k == BA_KERNEL_AUTO) k = (tc_ok && p->N >= kAutoMinKeysTc) ? BA_KERNEL_TCGEN05 : BA_KERNEL_SIMT;
    if (k == BA_KERNEL_TCGEN05 && !tc_ok) return fail(BA_ERR_UNSUPPORTED, "tcgen05 kernel: %s", why);
    if (k != BA_KERNEL_TCGEN05 && k != BA_KERNEL_SIMT) return fail(BA_ERR_VALIDATION, "unknown kernel id");
    *kernel = k;
    return BA_OK;
}

int ba_binary_attention_fwd(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                            const void* bias, void* O, float* row_max, float* row_sum, void* workspace,
                            void* stream_) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, true);
    if (rc) return rc;
    if (!Q || !K || !V || !O) return fail(BA_ERR_SHAPE, "attention: Q, K, V and O must be non-NULL");
    if (p->bias_mode == BA_BIAS_DENSE && !bias) return fail(BA_ERR_SHAPE, "bias: dense table must be N x N (got NULL)");
    if (p->bias_mode == BA_BIAS_REL1D && !bias)
        return fail(BA_ERR_SHAPE, "bias: relative-1d offsets must have length 2N-1 (got NULL)");
    if (p->bias_mode == BA_BIAS_REL2D && !bias)
        return fail(BA_ERR_SHAPE, "bias: relative-2d tables must have length 2*sqrt(N)-1 (got NULL)");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    BA_BIND_DEVICE(h);
    int kernel = 0;
    if ((rc = resolve_kernel(p, &kernel))) return rc;
    ba_params padded_params;
    if ((rc = maybe_pad_bias(h, p, kernel, &bias, &padded_params, stream))) return rc;
    p = &padded_params;
    const Layout L = make_layout(p);
    if (!workspace) {
        if ((rc = ensure(&h->ws, &h->ws_bytes, L.total, false))) return rc;
        workspace = h->ws;
    }
    if ((rc = ensure_tickets(h, 2 * (size_t)L.BH))) return rc;
    const bool prof = h->prof_ev && h->prof_n < h->prof_cap;
    if (p->unit_end > p->unit_begin) {
        // unit-sharded call: K1 (and K, V, the scales) for every head the range touches, the attention kernel for the range only
        const int upb = ba::units_per_head(p->N);
        const int64_t hb = p->unit_begin / upb, he = (p->unit_end - 1) / upb + 1;
        const size_t in_head = (size_t)p->N * p->d * ba::dtype_size(p->in_dtype), out_head = (size_t)p->N * p->d * (p->out_bf16 ? 2 : sizeof(float));
        return fwd_range(h, p, kernel, hb, he - hb, static_cast<const char*>(Q) + hb * in_head, static_cast<const char*>(K) + hb * in_head,
                         static_cast<const char*>(V) + hb * in_head, bias, static_cast<char*>(O) + hb * out_head,
                         row_max ? row_max + hb * p->N : nullptr, row_sum ? row_sum + hb * p->N : nullptr,
                         static_cast<char*>(workspace), h->tickets, stream, prof, (int)(p->unit_begin - hb * upb),
                         (int)(p->unit_end - hb * upb));
    }
    if (p->unit_begin != 0 || p->unit_end != 0) return BA_OK;  // empty range
    return fwd_range(h, p, kernel, 0, L.BH, Q, K, V, bias, O, row_max, row_sum, static_cast<char*>(workspace), h->tickets,
                     stream, prof);
}

// Host-buffer call: the head grid is cut into chunks that flow through three streams -- H2D copies, K1+K2, D2H copies
// -- so the two PCIe directions and the kernels overlap (the copies are asynchronous only for pinned host memory).
int ba_binary_attention_host(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                             const void* bias, void* O, float* row_max, float* row_sum) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, true);
    if (rc) return rc;
    if (!Q || !K || !V || !O) return fail(BA_ERR_SHAPE, "attention: Q, K, V and O must be non-NULL");
    if (p->bias_mode != BA_BIAS_NONE && !bias) return fail(BA_ERR_SHAPE, "bias: table / offsets pointer is NULL");
    if (p->unit_begin != 0 || p->unit_end != 0) return fail(BA_ERR_UNSUPPORTED, "the host-buffer call takes whole batches (no unit range)");
    BA_BIND_DEVICE(h);
    int kernel = 0;
    if ((rc = resolve_kernel(p, &kernel))) return rc;
    const size_t BH = (size_t)p->B * p->H;
    const size_t head_in = (size_t)p->N * p->d * ba::dtype_size(p->in_dtype);  // bytes of one head of Q, K or V
    const size_t head_out = (size_t)p->N * p->d * (p->out_bf16 ? 2 : sizeof(float));
    const size_t head_row = (size_t)p->N * sizeof(float);
    const size_t ld = p->bias_ld ? p->bias_ld : p->N;
    const size_t bias_bytes =
        p->bias_mode == BA_BIAS_DENSE   ? (size_t)p->bias_heads * p->N * ld * ba::dtype_size(p->bias_dtype)
        : p->bias_mode == BA_BIAS_REL1D ? (size_t)p->bias_heads * (2 * (size_t)p->N - 1) * ba::dtype_size(p->bias_dtype)
        : p->bias_mode == BA_BIAS_REL2D ? (size_t)p->bias_heads * 2 * (2 * (size_t)grid_side(p->N) - 1) * ba::dtype_size(p->bias_dtype)
                                        : 0;
    // chunk plan: sizes ramp up 2 -> 4 -> 8 -> 16 MB (of EACH input) and back down at the end, so the pipeline fills and
    // drains on small chunks while the bulk moves in few large copies (measured on C2: 5.9 ms with uniform 4 MB chunks,
    // 5.5 ms with uniform 16 MB; every copy costs ~10 us of DMA setup, every chunk two kernel launches)
    static const size_t chunk_bytes = [] {  // dev knob: BA_HOST_CHUNK_MB = size of the large chunks
        const char* e = getenv("BA_HOST_CHUNK_MB");
        const long mb = e ? atol(e) : 0;
        return (size_t)(mb > 0 ? mb : 16) << 20;
    }();
    size_t plan[kHostChunksMax];
    int chunks = 0;
    {
        const size_t big = std::max<size_t>(1, chunk_bytes / head_in);
        const size_t small = std::max<size_t>(1, big / 8);
        size_t done = 0, up = small;
        size_t tail[4];
        int ntail = 0;
        size_t reserve = 0;  // heads kept for the ramp down: big/2, big/4, big/8
        for (size_t t = big / 2; t >= small && ntail < 3 && t >= 1; t /= 2) {
            tail[ntail++] = t;
            reserve += t;
            if (t == 1) break;
        }
        if (reserve * 2 > BH) {  // small problem: no ramp down
            ntail = 0;
            reserve = 0;
        }
        while (done < BH - reserve && chunks < kHostChunksMax - ntail - 1) {
            const size_t n = std::min(up, BH - reserve - done);
            plan[chunks++] = n;
            done += n;
            up = std::min(big, up * 2);
        }
        if (done < BH - reserve) {  // out of slots: one last big chunk takes the rest of the bulk
            plan[chunks++] = BH - reserve - done;
            done = BH - reserve;
        }
        for (int i = 0; i < ntail; ++i) plan[chunks++] = tail[i];
    }
    size_t per = 0;  // largest chunk (workspace slices are sized for it)
    for (int c = 0; c < chunks; ++c) per = std::max(per, plan[c]);
    const Layout Lc = make_layout(p, (int64_t)per);
    const bool bias_dev = p->bias_on_device != 0 && bias_bytes;  // the table already lives on this device
    const size_t need[8] = {BH * head_in, BH * head_in, BH * head_in, bias_dev ? 0 : bias_bytes, BH * head_out,
                            row_max ? BH * head_row : 0, row_sum ? BH * head_row : 0, (size_t)chunks * Lc.total};
    for (int i = 0; i < 8; ++i)
        if (need[i] && (rc = ensure(&h->stage[i], &h->stage_bytes[i], need[i], false))) return rc;
    if ((rc = ensure_tickets(h, 2 * BH))) return rc;
    char* const dQ = static_cast<char*>(h->stage[0]);
    char* const dK = static_cast<char*>(h->stage[1]);
    char* const dV = static_cast<char*>(h->stage[2]);
    char* const dO = static_cast<char*>(h->stage[4]);
    char* const dM = static_cast<char*>(h->stage[5]);
    char* const dL = static_cast<char*>(h->stage[6]);
    if (bias_bytes && !bias_dev) BA_CUDA(cudaMemcpyAsync(h->stage[3], bias, bias_bytes, cudaMemcpyHostToDevice, h->stream_in));
    // the table on the device, once per call (re-laid with 16-byte rows when the TMA tile loads need that), on the copy stream:
    // every chunk's kernels wait for an event recorded on it after this point
    const void* dbias = bias_dev ? bias : (bias_bytes ? h->stage[3] : nullptr);
    ba_params padded_params;
    if ((rc = maybe_pad_bias(h, p, kernel, &dbias, &padded_params, h->stream_in))) return rc;
    p = &padded_params;
    size_t h0 = 0;
    for (int c = 0; c < chunks; h0 += plan[c], ++c) {
        const size_t nh = plan[c];
        BA_CUDA(cudaMemcpyAsync(dQ + h0 * head_in, static_cast<const char*>(Q) + h0 * head_in, nh * head_in,
                                cudaMemcpyHostToDevice, h->stream_in));
        BA_CUDA(cudaMemcpyAsync(dK + h0 * head_in, static_cast<const char*>(K) + h0 * head_in, nh * head_in,
                                cudaMemcpyHostToDevice, h->stream_in));
        BA_CUDA(cudaMemcpyAsync(dV + h0 * head_in, static_cast<const char*>(V) + h0 * head_in, nh * head_in,
                                cudaMemcpyHostToDevice, h->stream_in));
        BA_CUDA(cudaEventRecord(h->ev_in[c], h->stream_in));
        BA_CUDA(cudaStreamWaitEvent(h->stream, h->ev_in[c], 0));
        rc = fwd_range(h, p, kernel, (int64_t)h0, (int64_t)nh, dQ + h0 * head_in, dK + h0 * head_in, dV + h0 * head_in,
                       dbias, dO + h0 * head_out,
                       row_max ? reinterpret_cast<float*>(dM + h0 * head_row) : nullptr,
                       row_sum ? reinterpret_cast<float*>(dL + h0 * head_row) : nullptr,
                       static_cast<char*>(h->stage[7]) + (size_t)c * Lc.total, h->tickets + 2 * h0, h->stream, false);
        if (rc) {  // copies from / to the caller's buffers may still be in flight: drain before handing them back
            cudaStreamSynchronize(h->stream_in);
            cudaStreamSynchronize(h->stream);
            cudaStreamSynchronize(h->stream_out);
            return rc;
        }
        BA_CUDA(cudaEventRecord(h->ev_done[c], h->stream));
        BA_CUDA(cudaStreamWaitEvent(h->stream_out, h->ev_done[c], 0));
        BA_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(O) + h0 * head_out, dO + h0 * head_out, nh * head_out,
                                cudaMemcpyDeviceToHost, h->stream_out));
        if (row_max)
            BA_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(row_max) + h0 * head_row, dM + h0 * head_row, nh * head_row,
                                    cudaMemcpyDeviceToHost, h->stream_out));
        if (row_sum)
            BA_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(row_sum) + h0 * head_row, dL + h0 * head_row, nh * head_row,
                                    cudaMemcpyDeviceToHost, h->stream_out));
    }
    BA_CUDA(cudaStreamSynchronize(h->stream_out));
    BA_CUDA(cudaStreamSynchronize(h->stream));
    BA_CUDA(cudaStreamSynchronize(h->stream_in));
    return BA_OK;
}

}  // extern "C"
