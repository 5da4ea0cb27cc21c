// binattn_cuda.cu -- host side of the C ABI declared in include/binattn_cuda.h.
//
// Thin by design: validates the call the way binattn::check_shapes does (proj/src/attention.cpp:17-29),
// lays the workspace out, and launches K1 (pack_signs.cu) followed by one fused K2 kernel
// (attn_tcgen05.cu or attn_simt.cu).  No CPU fallback exists: every compute entry point ends in a
// CUDA kernel launch or an error code.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ba_common.cuh"

namespace ba {
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

struct Layout {
    size_t q_words, k_words, mu_q, mu_k, partials, total;
    int64_t BH;
    int W64, chunks;
};

Layout make_layout(const ba_params* p) {
    Layout L{};
    L.BH = (int64_t)p->B * p->H;
    L.W64 = (p->d + 63) / 64;
    L.chunks = ba::pack_partials_per_head(p->N, p->d, p->in_dtype);
    const size_t plane = align_up((size_t)L.BH * p->N * L.W64 * sizeof(uint64_t), 256);
    size_t off = 0;
    L.q_words = off; off += plane;
    L.k_words = off; off += plane;
    L.mu_q = off; off += align_up((size_t)L.BH * sizeof(float), 256);
    L.mu_k = off; off += align_up((size_t)L.BH * sizeof(float), 256);
    L.partials = off; off += align_up(2 * (size_t)L.BH * L.chunks * sizeof(float), 256);
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
    if (p->bias_mode != BA_BIAS_NONE && p->bias_mode != BA_BIAS_DENSE)
        return fail(BA_ERR_VALIDATION, "bias_mode must be BA_BIAS_NONE or BA_BIAS_DENSE");
    if (p->bias_mode == BA_BIAS_DENSE) {
        if (p->bias_heads != 1 && p->bias_heads != p->H)  // attention.cpp:60-61 (table must match the head)
            return fail(BA_ERR_SHAPE, "bias: dense table must be [1 or H, N, N]");
        if (p->bias_ld != 0 && p->bias_ld < p->N) return fail(BA_ERR_SHAPE, "bias: bias_ld must be >= N");
        if (p->bias_dtype != BA_BF16 && p->bias_dtype != BA_F32)
            return fail(BA_ERR_VALIDATION, "bias_dtype must be BA_BF16 or BA_F32");
    }
    if (p->d > 256) return fail(BA_ERR_UNSUPPORTED, "head dim %d > 256 is not supported", p->d);
    return BA_OK;
}

}  // namespace

struct ba_handle {
    int device = 0;
    int64_t launches = 0;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    unsigned int* tickets = nullptr;
    size_t tickets_n = 0;
    float* partials = nullptr;  // for standalone ba_pack_signs
    size_t partials_n = 0;
    // host-buffer path
    cudaStream_t stream = nullptr;
    void* stage[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t stage_bytes[7] = {0, 0, 0, 0, 0, 0, 0};
    // per-kernel profiling (ba_profile_begin/end)
    cudaEvent_t* prof_ev = nullptr;
    int prof_cap = 0, prof_n = 0;
};

namespace {

int ensure(void** ptr, size_t* have, size_t need, bool zero) {
    if (*have >= need && *ptr) return BA_OK;
    if (*ptr) BA_CUDA(cudaFree(*ptr));
    *ptr = nullptr;
    *have = 0;
    BA_CUDA(cudaMalloc(ptr, need));
    if (zero) BA_CUDA(cudaMemset(*ptr, 0, need));
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
    BA_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    BA_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(BA_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device,
                    prop.major, prop.minor);
    ba_handle* h = new ba_handle();
    h->device = device;
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete h;
        return fail(BA_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    *out = h;
    return BA_OK;
}

int ba_destroy(ba_handle* h) {
    if (!h) return BA_OK;
    cudaSetDevice(h->device);
    if (h->ws) cudaFree(h->ws);
    if (h->tickets) cudaFree(h->tickets);
    if (h->partials) cudaFree(h->partials);
    for (void* s : h->stage)
        if (s) cudaFree(s);
    if (h->stream) cudaStreamDestroy(h->stream);
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
    BA_CUDA(cudaSetDevice(h->device));
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

int ba_select_kernel(const ba_params* p) {
    if (check_params(p, true) != BA_OK) return -1;
    const char* why = nullptr;
    if (p->kernel == BA_KERNEL_SIMT) return BA_KERNEL_SIMT;
    return ba::tcgen05_supported(p, &why) ? BA_KERNEL_TCGEN05 : (p->kernel == BA_KERNEL_TCGEN05 ? -1 : BA_KERNEL_SIMT);
}

int ba_pack_signs(ba_handle* h, const ba_params* p, const void* X, uint64_t* words, float* mu, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, false);
    if (rc) return rc;
    if (!X || !words) return fail(BA_ERR_SHAPE, "pack_signs: X and words must be non-NULL");
    BA_CUDA(cudaSetDevice(h->device));
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

int ba_binary_logits(ba_handle* h, const ba_params* p, const uint64_t* q_words, const uint64_t* k_words,
                     int64_t head_index, int32_t* S, void* stream) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, false);
    if (rc) return rc;
    if (!q_words || !k_words || !S) return fail(BA_ERR_SHAPE, "binary_logits: NULL pointer");
    const int64_t BH = (int64_t)p->B * p->H;
    if (head_index < 0 || head_index >= BH) return fail(BA_ERR_SHAPE, "binary_logits: head %lld outside [0,%lld)",
                                                        (long long)head_index, (long long)BH);
    BA_CUDA(cudaSetDevice(h->device));
    const int W64 = (p->d + 63) / 64;
    const int64_t off = head_index * p->N * W64;
    const int n = ba::launch_binary_logits(q_words + off, k_words + off, p->N, p->d, S, static_cast<cudaStream_t>(stream));
    if (n < 0) return fail(BA_ERR_CUDA, "binary_logits launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    return BA_OK;
}

int ba_binary_attention_fwd(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                            const void* bias, float* O, float* row_max, float* row_sum, void* workspace,
                            void* stream_) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, true);
    if (rc) return rc;
    if (!Q || !K || !V || !O) return fail(BA_ERR_SHAPE, "attention: Q, K, V and O must be non-NULL");
    if (p->bias_mode == BA_BIAS_DENSE && !bias) return fail(BA_ERR_SHAPE, "bias: dense table must be N x N (got NULL)");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    BA_CUDA(cudaSetDevice(h->device));

    const char* why = "";
    const bool tc_ok = ba::tcgen05_supported(p, &why);
    int kernel = p->kernel;
    if (kernel == BA_KERNEL_AUTO) kernel = tc_ok ? BA_KERNEL_TCGEN05 : BA_KERNEL_SIMT;
    if (kernel == BA_KERNEL_TCGEN05 && !tc_ok) return fail(BA_ERR_UNSUPPORTED, "tcgen05 kernel: %s", why);
    if (kernel != BA_KERNEL_TCGEN05 && kernel != BA_KERNEL_SIMT) return fail(BA_ERR_VALIDATION, "unknown kernel id");

    const Layout L = make_layout(p);
    if (!workspace) {
        if ((rc = ensure(&h->ws, &h->ws_bytes, L.total, false))) return rc;
        workspace = h->ws;
    }
    if ((rc = ensure_tickets(h, 2 * (size_t)L.BH))) return rc;
    char* ws = static_cast<char*>(workspace);

    ba::FwdArgs a{};
    a.V = V;
    a.q_words = reinterpret_cast<uint64_t*>(ws + L.q_words);
    a.k_words = reinterpret_cast<uint64_t*>(ws + L.k_words);
    a.mu_q = reinterpret_cast<float*>(ws + L.mu_q);
    a.mu_k = reinterpret_cast<float*>(ws + L.mu_k);
    a.bias = p->bias_mode == BA_BIAS_DENSE ? bias : nullptr;
    a.O = O;
    a.row_max = row_max;
    a.row_sum = row_sum;
    a.bias_ld = p->bias_ld ? p->bias_ld : p->N;
    a.BH = (int)L.BH;
    a.H = p->H;
    a.N = p->N;
    a.d = p->d;
    a.W64 = L.W64;
    a.bias_heads = p->bias_mode == BA_BIAS_DENSE ? p->bias_heads : 1;
    a.bias_dtype = p->bias_dtype;
    a.in_dtype = p->in_dtype;
    a.inv_tau = p->inv_tau;

    const bool prof = h->prof_ev && h->prof_n < h->prof_cap;
    cudaEvent_t* ev = prof ? h->prof_ev + 3 * h->prof_n : nullptr;
    if (prof) BA_CUDA(cudaEventRecord(ev[0], stream));
    int n = ba::launch_pack_signs_qk(Q, K, p->in_dtype, L.BH, p->N, p->d, const_cast<uint64_t*>(a.q_words),
                                     const_cast<uint64_t*>(a.k_words), const_cast<float*>(a.mu_q),
                                     const_cast<float*>(a.mu_k), reinterpret_cast<float*>(ws + L.partials), h->tickets,
                                     stream);
    if (n < 0) return fail(BA_ERR_CUDA, "pack_signs launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    if (prof) BA_CUDA(cudaEventRecord(ev[1], stream));
    n = kernel == BA_KERNEL_TCGEN05 ? ba::launch_attn_tcgen05(a, stream) : ba::launch_attn_simt(a, stream);
    if (n < 0) return fail(BA_ERR_CUDA, "attention launch: %s", cudaGetErrorString((cudaError_t)(-n)));
    h->launches += n;
    if (prof) {
        BA_CUDA(cudaEventRecord(ev[2], stream));
        h->prof_n++;
    }
    return BA_OK;
}

int ba_binary_attention_host(ba_handle* h, const ba_params* p, const void* Q, const void* K, const void* V,
                             const void* bias, float* O, float* row_max, float* row_sum) {
    if (!h) return fail(BA_ERR_VALIDATION, "handle is NULL");
    int rc = check_params(p, true);
    if (rc) return rc;
    if (!Q || !K || !V || !O) return fail(BA_ERR_SHAPE, "attention: Q, K, V and O must be non-NULL");
    if (p->bias_mode == BA_BIAS_DENSE && !bias) return fail(BA_ERR_SHAPE, "bias: dense table must be N x N (got NULL)");
    BA_CUDA(cudaSetDevice(h->device));
    const size_t BH = (size_t)p->B * p->H;
    const size_t in_bytes = BH * p->N * p->d * ba::dtype_size(p->in_dtype);
    const size_t out_bytes = BH * p->N * p->d * sizeof(float);
    const size_t ld = p->bias_ld ? p->bias_ld : p->N;
    const size_t bias_bytes =
        p->bias_mode == BA_BIAS_DENSE ? (size_t)p->bias_heads * p->N * ld * ba::dtype_size(p->bias_dtype) : 0;
    const size_t row_bytes = BH * p->N * sizeof(float);
    const size_t need[7] = {in_bytes, in_bytes, in_bytes, bias_bytes, out_bytes, row_max ? row_bytes : 0,
                            row_sum ? row_bytes : 0};
    for (int i = 0; i < 7; ++i)
        if (need[i] && (rc = ensure(&h->stage[i], &h->stage_bytes[i], need[i], false))) return rc;
    cudaStream_t s = h->stream;
    BA_CUDA(cudaMemcpyAsync(h->stage[0], Q, in_bytes, cudaMemcpyHostToDevice, s));
    BA_CUDA(cudaMemcpyAsync(h->stage[1], K, in_bytes, cudaMemcpyHostToDevice, s));
    BA_CUDA(cudaMemcpyAsync(h->stage[2], V, in_bytes, cudaMemcpyHostToDevice, s));
    if (bias_bytes) BA_CUDA(cudaMemcpyAsync(h->stage[3], bias, bias_bytes, cudaMemcpyHostToDevice, s));
    rc = ba_binary_attention_fwd(h, p, h->stage[0], h->stage[1], h->stage[2], bias_bytes ? h->stage[3] : nullptr,
                                 static_cast<float*>(h->stage[4]), row_max ? static_cast<float*>(h->stage[5]) : nullptr,
                                 row_sum ? static_cast<float*>(h->stage[6]) : nullptr, nullptr, s);
    if (rc) return rc;
    BA_CUDA(cudaMemcpyAsync(O, h->stage[4], out_bytes, cudaMemcpyDeviceToHost, s));
    if (row_max) BA_CUDA(cudaMemcpyAsync(row_max, h->stage[5], row_bytes, cudaMemcpyDeviceToHost, s));
    if (row_sum) BA_CUDA(cudaMemcpyAsync(row_sum, h->stage[6], row_bytes, cudaMemcpyDeviceToHost, s));
    BA_CUDA(cudaStreamSynchronize(s));
    return BA_OK;
}

}  // extern "C"
