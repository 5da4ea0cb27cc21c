// ref_shim.cpp -- extern "C" doorway into the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (same rule as binattn_oracle.c).  This file is ours;
// it is compiled together with the reference's own sources where they lie under
// /root/reference/proj/src (see oracle/Makefile) into oracle/_ref/libbinattn_ref.so.
// Nothing from the reference is copied into this repository.  The flat C
// signatures mirror binattn_oracle.c one-to-one so tests can diff the two.
#include <functional>
#include <cstring>
#include <cstdint>
#include <cstring>
#include <optional>
#include <thread>
#include <vector>

#include "binattn/attention.hpp"
#include "binattn/errors.hpp"
#include "binattn/tensor_file.hpp"
#include "binattn/bitops.hpp"
#include "binattn/fidelity.hpp"
#include "binattn/parallel.hpp"
#include "binattn/quantize.hpp"
#include "binattn/rng.hpp"

using namespace binattn;

namespace {

DenseMatrix dm(const double* p, std::size_t r, std::size_t c) {
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

int guarded(const std::function<void()>& fn) {
    try {
        fn();
        return 0;
    } catch (const ShapeError&) {
        return 1;
    } catch (const ValidationError&) {
        return 2;
    } catch (const Error&) {
        return 4;
    }
}

AttentionConfig mkcfg(std::size_t n, std::size_t d, double tau, std::size_t br, std::size_t bc, int qpv,
                      const double* bias) {
    AttentionConfig cfg;
    cfg.seq_len = n;
    cfg.head_dim = d;
    cfg.temperature = tau;
    cfg.block_rows = br;
    cfg.block_cols = bc;
    cfg.quantize_pv = qpv != 0;
    if (bias) cfg.bias = BiasSpec{DenseBias{dm(bias, n, n)}};
    return cfg;
}

void emit(const AttentionOutput& out, double* y, double* m, double* l) {
    std::memcpy(y, out.output.data().data(), out.output.size() * sizeof(double));
    if (m) std::memcpy(m, out.row_max.data(), out.row_max.size() * sizeof(double));
    if (l) std::memcpy(l, out.row_sum.data(), out.row_sum.size() * sizeof(double));
}

struct RngBox {
    std::mt19937_64 rng;
};

} // namespace

extern "C" {

void ref_set_max_threads(int n) { set_max_threads(n); }
int ref_max_threads() { return max_threads(); }

// rng.hpp make_rng + tests/oracles.hpp random_dense semantics (fresh GaussianSource per matrix).
void* ref_rng_new(std::uint64_t seed, std::uint64_t stream) { return new RngBox{make_rng(seed, stream)}; }
void ref_rng_free(void* r) { delete static_cast<RngBox*>(r); }
std::uint64_t ref_rng_u64(void* r) { return static_cast<RngBox*>(r)->rng(); }
void ref_random_dense(void* r, std::size_t count, double scale, double* out) {
    GaussianSource gauss(static_cast<RngBox*>(r)->rng);
    for (std::size_t i = 0; i < count; ++i) out[i] = scale * gauss();
}

int ref_pack_signs(const double* m, std::size_t rows, std::size_t d, std::uint64_t* words) {
    return guarded([&] {
        const BitMatrix b = pack_signs(dm(m, rows, d));
        std::memcpy(words, b.words().data(), b.words().size() * sizeof(std::uint64_t));
    });
}

int ref_binary_quantize(const double* m, std::size_t rows, std::size_t d, std::uint64_t* words, double* mu) {
    return guarded([&] {
        const ScaledBinary sb = binary_quantize(dm(m, rows, d));
        std::memcpy(words, sb.bits.words().data(), sb.bits.words().size() * sizeof(std::uint64_t));
        *mu = sb.scale;
    });
}

std::int64_t ref_xnor_popcount_dot(const std::uint64_t* a, const std::uint64_t* b, std::size_t d) {
    const std::size_t w = BitMatrix::words_needed(d);
    return xnor_popcount_dot(std::span<const std::uint64_t>(a, w), std::span<const std::uint64_t>(b, w), d);
}

std::uint64_t ref_hamming_distance(const std::uint64_t* a, const std::uint64_t* b, std::size_t d) {
    const std::size_t w = BitMatrix::words_needed(d);
    return hamming_distance(std::span<const std::uint64_t>(a, w), std::span<const std::uint64_t>(b, w), d);
}

int ref_binary_gemm(const std::uint64_t* s, std::size_t n, const std::uint64_t* t, std::size_t m, std::size_t d,
                    std::int32_t* out) {
    return guarded([&] {
        const std::size_t w = BitMatrix::words_needed(d);
        const BitMatrix a(n, d, std::vector<std::uint64_t>(s, s + n * w));
        const BitMatrix b(m, d, std::vector<std::uint64_t>(t, t + m * w));
        const Int32Matrix g = binary_gemm(a, b);
        std::memcpy(out, g.data.data(), g.data.size() * sizeof(std::int32_t));
    });
}

int ref_quantize_values(const double* v, std::size_t rows, std::size_t cols, std::int8_t* data, double* scales) {
    return guarded([&] {
        const QuantizedValues q = quantize_values(dm(v, rows, cols));
        std::memcpy(data, q.data().data(), rows * cols);
        std::memcpy(scales, q.channel_scales().data(), cols * sizeof(double));
    });
}

int ref_materialize_bias_rel1d(const double* offsets, std::size_t n, double* table) {
    return guarded([&] {
        const DenseMatrix b =
            materialize_bias(BiasSpec{Relative1dBias{std::vector<double>(offsets, offsets + 2 * n - 1)}}, n);
        std::memcpy(table, b.data().data(), n * n * sizeof(double));
    });
}

int ref_materialize_bias_rel2d(const double* row_off, const double* col_off, std::size_t g2m1, std::size_t n,
                               double* table) {
    return guarded([&] {
        const DenseMatrix b = materialize_bias(
            BiasSpec{Relative2dBias{std::vector<double>(row_off, row_off + g2m1),
                                    std::vector<double>(col_off, col_off + g2m1)}},
            n);
        std::memcpy(table, b.data().data(), n * n * sizeof(double));
    });
}

// fidelity.cpp:40-85 attention_fidelity -> {cos_sim, relative_l1, rmse, precision_at_k}
int ref_attention_fidelity(const double* p_ref, const double* p_other, std::size_t rows, std::size_t cols, std::size_t k,
                           double* out) {
    return guarded([&] {
        const FidelityReport r = attention_fidelity(dm(p_ref, rows, cols), dm(p_other, rows, cols), k);
        out[0] = r.cos_sim;
        out[1] = r.relative_l1;
        out[2] = r.rmse;
        out[3] = r.precision_at_k;
    });
}

int ref_reference_attention(const double* q, const double* k, const double* v, std::size_t n, std::size_t d,
                            double tau, const double* bias, double* y, double* m, double* l, double* probs) {
    return guarded([&] {
        const AttentionConfig cfg = mkcfg(n, d, tau, 1, 1, 0, bias);
        const AttentionOutput out = reference_attention(dm(q, n, d), dm(k, n, d), dm(v, n, d), cfg, probs != nullptr);
        emit(out, y, m, l);
        if (probs) std::memcpy(probs, out.probs->data().data(), n * n * sizeof(double));
    });
}

int ref_binary_attention_unfused(const double* q, const double* k, const double* v, std::size_t n, std::size_t d,
                                 double tau, int qpv, const double* bias, double* y, double* m, double* l,
                                 double* probs) {
    return guarded([&] {
        const AttentionConfig cfg = mkcfg(n, d, tau, 1, 1, qpv, bias);
        const AttentionOutput out =
            binary_attention_unfused(dm(q, n, d), dm(k, n, d), dm(v, n, d), cfg, probs != nullptr);
        emit(out, y, m, l);
        if (probs) std::memcpy(probs, out.probs->data().data(), n * n * sizeof(double));
    });
}

int ref_binary_attention_fused(const double* q, const double* k, const double* v, std::size_t n, std::size_t d,
                               double tau, std::size_t br, std::size_t bc, int qpv, const double* bias, double* y,
                               double* m, double* l) {
    return guarded([&] {
        const AttentionConfig cfg = mkcfg(n, d, tau, br, bc, qpv, bias);
        const AttentionOutput out = binary_attention_fused(dm(q, n, d), dm(k, n, d), dm(v, n, d), cfg, false);
        emit(out, y, m, l);
    });
}

// Heads are independent calls.  nthreads host threads each run whole heads with the
// library's intra-call parallelism capped by intra_threads (set_max_threads is process-global).
int ref_binary_attention_fused_heads(const double* q, const double* k, const double* v, std::size_t heads,
                                     std::size_t n, std::size_t d, double tau, std::size_t br, std::size_t bc,
                                     int qpv, const double* bias, std::size_t bias_heads, double* y, int nthreads,
                                     int intra_threads) {
    if (nthreads < 1) nthreads = 1;
    if (static_cast<std::size_t>(nthreads) > heads) nthreads = static_cast<int>(heads);
    set_max_threads(intra_threads);
    std::vector<int> rcs(static_cast<std::size_t>(nthreads), 0);
    std::vector<std::thread> pool;
    const std::size_t chunk = (heads + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        pool.emplace_back([&, t] {
            const std::size_t b = t * chunk, e = std::min(heads, b + chunk);
            for (std::size_t h = b; h < e; ++h) {
                const double* bh = bias ? bias + (h % (bias_heads ? bias_heads : 1)) * n * n : nullptr;
                const int rc = ref_binary_attention_fused(q + h * n * d, k + h * n * d, v + h * n * d, n, d, tau, br,
                                                          bc, qpv, bh, y + h * n * d, nullptr, nullptr);
                if (rc) rcs[t] = rc;
            }
        });
    }
    for (auto& th : pool) th.join();
    set_max_threads(0);
    for (int rc : rcs)
        if (rc) return rc;
    return 0;
}

// ---- BATF tensor files (tensor_file.hpp:11-23): the reference's own writer / reader, for byte-level interchange checks.
// Return 0 on success, 2 = FormatError, 3 = IoError, 1 = any other binattn::Error.
static int guard_file(const std::function<void()>& f) {
    try {
        f();
        return 0;
    } catch (const FormatError&) {
        return 2;
    } catch (const IoError&) {
        return 3;
    } catch (const Error&) {
        return 1;
    }
}
int ref_write_dense(const char* path, const double* data, std::size_t rows, std::size_t cols, int as_f32) {
    return guard_file([&] {
        write_tensor(path, DenseMatrix(rows, cols, std::vector<double>(data, data + rows * cols), as_f32 ? Dtype::f32 : Dtype::f64));
    });
}
int ref_write_bits(const char* path, const std::uint64_t* words, std::size_t rows, std::size_t cols) {
    return guard_file([&] {
        write_tensor(path, BitMatrix(rows, cols, std::vector<std::uint64_t>(words, words + rows * BitMatrix::words_needed(cols))));
    });
}
// Reads any BATF file with the reference reader; reports dtype code and dims, and copies the payload into the buffer that
// matches the dtype (dense -> f64 values, packed-bit -> u64 words, int8/uint8 -> bytes, int8 scales -> f64).
int ref_read_tensor(const char* path, int* dtype, std::size_t* rows, std::size_t* cols, double* dense, std::uint64_t* words,
                    unsigned char* bytes, double* scales) {
    return guard_file([&] {
        const TensorVariant t = read_tensor(path);
        if (const auto* m = std::get_if<DenseMatrix>(&t)) {
            *dtype = m->storage() == Dtype::f32 ? 0 : 1;
            *rows = m->rows();
            *cols = m->cols();
            if (dense) std::copy(m->data().begin(), m->data().end(), dense);
        } else if (const auto* b = std::get_if<BitMatrix>(&t)) {
            *dtype = 4;
            *rows = b->rows();
            *cols = b->logical_cols();
            if (words) std::copy(b->words().begin(), b->words().end(), words);
        } else if (const auto* q = std::get_if<QuantizedValues>(&t)) {
            *dtype = 2;
            *rows = q->rows();
            *cols = q->cols();
            if (bytes) std::memcpy(bytes, q->data().data(), q->data().size());
            if (scales) std::copy(q->channel_scales().begin(), q->channel_scales().end(), scales);
        } else {
            const auto& c = std::get<QuantizedCoeffs>(t);
            *dtype = 3;
            *rows = c.rows();
            *cols = c.cols();
            if (bytes) std::memcpy(bytes, c.data().data(), c.data().size());
        }
    });
}

} // extern "C"
