// binattn_b200.hpp -- C++ host-side mirror of the reference operator API over the C ABI (binattn_cuda.h).
//
// Mirrors, name for name, the part of the reference a caller of the hot path touches:
//   binattn::AttentionConfig / ::make        proj/include/binattn/attention.hpp:29-41, proj/src/attention.cpp:45-53
//   binattn::AttentionOutput                 attention.hpp:43-48
//   binattn::binary_attention_fused          attention.hpp:69-71 (attention.cpp:250-382)
//   binattn::ShapeError / ValidationError    proj/include/binattn/errors.hpp:16-25   (thrown for the same conditions:
//                                            attention.cpp:21-28 shapes / temperature / block sizes, :60-61 bias table)
// and BASELINE.json's operator shape  binary_attention(Q, K, V, bias, scale) -> O.
//
// Header-only and templated on the matrix type so it can be compiled against the reference's own
// binattn::DenseMatrix (tensor.hpp:25-53) without copying it: any type with rows(), cols(), data() (contiguous
// row-major doubles exposing .data()/.size()) and a (rows, cols, std::vector<double>) constructor works.
// The reference computes in fp64 on the host; this shim uploads the operands in the requested device precision:
//   Precision::f32  -- values rounded to fp32; sign bits identical to the reference unless |x| < 1.4e-45
//                      (CUDA-core kernel; use this when bit-identical packed signs matter for arbitrary doubles)
//   Precision::bf16 -- values rounded to bf16 (tcgen05 kernel; what the benchmarks use; inputs that already are
//                      bf16-representable -- e.g. activations of a bf16 model -- lose nothing)
// Output O is fp32 on the device, widened to double here.  with_probs is diagnostics-only in the reference and is not carried
// over (attention_probs / attention_fidelity cover its callers).
//
// !! ONE DELIBERATE DEVIATION FROM THE REFERENCE'S DEFAULTS: AttentionConfigT::quantize_pv defaults to FALSE here, the
// reference's AttentionConfig to TRUE (attention.hpp:35).  false = fp P.V, the mode the tensor-core product path implements
// and the one O-parity (<= 2e-3) is defined against (the reference's own int8 mode is 1.3e-3..5.5e-3
// away from its fp64 mode); true = the reference's u8 x s8 integer P.V, here on the tensor cores for bf16 inputs (d <= 128) and on the CUDA cores otherwise (same key-block
// semantics, within 1e-3 of the reference's result).  A caller porting `AttentionConfig::make(n, d)` who wants the
// reference's default arithmetic must set cfg.quantize_pv = true.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "binattn_cuda.h"

namespace binattn::b200 {

class Error : public std::runtime_error {  // errors.hpp:10-13
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class ShapeError : public Error {  // errors.hpp:16-19
public:
    explicit ShapeError(const std::string& msg) : Error(msg) {}
};
class ValidationError : public Error {  // errors.hpp:22-25
public:
    explicit ValidationError(const std::string& msg) : Error(msg) {}
};
class CudaError : public Error {
public:
    explicit CudaError(const std::string& msg) : Error(msg) {}
};
class UnsupportedError : public Error {
public:
    explicit UnsupportedError(const std::string& msg) : Error(msg) {}
};

inline void check(int rc) {
    if (rc == BA_OK) return;
    const std::string msg = ba_last_error();
    switch (rc) {
        case BA_ERR_SHAPE: throw ShapeError(msg);
        case BA_ERR_VALIDATION: throw ValidationError(msg);
        case BA_ERR_UNSUPPORTED: throw UnsupportedError(msg);
        default: throw CudaError(msg);
    }
}

enum class Precision { f32, bf16 };

// binattn::AttentionConfig (attention.hpp:29-41) with the dense form of BiasSpec (materialize_bias output).
template <class DenseMatrixT>
struct AttentionConfigT {
    std::size_t seq_len = 0;
    std::size_t head_dim = 0;
    double temperature = 1.0;
    std::size_t block_rows = 64;  // validated like the reference; the CUDA kernels choose their own tiles
    std::size_t block_cols = 64;
    bool quantize_pv = false;
    std::optional<DenseMatrixT> bias;  // DenseBias: N x N table (attention.hpp:15-17)
    std::vector<double> rel1d_offsets;  // Relative1dBias: 2N-1 offsets, b_ij = offsets[i-j+N-1] (attention.hpp:18-21); empty = unused
    std::vector<double> rel2d_row_offsets, rel2d_col_offsets;  // Relative2dBias: 2*sqrt(N)-1 each (attention.hpp:22-26); empty = unused
    Precision precision = Precision::f32;

    static AttentionConfigT make(std::size_t n, std::size_t d) {  // attention.cpp:45-53
        AttentionConfigT cfg;
        cfg.seq_len = n;
        cfg.head_dim = d;
        cfg.temperature = std::sqrt(static_cast<double>(d));
        cfg.block_rows = n < 64 ? n : 64;
        cfg.block_cols = n < 64 ? n : 64;
        return cfg;
    }
};

template <class DenseMatrixT>
struct AttentionOutputT {  // attention.hpp:43-48 (probs is never produced)
    DenseMatrixT output;
    std::vector<double> row_max;
    std::vector<double> row_sum;
};

inline std::uint16_t to_bf16_bits(double x) {  // round-to-nearest-even
    float f = static_cast<float>(x);
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<std::uint16_t>(u >> 16);
}

struct FidelityReport {  // fidelity.hpp:12-18
    double cos_sim = 0.0, relative_l1 = 0.0, rmse = 0.0, precision_at_k = 0.0;
    std::size_t k = 0;
};

// One ba_handle per device; not copyable.
class Engine {
public:
    explicit Engine(int device = 0) { check(ba_create(device, &h_)); }
    ~Engine() { ba_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ba_handle* handle() const { return h_; }

    // binattn::binary_attention_fused(q, k, v, cfg): one head, N x d matrices.
    template <class DenseMatrixT>
    AttentionOutputT<DenseMatrixT> binary_attention_fused(const DenseMatrixT& q, const DenseMatrixT& k,
                                                          const DenseMatrixT& v,
                                                          const AttentionConfigT<DenseMatrixT>& cfg) const {
        const std::size_t n = cfg.seq_len, d = cfg.head_dim;
        // check_shapes, attention.cpp:17-29 (same messages, same exception types)
        if (q.rows() != n || q.cols() != d) throw ShapeError("attention: Q must be N x d");
        if (k.rows() != n || k.cols() != d) throw ShapeError("attention: K must be N x d");
        if (v.rows() != n || v.cols() != d) throw ShapeError("attention: V must be N x d");
        if (!(cfg.temperature > 0.0)) throw ValidationError("attention: temperature must be positive");
        if (cfg.block_rows < 1 || cfg.block_rows > n || cfg.block_cols < 1 || cfg.block_cols > n)
            throw ValidationError("attention: block sizes must be in [1, N]");
        if (cfg.bias && (cfg.bias->rows() != n || cfg.bias->cols() != n))
            throw ShapeError("bias: dense table must be N x N");  // attention.cpp:60-61
        const bool rel1d = !cfg.rel1d_offsets.empty();
        const bool rel2d = !cfg.rel2d_row_offsets.empty() || !cfg.rel2d_col_offsets.empty();
        if ((rel1d ? 1 : 0) + (rel2d ? 1 : 0) + (cfg.bias ? 1 : 0) > 1)
            throw ValidationError("bias: give ONE of a dense table, relative-1d offsets, relative-2d tables");
        if (rel1d && cfg.rel1d_offsets.size() != 2 * n - 1)
            throw ShapeError("bias: relative-1d offsets must have length 2N-1");  // attention.cpp:66-67
        if (rel2d) {
            const std::size_t g = static_cast<std::size_t>(std::lround(std::sqrt(static_cast<double>(n))));
            if (g * g != n) throw ShapeError("bias: relative-2d requires N to be a perfect square");  // attention.cpp:79-81
            if (cfg.rel2d_row_offsets.size() != 2 * g - 1 || cfg.rel2d_col_offsets.size() != 2 * g - 1)
                throw ShapeError("bias: relative-2d tables must have length 2*sqrt(N)-1");  // attention.cpp:82-83
        }
        if (n == 0 || d == 0) throw ShapeError("binary_quantize: empty matrix");  // quantize.cpp:17

        ba_params p{};
        p.B = 1;
        p.H = 1;
        p.N = static_cast<int32_t>(n);
        p.d = static_cast<int32_t>(d);
        p.in_dtype = cfg.precision == Precision::bf16 ? BA_BF16 : BA_F32;
        p.bias_mode = cfg.bias ? BA_BIAS_DENSE : rel1d ? BA_BIAS_REL1D : rel2d ? BA_BIAS_REL2D : BA_BIAS_NONE;
        p.bias_heads = 1;
        p.bias_dtype = BA_F32;
        p.bias_ld = 0;
        p.inv_tau = static_cast<float>(1.0 / cfg.temperature);
        p.kernel = BA_KERNEL_AUTO;
        p.quantize_pv = cfg.quantize_pv ? 1 : 0;  // true: the reference's default integer P.V mode
        p.block_cols = static_cast<int32_t>(cfg.block_cols);

        std::vector<float> o(n * d), m(n), l(n), bias32;
        if (cfg.bias) bias32.assign(cfg.bias->data().data(), cfg.bias->data().data() + n * n);
        if (rel1d) bias32.assign(cfg.rel1d_offsets.begin(), cfg.rel1d_offsets.end());  // the kernels expand it, no N x N table
        if (rel2d) {  // [2, 2g-1]: row table then col table
            bias32.assign(cfg.rel2d_row_offsets.begin(), cfg.rel2d_row_offsets.end());
            bias32.insert(bias32.end(), cfg.rel2d_col_offsets.begin(), cfg.rel2d_col_offsets.end());
        }
        if (cfg.precision == Precision::bf16) {
            std::vector<std::uint16_t> hq(n * d), hk(n * d), hv(n * d);
            for (std::size_t i = 0; i < n * d; ++i) {
                hq[i] = to_bf16_bits(q.data().data()[i]);
                hk[i] = to_bf16_bits(k.data().data()[i]);
                hv[i] = to_bf16_bits(v.data().data()[i]);
            }
            check(ba_binary_attention_host(h_, &p, hq.data(), hk.data(), hv.data(), bias32.empty() ? nullptr : bias32.data(),
                                           o.data(), m.data(), l.data()));
        } else {
            std::vector<float> hq(q.data().data(), q.data().data() + n * d), hk(k.data().data(), k.data().data() + n * d),
                hv(v.data().data(), v.data().data() + n * d);
            check(ba_binary_attention_host(h_, &p, hq.data(), hk.data(), hv.data(), bias32.empty() ? nullptr : bias32.data(),
                                           o.data(), m.data(), l.data()));
        }
        return AttentionOutputT<DenseMatrixT>{DenseMatrixT(n, d, std::vector<double>(o.begin(), o.end())),
                                              std::vector<double>(m.begin(), m.end()),
                                              std::vector<double>(l.begin(), l.end())};
    }

    // Batched form of the same call: heads.size() independent (q, k, v) triples of one shape in ONE host round trip (the
    // reference leaves the loop over heads to its caller; looping over binary_attention_fused above costs one
    // synchronous H2D / launch / D2H round trip per head).  The bias (dense table or relative offsets) is shared by all heads.
    template <class DenseMatrixT>
    std::vector<AttentionOutputT<DenseMatrixT>> binary_attention_fused_batch(const std::vector<const DenseMatrixT*>& q,
                                                                             const std::vector<const DenseMatrixT*>& k,
                                                                             const std::vector<const DenseMatrixT*>& v,
                                                                             const AttentionConfigT<DenseMatrixT>& cfg) const {
        const std::size_t heads = q.size(), n = cfg.seq_len, d = cfg.head_dim;
        if (heads == 0 || k.size() != heads || v.size() != heads) throw ShapeError("attention: need as many K and V as Q matrices");
        for (std::size_t h = 0; h < heads; ++h) {
            if (q[h]->rows() != n || q[h]->cols() != d) throw ShapeError("attention: Q must be N x d");
            if (k[h]->rows() != n || k[h]->cols() != d) throw ShapeError("attention: K must be N x d");
            if (v[h]->rows() != n || v[h]->cols() != d) throw ShapeError("attention: V must be N x d");
        }
        if (!(cfg.temperature > 0.0)) throw ValidationError("attention: temperature must be positive");
        if (cfg.block_rows < 1 || cfg.block_rows > n || cfg.block_cols < 1 || cfg.block_cols > n)
            throw ValidationError("attention: block sizes must be in [1, N]");
        if (cfg.bias && (cfg.bias->rows() != n || cfg.bias->cols() != n)) throw ShapeError("bias: dense table must be N x N");
        if (!cfg.rel1d_offsets.empty() || !cfg.rel2d_row_offsets.empty())
            throw ValidationError("binary_attention_fused_batch: pass relative biases as the dense table they expand to");
        ba_params p{};
        p.B = 1;
        p.H = static_cast<int32_t>(heads);
        p.N = static_cast<int32_t>(n);
        p.d = static_cast<int32_t>(d);
        p.in_dtype = cfg.precision == Precision::bf16 ? BA_BF16 : BA_F32;
        p.bias_mode = cfg.bias ? BA_BIAS_DENSE : BA_BIAS_NONE;
        p.bias_heads = 1;
        p.bias_dtype = BA_F32;
        p.inv_tau = static_cast<float>(1.0 / cfg.temperature);
        p.kernel = BA_KERNEL_AUTO;
        p.quantize_pv = cfg.quantize_pv ? 1 : 0;
        p.block_cols = static_cast<int32_t>(cfg.block_cols);
        const std::size_t per = n * d;
        std::vector<float> o(heads * per), m(heads * n), l(heads * n), bias32;
        if (cfg.bias) bias32.assign(cfg.bias->data().data(), cfg.bias->data().data() + n * n);
        auto gather = [&](auto& dst, const std::vector<const DenseMatrixT*>& src, auto conv) {
            for (std::size_t h = 0; h < heads; ++h)
                for (std::size_t i = 0; i < per; ++i) dst[h * per + i] = conv(src[h]->data().data()[i]);
        };
        const void* hb = bias32.empty() ? nullptr : bias32.data();
        if (cfg.precision == Precision::bf16) {
            std::vector<std::uint16_t> hq(heads * per), hk(heads * per), hv(heads * per);
            gather(hq, q, to_bf16_bits), gather(hk, k, to_bf16_bits), gather(hv, v, to_bf16_bits);
            check(ba_binary_attention_host(h_, &p, hq.data(), hk.data(), hv.data(), hb, o.data(), m.data(), l.data()));
        } else {
            std::vector<float> hq(heads * per), hk(heads * per), hv(heads * per);
            auto f32 = [](double x) { return static_cast<float>(x); };
            gather(hq, q, f32), gather(hk, k, f32), gather(hv, v, f32);
            check(ba_binary_attention_host(h_, &p, hq.data(), hk.data(), hv.data(), hb, o.data(), m.data(), l.data()));
        }
        std::vector<AttentionOutputT<DenseMatrixT>> out;
        out.reserve(heads);
        for (std::size_t h = 0; h < heads; ++h)
            out.push_back({DenseMatrixT(n, d, std::vector<double>(o.begin() + h * per, o.begin() + (h + 1) * per)),
                           std::vector<double>(m.begin() + h * n, m.begin() + (h + 1) * n),
                           std::vector<double>(l.begin() + h * n, l.begin() + (h + 1) * n)});
        return out;
    }

    // BASELINE.json operator: binary_attention(Q, K, V, bias, scale) -> O, scale = 1 / temperature.
    template <class DenseMatrixT>
    DenseMatrixT binary_attention(const DenseMatrixT& q, const DenseMatrixT& k, const DenseMatrixT& v,
                                  const std::optional<DenseMatrixT>& bias, double scale,
                                  Precision precision = Precision::f32) const {
        if (!(scale > 0.0)) throw ValidationError("attention: temperature must be positive");
        AttentionConfigT<DenseMatrixT> cfg = AttentionConfigT<DenseMatrixT>::make(q.rows(), q.cols());
        cfg.temperature = 1.0 / scale;
        cfg.bias = bias;
        cfg.precision = precision;
        return binary_attention_fused(q, k, v, cfg).output;
    }

    // binattn::attention_fidelity(p_ref, p_other, k) (fidelity.hpp:40-41): same checks, same exception types.
    template <class DenseMatrixT>
    FidelityReport attention_fidelity(const DenseMatrixT& p_ref, const DenseMatrixT& p_other, std::size_t k) const {
        if (p_ref.rows() != p_other.rows() || p_ref.cols() != p_other.cols())
            throw ShapeError("attention_fidelity: shape mismatch");  // fidelity.cpp:42-43
        if (k == 0) throw ValidationError("attention_fidelity: k must be >= 1");  // fidelity.cpp:44
        ba_fidelity f{};
        check(ba_attention_fidelity_host(h_, p_ref.data().data(), p_other.data().data(), static_cast<int64_t>(p_ref.rows()),
                                         static_cast<int64_t>(p_ref.cols()), static_cast<int64_t>(k), &f));
        return FidelityReport{f.cos_sim, f.relative_l1, f.rmse, f.precision_at_k, k};
    }

private:
    ba_handle* h_ = nullptr;
};

}  // namespace binattn::b200
