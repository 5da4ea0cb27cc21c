// test_dropin.cpp -- the reference's own attention test cases (proj/tests/test_attention.cpp) pointed at the
// B200 path through include/binattn_b200.hpp, with the CPU oracle (oracle/binattn_oracle.c) as the checker.
// Built and run by tests/test_cpp_dropin.py (-m gpu).  The matrix type below is a stand-in with the same
// surface as binattn::DenseMatrix (tensor.hpp:25-53); the shim is templated so the real one works unchanged.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "binattn_b200.hpp"

extern "C" {
typedef struct bo_rng bo_rng;
size_t bo_rng_sizeof(void);
void bo_rng_init(void* r, uint64_t seed, uint64_t stream);
void bo_random_dense(void* r, size_t count, double scale, double* out);
int bo_binary_attention_fused(const double* q, const double* k, const double* v, size_t n, size_t d, double tau,
                              size_t br, size_t bc, int qpv, const double* bias, double* y, double* m, double* l);
int bo_reference_attention(const double* q, const double* k, const double* v, size_t n, size_t d, double tau,
                           const double* bias, double* y, double* m, double* l, double* probs);
int bo_binary_attention_unfused(const double* q, const double* k, const double* v, size_t n, size_t d, double tau, int qpv,
                                const double* bias, double* y, double* m, double* l, double* probs);
int bo_attention_fidelity(const double* p_ref, const double* p_other, size_t rows, size_t cols, size_t k, double* out);
}

struct Span {
    const double* p;
    std::size_t n;
    const double* data() const { return p; }
    std::size_t size() const { return n; }
};
class Mat {  // same surface as binattn::DenseMatrix
public:
    Mat(std::size_t r, std::size_t c, std::vector<double> d) : r_(r), c_(c), d_(std::move(d)) {}
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    Span data() const { return {d_.data(), d_.size()}; }
    double operator()(std::size_t i, std::size_t j) const { return d_[i * c_ + j]; }

private:
    std::size_t r_, c_;
    std::vector<double> d_;
};

using namespace binattn::b200;
using Cfg = AttentionConfigT<Mat>;
static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);    \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

static Mat random_dense(void* rng, std::size_t r, std::size_t c, double scale = 1.0) {  // oracles.hpp:19-25
    std::vector<double> d(r * c);
    bo_random_dense(rng, r * c, scale, d.data());
    return Mat(r, c, std::move(d));
}
static double bf16_round(double x) {
    uint32_t u = (uint32_t)to_bf16_bits(x) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
static Mat rounded(const Mat& m, Precision p) {
    std::vector<double> d(m.data().data(), m.data().data() + m.rows() * m.cols());
    for (double& x : d) x = p == Precision::bf16 ? bf16_round(x) : (double)(float)x;
    return Mat(m.rows(), m.cols(), std::move(d));
}

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    Engine eng(0);
    std::vector<unsigned char> rng(bo_rng_sizeof());

    {  // frozen fixture: d=1 N=2 binary attention by hand (test_attention.cpp:163-174)
        const Mat q(2, 1, {2.0, -1.0}), k(2, 1, {1.0, -3.0}), v(2, 1, {4.0, -2.0});
        Cfg cfg = Cfg::make(2, 1);
        const auto out = eng.binary_attention_fused(q, k, v, cfg);
        CHECK(std::fabs(out.row_max[0] - 3.0) < 1e-5);
        CHECK(std::fabs(out.output(0, 0) - 3.985164261060192) < 1e-5);
        CHECK(std::fabs(out.output(1, 0) - -1.9851642610601914) < 1e-5);
    }
    {  // shape mismatches raise ShapeError, bad block sizes ValidationError (test_attention.cpp:126-141)
        bo_rng_init(rng.data(), 33, 0);
        const Mat q = random_dense(rng.data(), 4, 3), bad = random_dense(rng.data(), 4, 2), v = random_dense(rng.data(), 4, 3);
        Cfg cfg = Cfg::make(4, 3);
        CHECK(throws<ShapeError>([&] { eng.binary_attention_fused(q, bad, v, cfg); }));
        CHECK(throws<ShapeError>([&] { eng.binary_attention_fused(bad, q, v, cfg); }));
        CHECK(throws<ShapeError>([&] { eng.binary_attention_fused(q, v, bad, cfg); }));
        Cfg big = cfg;
        big.block_rows = 9;
        CHECK(throws<ValidationError>([&] { eng.binary_attention_fused(q, q, v, big); }));
        Cfg cold = cfg;
        cold.temperature = 0.0;
        CHECK(throws<ValidationError>([&] { eng.binary_attention_fused(q, q, v, cold); }));
        Cfg b = cfg;
        b.bias = Mat(3, 3, std::vector<double>(9, 0.0));
        CHECK(throws<ShapeError>([&] { eng.binary_attention_fused(q, q, v, b); }));  // attention.cpp:60-61
    }
    // seeded cases of the reference suite + the BASELINE head shapes, both precisions, with and without dense bias
    struct Case { uint64_t seed; std::size_t n, d; double bias_scale; };
    const Case cases[] = {{35, 12, 16, 0.0}, {38, 48, 16, 0.4}, {40, 64, 32, 0.0}, {43, 50, 12, 0.0},
                          {0, 197, 64, 0.5}, {1, 256, 72, 0.5}, {2, 130, 128, 0.5}};
    for (const Case& c : cases) {
        for (Precision prec : {Precision::f32, Precision::bf16}) {
            bo_rng_init(rng.data(), c.seed, 0);
            const Mat q = rounded(random_dense(rng.data(), c.n, c.d), prec), k = rounded(random_dense(rng.data(), c.n, c.d), prec),
                      v = rounded(random_dense(rng.data(), c.n, c.d), prec);
            Cfg cfg = Cfg::make(c.n, c.d);
            cfg.precision = prec;
            if (c.bias_scale > 0) cfg.bias = rounded(random_dense(rng.data(), c.n, c.n, c.bias_scale), Precision::f32);
            const auto out = eng.binary_attention_fused(q, k, v, cfg);
            std::vector<double> y(c.n * c.d), m(c.n), l(c.n);
            const int rc = bo_binary_attention_fused(q.data().data(), k.data().data(), v.data().data(), c.n, c.d,
                                                     cfg.temperature, cfg.block_rows, cfg.block_cols, 0,
                                                     cfg.bias ? cfg.bias->data().data() : nullptr, y.data(), m.data(), l.data());
            CHECK(rc == 0);
            double worst = 0.0;
            for (std::size_t i = 0; i < c.n * c.d; ++i) worst = std::fmax(worst, std::fabs(out.output.data().data()[i] - y[i]));
            std::printf("seed %llu N=%zu d=%zu %s bias=%d  max_abs=%.3e\n", (unsigned long long)c.seed, c.n, c.d,
                        prec == Precision::bf16 ? "bf16" : "f32", c.bias_scale > 0, worst);
            CHECK(worst <= 2e-3);
            // operator form: binary_attention(Q, K, V, bias, scale)
            const Mat o2 = eng.binary_attention(q, k, v, cfg.bias, 1.0 / cfg.temperature, prec);
            for (std::size_t i = 0; i < c.n * c.d; ++i) CHECK(o2.data().data()[i] == out.output.data().data()[i]);
        }
    }
    {  // quantize_pv = true, the reference's default mode (attention.hpp:35; test_attention.cpp:300-314 shape: N=64 d=32, 16x16)
        for (Precision prec : {Precision::f32, Precision::bf16}) {
            const std::size_t n = 64, d = 32;
            bo_rng_init(rng.data(), 40, 0);
            const Mat q = rounded(random_dense(rng.data(), n, d), prec), k = rounded(random_dense(rng.data(), n, d), prec),
                      v = rounded(random_dense(rng.data(), n, d), prec);
            Cfg cfg = Cfg::make(n, d);
            cfg.precision = prec;
            cfg.quantize_pv = true;
            cfg.block_rows = 16;
            cfg.block_cols = 16;
            const auto out = eng.binary_attention_fused(q, k, v, cfg);
            std::vector<double> y(n * d), m(n), l(n);
            CHECK(bo_binary_attention_fused(q.data().data(), k.data().data(), v.data().data(), n, d, cfg.temperature, 16, 16, 1,
                                            nullptr, y.data(), m.data(), l.data()) == 0);
            double worst = 0.0;
            for (std::size_t i = 0; i < n * d; ++i) worst = std::fmax(worst, std::fabs(out.output.data().data()[i] - y[i]));
            std::printf("quantize_pv=true N=%zu d=%zu %s  max_abs=%.3e\n", n, d, prec == Precision::bf16 ? "bf16" : "f32", worst);
            CHECK(worst <= 1e-3);
        }
    }
    {  // Relative1dBias (attention.hpp:18-21, attention.cpp:65-76): offsets handed to the kernels, table built for the oracle
        for (Precision prec : {Precision::f32, Precision::bf16}) {
            const std::size_t n = 197, d = 64;
            bo_rng_init(rng.data(), 51, 0);
            const Mat q = rounded(random_dense(rng.data(), n, d), prec), k = rounded(random_dense(rng.data(), n, d), prec),
                      v = rounded(random_dense(rng.data(), n, d), prec);
            const Mat off = rounded(random_dense(rng.data(), 1, 2 * n - 1, 0.5), Precision::f32);
            Cfg cfg = Cfg::make(n, d);
            cfg.precision = prec;
            cfg.rel1d_offsets.assign(off.data().data(), off.data().data() + 2 * n - 1);
            const auto out = eng.binary_attention_fused(q, k, v, cfg);
            std::vector<double> table(n * n), y(n * d), m(n), l(n);
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t j = 0; j < n; ++j) table[i * n + j] = cfg.rel1d_offsets[i + n - 1 - j];
            CHECK(bo_binary_attention_fused(q.data().data(), k.data().data(), v.data().data(), n, d, cfg.temperature,
                                            cfg.block_rows, cfg.block_cols, 0, table.data(), y.data(), m.data(), l.data()) == 0);
            double worst = 0.0;
            for (std::size_t i = 0; i < n * d; ++i) worst = std::fmax(worst, std::fabs(out.output.data().data()[i] - y[i]));
            std::printf("relative-1d bias N=%zu d=%zu %s  max_abs=%.3e\n", n, d, prec == Precision::bf16 ? "bf16" : "f32", worst);
            CHECK(worst <= 2e-3);
            Cfg bad = cfg;
            bad.rel1d_offsets.pop_back();
            CHECK(throws<ShapeError>([&] { eng.binary_attention_fused(q, k, v, bad); }));  // attention.cpp:66-67
        }
    }
    {  // attention_fidelity (fidelity.cpp:40-85): the full-precision attention map against the binary one, and the KATs of
       // test_fidelity.cpp:80-87 (ties go to the lower column) and :163-170 (validation)
        const std::size_t n = 96, d = 32;
        bo_rng_init(rng.data(), 52, 0);
        const Mat q = rounded(random_dense(rng.data(), n, d), Precision::bf16), k = rounded(random_dense(rng.data(), n, d), Precision::bf16),
                  v = rounded(random_dense(rng.data(), n, d), Precision::bf16);
        std::vector<double> y(n * d), m(n), l(n), pf(n * n), pb(n * n), want(4);
        CHECK(bo_reference_attention(q.data().data(), k.data().data(), v.data().data(), n, d, std::sqrt((double)d), nullptr, y.data(),
                                     m.data(), l.data(), pf.data()) == 0);
        CHECK(bo_binary_attention_unfused(q.data().data(), k.data().data(), v.data().data(), n, d, std::sqrt((double)d), 0, nullptr,
                                          y.data(), m.data(), l.data(), pb.data()) == 0);
        const Mat p_full(n, n, pf), p_bin(n, n, pb);
        for (std::size_t kk : {std::size_t{1}, std::size_t{5}, std::size_t{500}}) {
            CHECK(bo_attention_fidelity(pf.data(), pb.data(), n, n, kk, want.data()) == 0);
            const FidelityReport r = eng.attention_fidelity(p_full, p_bin, kk);
            std::printf("attention_fidelity k=%zu  cos=%.6f rel_l1=%.6f rmse=%.3e prec@k=%.4f\n", kk, r.cos_sim, r.relative_l1, r.rmse,
                        r.precision_at_k);
            CHECK(r.precision_at_k == want[3] && r.k == kk);
            CHECK(std::fabs(r.cos_sim - want[0]) <= 1e-12 && std::fabs(r.relative_l1 - want[1]) <= 1e-12 * want[1] &&
                  std::fabs(r.rmse - want[2]) <= 1e-12 * want[2]);
        }
        std::vector<double> uni(16, 0.25), hot0(16, 0.0), hot2(16, 0.0), half(16, 0.5);
        for (int i = 0; i < 4; ++i) hot0[i * 4] = 1.0, hot2[i * 4 + 2] = 1.0;
        CHECK(eng.attention_fidelity(Mat(4, 4, hot0), Mat(4, 4, uni), 1).precision_at_k == 1.0);
        CHECK(eng.attention_fidelity(Mat(4, 4, hot2), Mat(4, 4, uni), 1).precision_at_k == 0.0);
        CHECK(throws<ShapeError>([&] { eng.attention_fidelity(Mat(4, 4, uni), Mat(2, 8, uni), 2); }));
        CHECK(throws<ValidationError>([&] { eng.attention_fidelity(Mat(4, 4, uni), Mat(4, 4, half), 2); }));
        CHECK(throws<ValidationError>([&] { eng.attention_fidelity(Mat(4, 4, uni), Mat(4, 4, uni), 0); }));
    }
    std::printf(failures ? "FAILED (%d)\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
