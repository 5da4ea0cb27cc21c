// test_integration_ref.cpp -- INTEGRATION.md section 2's binding (tests/cpp/attention_b200.cpp, verbatim) compiled against the
// REAL reference headers (/root/reference/proj/include) and linked with the compiled reference (oracle/_ref) and
// libbinattn_cuda.so; runs the reference's own known-answer tests for the path through it:
//   test_attention.cpp:163-174   frozen fixture d=1 N=2 (mu_q = 1.5, mu_k = 2, Y = [3.985164261060192, -1.9851642610601914])
//   test_attention.cpp:234-252   seeds of the single-block cases (7x16, 64x16, 33x5), here: b200 path vs the reference's fused
// plus each BiasSpec alternative and the exception mapping.  Built by `make -C oracle reftest` where /root/reference exists;
// the binary travels to the GPU box in oracle/_ref/ (test infrastructure, like the rest of oracle/).
#include <cmath>
#include <cstdio>
#include <random>

#include "binattn/attention.hpp"
#include "binattn/errors.hpp"
#include "binattn/rng.hpp"
#include "oracles.hpp"  // proj/tests: random_dense

namespace binattn {
AttentionOutput binary_attention_fused_b200(const DenseMatrix& q, const DenseMatrix& k, const DenseMatrix& v, const AttentionConfig& cfg);
}
using namespace binattn;

static int failures = 0;
#define CHECK(cond)                                                    \
    do {                                                               \
        if (!(cond)) {                                                 \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                \
        }                                                              \
    } while (0)

static double max_abs(const DenseMatrix& a, const DenseMatrix& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.data().size(); ++i) m = std::fmax(m, std::fabs(a.data()[i] - b.data()[i]));
    return m;
}

int main() {
    {  // test_attention.cpp:163-174
        const DenseMatrix q(2, 1, {2.0, -1.0}), k(2, 1, {1.0, -3.0}), v(2, 1, {4.0, -2.0});
        AttentionConfig cfg = AttentionConfig::make(2, 1);  // tau = 1
        cfg.quantize_pv = false;
        const AttentionOutput out = binary_attention_fused_b200(q, k, v, cfg);
        CHECK(std::fabs(out.row_max[0] - 3.0) < 1e-5);
        CHECK(std::fabs(out.output(0, 0) - 3.985164261060192) < 1e-5);
        CHECK(std::fabs(out.output(1, 0) - (-1.9851642610601914)) < 1e-5);
        std::printf("fixture d=1: Y = [%.9f, %.9f], row_max[0] = %.6f\n", out.output(0, 0), out.output(1, 0), out.row_max[0]);
    }
    {  // test_attention.cpp:234-252 (same seed and shapes); fp32 upload -> CUDA-core kernel: ~1e-6 of the fp64 reference
        std::mt19937_64 rng = make_rng(37);
        for (const auto& [n, d] : {std::pair<std::size_t, std::size_t>{7, 16}, {64, 16}, {33, 5}}) {
            const DenseMatrix q = oracle::random_dense(n, d, rng), k = oracle::random_dense(n, d, rng), v = oracle::random_dense(n, d, rng);
            AttentionConfig cfg = AttentionConfig::make(n, d);
            cfg.quantize_pv = false;
            cfg.block_rows = n;
            cfg.block_cols = n;
            const AttentionOutput a = binary_attention_fused(q, k, v, cfg);
            const AttentionOutput b = binary_attention_fused_b200(q, k, v, cfg);
            const double e = max_abs(a.output, b.output);
            std::printf("seed 37 N=%zu d=%zu: max|Y_b200 - Y_ref| = %.3e\n", n, d, e);
            CHECK(e <= 2e-5);
        }
    }
    {  // every BiasSpec alternative (attention.hpp:15-27), N = 64 = 8 x 8
        std::mt19937_64 rng = make_rng(38);
        const std::size_t n = 64, d = 32, g = 8;
        const DenseMatrix q = oracle::random_dense(n, d, rng), k = oracle::random_dense(n, d, rng), v = oracle::random_dense(n, d, rng);
        GaussianSource gs(rng);
        std::vector<double> off1(2 * n - 1), row(2 * g - 1), col(2 * g - 1);
        for (double& x : off1) x = 0.5 * gs();
        for (double& x : row) x = 0.5 * gs();
        for (double& x : col) x = 0.5 * gs();
        const BiasSpec specs[3] = {DenseBias{oracle::random_dense(n, n, rng, 0.4)}, Relative1dBias{off1}, Relative2dBias{row, col}};
        for (int i = 0; i < 3; ++i) {
            AttentionConfig cfg = AttentionConfig::make(n, d);
            cfg.quantize_pv = false;
            cfg.bias = specs[i];
            const double e = max_abs(binary_attention_fused(q, k, v, cfg).output, binary_attention_fused_b200(q, k, v, cfg).output);
            std::printf("BiasSpec alternative %d: max|Y_b200 - Y_ref| = %.3e\n", i + 1, e);
            CHECK(e <= 2e-5);
        }
        AttentionConfig cfg = AttentionConfig::make(n, d);  // the reference's default mode (quantize_pv = true)
        const double e8 = max_abs(binary_attention_fused(q, k, v, cfg).output, binary_attention_fused_b200(q, k, v, cfg).output);
        std::printf("quantize_pv=true (reference default): max|Y_b200 - Y_ref| = %.3e\n", e8);
        CHECK(e8 <= 1e-3);
    }
    {  // exception mapping (attention.cpp:21-28)
        const DenseMatrix q(4, 3, std::vector<double>(12, 1.0)), bad(3, 3, std::vector<double>(9, 1.0));
        AttentionConfig cfg = AttentionConfig::make(4, 3);
        bool shape = false, valid = false;
        try { binary_attention_fused_b200(q, bad, q, cfg); } catch (const ShapeError&) { shape = true; }
        cfg.temperature = -1.0;
        try { binary_attention_fused_b200(q, q, q, cfg); } catch (const ValidationError&) { valid = true; }
        CHECK(shape && valid);
    }
    std::printf(failures ? "FAILED (%d)\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
