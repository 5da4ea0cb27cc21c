// proj/src/attention_b200.cpp  (new file in the reference tree, compiled when BINATTN_WITH_B200 is set)
#include "binattn/attention.hpp"
#include "binattn_b200.hpp"            // from this repo's include/

namespace binattn {

AttentionOutput binary_attention_fused_b200(const DenseMatrix& q, const DenseMatrix& k, const DenseMatrix& v,
                                            const AttentionConfig& cfg) {
    static b200::Engine engine(/*device=*/0);                       // one ba_handle per device
    b200::AttentionConfigT<DenseMatrix> c = b200::AttentionConfigT<DenseMatrix>::make(cfg.seq_len, cfg.head_dim);
    c.temperature = cfg.temperature;
    c.block_rows  = cfg.block_rows;                                 // validated like attention.cpp:26-28
    c.block_cols  = cfg.block_cols;
    c.quantize_pv = cfg.quantize_pv;                                // true -> the integer P.V mode (K2b-I8 / K2q)             
    if (const auto* dense = std::get_if<DenseBias>(&cfg.bias)) {
        c.bias = dense->table;                                      // N x N table (attention.cpp:59-63)
    } else if (const auto* r1 = std::get_if<Relative1dBias>(&cfg.bias)) {
        c.rel1d_offsets = r1->offsets;                              // generated in-kernel: no N x N table (attention.cpp:65-76)
    } else if (const auto* r2 = std::get_if<Relative2dBias>(&cfg.bias)) {
        c.rel2d_row_offsets = r2->row_offsets;                      // generated in-kernel or expanded on the device
        c.rel2d_col_offsets = r2->col_offsets;                      // (attention.cpp:78-96)
    }
    try {
        auto out = engine.binary_attention_fused(q, k, v, c);       // DenseMatrix satisfies the shim's matrix concept
        return AttentionOutput{std::move(out.output), std::move(out.row_max), std::move(out.row_sum), std::nullopt};
    } catch (const b200::ShapeError& e)      { throw ShapeError(e.what()); }
      catch (const b200::ValidationError& e) { throw ValidationError(e.what()); }
}

} // namespace binattn
