// attn_tc2.cu -- host side of the second-generation K2 (attn_tc2.cuh): shape gate, ring depths, tensor maps, dispatch.
#include <cmath>

#include "attn_tc2.cuh"

namespace ba {

namespace tc {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn();  // attn_tcgen05.cu
}  // namespace tc

static int launch_tc2_any(const FwdArgs& a, const int8_t* vq, int ldq, int vcol0, const double* vscales, int32_t* dbg_S, int dbg_head,
                          long long* dbg_T, cudaStream_t stream);

// Returns the number of kernels launched (> 0), a negative cudaError_t, or 0 when this kernel does not take the shape
// (the caller then runs the first-generation kernel).
int launch_attn_tc2(const FwdArgs& a, int32_t* dbg_S, int dbg_head, long long* dbg_T, cudaStream_t stream) {
    return launch_tc2_any(a, nullptr, 0, 0, nullptr, dbg_S, dbg_head, dbg_T, stream);
}

// quantize_pv = true on the tensor cores (the I8 mode of attn_tc2_kernel): vq = s8 value levels [BH, N, d], vscales = their
// per-channel fp64 scales [BH, d] (K1v), level rows ldq bytes apart (a multiple of 16).  Takes block_cols = 64 (one key tile per
// block, the reference's default for N >= 64), bf16-packed inputs with d % 8 == 0, d <= 128, N >= 128 and no bias or a TMA-able
// dense bf16 table; 0 otherwise (the caller then runs the CUDA-core kernel).  The fp32 O and the s32 block accumulator of a
// query tile share 128 TMEM columns, so one launch covers 64 columns of V: wider heads take a second pass over the other
// columns (logits and weights recomputed).
int launch_attn_tc2_i8(const FwdArgs& a, const int8_t* vq, int ldq, const double* vscales, int block_cols, cudaStream_t stream) {
    if (tc::env_long("BA_TC2_I8", 1) == 0 || block_cols != 64 || !vq || !vscales) return 0;
    if (!tc2_i8_shape_ok(a.in_dtype, a.N, a.d) || reinterpret_cast<uintptr_t>(vq) % 16 != 0 || ldq % 16 != 0) return 0;
    int total = 0;
    for (int c0 = 0; c0 < a.d; c0 += 64) {
        const int n = launch_tc2_any(a, vq, ldq, c0, vscales, nullptr, 0, nullptr, stream);
        if (n <= 0) return c0 == 0 ? n : -(int)cudaErrorUnknown;  // (the gate is the same for every slice)
        total += n;
    }
    return total;
}

static int launch_tc2_any(const FwdArgs& a, const int8_t* vq, int ldq, int vcol0, const double* vscales, int32_t* dbg_S, int dbg_head,
                          long long* dbg_T, cudaStream_t stream) {
    using namespace tc2;
    const bool i8 = vq != nullptr;
    if (env_long("BA_TC2", 1) == 0 && !i8) return 0;
    if (!(i8 || tc2_shape_ok(a.in_dtype, a.N, a.d)) || !a.k_exp || !a.q_exp) return 0;
    if (dbg_S && a.N % TN != 0) return 0;  // (the logits dump has no ragged instantiation)
    if (a.d % 8 != 0 || a.d > 128) return 0;
    if (!i8 && (reinterpret_cast<uintptr_t>(a.V) % 16 != 0 || reinterpret_cast<uintptr_t>(a.O) % (a.out_bf16 ? 16 : 32) != 0)) return 0;
    int bias_mode = 0;
    int g = 0;
    if (a.bias && a.bias_kind == BA_BIAS_REL2D) {
        if (i8) return 0;
        g = (int)std::lround(std::sqrt((double)a.N));
        if ((long long)g * g != a.N || g % 32 != 0 || g > 128) return 0;  // (the C-ABI layer expands the table for these)
        bias_mode = 4;
    } else if (a.bias) {
        if (a.bias_kind != BA_BIAS_DENSE) return 0;
        const bool tma_ok = a.bias_dtype == BA_BF16 && (a.bias_ld * 2) % 16 == 0 && reinterpret_cast<uintptr_t>(a.bias) % 16 == 0;
        if (!tma_ok) return 0;
        if (!i8 && a.N < env_long("BA_TC2_MIN_N_BIAS", 2048)) return 0;  // with a dense bias the first-generation kernel is level or ahead below ~2048 keys (measured)
        bias_mode = 1;
    }
    tc::EncodeTiledFn enc = tc::get_encode_fn();
    if (!enc) return 0;
    Params2 prm{};
    prm.a = a;
    prm.tiles = (a.N + TN - 1) / TN;
    prm.ublocks = (a.N + 2 * TM - 1) / (2 * TM);
    prm.units = a.BH * prm.ublocks;
    prm.unit0 = 0;
    if (a.unit1 > 0) {  // unit-sharded call: the shard unit IS this kernel's unit
        prm.unit0 = a.unit0;
        prm.units = std::min(a.unit1, a.BH * prm.ublocks);
        if (prm.units <= prm.unit0) return 0;
    }
    prm.vcol0 = vcol0;
    prm.dsl = i8 ? std::min(64, a.d - vcol0) : a.d;
    prm.dvp = (prm.dsl + 15) / 16 * 16;
    prm.nbox = (prm.dsl + 63) / 64;
    prm.dbg_S = dbg_S;
    prm.dbg_head = dbg_head;
    prm.g = g;
    prm.dbg_T = dbg_T;
    prm.vbox = i8 ? kVBox8 : kVBox;
    prm.vscales = vscales;
    const int kpad = (a.d + 31) / 32 * 32;
    // ring depths: as deep as 227 KB allow; the bias ring must cover the HBM latency of the N x N stream
    prm.kst = 4;
    prm.vst = 4;
    prm.qst = 2;
    prm.bst = bias_mode == 1 ? 6 : 0;
    // the staged (TMA store) epilogue matters when units are short; long units (>= 64 key tiles) keep their deeper rings instead
    prm.o_stage = (env_long("BA_O_STAGE", 1) && prm.tiles < 64) ? 1 : 0;
    if (smem_bytes2(prm, kpad) > kSmemMax2) prm.kst = 3;
    if (smem_bytes2(prm, kpad) > kSmemMax2 && prm.bst > 5) prm.bst = 5;
    if (smem_bytes2(prm, kpad) > kSmemMax2 && prm.o_stage) prm.vst = 3;
    if (smem_bytes2(prm, kpad) > kSmemMax2 && prm.o_stage && prm.bst > 4) prm.bst = 4;
    if (smem_bytes2(prm, kpad) > kSmemMax2) prm.o_stage = 0;
    if (smem_bytes2(prm, kpad) > kSmemMax2) prm.qst = 1;
    if (smem_bytes2(prm, kpad) > kSmemMax2) prm.vst = 3;
    if (smem_bytes2(prm, kpad) > kSmemMax2 && prm.bst > 4) prm.bst = 4;
    if (smem_bytes2(prm, kpad) > kSmemMax2) return 0;
    // dev knobs: shallower rings than the shared memory allows (to reproduce one shape's ring depths on another)
    if (env_long("BA_QST", 0) > 0) prm.qst = (int)std::min<long>(prm.qst, env_long("BA_QST", 0));
    if (env_long("BA_KST", 0) > 0) prm.kst = (int)std::min<long>(prm.kst, env_long("BA_KST", 0));
    if (env_long("BA_VST", 0) > 0) prm.vst = (int)std::min<long>(prm.vst, env_long("BA_VST", 0));
    if (env_long("BA_BST", 0) > 0) prm.bst = (int)std::min<long>(prm.bst, env_long("BA_BST", 0));

    CUtensorMap vmap, bmap, omap;
    const cuuint32_t estr[3] = {1, 1, 1};
    if (i8) {  // s8 value levels [BH, N, d]: boxes of 64 keys x 64 channels (64 B rows, 64B swizzle; channels past d read as 0)
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)ldq, (cuuint64_t)a.N * ldq};
        const cuuint32_t box[3] = {64, (cuuint32_t)TN, 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(vq), gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    } else {
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)a.N * a.d * 2};
        const cuuint32_t box[3] = {64, (cuuint32_t)TN, 1};
        if (enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.V), gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    {   // O: [BH, N, d] fp32 (or bf16, ba_params.out_bf16); per-warp boxes of 32 rows x 16 elements (64 B with the 64B swizzle,
        // or 32 B with the 32B swizzle), clipped at N and d by the hardware
        const cuuint64_t esz = a.out_bf16 ? 2 : 4;
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * esz, (cuuint64_t)a.N * a.d * esz};
        const cuuint32_t box[3] = {16, 32, 1};
        if (enc(&omap, a.out_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a.O, gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, a.out_bf16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    bmap = vmap;
    if (bias_mode == 1) {
        const cuuint64_t gdim[3] = {(cuuint64_t)a.N, (cuuint64_t)a.N, (cuuint64_t)a.bias_heads};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.bias_ld * 2, (cuuint64_t)a.N * a.bias_ld * 2};
        const cuuint32_t box[3] = {64, (cuuint32_t)TM, 1};
        if (enc(&bmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.bias), gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                // 256-byte L2 promotion: a tile row is 128 B of a 2N-byte table row, and the next key tile reads the 128 B beside it --
                // fetching both at once halves the DRAM page activations of the N x N stream (measured 1-5% on the whole kernel)
                env_long("BA_BIAS_L2", 256) == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    if (i8) {
        switch (kpad) {
            case 32: return launch_i8<32>(prm, bias_mode, vmap, bmap, omap, stream);
            case 64: return launch_i8<64>(prm, bias_mode, vmap, bmap, omap, stream);
            case 96: return launch_i8<96>(prm, bias_mode, vmap, bmap, omap, stream);
            case 128: return launch_i8<128>(prm, bias_mode, vmap, bmap, omap, stream);
        }
        return 0;
    }
    switch (kpad) {
        case 32: return launch_kpad2<32>(prm, bias_mode, vmap, bmap, omap, stream);
        case 64: return launch_kpad2<64>(prm, bias_mode, vmap, bmap, omap, stream);
        case 96: return launch_kpad2<96>(prm, bias_mode, vmap, bmap, omap, stream);
        case 128: return launch_kpad2<128>(prm, bias_mode, vmap, bmap, omap, stream);
    }
    return 0;
}

}  // namespace ba
