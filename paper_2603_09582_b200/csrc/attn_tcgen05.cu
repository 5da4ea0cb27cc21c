// attn_tcgen05.cu -- host side of K2 (tensor-core variant): shape checks, ring depths, tensor maps, variant dispatch.
// The kernel and its launch templates live in attn_tcgen05.cuh; attn_tcgen05_k{32,64,96,128}.cu instantiate them.
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

EncodeTiledFn get_encode_fn() { return get_encode(); }  // shared with attn_tc2.cu

static int32_t* g_dbg_S = nullptr;
static int g_dbg_head = -1;
static long long* g_dbg_T = nullptr;
}  // namespace tc

bool tcgen05_supported(const ba_params* p, const char** why) {
    const char* w = nullptr;
    if (p->in_dtype != BA_BF16) w = "inputs must be bf16";
    else if (p->d % 8 != 0) w = "head dim must be a multiple of 8 (16-byte TMA row stride)";
    else if (p->d > 128) w = "head dim must be <= 128";
    else if (!tc::get_encode()) w = "cuTensorMapEncodeTiled is unavailable in this driver";
    if (why) *why = w ? w : "";
    return w == nullptr;
}

int launch_attn_tc2(const FwdArgs& a, int32_t* dbg_S, int dbg_head, long long* dbg_T, cudaStream_t stream);  // attn_tc2.cu

int launch_attn_tcgen05(const FwdArgs& a, cudaStream_t stream) {
    using namespace tc;
    // long sequences in whole 128-key tiles: the second-generation kernel (one CTA per SM, two query tiles in flight)
    {
        const int n2 = launch_attn_tc2(a, g_dbg_S, g_dbg_head, g_dbg_T, stream);
        if (n2 != 0) return n2;
    }
    if (a.bias && a.bias_kind == BA_BIAS_REL2D) return -(int)cudaErrorNotSupported;  // (the C-ABI layer expands the table for this kernel)
    if (reinterpret_cast<uintptr_t>(a.V) % 16 != 0 || reinterpret_cast<uintptr_t>(a.O) % 16 != 0)
        return -(int)cudaErrorMisalignedAddress;
    EncodeTiledFn enc = get_encode();
    if (!enc) return -(int)cudaErrorNotSupported;
    Params prm{};
    prm.a = a;
    prm.mblocks = (a.N + BM - 1) / BM;
    prm.tiles = (a.N + BN - 1) / BN;
    // tail folding: when only 1..8 keys spill past the last full tile (N = 197: 5), they do not get a tile of their own
    // -- a tile costs the same pipeline round trip whether it holds 5 keys or 64 -- but ride along with the last full
    // tile: logits by xor/popc on the CUDA cores, weights in P columns 32..39, V rows in a fifth P.V k-step
    prm.fold = 0;
    if (a.N > BN && a.N % BN >= 1 && a.N % BN <= kFoldMax && env_long("BA_FOLD", 1)) {
        prm.fold = a.N % BN;
        prm.tiles = a.N / BN;
    }
    prm.vbox = prm.fold ? 8192 + 2048 : 8192;
    prm.units = a.BH * prm.mblocks;
    prm.unit0 = 0;
    if (a.unit1 > 0) {  // unit-sharded call: the 128-row units covered by the 256-row shard units [unit0, unit1) of this call's heads
        const int upb = units_per_head(a.N);
        auto first128 = [&](int g) { return g >= a.BH * upb ? a.BH * prm.mblocks : (g / upb) * prm.mblocks + std::min(2 * (g % upb), prm.mblocks); };
        prm.unit0 = first128(a.unit0);
        prm.units = first128(a.unit1);
        if (prm.units <= prm.unit0) return 1 - 1;  // nothing to do
    }
    prm.dvp = (a.d + 15) / 16 * 16;
    prm.nbox = (a.d + 63) / 64;
    prm.o_vec8 = reinterpret_cast<uintptr_t>(a.O) % 32 == 0 ? 1 : 0;  // d % 8 == 0 keeps every row 32-byte aligned
    prm.dbg_S = g_dbg_S;
    prm.dbg_head = g_dbg_head;
    prm.dbg_T = g_dbg_T;
    const int kpad = (a.d + 31) / 32 * 32;

    // bias path: a bf16 table with 16-byte aligned rows is staged tile by tile with TMA; anything else is read directly
    int bias_mode = 0;
    if (a.bias && a.bias_kind == BA_BIAS_REL1D) {
        bias_mode = 3;  // relative-1d offsets: a 191-entry window per tile is staged by the producer warp
    } else if (a.bias) {
        const bool tma_ok = a.bias_dtype == BA_BF16 && (a.bias_ld * 2) % 16 == 0 &&
                            reinterpret_cast<uintptr_t>(a.bias) % 16 == 0;
        bias_mode = tma_ok ? 1 : 2;
    }
    // ring depths: as deep as fits two CTAs per SM; the asynchronous epilogue staging matters most when units are short
    prm.qst = 2;
    prm.kst = 3;
    prm.vst = 3;
    prm.bst = bias_mode == 1 ? 2 : bias_mode == 3 ? 4 : 0;
    prm.bstride = bias_mode == 3 ? kRelStage : 16384;
    prm.o_stage = env_long("BA_O_STAGE", 1) ? 1 : 0;
    if (smem_bytes(prm, kpad) > kSmemBudget) prm.vst = 2;
    if (smem_bytes(prm, kpad) > kSmemBudget) prm.kst = 2;
    if (smem_bytes(prm, kpad) > kSmemBudget) prm.qst = 1;
    if (smem_bytes(prm, kpad) > kSmemBudget && prm.tiles >= 16) prm.o_stage = 0;  // long units: the epilogue is rare
    if (smem_bytes(prm, kpad) > kSmemBudget && prm.bst == 2) prm.bst = 1;
    if (smem_bytes(prm, kpad) > kSmemBudget) prm.o_stage = 0;
    if (smem_bytes(prm, kpad) > kSmemBudget) return -(int)cudaErrorInvalidConfiguration;

    Maps m;
    const cuuint32_t estr[3] = {1, 1, 1};
    {
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)a.N * a.d * 2};
        const cuuint32_t box[3] = {64, (cuuint32_t)BN, 1};
        if (enc(&m.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.V), gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    m.v16 = m.v;
    if (prm.fold) {  // 16-key boxes for the folded tail rows (zero fill past N)
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)a.N * a.d * 2};
        const cuuint32_t box[3] = {64, 16, 1};
        if (enc(&m.v16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.V), gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    {   // O: [BH, N, d] fp32 (or bf16, ba_params.out_bf16); per-warp boxes of 32 rows x 32 elements (128 B with the 128B
        // swizzle, or 64 B with the 64B swizzle), clipped at N and d by the hardware
        const cuuint64_t esz = a.out_bf16 ? 2 : 4;
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * esz, (cuuint64_t)a.N * a.d * esz};
        const cuuint32_t box[3] = {32, 32, 1};
        if (enc(&m.o, a.out_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a.O, gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, a.out_bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    m.b = m.v;
    if (bias_mode == 1) {
        const cuuint64_t gdim[3] = {(cuuint64_t)a.N, (cuuint64_t)a.N, (cuuint64_t)a.bias_heads};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.bias_ld * 2, (cuuint64_t)a.N * a.bias_ld * 2};
        const cuuint32_t box[3] = {(cuuint32_t)BN, (cuuint32_t)BM, 1};
        if (enc(&m.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.bias), gdim, gstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -(int)cudaErrorInvalidValue;
    }
    const bool timeline = g_dbg_T != nullptr;  // dev tool: stamped builds of a few representative variants
    switch (kpad) {
        case 32: return launch_tc_k32(prm, bias_mode, m, stream, timeline);
        case 64: return launch_tc_k64(prm, bias_mode, m, stream, timeline);
        case 96: return launch_tc_k96(prm, bias_mode, m, stream, timeline);
        case 128: return launch_tc_k128(prm, bias_mode, m, stream, timeline);
    }
    return -(int)cudaErrorInvalidValue;
}

}  // namespace ba

// Test hook (not part of include/binattn_cuda.h): dump the tensor-core logits of one head as int32 [N,N].
extern "C" void ba_debug_tcgen05_logits(int32_t* dev_S, int head) {
    ba::tc::g_dbg_S = dev_S;
    ba::tc::g_dbg_head = head;
}
// Dev hook: per-CTA clock64 timeline, [ctas][4 roles][256] int64 (zero-filled by the caller).
extern "C" void ba_debug_tcgen05_timeline(long long* dev_T) { ba::tc::g_dbg_T = dev_T; }
