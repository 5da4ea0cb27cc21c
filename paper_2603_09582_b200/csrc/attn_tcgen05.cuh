// attn_tcgen05.cuh -- K2 (tensor-core variant): fused BinaryAttention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Follows binattn::binary_attention_fused with quantize_pv = false (proj/src/attention.cpp:250-382), Algorithm 1 of
// the paper:
//   S = Q^ K^T            exact +-1 contraction (== d - 2*popc(q xor k), bitops.cpp:59-67): the packed sign planes
//                         written by K1 are expanded in shared memory to e4m3 +-1.0 bytes (pad columns = 0) and
//                         multiplied by tcgen05.mma.kind::f8f6f4 into fp32 TMEM accumulators.  Every product is
//                         +-1 and |sum| <= d <= 128, so the fp32 accumulator holds the integer logit exactly.
//   x = S*mu_q*mu_k/tau + bias   (attention.cpp:34-36), softmax in the base-2 domain, fp32
//   O += P V              bf16 tcgen05.mma.kind::f16 with the A operand (P) read straight from TENSOR MEMORY: the
//                         softmax warps overwrite the S tile they just read with the bf16 weights (tcgen05.st), so P
//                         never touches shared memory; V tiles come by TMA (128B swizzle), consumed MN-major
//   O / l                 epilogue (attention.cpp:354-364): TMEM -> registers -> 32-byte vector stores
//
// PERSISTENT kernel: grid = min(units, 2 x SMs) CTAs, each walks units u = blockIdx.x, +gridDim.x, ... where one
// unit = one (head, 128-query block); key/value tiles of 64.  All pipelines (mbarrier rings) run straight across unit
// boundaries, so the loads, the K/Q expansion and the S MMAs of the next unit overlap the tail and the epilogue of the
// current one, and TMEM allocation / barrier setup / the lookup table are paid once per CTA.  256 threads:
//   warps 0-3  softmax + epilogue (thread r owns query row r == TMEM lane r)
//   warp  4    TMEM allocation + tcgen05.mma issue (warp-uniform control flow, one elected lane issues)
//   warp  5    TMA producer for V and bias tiles
//   warps 6-7  Q / K expanders (bit plane -> e4m3 bytes through a shared lookup table)
// TMEM (256 columns): S0 [0,64) | S1 [64,128) (P aliases the first 32 columns of its S stage) | O [128,128+dvp) |
// denominator block [128+dvp,+16).  tcgen05.mma instructions execute in issue order, and the issue order is
// S(g+1), PV(g), S(g+2), ... so the S MMA that recycles a stage always follows the PV MMA that read P from it.
// The running max uses the lazy-rescale rule: O/l are rescaled only when a row max grows by more than 2^8, which keeps
// TMEM read-modify-write traffic off the common path; the final O/l is unaffected (both carry the same reference max).
#pragma once
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ba_common.cuh"

namespace ba {
namespace tc {

constexpr int BM = 128;          // query rows per unit (UMMA M)
constexpr int BN = 64;           // keys per tile (UMMA N of the S MMA, K extent of the P.V MMA)
constexpr int kThreads = 256;
constexpr int kTmemCols = 256;
constexpr int kColS = 0, kColO = 128;
constexpr int kMaxStages = 4;
constexpr int kRelWin = 200;        // floats of the relative-1d bias window of one tile: 8 (folded keys) + 128 + 64 - 1, padded
constexpr int kRelStage = 1024;    // bytes of one window stage
constexpr int kFoldMax = 8;        // trailing keys that can be folded into the last full tile (CUDA-core logits, 5th P.V k-step)
constexpr int kRegsSoftmax = 200, kRegsCtrl = 56;  // setmaxnreg split of the 2 x 128 x 128 register pool (folded-tail kernels;
                                                  // the others run 192 / 64, which is what keeps each side free of spills)
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kSuspendHint = 0x989680;  // try_wait may sleep this long before re-polling (cuts spin instructions)

// ------------------------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// One arrival on behalf of the whole warp: every lane's preceding work is ordered before it by the warp barrier
// (128 per-thread arrivals on one mbarrier serialise in the shared-memory atomic unit and slow every barrier op).
__device__ __forceinline__ void warp_arrive(uint64_t* bar, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Non-blocking poll; the predicate lands asynchronously, so issuing it early hides the ~170-cycle round trip.
__device__ __forceinline__ uint32_t mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done;
}
// Truly non-blocking phase test (try_wait may sleep up to a hardware time limit when the phase is still open).
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done;
}
// Bounded wait: a protocol bug traps (clean launch failure) after 2^26 polls -- each poll sleeps in hardware up to
// kSuspendHint ns or until the barrier moves, so that is seconds -- instead of hanging the GPU.
#ifndef BA_WAIT_SPINS
#define BA_WAIT_SPINS (1u << 26)  // dev builds lower this (BA_NVCC_FLAGS=-DBA_WAIT_SPINS=...) so a deadlock traps in seconds
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0, spins = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(kSuspendHint)
            : "memory");
        if (done) break;
        if (++spins == BA_WAIT_SPINS) __trap();
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One lane of a converged warp (elect.sync): the MMA warp runs its waits as a whole warp and wraps every block of
// tcgen05.mma / tcgen05.commit instructions in `if (elect_one())`, so ptxas emits one ELECT + branch per block and the
// operands stay in uniform registers (a per-instruction lane predicate makes it wrap each MMA in its own elect loop).
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
        "elect.sync rx|px, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, px;\n\t}"
        : "=r"(pred));
    return pred;
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mma_f8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: the A operand (bf16, K-major: lane = row, one 32-bit column = two K elements).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

// Shared-memory matrix descriptor (cute::UMMA::SmemDescriptor bit layout, mma_sm100_desc.hpp):
// [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 | [61,64) layout (0 none, 2 = 128B swizzle).
// Advancing the start address by X bytes is `desc + (X >> 4)` (all tiles live below 256 KB, so no carry leaves the field).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo_bytes >> 4) << 16) | ((uint64_t)(sbo_bytes >> 4) << 32) |
           (1ull << 46) | ((uint64_t)layout << 61);
}

#define BA_TMEM_LD16(taddr, v, o)                                                                                  \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=f"(v[o + 0]), "=f"(v[o + 1]), "=f"(v[o + 2]), "=f"(v[o + 3]), "=f"(v[o + 4]), "=f"(v[o + 5]),   \
                   "=f"(v[o + 6]), "=f"(v[o + 7]), "=f"(v[o + 8]), "=f"(v[o + 9]), "=f"(v[o + 10]), "=f"(v[o + 11]), \
                   "=f"(v[o + 12]), "=f"(v[o + 13]), "=f"(v[o + 14]), "=f"(v[o + 15])                              \
                 : "r"(taddr)                                                                                      \
                 : "memory")

#define BA_TMEM_ST16(taddr, v, o)                                                                                  \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15};" \
                 ::"f"(v[o + 0]), "f"(v[o + 1]), "f"(v[o + 2]), "f"(v[o + 3]), "f"(v[o + 4]), "f"(v[o + 5]),         \
                   "f"(v[o + 6]), "f"(v[o + 7]), "f"(v[o + 8]), "f"(v[o + 9]), "f"(v[o + 10]), "f"(v[o + 11]),       \
                   "f"(v[o + 12]), "f"(v[o + 13]), "f"(v[o + 14]), "f"(v[o + 15]), "r"(taddr)                       \
                 : "memory")

#define BA_TMEM_ST16U(taddr, v)                                                                                    \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15};" \
                 ::"r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), \
                   "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(taddr)     \
                 : "memory")

__device__ __forceinline__ float ex2(float x) {
#ifdef BA_EXP_NOMUFU
    return x * 0.001f;  // dev experiment: wrong numbers, no MUFU
#else
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#endif
}
// 2^x on the FMA / ALU pipes (Cody-Waite split + degree-3 minimax polynomial, max relative error 7.5e-5 -- far below
// the bf16 rounding of P): a fixed share of the exponentials of every tile goes here instead of the 16-per-clock MUFU
// unit, which is the pipe the softmax warps queue on.  x <= ~8 by the lazy-rescale rule; x below -125 is clamped
// (2^-125 is zero for every purpose here and keeps the exponent arithmetic in range).
#ifndef BA_POLY_NOBIAS
#define BA_POLY_NOBIAS 0  // of every 16 exponentials, without a bias tile (measured: any share > 0 is slower)
#endif
#ifndef BA_POLY_BIAS
#define BA_POLY_BIAS 0    // of every 16 exponentials, with a bias tile
#endif
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;        // 1.5 * 2^23: round(x) lands in the low mantissa bits
    const float f = x - (t - 12582912.0f);  // [-0.5, 0.5]
    float p = fmaf(0.0551717501f, f, 0.242611319f);
    p = fmaf(p, f, 0.693260968f);
    p = fmaf(p, f, 0.999928057f);
    return __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23));  // p * 2^round(x)
}
template <int POLY>
__device__ __forceinline__ float ex2_mix(float x, int i) {  // i is a compile-time column index after unrolling
    return (((i & 15) * POLY) & 15) < POLY ? ex2_poly(x) : ex2(x);
}
// Packed fp32 FMA (Blackwell FFMA2): two independent a*b+c per instruction.  The softmax warps are bound by issue
// slots and latency, not by FMA throughput, so halving the FFMA count of the score and exponent-argument math pays.
__device__ __forceinline__ void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
#ifdef BA_EXP_NOF2FP
    // round-half-up on the integer pipe: add half an ulp, keep the top halves (one PRMT)
    return __byte_perm(__float_as_uint(lo) + 0x8000u, __float_as_uint(hi) + 0x8000u, 0x7632);
#else
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
#endif
}
__device__ __forceinline__ void stg_256(float* p, const float* v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]),
                 "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// 8 sign bits (bit = 1 -> +1.0) -> 8 e4m3 bytes: +1.0 = 0x38, -1.0 = 0xB8.  Used once per CTA to build the
// 256-entry lookup table the expanders read (one 8-byte shared-memory load per 8 elements).
__device__ __forceinline__ uint2 expand_byte(uint32_t b) {
    uint2 v;
    v.x = 0xB8B8B8B8u ^ (((b & 0xF) * 0x10204080u) & 0x80808080u);
    v.y = 0xB8B8B8B8u ^ ((((b >> 4) & 0xF) * 0x10204080u) & 0x80808080u);
    return v;
}

struct Smem {
    uint64_t qfull[2], qfree[2];                    // Q tile expanded / every S MMA of its unit retired
    uint64_t kfull[kMaxStages], kfree[kMaxStages];  // K tile expanded / its S MMA retired
    uint64_t vfull[kMaxStages], vfree[kMaxStages];  // V tile landed (TMA) / its P.V MMA retired
    uint64_t bfull[kMaxStages], bfree[kMaxStages];  // bias tile landed (TMA) / read out by the four softmax warps
    uint64_t sfull[2];                              // S tile ready in TMEM (tcgen05.commit)
    uint64_t pfull[2];                              // P tile written to TMEM by the four softmax warps
    uint64_t pvdone[2];                             // P.V MMA of a tile retired (O and the denominators are up to date)
    uint64_t ofree;                                 // O of the finished unit read out by the four softmax warps
    uint64_t ffull[2], ffree[2];                    // packed words of the folded tail keys staged / read out (by unit parity)
    uint64_t kbits[2][kFoldMax][2];                 // those words: [unit parity][key][64-bit word]
    uint2 lut[256];                                 // byte of sign bits -> 8 e4m3 +-1.0 bytes
    uint32_t tmem_base;
};

constexpr int kTlStamps = 256;

struct Params {
    FwdArgs a;
    int mblocks;       // ceil(N / BM)
    int tiles;         // ceil(N / BN)
    int units;         // END (exclusive) of this call's range of (head, 128-query block) units: BH * mblocks unless unit-sharded
    int unit0;         // first unit of the range (0 unless unit-sharded, ba_params.unit_begin)
    int dvp;           // d rounded up to 16 (UMMA N of P.V)
    int nbox;          // ceil(d / 64) TMA boxes per V tile
    int qst, kst, vst, bst;  // ring depths in shared memory
    int bstride;       // bytes of one bias stage: 16384 (dense tile by TMA) or kRelStage (relative-1d window)
    int o_vec8;        // O rows are 32-byte aligned (256-bit stores)
    int fold;          // 1..8: that many trailing keys (N % 64) ride along with the last full tile instead of a tile of their own
    int vbox;          // bytes of one 64-column V box in shared memory (64 keys, or 80 with folding)
    int o_stage;       // epilogue goes through the shared-memory staging boxes + TMA stores (asynchronous)
    int32_t* dbg_S;    // optional [N,N] int32 dump of the logits of head dbg_head (tests only)
    int dbg_head;
    long long* dbg_T;  // optional timeline: [cta][role 0..3][kTlStamps] clock64 stamps (dev tool, TL kernels only)
};

// Position in an mbarrier ring: consumers wait full[stage] with `phase`, producers wait free[stage] with phase ^ 1
// (which passes at once on the first lap, when the barrier is still in its initial phase).
struct Ring {
    int stage = 0;
    uint32_t phase = 0;
    __device__ __forceinline__ void next(int depth) {
        if (++stage == depth) {
            stage = 0;
            phase ^= 1u;
        }
    }
};

// Packed sign words of one row -> KPAD/32 32-bit registers (zeros when !valid).
template <int KPAD>
__device__ __forceinline__ void load_words(uint32_t (&w32)[KPAD / 32], const uint64_t* words, int w64, bool valid) {
#pragma unroll
    for (int i = 0; i < (KPAD + 63) / 64; ++i) {
        const uint64_t w = (valid && i < w64) ? __ldg(words + i) : 0ull;
        w32[2 * i] = (uint32_t)w;
        if (2 * i + 1 < KPAD / 32) w32[2 * i + 1] = (uint32_t)(w >> 32);
    }
}

// Expand one row into a K-major no-swizzle e4m3 tile through the lookup table:
// byte (r, kb) lives at (kb/16) * (rows*16) + r*16 + kb%16   (8x16B core matrices, SBO = 128, LBO = rows*16).
// d % 8 == 0, so validity is decided per 8-element group; groups at or past d (and whole invalid rows) store 0.0.
template <int KPAD>
__device__ __forceinline__ void expand_store(unsigned char* tile, int rows, int r, const uint32_t (&w32)[KPAD / 32],
                                             int d, bool valid, const uint2* lut) {
#pragma unroll
    for (int c = 0; c < KPAD / 16; ++c) {
        const uint32_t bits16 = w32[c / 2] >> (16 * (c & 1));
        const uint2 lo = (valid && 16 * c < d) ? lut[bits16 & 0xFF] : make_uint2(0, 0);
        const uint2 hi = (valid && 16 * c + 8 < d) ? lut[(bits16 >> 8) & 0xFF] : make_uint2(0, 0);
        *reinterpret_cast<uint4*>(tile + (size_t)c * rows * 16 + r * 16) = make_uint4(lo.x, lo.y, hi.x, hi.y);
    }
}

#define BA_STAMP(role)                                                                         \
    do {                                                                                       \
        if (TL && tl_buf && tl_n < kTlStamps) tl_buf[(role) * kTlStamps + tl_n++] = clock64(); \
    } while (0)

// ------------------------------------------------------------------------------------------------ softmax pieces
// Scores of one 16-column chunk: x = dot*sc + bias.  BIAS 1 reads the bf16 tile staged by TMA (row `tid` of a
// 128 x 64 tile, 128B swizzle), BIAS 2 reads the table directly.
template <int BIAS>
__device__ __forceinline__ void bias_chunk(float (&x)[BN], int c16, float sc, const unsigned char* brow, int tid,
                                           const char* bias_row, int bias_dtype, int col0, int nk) {
    if (BIAS == 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = 2 * c16 + h;  // 16-byte chunk = 8 bf16
            const uint4 b = *reinterpret_cast<const uint4*>(brow + ((c ^ (tid & 7)) << 4));
            const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                fma2(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], sc, sc,
                     __uint_as_float(bw[e] << 16), __uint_as_float(bw[e] & 0xFFFF0000u));
        }
    } else if (BIAS == 2) {
#pragma unroll
        for (int i = 16 * c16; i < 16 * c16 + 16; ++i) {
            const float bv = (bias_row && i < nk) ? load_as_float(bias_row, bias_dtype, col0 + i) : 0.f;
            x[i] = fmaf(x[i], sc, bv);
        }
    }
}

// Row maximum over chunks [0, nch) of 16 columns (4 independent chains); MASKED ignores columns >= nk.
template <bool MASKED>
__device__ __forceinline__ float tile_max(const float (&x)[BN], int nk, int nch) {
    float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
    for (int c = 0; c < BN / 16; ++c) {
        if (!MASKED || c < nch) {  // (a guarded body, not a break: the loop must unroll so x[] stays in registers)
#pragma unroll
            for (int i = 16 * c; i < 16 * c + 16; i += 4) {
                m0 = fmaxf(m0, (!MASKED || i + 0 < nk) ? x[i + 0] : -INFINITY);
                m1 = fmaxf(m1, (!MASKED || i + 1 < nk) ? x[i + 1] : -INFINITY);
                m2 = fmaxf(m2, (!MASKED || i + 2 < nk) ? x[i + 2] : -INFINITY);
                m3 = fmaxf(m3, (!MASKED || i + 3 < nk) ? x[i + 3] : -INFINITY);
            }
        }
    }
    return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
}

// p = 2^(x*ea - m_ref), rounded to bf16 and stored over the S tile just read: TMEM column c of the stage holds keys
// 2c (low half) and 2c+1, the K-major A-operand layout of the P.V MMA.  SUM adds the fp32 row sum (otherwise the
// tensor core sums the bf16 values through the ones block).  MASKED zeroes columns >= nk and skips the 32-key halves
// the MMA will not read.
// ROLLING REFILL (unmasked tiles): as soon as a 16-column quarter of x has been through ex2, the same registers are
// reloaded with the NEXT tile's scores (other S stage) if that tile is already complete (`refill`), so the TMEM load
// latency and the barrier round trip of the next tile hide behind this tile's exponentials.
template <bool MASKED, bool SUM, int POLY>
__device__ __forceinline__ float exp_store(float (&x)[BN], int nk, int nch, float ea, float nm, uint32_t p_addr, bool refill,
                                           uint32_t next_addr) {
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!MASKED || 2 * h < nch) {  // (a guarded body, not a break: the loop must unroll so x[] stays in registers)
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
                for (int e = 8 * q; e < 8 * q + 8; ++e) {
                    const int i = 32 * h + 2 * e;
                    float a0, a1;
                    fma2(a0, a1, x[i], x[i + 1], ea, ea, nm, nm);
                    float p0 = ex2_mix<POLY>(a0, i);
                    float p1 = ex2_mix<POLY>(a1, i + 1);
                    if (MASKED) {
                        p0 = (i < nk) ? p0 : 0.f;
                        p1 = (i + 1 < nk) ? p1 : 0.f;
                    }
                    if (SUM) {
                        l0 += p0;
                        l1 += p1;
                    }
                    pk[e] = pack_bf16(p0, p1);
                }
                if (!MASKED && refill) {
                    if (h == 0 && q == 0) BA_TMEM_LD16(next_addr + 0, x, 0);
                    if (h == 0 && q == 1) BA_TMEM_LD16(next_addr + 16, x, 16);
                    if (h == 1 && q == 0) BA_TMEM_LD16(next_addr + 32, x, 32);
                    if (h == 1 && q == 1) BA_TMEM_LD16(next_addr + 48, x, 48);
                }
            }
            BA_TMEM_ST16U(p_addr + 16 * h, pk);
        }
    }
    return l0 + l1;
}

// O (and the denominator block) of one row times alpha, in tensor memory.  Rare (lazy rescale) and kept out of line so
// its loop does not sit in the middle of the per-tile code.
static __device__ __noinline__ void rescale_o(uint32_t o_addr, int ocols, float alpha) {
    tc_fence_after();
    for (int c = 0; c < ocols; c += 16) {
        float o[16];
        BA_TMEM_LD16(o_addr + c, o, 0);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] *= alpha;
        BA_TMEM_ST16(o_addr + c, o, 0);
    }
}

struct RowState {
    float m_ref, m_true, l;  // base-2 units: reference max used in the exponent, true running max, running denominator
};

// One 64-key tile of the online softmax for one query row: x (raw scores, already in registers) -> P (TMEM, over S).
// FULL = all 64 keys valid: straight-line code.  The caller has waited for the bias stage; `refill` says the next S tile
// is complete, in which case x leaves holding the next tile's raw scores (loads in flight).
template <int BIAS, bool ROWSUM, bool FULL, bool DBG, bool TL>
__device__ __forceinline__ void softmax_tile(long long* tl_buf, int& tl_n, Smem* sm, RowState& rs, float (&x)[BN], uint32_t s_addr, uint32_t lane_base,
                                             const unsigned char* brow, int bstage, const char* bias_row, int bias_dtype,
                                             int j, uint32_t g, int nk, float sc, float ea, int ocols, int tid, int lane,
                                             int32_t* dbg_row, uint64_t* next_bar, uint32_t next_par, bool has_next, uint32_t next_addr, bool& refilled,
                                             const float (&xt)[kFoldMax], int nt) {
    const int nch = FULL ? BN / 16 : (nk + 15) >> 4;
    if (DBG && dbg_row) {
#pragma unroll
        for (int i = 0; i < BN; ++i)
            if (i < nk) dbg_row[i] = (int)x[i];
    }
    if (BIAS == 1 && FULL) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint4 b = *reinterpret_cast<const uint4*>(brow + ((c ^ (tid & 7)) << 4));
            const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                fma2(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], sc, sc,
                     __uint_as_float(bw[e] << 16), __uint_as_float(bw[e] & 0xFFFF0000u));
        }
        warp_arrive(&sm->bfree[bstage], lane);
    } else if (BIAS == 1) {
#pragma unroll
        for (int c = 0; c < BN / 16; ++c)
            if (c < nch) bias_chunk<1>(x, c, sc, brow, tid, nullptr, 0, 0, nk);
        warp_arrive(&sm->bfree[bstage], lane);
    } else if (BIAS == 2) {
#pragma unroll
        for (int c = 0; c < BN / 16; ++c)
            if (c < nch) bias_chunk<2>(x, c, sc, nullptr, tid, bias_row, bias_dtype, j * BN, nk);
    } else if (BIAS == 3) {
        // relative-1d bias (attention.cpp:65-76): b(row, col) = offsets[row - col + N - 1]; the producer warp staged the
        // 191 entries this tile can touch, win[8 + r + 63 - c] for row r and column c of the tile (lanes read
        // consecutive words: no bank conflicts)
        const float* win = reinterpret_cast<const float*>(brow) + 8 + tid + 63;
#pragma unroll
        for (int i = 0; i < BN; ++i)
            if (FULL || i < nk) x[i] = fmaf(x[i], sc, win[-i]);
        warp_arrive(&sm->bfree[bstage], lane);
    }
    BA_STAMP(0);
    float tmax = tile_max<!FULL>(x, nk, nch);
    if (FULL && nt > 0) {  // folded trailing keys (xt already holds dot*sc + bias, -inf past nt)
#pragma unroll
        for (int i = 0; i < kFoldMax; ++i) tmax = fmaxf(tmax, xt[i]);
    }
    tmax *= ea;  // ea >= 0, so the max commutes with the scaling
    rs.m_true = fmaxf(rs.m_true, tmax);
    // lazy rescale (first tile: m_ref = -inf forces it with alpha = 0 on the still-unwritten O)
    const bool need = tmax > rs.m_ref + kRescaleThreshold;
    if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? tmax : rs.m_ref;
        const float alpha = need ? ex2(rs.m_ref - m_new) : 1.0f;
        if (j > 0) {
            mbar_wait(&sm->pvdone[(g - 1) & 1u], ((g - 1) >> 1) & 1u);  // P.V of the previous tile has landed in O
            rescale_o(lane_base + kColO, ocols, alpha);
        }
        rs.l *= alpha;
        rs.m_ref = m_new;
    }
    BA_STAMP(0);
    // is the next S tile complete by now?  (uniform across the warp: one barrier, one instruction)
    refilled = FULL && has_next && mbar_test(next_bar, next_par);
    if (refilled) tc_fence_after();
    rs.l += exp_store<!FULL, !ROWSUM, (BIAS == 0 ? BA_POLY_NOBIAS : BA_POLY_BIAS)>(x, nk, nch, ea, -rs.m_ref, s_addr, refilled, next_addr);
    if (FULL && nt > 0) {  // weights of the folded keys: P columns 32..39 (keys 64..79 of this tile; -inf -> 0)
        uint32_t pk[8];
        float lt = 0.f;
#pragma unroll
        for (int e = 0; e < kFoldMax / 2; ++e) {
            const float p0 = ex2(fmaf(xt[2 * e], ea, -rs.m_ref)), p1 = ex2(fmaf(xt[2 * e + 1], ea, -rs.m_ref));
            lt += p0 + p1;
            pk[e] = pack_bf16(p0, p1);
        }
#pragma unroll
        for (int e = kFoldMax / 2; e < 8; ++e) pk[e] = 0u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%8], {%0,%1,%2,%3,%4,%5,%6,%7};" ::"r"(pk[0]), "r"(pk[1]), "r"(pk[2]),
                     "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]), "r"(s_addr + 32)
                     : "memory");
        if (!ROWSUM) rs.l += lt;
    }
    BA_STAMP(0);
}

struct Epilogue {
    RowState rs;
    uint32_t g_last;  // CTA-wide index of the unit's last tile
    int head, row;
    bool pending, warp_ok, row_ok;
};

// O / l -> global for one finished unit, then tell the MMA warp that O may be overwritten.
// Staged path (o_stage): each warp owns two 4 KB staging boxes of [32 rows][32 floats] (128B-swizzled like the O tensor
// map); a box is written, handed to a TMA store and only waited for when the SAME buffer is needed again (normally one
// whole unit later), so the softmax warps never sit on the store queue -- direct stores cost ~25% of the kernel at
// N=197.  The hardware clips the boxes at N and d.
template <bool ROWSUM>
__device__ __forceinline__ void run_epilogue(Smem* sm, const Params& prm, const CUtensorMap* omap, unsigned char* stage,
                                             Epilogue& ep, uint32_t lane_base, int warp, int lane) {
    const FwdArgs& a = prm.a;
    mbar_wait(&sm->pvdone[ep.g_last & 1u], (ep.g_last >> 1) & 1u);  // every MMA of the unit has retired
    if (ep.warp_ok) {
        tc_fence_after();
        float l = ep.rs.l;
        float* orow = a.O + ((int64_t)ep.head * a.N + ep.row) * a.d;
        __nv_bfloat16* orow16 = reinterpret_cast<__nv_bfloat16*>(a.O) + ((int64_t)ep.head * a.N + ep.row) * a.d;  // (out_bf16)
        for (int c = 0; c < prm.dvp; c += 32) {
            float o[32], den[16];
            const bool two = c + 16 < prm.dvp;
            if (ROWSUM && c == 0) BA_TMEM_LD16(lane_base + kColO + prm.dvp, den, 0);
            BA_TMEM_LD16(lane_base + kColO + c, o, 0);
            if (two) BA_TMEM_LD16(lane_base + kColO + c + 16, o, 16);
            if (prm.o_stage && c == 0) {  // both staging boxes are free again (their stores were issued a unit ago);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // overlaps the TMEM loads
                __syncwarp();
            }
            tc_wait_ld();
            if (ROWSUM && c == 0) l = den[0];  // sum of the bf16 weights the MMA used (first column of the ones block)
            const float inv_l = 1.0f / l;
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= inv_l;
            if (prm.o_stage) {
                const int bi = (c >> 5) & 1;
                unsigned char* box = stage + (warp * 2 + bi) * 4096;
                if (c >= 64 && bi == 0) {  // a wide head reuses the two boxes inside the same epilogue
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
                if (a.out_bf16) {  // [32 rows][32 bf16]: 64-byte rows, 64B swizzle (chunk q of row r sits at q ^ ((r >> 1) & 3))
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<uint4*>(box + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
                            make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                                       pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        *reinterpret_cast<float4*>(box + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                            make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
                }
                if (bi == 1 || c + 32 >= prm.dvp) {  // one proxy fence and one bulk group per pair of boxes
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        if (bi == 1) tma_store_3d(omap, box - 4096, c - 32, ep.row - lane, ep.head);
                        tma_store_3d(omap, box, c, ep.row - lane, ep.head);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
            } else if (ep.row_ok) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int cc = c + 8 * q;
                    if (cc + 8 <= a.d) {
                        if (a.out_bf16) {  // 8 bf16 = 16 bytes (d % 8 == 0 and a 16-byte aligned O keep every chunk aligned)
                            *reinterpret_cast<uint4*>(orow16 + cc) =
                                make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                                           pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
                        } else if (prm.o_vec8) {
                            stg_256(orow + cc, o + 8 * q);
                        } else {
                            *reinterpret_cast<float4*>(orow + cc) = make_float4(o[8 * q], o[8 * q + 1], o[8 * q + 2], o[8 * q + 3]);
                            *reinterpret_cast<float4*>(orow + cc + 4) = make_float4(o[8 * q + 4], o[8 * q + 5], o[8 * q + 6], o[8 * q + 7]);
                        }
                    }
                }
            }
        }
        tc_fence_before();
        if (ep.row_ok) {
            if (a.row_max) a.row_max[(int64_t)ep.head * a.N + ep.row] = ep.rs.m_true * kLn2;
            if (a.row_sum) a.row_sum[(int64_t)ep.head * a.N + ep.row] = l * ex2(ep.rs.m_ref - ep.rs.m_true);
        }
    }
    warp_arrive(&sm->ofree, lane);
    ep.pending = false;
}


// BIAS: 0 = none, 1 = bf16 tile staged by TMA (128B swizzle), 2 = direct global loads (fp32 / unaligned rows),
//       3 = relative-1d offsets (b_ij = offsets[i-j+N-1]) generated from a per-tile window in shared memory
// MODE: 0 = general (the last key tile may be partial), 1 = 1..8 trailing keys folded into the last full tile,
//       2 = N is a multiple of 64.  Modes 1 and 2 have no partial tile, so the masked code path is not even compiled in:
//       the hot loop of the persistent kernel is instruction-fetch sensitive (ncu: ~1/4 of the softmax warps' samples
//       sit on control flow / no_inst stalls), and the masked variant, the logits dump (DBG, tests only) and the rescale
//       loop used to sit in the middle of it.
template <int KPAD, int BIAS, int MODE, bool DBG = false, bool TL = false>
__global__ void __launch_bounds__(kThreads, 2)
attn_tc_kernel(const __grid_constant__ Params prm, const __grid_constant__ CUtensorMap vmap,
               const __grid_constant__ CUtensorMap bmap, const __grid_constant__ CUtensorMap omap,
               const __grid_constant__ CUtensorMap vmap16) {
    // d <= 96 leaves 16 spare TMEM columns next to O: the softmax denominator is then accumulated by the tensor
    // core (P x ones), which removes one FADD per score from the softmax warps.
    constexpr bool ROWSUM = KPAD <= 96;
    constexpr bool FOLD = MODE == 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FwdArgs& a = prm.a;
    // carve shared memory: V ring | bias ring | O staging (all 1024-aligned for the 128B swizzle) | Q ring | K ring | ones | barriers + table
    unsigned char* sV = smem_raw;                                   // vst x nbox x vbox (8192, or 10240 with folding)
    unsigned char* sB = sV + prm.vst * prm.nbox * prm.vbox;         // bst x 16384
    unsigned char* sO = sB + prm.bst * prm.bstride;                       // o_stage x 32768: epilogue staging boxes (4 warps x 2 x 4 KB)
    unsigned char* sQ = sO + prm.o_stage * 32768;                   // qst x BM x KPAD
    unsigned char* sK = sQ + prm.qst * BM * KPAD;                   // kst x BN x KPAD
    unsigned char* sOnes = sK + prm.kst * BN * KPAD;                // 512 B of bf16 1.0 (B operand of the row-sum MMA)
    Smem* sm = reinterpret_cast<Smem*>(sOnes + 512);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = a.N, d = a.d, w64 = a.W64, T = prm.tiles;
    const int G = gridDim.x;
    const int ub0 = prm.unit0 + (int)blockIdx.x;  // this CTA's first unit
    const int ocols = prm.dvp + (ROWSUM ? 16 : 0);  // TMEM columns of the O accumulator (+ denominator block)
    long long* tl_buf = (TL && prm.dbg_T) ? prm.dbg_T + (size_t)blockIdx.x * 4 * kTlStamps : nullptr;
    int tl_n = 0;
    (void)tl_buf; (void)tl_n;
    if (TL && !(tid == 0 || tid == 128 || tid == 160 || tid == 192)) tl_buf = nullptr;  // one stamper per role
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);

    // ---------------------------------------------------------------- prologue (once per CTA)
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->qfull[s], 2);     // one elected arrival per expander warp
            mbar_init(&sm->qfree[s], 1);     // tcgen05.commit after the last S MMA of the unit
            mbar_init(&sm->sfull[s], 1);     // tcgen05.commit after the S MMA of a tile
            mbar_init(&sm->pfull[s], 4);     // one elected arrival per softmax warp (P tile written to TMEM)
            mbar_init(&sm->pvdone[s], 1);    // tcgen05.commit after the P.V MMA of a tile
        }
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(&sm->kfull[s], 2);     // one elected arrival per expander warp
            mbar_init(&sm->kfree[s], 1);     // tcgen05.commit after the S MMA that read the stage
            mbar_init(&sm->vfull[s], 1);     // expect_tx arrive + TMA bytes
            mbar_init(&sm->vfree[s], 1);     // tcgen05.commit after the P.V MMA that read the stage
            mbar_init(&sm->bfull[s], BIAS == 3 ? 64 : 1);  // expect_tx arrive + TMA bytes, or one arrival per expander thread (window)
            mbar_init(&sm->bfree[s], 4);     // one elected arrival per softmax warp (bias stage read out)
        }
        mbar_init(&sm->ofree, 4);            // one elected arrival per softmax warp (O read out by the epilogue)
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->ffull[s], kFoldMax);  // one arrival per writing lane of the first expander warp (keys 0..7 past the last full tile)
            mbar_init(&sm->ffree[s], 4);     // one elected arrival per softmax warp
        }
        fence_barrier_init();
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm->tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 5 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        if (BIAS == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
        if (prm.o_stage) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&omap)) : "memory");
    }
    sm->lut[tid] = expand_byte((uint32_t)tid);
    if (tid < 128) reinterpret_cast<uint32_t*>(sOnes)[tid] = 0x3F803F80u;  // bf16 1.0 pairs
    fence_proxy_async();  // the ones block is read by the tensor core (async proxy)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm->tmem_base;
    // Programmatic dependent launch: everything above (barriers, TMEM, table) ran while K1 was still draining; K1's packed
    // words and scales are only read from here on.  (A no-op when the kernel was not launched as a dependent.)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);
    // register rebalancing between the two warpgroups (the pool is 256 x 128 per CTA): the softmax threads hold a
    // 64-column score row plus the bias row, the control warps need very little
    if (warp >= 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(MODE == 1 ? kRegsCtrl : kRegsCtrl + 8));
    if (warp == 4) {
        // ============================================================ MMA issuer (whole warp, uniform control flow)
        // instruction descriptors (cute::UMMA::InstrDescriptor bit layout)
        const uint32_t idesc_s = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);  // e4m3 x e4m3 -> f32, K-major A/B
        const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |                      // bf16 x bf16 -> f32, B MN-major
                                  ((uint32_t)(prm.dvp >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        const uint32_t idesc_l = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) |      // bf16 x ones(K-major) -> f32, N = 16
                                 ((uint32_t)(BM >> 4) << 24);
        const uint64_t q_desc = make_desc(smem_u32(sQ), BM * 16, 128, 0);     // K-major no swizzle; +ks*2*BM*16 per K step
        const uint64_t k_desc = make_desc(smem_u32(sK), BN * 16, 128, 0);     // +s*BN*KPAD per stage, +ks*2*BN*16 per K step
        const uint64_t v_desc = make_desc(smem_u32(sV), (uint32_t)prm.vbox, 1024, 2);  // MN-major 128B swizzle; +ks*2048 per 16 keys
        const uint64_t ones_desc = make_desc(smem_u32(sOnes), 256, 128, 0);   // 16 x 16 block of ones: any layout reads 1.0
        Ring qr, kr, vr;
        uint32_t g = 0;  // tiles issued so far by this CTA (S stage = g & 1)
        // the P.V MMA of a tile is issued one tile late, after the S MMA of the next tile (also across unit boundaries)
        int pend = 0, pend_nk = 0, pend_j = 0, pend_unit = 0;
        uint32_t pend_g = 0;
        auto issue_pv = [&]() {
            const uint32_t s = pend_g & 1u;
            const uint32_t v_ok = mbar_try(&sm->vfull[vr.stage], vr.phase);
            mbar_wait(&sm->pfull[s], (pend_g >> 1) & 1u);
            if (!v_ok) mbar_wait(&sm->vfull[vr.stage], vr.phase);
            // the first tile of a unit overwrites O: the epilogue of the previous unit must have read it out
            if (pend_j == 0 && pend_unit > 0) mbar_wait(&sm->ofree, (uint32_t)(pend_unit - 1) & 1u);
            BA_STAMP(1);
            tc_fence_after();
            const int ksteps = (pend_nk + 15) >> 4;
            const uint32_t p_tmem = tmem + kColS + s * BN;
            const uint64_t vd = v_desc + (uint64_t)((vr.stage * prm.nbox * prm.vbox) >> 4);
            if (elect_one()) {
#pragma unroll
                for (int ks = 0; ks < BN / 16 + (FOLD ? 1 : 0); ++ks) {  // (the fifth step only exists for a folded tail)
                    if (ks < ksteps) {
                        const uint32_t acc = (pend_j > 0 || ks > 0) ? 1u : 0u;
                        mma_bf16_ts(tmem + kColO, p_tmem + ks * 8, vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv, acc);
                        if (ROWSUM) mma_bf16_ts(tmem + kColO + prm.dvp, p_tmem + ks * 8, ones_desc, idesc_l, acc);
                    }
                }
                tc_commit(&sm->pvdone[s]);
                tc_commit(&sm->vfree[vr.stage]);
            }
            __syncwarp();
            vr.next(prm.vst);
            BA_STAMP(1);
        };
        int unit_i = 0;
        for (int u = ub0; u < prm.units; u += G, ++unit_i) {
            mbar_wait(&sm->qfull[qr.stage], qr.phase);
            const uint64_t qd = q_desc + (uint64_t)((qr.stage * BM * KPAD) >> 4);
            for (int j = 0; j < T; ++j) {
                mbar_wait(&sm->kfull[kr.stage], kr.phase);
                BA_STAMP(1);
                tc_fence_after();
                const uint64_t kd = k_desc + (uint64_t)((kr.stage * BN * KPAD) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < KPAD / 32; ++ks)
                        mma_f8(tmem + kColS + (g & 1u) * BN, qd + (uint64_t)(ks * ((2 * BM * 16) >> 4)),
                               kd + (uint64_t)(ks * ((2 * BN * 16) >> 4)), idesc_s, ks > 0 ? 1u : 0u);
                    tc_commit(&sm->sfull[g & 1u]);
                    tc_commit(&sm->kfree[kr.stage]);
                    if (j == T - 1) tc_commit(&sm->qfree[qr.stage]);
                }
                __syncwarp();
                kr.next(prm.kst);
                BA_STAMP(1);
                if (pend) issue_pv();
                pend = 1;
                pend_g = g;
                pend_j = j;
                pend_unit = unit_i;
                pend_nk = (FOLD && j == T - 1) ? BN + prm.fold : min(BN, N - j * BN);
                ++g;
            }
            qr.next(prm.qst);
        }
        if (pend) issue_pv();
    } else if (warp == 5) {
        // ============================================================ TMA producer (V tiles, bias tiles / windows)
        if (lane == 0) {
            Ring vr, br;
            for (int u = ub0; u < prm.units; u += G) {
                const int head = u / prm.mblocks;
                const int row0 = (u - head * prm.mblocks) * BM;
                const int bh = (a.head0 + head) % a.H % a.bias_heads;
                for (int j = 0; j < T; ++j) {
                    if (BIAS == 1) {
                        mbar_wait(&sm->bfree[br.stage], br.phase ^ 1u);
                        mbar_expect_tx(&sm->bfull[br.stage], 16384);
                        tma_load_3d(&bmap, &sm->bfull[br.stage], sB + br.stage * 16384, j * BN, row0, bh);
                        br.next(prm.bst);
                    }
                    if (lane == 0) {
                        BA_STAMP(2);
                        mbar_wait(&sm->vfree[vr.stage], vr.phase ^ 1u);
                        BA_STAMP(2);
                        const bool folded = FOLD && j == T - 1;  // this tile carries the 1..8 trailing keys as 16 more V rows
                        mbar_expect_tx(&sm->vfull[vr.stage], prm.nbox * (folded ? 8192 + 2048 : 8192));
                        for (int b = 0; b < prm.nbox; ++b) {
                            unsigned char* dst = sV + (vr.stage * prm.nbox + b) * prm.vbox;
                            tma_load_3d(&vmap, &sm->vfull[vr.stage], dst, b * 64, j * BN, head);
                            if (folded) tma_load_3d(&vmap16, &sm->vfull[vr.stage], dst + 8192, b * 64, (j + 1) * BN, head);
                        }
                        vr.next(prm.vst);
                    }
                }
            }
        }
    } else if (warp >= 6) {
        // ============================================================ Q / K expanders
        const int t = tid - 6 * 32;  // 0..63: key t of every K tile, query rows t and t + 64 of every Q tile
        Ring qr, kr, wr, fr;
        uint32_t wq0[KPAD / 32], wq1[KPAD / 32], wk[KPAD / 32];
        uint32_t wf[FOLD ? KPAD / 32 : 1];  // folded tail: thread t < fold holds the packed words of key T*64 + t
        if (ub0 < prm.units) {  // words of the first unit
            const int head = ub0 / prm.mblocks;
            const int row0 = (ub0 - head * prm.mblocks) * BM;
            if constexpr (FOLD)
                if (warp == 6) load_words<KPAD>(wf, a.k_words + ((int64_t)head * N + T * BN + t) * w64, w64, t < prm.fold);
            load_words<KPAD>(wq0, a.q_words + ((int64_t)head * N + row0 + t) * w64, w64, row0 + t < N);
            load_words<KPAD>(wq1, a.q_words + ((int64_t)head * N + row0 + t + 64) * w64, w64, row0 + t + 64 < N);
            load_words<KPAD>(wk, a.k_words + ((int64_t)head * N + t) * w64, w64, t < N);
        }
        for (int u = ub0; u < prm.units; u += G) {
            const int head = u / prm.mblocks;
            const int row0 = (u - head * prm.mblocks) * BM;
            mbar_wait(&sm->qfree[qr.stage], qr.phase ^ 1u);
            unsigned char* qt = sQ + qr.stage * BM * KPAD;
            expand_store<KPAD>(qt, BM, t, wq0, d, row0 + t < N, sm->lut);
            expand_store<KPAD>(qt, BM, t + 64, wq1, d, row0 + t + 64 < N, sm->lut);
            fence_proxy_async();
            warp_arrive(&sm->qfull[qr.stage], lane);
            qr.next(prm.qst);
            const int un = u + G;
            const int hn = un / prm.mblocks;
            if constexpr (FOLD) {
                // the folded keys' packed words go to the softmax threads through shared memory (they used to prefetch
                // them from global memory into 16 registers each, which cost the tile loop a spill)
                if (warp == 6) {
                    mbar_wait(&sm->ffree[fr.stage], fr.phase ^ 1u);
                    if (t < kFoldMax) {
#pragma unroll
                        for (int w = 0; w < 2; ++w) {
                            const uint32_t lo = 2 * w < KPAD / 32 ? wf[(2 * w) % (KPAD / 32)] : 0u;
                            const uint32_t hi = 2 * w + 1 < KPAD / 32 ? wf[(2 * w + 1) % (KPAD / 32)] : 0u;
                            sm->kbits[fr.stage][t][w] = ((uint64_t)hi << 32) | lo;
                        }
                        mbar_arrive(&sm->ffull[fr.stage]);  // each writer releases its own words (keeps racecheck's model simple)
                    }
                    fr.next(2);
                    if (un < prm.units) load_words<KPAD>(wf, a.k_words + ((int64_t)hn * N + T * BN + t) * w64, w64, t < prm.fold);
                }
            }
            // Q words of the next unit: their latency hides behind this unit's K tiles
            if (un < prm.units) {
                const int rn = (un - hn * prm.mblocks) * BM;
                load_words<KPAD>(wq0, a.q_words + ((int64_t)hn * N + rn + t) * w64, w64, rn + t < N);
                load_words<KPAD>(wq1, a.q_words + ((int64_t)hn * N + rn + t + 64) * w64, w64, rn + t + 64 < N);
            }
            for (int j = 0; j < T; ++j) {
                const int key = j * BN + t;
                if (BIAS == 3) {
                    // relative-1d bias: stage the window of the head's 2N-1 offsets this tile can touch (zero outside the
                    // table); win[0] is entry row0 - 64j - 63 + N - 1 - 8.  The expanders run two to three tiles ahead of
                    // the softmax, so the L2 round trip of these loads is hidden; all loads are issued before any store.
                    mbar_wait(&sm->bfree[wr.stage], wr.phase ^ 1u);
                    float* win = reinterpret_cast<float*>(sB + wr.stage * kRelStage);
                    const int bh = (a.head0 + head) % a.H % a.bias_heads;
                    const char* off = static_cast<const char*>(a.bias) + (int64_t)bh * (2 * (int64_t)N - 1) * dtype_size(a.bias_dtype);
                    const int base = row0 - j * BN - 63 + N - 1 - 8;
                    constexpr int PER = (kRelWin + 63) / 64;
                    float wv[PER];
#pragma unroll
                    for (int q = 0; q < PER; ++q) {
                        const int idx = base + t + 64 * q;
                        wv[q] = 0.f;
                        if (t + 64 * q < kRelWin && idx >= 0 && idx <= 2 * N - 2) {
                            if (a.bias_dtype == BA_F32) wv[q] = __ldg(reinterpret_cast<const float*>(off) + idx);
                            else wv[q] = __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(off) + idx) << 16);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < PER; ++q)
                        if (t + 64 * q < kRelWin) win[t + 64 * q] = wv[q];
                    mbar_arrive(&sm->bfull[wr.stage]);  // every writer releases its own entries
                    wr.next(prm.bst);
                }
                mbar_wait(&sm->kfree[kr.stage], kr.phase ^ 1u);
                BA_STAMP(3);
                expand_store<KPAD>(sK + kr.stage * BN * KPAD, BN, t, wk, d, key < N, sm->lut);
                fence_proxy_async();
                warp_arrive(&sm->kfull[kr.stage], lane);
                kr.next(prm.kst);
                BA_STAMP(3);
                // prefetch the next tile's words (the next unit's first tile after the last one)
                if (j + 1 < T) load_words<KPAD>(wk, a.k_words + ((int64_t)head * N + key + BN) * w64, w64, key + BN < N);
                else if (un < prm.units) load_words<KPAD>(wk, a.k_words + ((int64_t)hn * N + t) * w64, w64, t < N);
            }
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MODE == 1 ? kRegsSoftmax : kRegsSoftmax - 8));
        // ============================================================ softmax + epilogue (thread = query row)
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        Ring br, fr;
        uint32_t g = 0;  // tiles consumed so far (S stage = g & 1)
        // per-head scales are fetched one unit ahead and only combined when used (an early multiply would stall this
        // in-order thread on the global loads)
        float muq_next = 0.f, muk_next = 0.f;
        if (ub0 < prm.units) {
            const int head = ub0 / prm.mblocks;
            muq_next = __ldg(a.mu_q + head);
            muk_next = __ldg(a.mu_k + head);
        }
        // The epilogue of a unit is deferred until the first tile of the NEXT unit has been through the softmax, so the
        // latency of the unit's last P.V MMA hides behind useful work (the MMA warp holds that next tile's P.V back until
        // `ofree` says O has been read out).
        Epilogue ep{};
        ep.pending = false;
        // x holds the raw scores of the tile about to be processed; its TMEM loads are issued one tile ahead (by the
        // rolling refill inside the previous tile's exponentials when S was ready in time, else right after that tile)
        float x[BN];
        const int my_units = (prm.units - ub0 + G - 1) / G;
        const uint32_t total_tiles = (uint32_t)(my_units > 0 ? my_units : 0) * (uint32_t)T;
        if (total_tiles > 0) {
            mbar_wait(&sm->sfull[0], 0);
            tc_fence_after();
            BA_TMEM_LD16(lane_base + kColS + 0, x, 0);
            BA_TMEM_LD16(lane_base + kColS + 16, x, 16);
            BA_TMEM_LD16(lane_base + kColS + 32, x, 32);
            BA_TMEM_LD16(lane_base + kColS + 48, x, 48);
        }
        // (head, query block, bias table) of the unit are carried incrementally: this thread is alone on its critical
        // path, and the divisions / modulos of a fresh decomposition cost several hundred cycles per unit
        const int step_h = G / prm.mblocks, step_m = G - step_h * prm.mblocks;
        int head = ub0 / prm.mblocks, mb = ub0 - head * prm.mblocks;
        int tab = (a.head0 + head) % a.H;             // head index inside the batch element
        const int step_t = step_h % a.H;
        for (int u = ub0; u < prm.units; u += G) {
            const int row0 = mb * BM;
            const int row = row0 + tid;
            const bool row_ok = row < N;
            const bool warp_ok = row0 + warp * 32 < N;  // warps whose 32 rows are all past N only keep the barriers moving
            const int bias_tab = a.bias_heads == 1 ? 0 : tab;  // bias_heads is 1 or H
            const float sc = muq_next * muk_next * a.inv_tau;  // natural-log units per unit of dot
            // next unit of this CTA
            int head_n = head + step_h, mb_n = mb + step_m, tab_n = tab + step_t;
            if (mb_n >= prm.mblocks) {
                mb_n -= prm.mblocks;
                ++head_n;
                ++tab_n;
            }
            if (tab_n >= a.H) tab_n -= a.H;
            if (tab_n >= a.H) tab_n -= a.H;
            if (u + G < prm.units) {
                muq_next = __ldg(a.mu_q + head_n);
                muk_next = __ldg(a.mu_k + head_n);
            }
            // BIAS == 0 keeps x = raw integer dot and folds sc*log2e into the exponent FMA; otherwise x = dot*sc + bias
            const float ea = (BIAS == 0) ? sc * kLog2e : kLog2e;
            const char* bias_row = nullptr;
            if (BIAS == 2 && row_ok)
                bias_row = static_cast<const char*>(a.bias) + ((int64_t)bias_tab * N + row) * a.bias_ld * dtype_size(a.bias_dtype);
            RowState rs{-INFINITY, -INFINITY, 0.f};
            const bool dump = DBG && prm.dbg_S && head == prm.dbg_head && row_ok;
            // folded tail keys (prm.fold of them): this row's packed query and those keys' packed words / bias values are
            // requested now and only turned into logits at the unit's last tile, so the loads cost no wait
            constexpr int W = (KPAD + 63) / 64;
            constexpr int NF = FOLD ? kFoldMax : 1;
            uint64_t fq[W];
            float fb[NF];                       // BIAS 2: values; BIAS 1: unused (the raw 16-byte vector fbraw is unpacked at use --
            uint4 fbraw = make_uint4(0, 0, 0, 0);  // converting here would stall this in-order thread on the load)
            if (FOLD && warp_ok) {
#pragma unroll
                for (int w = 0; w < W; ++w) fq[w] = (row_ok && w < w64) ? __ldg(a.q_words + (uint32_t)((head * N + row) * w64 + w)) : 0ull;
#pragma unroll
                for (int i = 0; i < NF; ++i) fb[i] = 0.f;
                if ((BIAS == 1 || BIAS == 2) && row_ok) {
                    const char* brow_g = static_cast<const char*>(a.bias) + ((int64_t)bias_tab * N + row) * a.bias_ld * dtype_size(a.bias_dtype);
                    if (BIAS == 1) {  // bf16 rows padded to 16 bytes: the 8 columns after the last full tile are one vector
                        fbraw = __ldg(reinterpret_cast<const uint4*>(brow_g + (size_t)T * BN * 2));
                    } else {
#pragma unroll
                        for (int i = 0; i < NF; ++i)
                            if (i < prm.fold) fb[i] = load_as_float(brow_g, a.bias_dtype, T * BN + i);
                    }
                }
            }

            for (int j = 0; j < T; ++j, ++g) {
                const uint32_t s = g & 1u;
                const int nk = MODE != 0 ? BN : min(BN, N - j * BN);  // (folded / exact-multiple kernels only see full tiles)
                const bool has_next = g + 1 < total_tiles;
                const uint32_t next_addr = lane_base + kColS + (s ^ 1u) * BN;
                uint64_t* next_bar = &sm->sfull[s ^ 1u];
                const uint32_t next_par = ((g + 1) >> 1) & 1u;
                bool refilled = false;
                BA_STAMP(0);
                tc_wait_ld();  // S(g) is in x
                BA_STAMP(0);
                if (!warp_ok) {  // stay in lock-step with the pipelines, do no math
                    if (BIAS == 1 || BIAS == 3) {
                        mbar_wait(&sm->bfull[br.stage], br.phase);
                        warp_arrive(&sm->bfree[br.stage], lane);
                        br.next(prm.bst);
                    }
                    if (FOLD && j == T - 1) {
                        mbar_wait(&sm->ffull[fr.stage], fr.phase);
                        warp_arrive(&sm->ffree[fr.stage], lane);
                        fr.next(2);
                    }
                    tc_fence_before();
                    warp_arrive(&sm->pfull[s], lane);
                } else {
                    const unsigned char* brow = nullptr;
                    if (BIAS == 1) {
                        mbar_wait(&sm->bfull[br.stage], br.phase);
                        brow = sB + br.stage * 16384 + tid * 128;  // row tid of the 128 x 64 bf16 tile
                    } else if (BIAS == 3) {
                        mbar_wait(&sm->bfull[br.stage], br.phase);
                        brow = sB + br.stage * kRelStage;         // the tile's window of relative-1d offsets
                    }
                    const uint32_t s_addr = lane_base + kColS + s * BN;
                    int32_t* dbg_row = dump ? prm.dbg_S + (int64_t)row * N + j * BN : nullptr;
                    float xt[kFoldMax];
                    int nt = 0;
#pragma unroll
                    for (int i = 0; i < kFoldMax; ++i) xt[i] = -INFINITY;
                    if (FOLD && j == T - 1) {  // logits of the folded keys: d - 2*popc(q xor k) (bitops.cpp:59-67)
                        nt = prm.fold;
                        // pin the use of the prefetched words to this tile: the logits below do not depend on j, so the
                        // compiler would otherwise hoist them to the unit header and stall there on the loads
#pragma unroll
                        for (int w = 0; w < W; ++w) asm volatile("" : "+l"(fq[w]));
                        // the keys' words were staged by the expander warp (zeros past prm.fold and past w64)
                        uint64_t fk[NF][W];
                        mbar_wait(&sm->ffull[fr.stage], fr.phase);
#pragma unroll
                        for (int i = 0; i < NF; ++i)
#pragma unroll
                            for (int w = 0; w < W; ++w) fk[i][w] = sm->kbits[fr.stage][i][w];
                        asm volatile("" : "+r"(fbraw.x), "+r"(fbraw.y), "+r"(fbraw.z), "+r"(fbraw.w));
                        if (BIAS == 1) {
                            const uint32_t bw[4] = {fbraw.x, fbraw.y, fbraw.z, fbraw.w};
#pragma unroll
                            for (int e = 0; e < NF / 2; ++e) {
                                fb[2 * e] = __uint_as_float(bw[e] << 16);
                                fb[2 * e + 1] = __uint_as_float(bw[e] & 0xFFFF0000u);
                            }
                        }
#pragma unroll
                        for (int i = 0; i < NF; ++i) {
                            int pc = 0;
#pragma unroll
                            for (int w = 0; w < W; ++w) pc += __popcll(fq[w] ^ fk[i][w]);
                            const float dot = (float)(d - 2 * pc);
                            if (i < nt) {
                                // relative-1d: column 64 + i of this tile is window entry 8 + r + 63 - (64 + i)
                                const float bvv = (BIAS == 3) ? reinterpret_cast<const float*>(brow)[8 + tid - 1 - i] : fb[i];
                                xt[i] = (BIAS == 0) ? dot : fmaf(dot, sc, bvv);
                                if (DBG && dbg_row) dbg_row[BN + i] = d - 2 * pc;
                            }
                        }
                        warp_arrive(&sm->ffree[fr.stage], lane);
                        fr.next(2);
                    }
                    if (MODE != 0 || nk == BN)
                        softmax_tile<BIAS, ROWSUM, true, DBG, TL>(tl_buf, tl_n, sm, rs, x, s_addr, lane_base, brow, br.stage, bias_row,
                                                                  a.bias_dtype, j, g, nk, sc, ea, ocols, tid, lane, dbg_row, next_bar, next_par,
                                                                  has_next, next_addr, refilled, xt, nt);
                    else if (MODE == 0)
                        softmax_tile<BIAS, ROWSUM, false, DBG, TL>(tl_buf, tl_n, sm, rs, x, s_addr, lane_base, brow, br.stage, bias_row,
                                                                   a.bias_dtype, j, g, nk, sc, ea, ocols, tid, lane, dbg_row, next_bar, next_par,
                                                                   has_next, next_addr, refilled, xt, nt);
                    if (BIAS == 1 || BIAS == 3) br.next(prm.bst);
                    tc_wait_st();
                    BA_STAMP(0);
                    tc_fence_before();
                    warp_arrive(&sm->pfull[s], lane);
                }
                BA_STAMP(0);
                if (has_next && !refilled) {  // the next tile was not ready in time (or this warp idles): load it now
                    mbar_wait(next_bar, next_par);
                    tc_fence_after();
                    BA_TMEM_LD16(next_addr + 0, x, 0);
                    BA_TMEM_LD16(next_addr + 16, x, 16);
                    BA_TMEM_LD16(next_addr + 32, x, 32);
                    BA_TMEM_LD16(next_addr + 48, x, 48);
                }
                BA_STAMP(0);
                if (j == 0 && ep.pending) {
                    run_epilogue<ROWSUM>(sm, prm, &omap, sO, ep, lane_base, warp, lane);
                    BA_STAMP(0);
                }
            }
            ep.pending = true;
            ep.warp_ok = warp_ok;
            ep.row_ok = row_ok;
            ep.head = head;
            ep.row = row;
            ep.g_last = g - 1;
            ep.rs = rs;
            head = head_n;
            mb = mb_n;
            tab = tab_n;
        }
        if (ep.pending) run_epilogue<ROWSUM>(sm, prm, &omap, sO, ep, lane_base, warp, lane);
        if (prm.o_stage && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem may be released
        BA_STAMP(0);
    }
    tc_fence_before();
    __syncthreads();
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// ---------------------------------------------------------------------------------------------------- launch templates
// (the kernel is instantiated per padded head dim in attn_tcgen05_k{32,64,96,128}.cu so the four sets compile in parallel)
constexpr size_t kSmemBudget = 113 * 1024;  // two CTAs per SM (227 KB usable, 1 KB reserved per CTA)

inline long env_long(const char* name, long dflt) {
    const char* e = getenv(name);
    return e ? atol(e) : dflt;
}
inline size_t smem_bytes(const Params& prm, int kpad) {
    return (size_t)prm.vst * prm.nbox * prm.vbox + (size_t)prm.bst * prm.bstride + (size_t)prm.o_stage * 32768 + (size_t)prm.qst * BM * kpad +
           (size_t)prm.kst * BN * kpad + 512 + sizeof(Smem);
}

struct Maps {
    CUtensorMap v, b, o, v16;
};

constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return (dev >= 0 && dev < kMaxDevices) ? dev : 0;
}
inline int sm_count() {  // per device: one process may hold handles on several GPUs
    static int n[kMaxDevices] = {};
    const int dev = current_device();
    if (!n[dev]) {
        cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
        if (n[dev] <= 0) n[dev] = 148;
    }
    return n[dev];
}

template <int KPAD, int BIAS, int MODE, bool DBG, bool TL>
static int launch_variant(const Params& prm, const Maps& m, cudaStream_t stream) {
    static bool configured[kMaxDevices] = {};  // the attribute is per device
    const int dev = current_device();
    if (!configured[dev]) {
        const cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<KPAD, BIAS, MODE, DBG, TL>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
        if (e != cudaSuccess) return -(int)e;
        configured[dev] = true;
    }
    const long per_sm = env_long("BA_CTAS_PER_SM", 2);  // dev knob
    const long count = prm.units - prm.unit0;
    int grid = (int)std::min<long>(count, per_sm * sm_count());
    if (env_long("BA_GRID", 0) > 0) grid = (int)std::min<long>(count, env_long("BA_GRID", 0));  // dev knob
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_bytes(prm, KPAD);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap this kernel's prologue with K1's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // Only for many-wave launches.  With few units per CTA the static unit assignment makes the runtime depend on WHICH two
    // CTAs share an SM: a normal launch places CTA b and b + #SMs together, which pairs a CTA that has one unit more with one
    // that has one less (the survivor then finishes alone, up to 1.8x faster); a programmatic launch fills SMs as K1's CTAs
    // retire and pairs neighbours instead -- measured 7-12% slower at 1024 units (3.46 per CTA), 1-2.6% faster at >= 6.9.
    const long pdl_default = count >= 6L * grid ? 1 : 0;
    cfg.numAttrs = env_long("BA_PDL", pdl_default) ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_tc_kernel<KPAD, BIAS, MODE, DBG, TL>, prm, m.v, m.b, m.o, m.v16);
    return e == cudaSuccess ? 1 : -(int)e;
}

template <int KPAD, int MODE>
static int launch_mode(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream) {
    if (prm.dbg_S && bias_mode == 0) return launch_variant<KPAD, 0, MODE, true, false>(prm, m, stream);  // logits dump (tests)
    switch (bias_mode) {
        case 0: return launch_variant<KPAD, 0, MODE, false, false>(prm, m, stream);
        case 1: return launch_variant<KPAD, 1, MODE, false, false>(prm, m, stream);
        case 3: return launch_variant<KPAD, 3, MODE, false, false>(prm, m, stream);
        default: return launch_variant<KPAD, 2, MODE, false, false>(prm, m, stream);
    }
}

template <int KPAD>
static int launch_kpad(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream) {
    if (prm.fold) return launch_mode<KPAD, 1>(prm, bias_mode, m, stream);
    if (prm.a.N % BN == 0) return launch_mode<KPAD, 2>(prm, bias_mode, m, stream);
    return launch_mode<KPAD, 0>(prm, bias_mode, m, stream);
}


// Defined in attn_tcgen05_k<KPAD>.cu: every kernel variant of one padded head dim (timeline = dev-tool build with stamps).
int launch_tc_k32(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline);
int launch_tc_k64(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline);
int launch_tc_k96(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline);
int launch_tc_k128(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline);

}  // namespace tc
}  // namespace ba
