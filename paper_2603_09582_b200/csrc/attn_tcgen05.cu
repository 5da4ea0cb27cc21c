// attn_tcgen05.cu -- K2 (tensor-core variant): fused BinaryAttention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Follows binattn::binary_attention_fused with quantize_pv = false (proj/src/attention.cpp:250-382), Algorithm 1 of
// the paper:
//   S = Q^ K^T            exact +-1 contraction (== d - 2*popc(q xor k), bitops.cpp:59-67): the packed sign planes
//                         written by K1 are expanded in shared memory to e4m3 +-1.0 bytes (pad columns = 0) and
//                         multiplied by tcgen05.mma.kind::f8f6f4 into fp32 TMEM accumulators.  Every product is
//                         +-1 and |sum| <= d <= 128, so the fp32 accumulator holds the integer logit exactly.
//   x = S*mu_q*mu_k/tau + bias   (attention.cpp:34-36), softmax in the base-2 domain, fp32
//   O += P V              bf16 tcgen05.mma.kind::f16, P staged by the softmax warps in shared memory (K-major),
//                         V tiles brought by TMA (128B swizzle) and consumed MN-major; O accumulates in TMEM
//   O / l                 epilogue (attention.cpp:354-364), staged in swizzled shared memory and written by TMA
//
// One CTA = one (head, 128-query block); key/value tiles of 64.  256 threads:
//   warps 0-3  softmax + epilogue (thread r owns query row r == TMEM lane r)
//   warp  4    TMEM allocation + tcgen05.mma issue (warp-uniform control flow, one elected lane issues)
//   warp  5    TMA producer for V and bias tiles
//   warps 6-7  K-tile expanders (bit plane -> e4m3 bytes through a shared lookup table, one key per thread)
// Pipelines (mbarriers): K bytes 2 stages, V 2 stages, S (TMEM) 2 stages, P (smem) 1-2 stages, bias tile (bf16,
// TMA, 128B swizzle) 1-2 stages -- the stage counts are picked on the host so that two CTAs fit one SM.  Two
// completion barriers per tile are signalled by tcgen05.commit: sdone (S ready for the softmax warps == K stage free
// for the expanders) and pvdone (O updated / P stage free for the softmax warps == V stage free for the TMA warp).
// The running max uses the lazy-rescale rule: O/l are rescaled only when a row max grows by more than 2^8, which keeps
// TMEM read-modify-write traffic off the common path; the final O/l is unaffected (both carry the same reference max).
#include <cuda.h>

#include <cstdlib>

#include "ba_common.cuh"

namespace ba {
namespace tc {

constexpr int BM = 128;          // query rows per CTA (UMMA M)
constexpr int BN = 64;           // keys per tile (UMMA N of the S MMA, K extent of the P.V MMA)
constexpr int kThreads = 256;
constexpr int kTmemCols = 256;   // S0 [0,64) | S1 [64,128) | O [128, 128+dvp) | denominator block [128+dvp, +16)
constexpr int kColS = 0, kColO = 128;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint64_t kHangNs = 4000000000ull;
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
// Bounded wait: a protocol bug traps after ~4 s (clean launch failure) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    uint64_t t0 = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(kSuspendHint)
            : "memory");
        if (done) break;
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > kHangNs) __trap();
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// The next three are executed by the whole MMA warp in uniform control flow (so their operands live in uniform
// registers); `leader` predicates the instruction itself down to one lane.
__device__ __forceinline__ void tc_commit(uint64_t* bar, uint32_t leader) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(smem_u32(bar)), "r"(leader)
        : "memory");
}
__device__ __forceinline__ void mma_f8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc,
                                       uint32_t leader) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(leader)
        : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc,
                                         uint32_t leader) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc), "r"(leader)
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

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
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
    uint64_t kfull[2], vfull[2], sdone[2], sempty[2], pfull[2], pvdone[2], bfull[2], bempty[2];
    uint2 lut[256];  // byte of sign bits -> 8 e4m3 +-1.0 bytes
    uint32_t tmem_base;
};

struct Params {
    FwdArgs a;
    int mblocks;       // ceil(N / BM)
    int tiles;         // ceil(N / BN)
    int dvp;           // d rounded up to 16 (UMMA N of P.V)
    int nbox;          // ceil(d / 64) TMA boxes per V tile
    int pstages;       // P stages in shared memory (1 or 2)
    int bstages;       // bias-tile stages (0 = no TMA bias, 1 or 2)
    int32_t* dbg_S;    // optional [N,N] int32 dump of the logits of head dbg_head (tests only)
    int dbg_head;
    long long* dbg_T;  // optional timeline: [cta][role 0..3][128] clock64 stamps (dev tool, TL kernels only)
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
            for (int e = 0; e < 4; ++e) {
                x[c * 8 + 2 * e] = fmaf(x[c * 8 + 2 * e], sc, __uint_as_float(bw[e] << 16));
                x[c * 8 + 2 * e + 1] = fmaf(x[c * 8 + 2 * e + 1], sc, __uint_as_float(bw[e] & 0xFFFF0000u));
            }
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

// p = 2^(x*ea - m_ref), rounded to bf16 and stored straight into the P stage (row `prow`, 8-key chunks 2048 B apart:
// K-major core matrices).  SUM adds the fp32 row sum (otherwise the tensor core sums the bf16 values through the
// ones block).  MASKED zeroes columns >= nk and stops after nch 16-column chunks.
template <bool MASKED, bool SUM>
__device__ __forceinline__ float exp_store(const float (&x)[BN], int nk, int nch, float ea, float nm,
                                           unsigned char* prow) {
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int c = 0; c < BN / 8; ++c) {
        if (!MASKED || c < 2 * nch) {  // (a guarded body, not a break: the loop must unroll so x[] stays in registers)
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 8 * c + 2 * e;
                float p0 = ex2(fmaf(x[i], ea, nm));
                float p1 = ex2(fmaf(x[i + 1], ea, nm));
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
            *reinterpret_cast<uint4*>(prow + c * (BM * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
    }
    return l0 + l1;
}

#define BA_STAMP(role)                                                                  \
    do {                                                                                \
        if (TL && tl_buf && tl_n < 128) tl_buf[(role) * 128 + tl_n++] = clock64();      \
    } while (0)

// BIAS: 0 = none, 1 = bf16 tile staged by TMA (128B swizzle), 2 = direct global loads (fp32 / unaligned rows)
template <int KPAD, int BIAS, bool TL = false>
__global__ void __launch_bounds__(kThreads, 2)
attn_tc_kernel(const __grid_constant__ Params prm, const __grid_constant__ CUtensorMap vmap,
               const __grid_constant__ CUtensorMap bmap, const __grid_constant__ CUtensorMap omap) {
    // d <= 96 leaves 16 spare TMEM columns next to O: the softmax denominator is then accumulated by the tensor
    // core (P x ones), which removes one FADD per score from the softmax warps.
    constexpr bool ROWSUM = KPAD <= 96;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FwdArgs& a = prm.a;
    // carve shared memory: V stages | bias stages | P stages (1024-aligned; the O staging of the epilogue reuses this
    // region once every MMA has retired) | Q tile | K stages | ones | barriers + table
    unsigned char* sV = smem_raw;                                   // 2 x nbox x 8192
    unsigned char* sB = sV + 2 * prm.nbox * 8192;                   // bstages x 16384
    unsigned char* sP = sB + prm.bstages * 16384;                   // pstages x 16384
    unsigned char* sQ = sP + prm.pstages * 16384;                   // BM x KPAD
    unsigned char* sK = sQ + BM * KPAD;                             // 2 x BN x KPAD
    unsigned char* sOnes = sK + 2 * BN * KPAD;                      // 512 B of bf16 1.0 (B operand of the row-sum MMA)
    Smem* sm = reinterpret_cast<Smem*>(sOnes + 512);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int head = blockIdx.x / prm.mblocks;
    const int mb = blockIdx.x - head * prm.mblocks;
    const int N = a.N, d = a.d, w64 = a.W64, T = prm.tiles;
    const int row0 = mb * BM;
    const int pst = prm.pstages;
    const bool b2 = prm.bstages == 2;
    const int ocols = prm.dvp + (ROWSUM ? 16 : 0);  // TMEM columns of the O accumulator (+ denominator block)
    long long* tl_buf = (TL && prm.dbg_T) ? prm.dbg_T + (size_t)blockIdx.x * 4 * 128 : nullptr;
    int tl_n = 0;
    (void)tl_buf; (void)tl_n;
    if (TL && !(tid == 0 || tid == 128 || tid == 160 || tid == 192)) tl_buf = nullptr;  // one stamper per role
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);

    // ---------------------------------------------------------------- prologue
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->kfull[s], 2);     // one elected arrival per expander warp
            mbar_init(&sm->vfull[s], 1);     // expect_tx arrive + TMA bytes
            mbar_init(&sm->sdone[s], 1);     // tcgen05.commit after the S MMA of a tile
            mbar_init(&sm->sempty[s], 4);    // one elected arrival per softmax warp (S stage read out)
            mbar_init(&sm->pfull[s], 4);     // one elected arrival per softmax warp (P stage written)
            mbar_init(&sm->pvdone[s], 1);    // tcgen05.commit after the P.V MMA of a tile
            mbar_init(&sm->bfull[s], 1);     // expect_tx arrive + TMA bytes
            mbar_init(&sm->bempty[s], 4);    // one elected arrival per softmax warp (bias stage read out)
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
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&omap)) : "memory");
        if (BIAS == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
    }
    sm->lut[tid] = expand_byte((uint32_t)tid);
    if (tid < 128) reinterpret_cast<uint32_t*>(sOnes)[tid] = 0x3F803F80u;  // bf16 1.0 pairs
    // the first packed words are fetched before the barrier so their latency overlaps the table build
    uint32_t w32[KPAD / 32];
    if (tid < BM) load_words<KPAD>(w32, a.q_words + ((int64_t)head * N + row0 + tid) * w64, w64, row0 + tid < N);
    else if (warp >= 6) load_words<KPAD>(w32, a.k_words + ((int64_t)head * N + (tid - 192)) * w64, w64, tid - 192 < N);
    float sc = 0.f;
    if (tid < BM) sc = __ldg(a.mu_q + head) * __ldg(a.mu_k + head) * a.inv_tau;  // natural-log units per unit of dot
    __syncthreads();
    if (tid < BM) expand_store<KPAD>(sQ, BM, tid, w32, d, row0 + tid < N, sm->lut);  // Q tile: thread r = query row
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm->tmem_base;
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);

    if (warp == 4) {
        // ============================================================ MMA issuer (whole warp, uniform control flow)
        const uint32_t leader = lane == 0 ? 1u : 0u;
        // instruction descriptors (cute::UMMA::InstrDescriptor bit layout)
        const uint32_t idesc_s = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);  // e4m3 x e4m3 -> f32, K-major A/B
        const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |                      // bf16 x bf16 -> f32, B MN-major
                                  ((uint32_t)(prm.dvp >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        const uint32_t idesc_l = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) |      // bf16 x ones(K-major) -> f32, N = 16
                                 ((uint32_t)(BM >> 4) << 24);
        const uint64_t q_desc = make_desc(smem_u32(sQ), BM * 16, 128, 0);     // K-major no swizzle; +ks*2*BM*16 per K step
        const uint64_t k_desc = make_desc(smem_u32(sK), BN * 16, 128, 0);     // +s*BN*KPAD per stage, +ks*2*BN*16 per K step
        const uint64_t p_desc = make_desc(smem_u32(sP), 2048, 128, 0);        // +ps*16384 per stage, +ks*4096 per K step
        const uint64_t v_desc = make_desc(smem_u32(sV), 8192, 1024, 2);       // MN-major 128B swizzle; +ks*2048 per 16 keys
        const uint64_t ones_desc = make_desc(smem_u32(sOnes), 256, 128, 0);   // 16 x 16 block of ones: any layout reads 1.0
        auto issue_pv = [&](int t) {
            const int s = t & 1, n = t >> 1;
            const int ps = pst == 2 ? s : 0, pn = pst == 2 ? n : t;
            const uint32_t v_ok = mbar_try(&sm->vfull[s], n & 1);
            mbar_wait(&sm->pfull[ps], pn & 1);
            if (!v_ok) mbar_wait(&sm->vfull[s], n & 1);
            BA_STAMP(1);
            tc_fence_after();
            const int nk = min(BN, N - t * BN);
            const int ksteps = (nk + 15) >> 4;
            const uint64_t pd = p_desc + (uint64_t)((ps * 16384) >> 4);
            const uint64_t vd = v_desc + (uint64_t)((s * prm.nbox * 8192) >> 4);
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint32_t acc = (t > 0 || ks > 0) ? 1u : 0u;
                mma_bf16(tmem + kColO, pd + (uint64_t)(ks * (4096 >> 4)), vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv, acc, leader);
                if (ROWSUM) mma_bf16(tmem + kColO + prm.dvp, pd + (uint64_t)(ks * (4096 >> 4)), ones_desc, idesc_l, acc, leader);
            }
            tc_commit(&sm->pvdone[s], leader);
            BA_STAMP(1);
        };
        for (int j = 0; j < T; ++j) {
            const int s = j & 1, n = j >> 1;
            const uint32_t s_ok = n > 0 ? mbar_try(&sm->sempty[s], (n & 1) ^ 1) : 1u;  // first use: stage is free
            mbar_wait(&sm->kfull[s], n & 1);
            if (!s_ok) mbar_wait(&sm->sempty[s], (n & 1) ^ 1);
            BA_STAMP(1);
            tc_fence_after();
            const uint64_t kd = k_desc + (uint64_t)((s * BN * KPAD) >> 4);
#pragma unroll
            for (int ks = 0; ks < KPAD / 32; ++ks)
                mma_f8(tmem + kColS + s * BN, q_desc + (uint64_t)(ks * ((2 * BM * 16) >> 4)),
                       kd + (uint64_t)(ks * ((2 * BN * 16) >> 4)), idesc_s, ks > 0 ? 1u : 0u, leader);
            tc_commit(&sm->sdone[s], leader);
            BA_STAMP(1);
            if (j > 0) issue_pv(j - 1);
        }
        issue_pv(T - 1);
    } else if (warp == 5) {
        // ============================================================ TMA producer (V tiles, bias tiles)
        if (lane == 0) {
            const int bh = (a.head0 + head) % a.H % a.bias_heads;
            for (int j = 0; j < T; ++j) {
                const int s = j & 1, n = j >> 1;
                if (BIAS == 1) {
                    const int bs = b2 ? s : 0, bn = b2 ? n : j;
                    if (bn > 0) mbar_wait(&sm->bempty[bs], (bn & 1) ^ 1);
                    mbar_expect_tx(&sm->bfull[bs], 16384);
                    tma_load_3d(&bmap, &sm->bfull[bs], sB + bs * 16384, j * BN, row0, bh);
                }
                BA_STAMP(2);
                if (n > 0) mbar_wait(&sm->pvdone[s], (n & 1) ^ 1);  // P.V of tile j-2 released this V stage
                BA_STAMP(2);
                mbar_expect_tx(&sm->vfull[s], prm.nbox * 8192);
                for (int b = 0; b < prm.nbox; ++b)
                    tma_load_3d(&vmap, &sm->vfull[s], sV + (s * prm.nbox + b) * 8192, b * 64, j * BN, head);
            }
        }
    } else if (warp >= 6) {
        // ============================================================ K expanders (one key per thread)
        const int t = tid - 6 * 32;
        for (int j = 0; j < T; ++j) {
            const int s = j & 1, n = j >> 1;
            const int key = j * BN + t;
            if (n > 0) mbar_wait(&sm->sdone[s], (n & 1) ^ 1);  // S MMA of tile j-2 released this K stage
            BA_STAMP(3);
            expand_store<KPAD>(sK + s * BN * KPAD, BN, t, w32, d, key < N, sm->lut);
            BA_STAMP(3);
            fence_proxy_async();
            warp_arrive(&sm->kfull[s], lane);
            BA_STAMP(3);
            // prefetch the next tile's words so their L2 latency hides behind the next wait
            if (j + 1 < T) load_words<KPAD>(w32, a.k_words + ((int64_t)head * N + key + BN) * w64, w64, key + BN < N);
        }
    } else {
        // ============================================================ softmax + epilogue (thread = query row)
        const int row = row0 + tid;
        const bool row_ok = row < N;
        const bool warp_ok = row0 + warp * 32 < N;  // warps whose 32 rows are all past N only keep the barriers moving
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        // BIAS == 0 keeps x = raw integer dot and folds sc*log2e into the exponent FMA; otherwise x = dot*sc + bias
        const float ea = (BIAS == 0) ? sc * kLog2e : kLog2e;
        const char* bias_row = nullptr;
        if (BIAS == 2 && row_ok)
            bias_row = static_cast<const char*>(a.bias) +
                       ((int64_t)((a.head0 + head) % a.H % a.bias_heads) * N + row) * a.bias_ld * dtype_size(a.bias_dtype);
        float m_ref = -INFINITY, m_true = -INFINITY, l = 0.f;  // base-2 units
        uint32_t s_ok = mbar_try(&sm->sdone[0], 0);

        for (int j = 0; j < T; ++j) {
            const int s = j & 1, n = j >> 1;
            const int ps = pst == 2 ? s : 0;
            const int bs = b2 ? s : 0, bn = b2 ? n : j;
            const int nk = min(BN, N - j * BN);
            const int nch = (nk + 15) >> 4;
            // "P stage free" = P.V of tile j-pstages retired (always true for the first pstages tiles)
            const int jf = j - pst;
            BA_STAMP(0);
            if (!s_ok) mbar_wait(&sm->sdone[s], n & 1);
            BA_STAMP(0);
            if (!warp_ok) {  // stay in lock-step with the pipelines, do no math
                warp_arrive(&sm->sempty[s], lane);
                if (BIAS == 1) {
                    mbar_wait(&sm->bfull[bs], bn & 1);
                    warp_arrive(&sm->bempty[bs], lane);
                }
                if (jf >= 0) mbar_wait(&sm->pvdone[jf & 1], (jf >> 1) & 1);
                warp_arrive(&sm->pfull[ps], lane);
                s_ok = (j + 1 < T) ? mbar_try(&sm->sdone[s ^ 1], ((j + 1) >> 1) & 1) : 1u;
                continue;
            }
            float x[BN];
            tc_fence_after();
            const uint32_t s_addr = lane_base + kColS + s * BN;
            BA_TMEM_LD16(s_addr + 0, x, 0);
            if (nch > 1) BA_TMEM_LD16(s_addr + 16, x, 16);
            if (nch > 2) BA_TMEM_LD16(s_addr + 32, x, 32);
            if (nch > 3) BA_TMEM_LD16(s_addr + 48, x, 48);
            uint32_t b_ok = 1;
            if (BIAS == 1) b_ok = mbar_try(&sm->bfull[bs], bn & 1);  // these polls overlap the TMEM load
            const uint32_t p_ok = jf >= 0 ? mbar_try(&sm->pvdone[jf & 1], (jf >> 1) & 1) : 1u;
            tc_wait_ld();
            tc_fence_before();
            warp_arrive(&sm->sempty[s], lane);
            BA_STAMP(0);

            if (prm.dbg_S && head == prm.dbg_head && row_ok) {
#pragma unroll
                for (int i = 0; i < BN; ++i)
                    if (i < nk) prm.dbg_S[(int64_t)row * N + j * BN + i] = (int)x[i];
            }
            if (BIAS == 1) {
                if (!b_ok) mbar_wait(&sm->bfull[bs], bn & 1);
                const unsigned char* brow = sB + bs * 16384 + tid * 128;  // row tid of the 128 x 64 bf16 tile
#pragma unroll
                for (int c = 0; c < BN / 16; ++c)
                    if (c < nch) bias_chunk<1>(x, c, sc, brow, tid, nullptr, 0, 0, nk);
                warp_arrive(&sm->bempty[bs], lane);
            } else if (BIAS == 2) {
#pragma unroll
                for (int c = 0; c < BN / 16; ++c)
                    if (c < nch) bias_chunk<2>(x, c, sc, nullptr, tid, bias_row, a.bias_dtype, j * BN, nk);
            }
            BA_STAMP(0);
            float tmax = (nk == BN) ? tile_max<false>(x, nk, nch) : tile_max<true>(x, nk, nch);
            tmax *= ea;  // ea >= 0, so the max commutes with the scaling
            m_true = fmaxf(m_true, tmax);
            // lazy rescale (first tile: m_ref = -inf forces it with alpha = 0 on the still-unwritten O)
            const bool need = tmax > m_ref + kRescaleThreshold;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? tmax : m_ref;
                const float alpha = need ? ex2(m_ref - m_new) : 1.0f;
                if (j > 0) {
                    mbar_wait(&sm->pvdone[(j - 1) & 1], ((j - 1) >> 1) & 1);  // P.V of tile j-1 has landed in O
                    tc_fence_after();
                    for (int c = 0; c < ocols; c += 16) {
                        float o[16];
                        BA_TMEM_LD16(lane_base + kColO + c, o, 0);
                        tc_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) o[i] *= alpha;
                        BA_TMEM_ST16(lane_base + kColO + c, o, 0);
                    }
                    tc_wait_st();
                    tc_fence_before();
                }
                l *= alpha;
                m_ref = m_new;
            }
            if (!p_ok) mbar_wait(&sm->pvdone[jf & 1], (jf >> 1) & 1);  // the previous P.V on this stage no longer reads it
            BA_STAMP(0);
            unsigned char* prow = sP + ps * 16384 + tid * 16;
            if (nk == BN) l += exp_store<false, !ROWSUM>(x, nk, nch, ea, -m_ref, prow);
            else l += exp_store<true, !ROWSUM>(x, nk, nch, ea, -m_ref, prow);
            BA_STAMP(0);
            fence_proxy_async();
            warp_arrive(&sm->pfull[ps], lane);
            s_ok = (j + 1 < T) ? mbar_try(&sm->sdone[s ^ 1], ((j + 1) >> 1) & 1) : 1u;
            BA_STAMP(0);
        }
        // ---------------------------------------------------------------- epilogue: O / l -> swizzled smem -> TMA store
        mbar_wait(&sm->pvdone[(T - 1) & 1], ((T - 1) >> 1) & 1);  // every MMA has retired: all tile smem is free
        BA_STAMP(0);
        if (warp_ok) {
            tc_fence_after();
            if (ROWSUM) {  // denominator = first column of the ones block (sum of the bf16 weights the MMA used)
                float o[16];
                BA_TMEM_LD16(lane_base + kColO + prm.dvp, o, 0);
                tc_wait_ld();
                l = o[0];
            }
            const float inv_l = 1.0f / l;
            // staging: per warp, boxes of [32 rows][32 floats] = 4 KB, 128B-swizzled like the O tensor map
            const int nobox = (d + 31) >> 5;
            unsigned char* stage = smem_raw + warp * nobox * 4096;
            for (int c = 0; c < prm.dvp; c += 16) {
                float o[16];
                BA_TMEM_LD16(lane_base + kColO + c, o, 0);
                tc_wait_ld();
                unsigned char* box = stage + (c >> 5) * 4096 + lane * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int chunk = ((c & 16) >> 2) + q;  // 16-byte chunk inside the 128-byte box row
                    *reinterpret_cast<float4*>(box + ((chunk ^ (lane & 7)) << 4)) =
                        make_float4(o[4 * q] * inv_l, o[4 * q + 1] * inv_l, o[4 * q + 2] * inv_l, o[4 * q + 3] * inv_l);
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                for (int b = 0; b < nobox; ++b) tma_store_3d(&omap, stage + b * 4096, b * 32, row0 + warp * 32, head);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (row_ok) {
                if (a.row_max) a.row_max[(int64_t)head * N + row] = m_true * kLn2;
                if (a.row_sum) a.row_sum[(int64_t)head * N + row] = l * ex2(m_ref - m_true);
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem may be released
            tc_fence_before();
        }
        BA_STAMP(0);
    }
    __syncthreads();
    BA_STAMP(tid == 0 ? 0 : tid == 128 ? 1 : tid == 160 ? 2 : 3);
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// ---------------------------------------------------------------------------------------------------- host side
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

static int32_t* g_dbg_S = nullptr;
static int g_dbg_head = -1;
static long long* g_dbg_T = nullptr;
constexpr size_t kSmemBudget = 113 * 1024;
constexpr size_t kSmemMax = 227 * 1024;  // two CTAs per SM (227 KB usable, 1 KB reserved per CTA)

static size_t smem_pad() {  // dev knob: BA_SMEM_PAD=<bytes> forces lower occupancy for experiments
    static long pad = -1;
    if (pad < 0) { const char* e = getenv("BA_SMEM_PAD"); pad = e ? atol(e) : 0; }
    return (size_t)pad;
}
static size_t smem_bytes(const Params& prm, int kpad) {
    return smem_pad() + 2 * (size_t)prm.nbox * 8192 + (size_t)prm.bstages * 16384 + (size_t)prm.pstages * 16384 + (size_t)BM * kpad +
           2 * (size_t)BN * kpad + 512 + sizeof(Smem);
}

struct Maps {
    CUtensorMap v, b, o;
};

template <int KPAD, int BIAS>
static int launch_variant(const Params& prm, const Maps& m, cudaStream_t stream) {
    static bool configured = false;
    if (!configured) {
        const cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<KPAD, BIAS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)kSmemMax);
        if (e != cudaSuccess) return -(int)e;
        configured = true;
    }
    attn_tc_kernel<KPAD, BIAS><<<(unsigned)(prm.a.BH * prm.mblocks), kThreads, smem_bytes(prm, KPAD), stream>>>(prm, m.v, m.b, m.o);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

// Timeline build of three representative variants (dev tool; selected when a timeline buffer is registered).
template <int KPAD, int BIAS>
static int launch_timeline(const Params& prm, const Maps& m, cudaStream_t stream) {
    cudaFuncSetAttribute(attn_tc_kernel<KPAD, BIAS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget);
    attn_tc_kernel<KPAD, BIAS, true><<<(unsigned)(prm.a.BH * prm.mblocks), kThreads, smem_bytes(prm, KPAD), stream>>>(prm, m.v, m.b, m.o);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

template <int KPAD>
static int launch_kpad(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream) {
    switch (bias_mode) {
        case 0: return launch_variant<KPAD, 0>(prm, m, stream);
        case 1: return launch_variant<KPAD, 1>(prm, m, stream);
        default: return launch_variant<KPAD, 2>(prm, m, stream);
    }
}

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

int launch_attn_tcgen05(const FwdArgs& a, cudaStream_t stream) {
    using namespace tc;
    if (reinterpret_cast<uintptr_t>(a.V) % 16 != 0 || reinterpret_cast<uintptr_t>(a.O) % 16 != 0)
        return -(int)cudaErrorMisalignedAddress;
    EncodeTiledFn enc = get_encode();
    if (!enc) return -(int)cudaErrorNotSupported;
    Params prm{};
    prm.a = a;
    prm.mblocks = (a.N + BM - 1) / BM;
    prm.tiles = (a.N + BN - 1) / BN;
    prm.dvp = (a.d + 15) / 16 * 16;
    prm.nbox = (a.d + 63) / 64;
    prm.dbg_S = g_dbg_S;
    prm.dbg_head = g_dbg_head;
    prm.dbg_T = g_dbg_T;
    const int kpad = (a.d + 31) / 32 * 32;

    // bias path: a bf16 table with 16-byte aligned rows is staged tile by tile with TMA; anything else is read directly
    int bias_mode = 0;
    if (a.bias) {
        const bool tma_ok = a.bias_dtype == BA_BF16 && (a.bias_ld * 2) % 16 == 0 &&
                            reinterpret_cast<uintptr_t>(a.bias) % 16 == 0;
        bias_mode = tma_ok ? 1 : 2;
    }
    // stage counts: as deep as fits two CTAs per SM
    prm.pstages = 2;
    prm.bstages = bias_mode == 1 ? 2 : 0;
    if (smem_bytes(prm, kpad) > kSmemBudget) prm.pstages = 1;
    if (smem_bytes(prm, kpad) > kSmemBudget && prm.bstages == 2) prm.bstages = 1;

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
    {   // O: fp32 [BH, N, d]; per-warp boxes of 32 rows x 32 floats (128 B), clipped at N and d by the hardware
        const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
        const cuuint64_t gstr[2] = {(cuuint64_t)a.d * 4, (cuuint64_t)a.N * a.d * 4};
        const cuuint32_t box[3] = {32, 32, 1};
        if (enc(&m.o, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a.O, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
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
    if (g_dbg_T) {
        if (kpad == 64 && bias_mode == 1) return launch_timeline<64, 1>(prm, m, stream);
        if (kpad == 64 && bias_mode == 0) return launch_timeline<64, 0>(prm, m, stream);
        if (kpad == 128 && bias_mode == 0) return launch_timeline<128, 0>(prm, m, stream);
    }
    switch (kpad) {
        case 32: return launch_kpad<32>(prm, bias_mode, m, stream);
        case 64: return launch_kpad<64>(prm, bias_mode, m, stream);
        case 96: return launch_kpad<96>(prm, bias_mode, m, stream);
        case 128: return launch_kpad<128>(prm, bias_mode, m, stream);
    }
    return -(int)cudaErrorInvalidValue;
}

}  // namespace ba

// Test hook (not part of include/binattn_cuda.h): dump the tensor-core logits of one head as int32 [N,N].
extern "C" void ba_debug_tcgen05_logits(int32_t* dev_S, int head) {
    ba::tc::g_dbg_S = dev_S;
    ba::tc::g_dbg_head = head;
}
// Dev hook: per-CTA clock64 timeline, [ctas][4 roles][128] int64 (zero-filled by the caller).
extern "C" void ba_debug_tcgen05_timeline(long long* dev_T) { ba::tc::g_dbg_T = dev_T; }
