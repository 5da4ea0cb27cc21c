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
//   O / l                 epilogue (attention.cpp:354-364)
//
// One CTA = one (head, 128-query block); key/value tiles of 64.  256 threads:
//   warps 0-3  softmax + epilogue (thread r owns query row r == TMEM lane r)
//   warp  4    TMEM allocation + single-thread tcgen05.mma issue
//   warp  5    TMA producer for V
//   warps 6-7  K-tile expanders (bit plane -> e4m3 bytes, one key per thread)
// Pipelines (mbarriers): K bytes 2 stages, V 2 stages, S (TMEM) 2 stages, P (smem) 2 stages.  The running max uses
// the lazy-rescale rule: O/l are rescaled only when a row max grows by more than 2^8, which keeps TMEM read-modify-
// write traffic off the common path; the final O/l is unaffected (both carry the same reference max).
#include <cuda.h>

#include "ba_common.cuh"

namespace ba {
namespace tc {

constexpr int BM = 128;          // query rows per CTA (UMMA M)
constexpr int BN = 64;           // keys per tile (UMMA N of the S MMA, K extent of the P.V MMA)
constexpr int kThreads = 256;
constexpr int kTmemCols = 256;   // S0 [0,64) | S1 [64,128) | O [128, 128+DVP)
constexpr int kColS = 0, kColO = 128;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr uint32_t kSpinLimit = 1u << 24;

// ------------------------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bounded spin: a protocol bug traps (clean launch failure) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0, spins = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) break;
        if (++spins > kSpinLimit) __trap();
    }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// D[tmem] (+)= A[smem desc] * B[smem desc]; issued by ONE thread.
__device__ __forceinline__ void mma_f8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

// Shared-memory matrix descriptor (cute::UMMA::SmemDescriptor bit layout, mma_sm100_desc.hpp):
// [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 | [61,64) layout (0 none, 2 = 128B swizzle)
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

// 4 sign bits (bit = 1 -> +1.0) -> 4 e4m3 bytes: +1.0 = 0x38, -1.0 = 0xB8.
__device__ __forceinline__ uint32_t expand_nibble(uint32_t nib) {
    return 0xB8B8B8B8u ^ ((nib * 0x10204080u) & 0x80808080u);
}
// 16 sign bits starting at element e0 of a row of logical width d -> 16 bytes (elements >= d become 0.0).
__device__ __forceinline__ uint4 expand16(uint32_t bits16, int e0, int d) {
    uint4 v;
    v.x = (e0 + 0 < d) ? expand_nibble(bits16 & 0xF) : 0u;
    v.y = (e0 + 4 < d) ? expand_nibble((bits16 >> 4) & 0xF) : 0u;
    v.z = (e0 + 8 < d) ? expand_nibble((bits16 >> 8) & 0xF) : 0u;
    v.w = (e0 + 12 < d) ? expand_nibble((bits16 >> 12) & 0xF) : 0u;
    return v;
}

struct Smem {
    // barriers first (8-byte aligned), tiles after (1024-byte aligned for the swizzled V stages)
    uint64_t kfull[2], kempty[2], vfull[2], vempty[2], sfull[2], sempty[2], pfull[2], pempty[2];
    uint32_t tmem_base;
};

struct Params {
    FwdArgs a;
    int mblocks;       // ceil(N / BM)
    int tiles;         // ceil(N / BN)
    int dvp;           // d rounded up to 16 (UMMA N of P.V)
    int nbox;          // ceil(d / 64) TMA boxes per V tile
    int32_t* dbg_S;    // optional [N,N] int32 dump of the logits of head dbg_head (tests only)
    int dbg_head;
};

// Expand row `row` (packed u64 words, or zeros when !valid) into a K-major no-swizzle e4m3 tile:
// byte (r, kb) lives at (kb/16) * (rows*16) + r*16 + kb%16   (8x16B core matrices, SBO = 128, LBO = rows*16).
template <int KPAD>
__device__ __forceinline__ void expand_row(unsigned char* tile, int rows, int r, const uint64_t* words, int w64, int d,
                                           bool valid) {
    uint32_t w32[KPAD / 32];
#pragma unroll
    for (int i = 0; i < KPAD / 64; ++i) {
        const uint64_t w = (valid && i < w64) ? __ldg(words + i) : 0ull;
        w32[2 * i] = (uint32_t)w;
        w32[2 * i + 1] = (uint32_t)(w >> 32);
    }
    if constexpr (KPAD % 64 != 0) {  // KPAD = 32 or 96: one extra 32-bit half word
        const int i = KPAD / 64;
        const uint64_t w = (valid && i < w64) ? __ldg(words + i) : 0ull;
        w32[KPAD / 32 - 1] = (uint32_t)w;
    }
#pragma unroll
    for (int c = 0; c < KPAD / 16; ++c) {
        const uint32_t bits16 = (w32[c / 2] >> (16 * (c & 1))) & 0xFFFFu;
        const uint4 v = valid ? expand16(bits16, 16 * c, d) : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(tile + (size_t)c * rows * 16 + r * 16) = v;
    }
}

template <int KPAD>
__global__ void __launch_bounds__(kThreads, 2)
attn_tc_kernel(const __grid_constant__ Params prm, const __grid_constant__ CUtensorMap vmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FwdArgs& a = prm.a;
    // carve shared memory: V stages (1024-aligned) | P stages | Q tile | K stages | barriers
    unsigned char* sV = smem_raw;                                   // 2 x nbox x 8192
    unsigned char* sP = sV + 2 * prm.nbox * 8192;                   // 2 x 16384
    unsigned char* sQ = sP + 2 * 16384;                             // BM x KPAD
    unsigned char* sK = sQ + BM * KPAD;                             // 2 x BN x KPAD
    Smem* sm = reinterpret_cast<Smem*>(sK + 2 * BN * KPAD);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int head = blockIdx.x / prm.mblocks;
    const int mb = blockIdx.x - head * prm.mblocks;
    const int N = a.N, d = a.d, w64 = a.W64, T = prm.tiles;
    const int row0 = mb * BM;

    // ---------------------------------------------------------------- prologue
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->kfull[s], 64);   // every expander thread arrives
            mbar_init(&sm->kempty[s], 1);   // tcgen05.commit
            mbar_init(&sm->vfull[s], 1);    // expect_tx arrive + TMA bytes
            mbar_init(&sm->vempty[s], 1);   // tcgen05.commit
            mbar_init(&sm->sfull[s], 1);    // tcgen05.commit
            mbar_init(&sm->sempty[s], 128); // every softmax thread arrives
            mbar_init(&sm->pfull[s], 128);  // every softmax thread arrives
            mbar_init(&sm->pempty[s], 1);   // tcgen05.commit
        }
        fence_barrier_init();
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm->tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 5 && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
    if (tid < BM) {  // Q tile: thread r expands query row row0 + r (zeros past N)
        const int row = row0 + tid;
        expand_row<KPAD>(sQ, BM, tid, a.q_words + ((int64_t)head * N + row) * w64, w64, d, row < N);
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm->tmem_base;

    if (warp == 4) {
        // ============================================================ MMA issuer
        if (lane == 0) {
            // instruction descriptors (cute::UMMA::InstrDescriptor bit layout)
            const uint32_t idesc_s = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);  // e4m3 x e4m3 -> f32, K-major A/B
            const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |                      // bf16 x bf16 -> f32, B MN-major
                                      ((uint32_t)(prm.dvp >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
            const uint32_t q_addr = smem_u32(sQ), k_addr = smem_u32(sK), p_addr = smem_u32(sP), v_addr = smem_u32(sV);
            auto issue_pv = [&](int t) {
                const int s = t & 1, n = t >> 1;
                mbar_wait(&sm->pfull[s], n & 1);
                mbar_wait(&sm->vfull[s], n & 1);
                tc_fence_after();
                const int nk = min(BN, N - t * BN);
                const int ksteps = (nk + 15) >> 4;
                for (int ks = 0; ks < ksteps; ++ks) {
                    // A = P (K-major, no swizzle): 16 bf16 per step = 2 core-matrix columns of 2048 B
                    const uint64_t ad = make_desc(p_addr + s * 16384 + ks * 4096, 2048, 128, 0);
                    // B = V tile (MN-major, 128B swizzle): 16 keys per step = 2048 B; next 64 columns = next TMA box
                    const uint64_t bd = make_desc(v_addr + s * prm.nbox * 8192 + ks * 2048, 8192, 1024, 2);
                    mma_bf16(tmem + kColO, ad, bd, idesc_pv, (t > 0 || ks > 0) ? 1u : 0u);
                }
                tc_commit(&sm->pempty[s]);
                tc_commit(&sm->vempty[s]);
            };
            for (int j = 0; j < T; ++j) {
                const int s = j & 1, n = j >> 1;
                mbar_wait(&sm->kfull[s], n & 1);
                mbar_wait(&sm->sempty[s], (n & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < KPAD / 32; ++ks) {
                    const uint64_t ad = make_desc(q_addr + ks * 2 * BM * 16, BM * 16, 128, 0);
                    const uint64_t bd = make_desc(k_addr + s * BN * KPAD + ks * 2 * BN * 16, BN * 16, 128, 0);
                    mma_f8(tmem + kColS + s * BN, ad, bd, idesc_s, ks > 0 ? 1u : 0u);
                }
                tc_commit(&sm->sfull[s]);
                tc_commit(&sm->kempty[s]);
                if (j > 0) issue_pv(j - 1);
            }
            issue_pv(T - 1);
        }
    } else if (warp == 5) {
        // ============================================================ TMA producer (V tiles)
        if (lane == 0) {
            for (int j = 0; j < T; ++j) {
                const int s = j & 1, n = j >> 1;
                mbar_wait(&sm->vempty[s], (n & 1) ^ 1);
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
            mbar_wait(&sm->kempty[s], (n & 1) ^ 1);
            const int key = j * BN + t;
            expand_row<KPAD>(sK + s * BN * KPAD, BN, t, a.k_words + ((int64_t)head * N + key) * w64, w64, d, key < N);
            fence_proxy_async();
            mbar_arrive(&sm->kfull[s]);
        }
    } else {
        // ============================================================ softmax + epilogue (thread = query row)
        const int row = row0 + tid;
        const bool row_ok = row < N;
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
        const float sc2 = a.mu_q[head] * a.mu_k[head] * a.inv_tau * kLog2e;
        const char* bias_row = nullptr;
        const int bsz = dtype_size(a.bias_dtype);
        if (a.bias && row_ok)
            bias_row = static_cast<const char*>(a.bias) + ((int64_t)(head % a.H % a.bias_heads) * N + row) * a.bias_ld * bsz;
        const bool bias_vec = bias_row && a.bias_dtype == BA_BF16 && (reinterpret_cast<uintptr_t>(bias_row) % 16 == 0);
        float m_ref = -INFINITY, m_true = -INFINITY, l = 0.f;

        for (int j = 0; j < T; ++j) {
            const int s = j & 1, n = j >> 1;
            const int nk = min(BN, N - j * BN);
            float x[BN];
            mbar_wait(&sm->sfull[s], n & 1);
            tc_fence_after();
            const uint32_t s_addr = lane_base + kColS + s * BN;
            BA_TMEM_LD16(s_addr + 0, x, 0);
            BA_TMEM_LD16(s_addr + 16, x, 16);
            BA_TMEM_LD16(s_addr + 32, x, 32);
            BA_TMEM_LD16(s_addr + 48, x, 48);
            tc_wait_ld();
            tc_fence_before();
            mbar_arrive(&sm->sempty[s]);

            if (prm.dbg_S && head == prm.dbg_head && row_ok) {
#pragma unroll
                for (int i = 0; i < BN; ++i)
                    if (i < nk) prm.dbg_S[(int64_t)row * N + j * BN + i] = (int)x[i];
            }
            // scores in the base-2 domain; masked columns -> -inf
            if (bias_row) {
#pragma unroll
                for (int c = 0; c < BN / 8; ++c) {
                    const int col = j * BN + c * 8;
                    if (bias_vec && col + 8 <= N) {
                        const uint4 b = __ldg(reinterpret_cast<const uint4*>(bias_row + (int64_t)col * 2));
                        const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            x[c * 8 + 2 * e] = fmaf(x[c * 8 + 2 * e], sc2, __uint_as_float(bw[e] << 16) * kLog2e);
                            x[c * 8 + 2 * e + 1] = fmaf(x[c * 8 + 2 * e + 1], sc2, __uint_as_float(bw[e] & 0xFFFF0000u) * kLog2e);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float bv = (col + e < N) ? load_as_float(bias_row, a.bias_dtype, col + e) : 0.f;
                            x[c * 8 + e] = fmaf(x[c * 8 + e], sc2, bv * kLog2e);
                        }
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < BN; ++i) x[i] *= sc2;
            }
            float tmax = -INFINITY;
#pragma unroll
            for (int i = 0; i < BN; ++i) {
                x[i] = (i < nk) ? x[i] : -INFINITY;
                tmax = fmaxf(tmax, x[i]);
            }
            m_true = fmaxf(m_true, tmax);
            // lazy rescale (first tile: m_ref = -inf forces it with alpha = 0 on the still-unwritten O)
            const bool need = tmax > m_ref + kRescaleThreshold;
            if (__any_sync(0xffffffffu, need)) {
                const float m_new = need ? tmax : m_ref;
                const float alpha = need ? ex2(m_ref - m_new) : 1.0f;
                if (j > 0) {
                    mbar_wait(&sm->pempty[(j - 1) & 1], ((j - 1) >> 1) & 1);  // P.V of tile j-1 has landed in O
                    tc_fence_after();
                    for (int c = 0; c < prm.dvp; c += 16) {
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
            mbar_wait(&sm->pempty[s], (n & 1) ^ 1);  // P.V of tile j-2 no longer reads this P stage
            unsigned char* prow = sP + s * 16384 + tid * 16;
#pragma unroll
            for (int c = 0; c < BN / 8; ++c) {
                float p[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    p[e] = ex2(x[c * 8 + e] - m_ref);
                    l += p[e];
                }
                uint4 v;
                v.x = pack_bf16(p[0], p[1]);
                v.y = pack_bf16(p[2], p[3]);
                v.z = pack_bf16(p[4], p[5]);
                v.w = pack_bf16(p[6], p[7]);
                *reinterpret_cast<uint4*>(prow + c * (BM * 16)) = v;  // column chunk c, row tid: K-major core matrices
            }
            fence_proxy_async();
            mbar_arrive(&sm->pfull[s]);
        }
        // ---------------------------------------------------------------- epilogue: O / l
        mbar_wait(&sm->pempty[(T - 1) & 1], ((T - 1) >> 1) & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l;
        float* orow = a.O + ((int64_t)head * N + row) * d;
        for (int c = 0; c < prm.dvp; c += 16) {
            float o[16];
            BA_TMEM_LD16(lane_base + kColO + c, o, 0);
            tc_wait_ld();
            if (row_ok) {
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    if (c + i < d)
                        *reinterpret_cast<float4*>(orow + c + i) =
                            make_float4(o[i] * inv_l, o[i + 1] * inv_l, o[i + 2] * inv_l, o[i + 3] * inv_l);
            }
        }
        if (row_ok) {
            if (a.row_max) a.row_max[(int64_t)head * N + row] = m_true * kLn2;
            if (a.row_sum) a.row_sum[(int64_t)head * N + row] = l * ex2(m_ref - m_true);
        }
        tc_fence_before();
    }
    __syncthreads();
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

template <int KPAD>
static int launch_kpad(const Params& prm, const CUtensorMap& vmap, cudaStream_t stream) {
    const size_t smem = 2 * (size_t)prm.nbox * 8192 + 2 * 16384 + (size_t)BM * KPAD + 2 * (size_t)BN * KPAD + sizeof(Smem);
    static bool configured = false;
    if (!configured) {
        const cudaError_t e =
            cudaFuncSetAttribute(attn_tc_kernel<KPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        if (e != cudaSuccess) return -(int)e;
        configured = true;
    }
    attn_tc_kernel<KPAD><<<(unsigned)(prm.a.BH * prm.mblocks), kThreads, smem, stream>>>(prm, vmap);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
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
    if (reinterpret_cast<uintptr_t>(a.V) % 16 != 0) return -(int)cudaErrorMisalignedAddress;
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

    CUtensorMap vmap;
    const cuuint64_t gdim[3] = {(cuuint64_t)a.d, (cuuint64_t)a.N, (cuuint64_t)a.BH};
    const cuuint64_t gstr[2] = {(cuuint64_t)a.d * 2, (cuuint64_t)a.N * a.d * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)BN, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.V), gdim, gstr, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -(int)cudaErrorInvalidValue;

    const int kpad = (a.d + 31) / 32 * 32;
    switch (kpad) {
        case 32: return launch_kpad<32>(prm, vmap, stream);
        case 64: return launch_kpad<64>(prm, vmap, stream);
        case 96: return launch_kpad<96>(prm, vmap, stream);
        case 128: return launch_kpad<128>(prm, vmap, stream);
    }
    return -(int)cudaErrorInvalidValue;
}

}  // namespace ba

// Test hook (not part of include/binattn_cuda.h): dump the tensor-core logits of one head as int32 [N,N].
extern "C" void ba_debug_tcgen05_logits(int32_t* dev_S, int head) {
    ba::tc::g_dbg_S = dev_S;
    ba::tc::g_dbg_head = head;
}
