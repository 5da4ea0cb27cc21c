// attn_tc2.cuh -- K2, second generation: fused BinaryAttention forward for sm_100a with ONE CTA per SM that keeps two
// 128-row query tiles in flight against 128-key tiles.
//
// Same arithmetic as attn_tcgen05.cuh (binattn::binary_attention_fused, quantize_pv = false, proj/src/attention.cpp:250-382):
//   S = Q^ K^T   exact +-1 contraction on tcgen05.mma.kind::f8f6f4 (== d - 2 popc(q xor k), bitops.cpp:59-67)
//   x = S*mu_q*mu_k/tau + bias (attention.cpp:34-36), online softmax in the base-2 domain (attention.cpp:306-324)
//   O += P V     bf16 tcgen05.mma.kind::f16, P read from tensor memory, V tiles by TMA; O / l epilogue (attention.cpp:354-364)
//
// Why a second kernel.  The first generation runs one softmax warp per scheduler and CTA (two CTAs per SM); its in-kernel
// timeline shows a 64-key tile costing ~2000 clk per warp, half of it outside the exponentials (barrier round trips,
// TMEM load/store waits, instruction fetch), so the MUFU pipe -- the floor of this kernel -- is ~50% busy.  A register
// loop of the same instructions reaches 15.9 of 16 ex2/clk/SM with two warps per scheduler (scripts/micro/pipe_bench.cu).
// This kernel therefore puts FOUR softmax warps on every scheduler:
//   unit        = (head, 256 query rows) = query tiles A and B; both use the same expanded K tile and the same V tile
//   softmax     = 16 warps: (tile A | B) x (key columns 0-63 | 64-127) x 4 lane quadrants; thread = one row x 64 keys
//   per tile    = one S wait, one P hand-over and one P.V commit per 128 keys (half the fixed cost of 64-key tiles)
//   MMA order   = PV_A(j-1), S_A(j), PV_B(j-1), S_B(j): tile A computes its softmax while the tensor core works for
//                 tile B and vice versa, so the MUFU pipe always sees two warps per scheduler in their exp phase
// 640 threads: warps 0-15 softmax (104 registers), 16 MMA issue + TMEM allocation, 17 TMA producer, 18-19 Q/K expanders.
// TMEM (512 columns): S_A [0,128) | S_B [128,256) | O_A [256,256+dvp) | O_B [384,384+dvp); the bf16 weights overwrite the
// S columns their thread has just read: keys 0-63 -> columns [0,32), keys 64-127 -> columns [64,96) of the tile's S block.
//
// Reference max.  The running max follows the lazy rule of the first kernel (O and l are rescaled only when a row max
// grows by more than 2^kThr2 over the reference used so far; O / l is unaffected).  The two threads of a row exchange a
// one-word "needs a new reference" flag per tile through shared memory and a 64-thread named barrier, and their half-row
// maxima only when the flag is up (always on the first tile of a unit).  Without a bias every logit is bounded a priori by
// |x| <= d*mu_q*mu_k/tau, so when that bound is below 2^32 the reference is the bound itself and the kernel computes no
// row max at all (FAST path; the row_max / row_sum outputs need the true max and take the general path).
#pragma once
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc2 {

using namespace ba::tc;  // PTX wrappers, descriptors, Ring, expand_store, rescale_o

constexpr int TM = 128;            // rows of one query tile (UMMA M)
constexpr int TN = 128;            // keys per tile (UMMA N of the S MMA)
constexpr int kThreads2 = 640;
constexpr int kColO2 = 256;        // first O column; tile X owns [256 + 128 X, +dvp)
constexpr int kVBox = 16384;       // one TMA box of V: 128 keys x 64 columns bf16, 128B swizzle
constexpr int kBSub = 16384;       // one bias sub-tile: 128 rows x 64 columns bf16, 128B swizzle
constexpr float kThr2 = 16.0f;     // lazy-rescale threshold, log2 units
constexpr float kFastBound = 32.0f;  // FAST path when d * mu_q mu_k / tau * log2(e) <= this (weights stay >= 2^-64)
constexpr int kRegsSoftmax2 = 104, kRegsCtrl2 = 64;  // the pool is what the launch allocated: 640 x 96 = 512 x 104 + 128 x 64

struct Smem2 {
    uint64_t qfull[2], qfree[2];  // Q tiles of a unit expanded / every S MMA of the unit retired
    uint64_t kfull[4], kfree[4];  // K tile expanded / its S MMAs retired
    uint64_t vfull[4], vfree[4];  // V tile landed (TMA) / its P.V MMAs retired
    uint64_t bfull[8], bfree[8];  // bias sub-tile landed (TMA) / read out by its four softmax warps
    uint64_t sfull[2];            // S of query tile X ready in TMEM
    uint64_t pfull[2];            // P of query tile X written by its eight softmax warps
    uint64_t pvdone[2];           // P.V MMA of query tile X retired
    uint64_t ofree[2];            // O of query tile X read out by the epilogue
    uint64_t stag;                // tile A is half way through its first softmax tile: S_B(0) may be issued (phase stagger)
    uint2 lut[256];               // byte of sign bits -> 8 e4m3 +-1.0 bytes
    float xch[2][2][TM];          // (query tile, column half, row): half-row max / partial denominator for the other half
    uint32_t flag[2][2][4][2];    // (tile parity, query tile, lane quadrant, column half): "my warp needs a new reference max"
    uint32_t tmem_base;
};

struct Params2 {
    FwdArgs a;
    int tiles;     // N / 128 key tiles
    int ublocks;   // ceil(N / 256) units per head
    int units;     // BH * ublocks
    int dvp;       // d rounded up to 16
    int nbox;      // ceil(d / 64) TMA boxes per V tile
    int qst, kst, vst, bst;
    int32_t* dbg_S;
    int dbg_head;
};

__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1) {
    asm("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
        "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1));
}
__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// BIAS: 0 = none, 1 = dense bf16 table staged by TMA.  N % 128 == 0.
template <int KPAD, int BIAS, bool DBG>
__global__ void __launch_bounds__(kThreads2, 1)
attn_tc2_kernel(const __grid_constant__ Params2 prm, const __grid_constant__ CUtensorMap vmap,
                const __grid_constant__ CUtensorMap bmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FwdArgs& a = prm.a;
    unsigned char* sV = smem_raw;                               // vst x nbox x 16 KB
    unsigned char* sB = sV + prm.vst * prm.nbox * kVBox;        // bst x 16 KB
    unsigned char* sQ = sB + prm.bst * kBSub;                   // qst x 256 x KPAD (tile A rows, then tile B rows)
    unsigned char* sK = sQ + prm.qst * 2 * TM * KPAD;           // kst x 128 x KPAD
    Smem2* sm = reinterpret_cast<Smem2*>(sK + prm.kst * TN * KPAD);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = a.N, d = a.d, w64 = a.W64, T = prm.tiles;
    const int G = gridDim.x;

    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->qfull[s], 2);
            mbar_init(&sm->qfree[s], 1);
            mbar_init(&sm->sfull[s], 1);
            mbar_init(&sm->pfull[s], 8);
            mbar_init(&sm->pvdone[s], 1);
            mbar_init(&sm->ofree[s], 8);
        }
        mbar_init(&sm->stag, 8);
        for (int s = 0; s < 4; ++s) {
            mbar_init(&sm->kfull[s], 2);
            mbar_init(&sm->kfree[s], 1);
            mbar_init(&sm->vfull[s], 1);
            mbar_init(&sm->vfree[s], 1);
        }
        for (int s = 0; s < 8; ++s) {
            mbar_init(&sm->bfull[s], 1);
            mbar_init(&sm->bfree[s], 4);
        }
        fence_barrier_init();
    }
    if (warp == 16) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm->tmem_base)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 17 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        if (BIAS == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
    }
    if (tid < 256) sm->lut[tid] = expand_byte((uint32_t)tid);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm->tmem_base;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's packed words and scales are read from here on

    if (warp >= 16) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtrl2));
        if (warp == 16) {
            // ======================================================== MMA issuer (whole warp, one elected lane issues)
            const uint32_t idesc_s = (1u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
            const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(prm.dvp >> 3) << 17) |
                                      ((uint32_t)(TM >> 4) << 24);
            const uint64_t q_desc = make_desc(smem_u32(sQ), TM * 16, 128, 0);
            const uint64_t k_desc = make_desc(smem_u32(sK), TN * 16, 128, 0);
            const uint64_t v_desc = make_desc(smem_u32(sV), kVBox, 1024, 2);
            Ring qr, kr, vr;
            uint32_t gp[2] = {0, 0};  // P tiles consumed per query tile
            uint32_t up[2] = {0, 0};  // units finished per query tile
            int pend = 0, pj = 0, pnact = 0, pvs = 0;
            bool staggered = false;
            uint32_t pvph = 0;
            // P.V of the pending key tile for query tile X (issued one S MMA late, see the header)
            auto issue_pv = [&](int X, bool last_of_tile) {
                mbar_wait(&sm->pfull[X], gp[X] & 1u);
                if (pj == 0 && up[X] > 0) mbar_wait(&sm->ofree[X], (up[X] - 1) & 1u);  // the epilogue has read the old O
                tc_fence_after();
                const uint64_t vd = v_desc + (uint64_t)((pvs * prm.nbox * kVBox) >> 4);
                const uint32_t p_tmem = tmem + X * TN;
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < TN / 16; ++ks)
                        mma_bf16_ts(tmem + kColO2 + X * 128, p_tmem + (ks >> 2) * 64 + (ks & 3) * 8, vd + (uint64_t)(ks * (2048 >> 4)),
                                    idesc_pv, (pj > 0 || ks > 0) ? 1u : 0u);
                    tc_commit(&sm->pvdone[X]);
                    if (last_of_tile) tc_commit(&sm->vfree[pvs]);
                }
                __syncwarp();
                ++gp[X];
                if (pj == T - 1) ++up[X];
            };
            for (int u = blockIdx.x; u < prm.units; u += G) {
                const int ub = u % prm.ublocks;
                const int nact = (ub * 2 * TM + TM < N) ? 2 : 1;
                mbar_wait(&sm->qfull[qr.stage], qr.phase);
                const uint64_t qd = q_desc + (uint64_t)((qr.stage * 2 * TM * KPAD) >> 4);
                for (int j = 0; j < T; ++j) {
                    if (pend) {
                        mbar_wait(&sm->vfull[pvs], pvph);
                        issue_pv(0, pnact == 1);
                    }
                    mbar_wait(&sm->kfull[kr.stage], kr.phase);
                    tc_fence_after();
                    const uint64_t kd = k_desc + (uint64_t)((kr.stage * TN * KPAD) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < KPAD / 32; ++ks)
                            mma_f8(tmem, qd + (uint64_t)(ks * ((2 * TM * 16) >> 4)), kd + (uint64_t)(ks * ((2 * TN * 16) >> 4)), idesc_s,
                                   ks > 0 ? 1u : 0u);
                        tc_commit(&sm->sfull[0]);
                        if (nact == 1) {
                            tc_commit(&sm->kfree[kr.stage]);
                            if (j == T - 1) tc_commit(&sm->qfree[qr.stage]);
                        }
                    }
                    __syncwarp();
                    if (pend && pnact == 2) issue_pv(1, true);
                    if (nact == 2) {
                        // The two query tiles must run in ANTI-phase (A in its exponentials while the tensor core works for
                        // B): the offset between them is neutrally stable, so it is set once, here, by holding B's first S
                        // back until A is half way through its first tile.
                        if (!staggered) {
                            mbar_wait(&sm->stag, 0);
                            staggered = true;
                        }
                        if (elect_one()) {
#pragma unroll
                            for (int ks = 0; ks < KPAD / 32; ++ks)
                                mma_f8(tmem + TN, qd + (uint64_t)((TM * KPAD) >> 4) + (uint64_t)(ks * ((2 * TM * 16) >> 4)),
                                       kd + (uint64_t)(ks * ((2 * TN * 16) >> 4)), idesc_s, ks > 0 ? 1u : 0u);
                            tc_commit(&sm->sfull[1]);
                            tc_commit(&sm->kfree[kr.stage]);
                            if (j == T - 1) tc_commit(&sm->qfree[qr.stage]);
                        }
                        __syncwarp();
                    }
                    pend = 1;
                    pj = j;
                    pnact = nact;
                    pvs = vr.stage;
                    pvph = vr.phase;
                    vr.next(prm.vst);
                    kr.next(prm.kst);
                }
                qr.next(prm.qst);
            }
            if (pend) {
                mbar_wait(&sm->vfull[pvs], pvph);
                issue_pv(0, pnact == 1);
                if (pnact == 2) issue_pv(1, true);
            }
        } else if (warp == 17) {
            // ======================================================== TMA producer: bias sub-tiles, V tiles
            if (lane == 0) {
                Ring vr, br;
                for (int u = blockIdx.x; u < prm.units; u += G) {
                    const int head = u / prm.ublocks;
                    const int ub = u - head * prm.ublocks;
                    const int nact = (ub * 2 * TM + TM < N) ? 2 : 1;
                    const int bh = (a.head0 + head) % a.H % a.bias_heads;
                    for (int j = 0; j < T; ++j) {
                        if (BIAS == 1) {
                            for (int s = 0; s < 2 * nact; ++s) {  // (tile A | B) x (columns 0-63 | 64-127), in consumption order
                                mbar_wait(&sm->bfree[br.stage], br.phase ^ 1u);
                                mbar_expect_tx(&sm->bfull[br.stage], kBSub);
                                tma_load_3d(&bmap, &sm->bfull[br.stage], sB + br.stage * kBSub, j * TN + (s & 1) * 64,
                                            ub * 2 * TM + (s >> 1) * TM, bh);
                                br.next(prm.bst);
                            }
                        }
                        mbar_wait(&sm->vfree[vr.stage], vr.phase ^ 1u);
                        mbar_expect_tx(&sm->vfull[vr.stage], prm.nbox * kVBox);
                        for (int b = 0; b < prm.nbox; ++b)
                            tma_load_3d(&vmap, &sm->vfull[vr.stage], sV + (vr.stage * prm.nbox + b) * kVBox, b * 64, j * TN, head);
                        vr.next(prm.vst);
                    }
                }
            }
        } else {
            // ======================================================== Q / K expanders (64 threads)
            const int t = tid - 18 * 32;
            Ring qr, kr;
            uint32_t wk0[KPAD / 32], wk1[KPAD / 32];
            if ((int)blockIdx.x < prm.units) {
                const int head = blockIdx.x / prm.ublocks;
                load_words<KPAD>(wk0, a.k_words + ((int64_t)head * N + t) * w64, w64, true);
                load_words<KPAD>(wk1, a.k_words + ((int64_t)head * N + t + 64) * w64, w64, true);
            }
            for (int u = blockIdx.x; u < prm.units; u += G) {
                const int head = u / prm.ublocks;
                const int row0 = (u - head * prm.ublocks) * 2 * TM;
                {   // the unit's 256 query rows (rows past N expand to zeros)
                    uint32_t wq[4][KPAD / 32];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        load_words<KPAD>(wq[i], a.q_words + ((int64_t)head * N + row0 + t + 64 * i) * w64, w64, row0 + t + 64 * i < N);
                    mbar_wait(&sm->qfree[qr.stage], qr.phase ^ 1u);
                    unsigned char* qt = sQ + qr.stage * 2 * TM * KPAD;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        expand_store<KPAD>(qt + (i >> 1) * TM * KPAD, TM, t + 64 * (i & 1), wq[i], d, row0 + t + 64 * i < N, sm->lut);
                    fence_proxy_async();
                    warp_arrive(&sm->qfull[qr.stage], lane);
                    qr.next(prm.qst);
                }
                const int un = u + G;
                const int hn = un / prm.ublocks;
                for (int j = 0; j < T; ++j) {
                    mbar_wait(&sm->kfree[kr.stage], kr.phase ^ 1u);
                    unsigned char* kt = sK + kr.stage * TN * KPAD;
                    expand_store<KPAD>(kt, TN, t, wk0, d, true, sm->lut);
                    expand_store<KPAD>(kt, TN, t + 64, wk1, d, true, sm->lut);
                    fence_proxy_async();
                    warp_arrive(&sm->kfull[kr.stage], lane);
                    kr.next(prm.kst);
                    if (j + 1 < T) {
                        load_words<KPAD>(wk0, a.k_words + ((int64_t)head * N + (j + 1) * TN + t) * w64, w64, true);
                        load_words<KPAD>(wk1, a.k_words + ((int64_t)head * N + (j + 1) * TN + t + 64) * w64, w64, true);
                    } else if (un < prm.units) {
                        load_words<KPAD>(wk0, a.k_words + ((int64_t)hn * N + t) * w64, w64, true);
                        load_words<KPAD>(wk1, a.k_words + ((int64_t)hn * N + t + 64) * w64, w64, true);
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax2));
        // ============================================================ softmax + epilogue: thread = (query row, 64 keys)
        const int X = warp >> 3, half = (warp >> 2) & 1, quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const uint32_t s_addr = lane_base + X * TN + half * 64;  // my 64 S columns; P goes over the first 32 of them
        const uint32_t o_addr = lane_base + kColO2 + X * 128;
        const int pair_id = 1 + X * 4 + quad;
        const int h16 = ((prm.dvp >> 1) + 15) & ~15;             // O columns [0,h16) belong to half 0, [h16,dvp) to half 1
        const int oc0 = half ? h16 : 0, oc1 = half ? prm.dvp : h16;
        const bool stats = a.row_max != nullptr || a.row_sum != nullptr;
        uint32_t gx = 0;      // key tiles this query tile has been through (parity of sfull / pfull / pvdone)
        uint32_t bcount = 0;  // bias sub-tiles the producer has issued before the current unit
        for (int u = blockIdx.x; u < prm.units; u += G) {
            const int head = u / prm.ublocks;
            const int ub = u - head * prm.ublocks;
            const int nact = (ub * 2 * TM + TM < N) ? 2 : 1;
            if (X >= nact) {  // tile B of the last unit of a head with an odd number of 128-row blocks: nothing to do
                bcount += (uint32_t)(T * 2 * nact);
                continue;
            }
            const int row = ub * 2 * TM + X * TM + r;
            const float sc = __ldg(a.mu_q + head) * __ldg(a.mu_k + head) * a.inv_tau;  // natural-log units per unit of dot
            const float ea = (BIAS == 0) ? sc * kLog2e : kLog2e;  // BIAS 0 keeps x = raw dot and folds the scale into the exponent
            const bool fast = BIAS == 0 && !stats && !DBG && sc * kLog2e * (float)d <= kFastBound;
            float m_ref = fast ? sc * kLog2e * (float)d : -INFINITY, m_true = -INFINITY;
            float l0 = 0.f, l1 = 0.f;
            const bool dump = DBG && prm.dbg_S && head == prm.dbg_head;
            for (int j = 0; j < T; ++j, ++gx) {
                float x[64];
                uint32_t bstage = 0;
                mbar_wait(&sm->sfull[X], gx & 1u);
                tc_fence_after();
                BA_TMEM_LD16(s_addr + 0, x, 0);
                BA_TMEM_LD16(s_addr + 16, x, 16);
                BA_TMEM_LD16(s_addr + 32, x, 32);
                BA_TMEM_LD16(s_addr + 48, x, 48);
                if (BIAS == 1) {
                    const uint32_t bi = bcount + (uint32_t)(j * 2 * nact + X * 2 + half);
                    const uint32_t lap = bi / (uint32_t)prm.bst;
                    bstage = bi - lap * (uint32_t)prm.bst;
                    mbar_wait(&sm->bfull[bstage], lap & 1u);
                }
                tc_wait_ld();
                if (DBG && dump) {
                    int32_t* drow = prm.dbg_S + (int64_t)row * N + j * TN + half * 64;
#pragma unroll
                    for (int i = 0; i < 64; ++i) drow[i] = (int)x[i];
                }
                if (BIAS == 1) {
                    const unsigned char* brow = sB + bstage * kBSub + r * 128;  // row r of the 128 x 64 bf16 sub-tile
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 b = *reinterpret_cast<const uint4*>(brow + ((c ^ (r & 7)) << 4));
                        const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            fma2(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], sc, sc,
                                 __uint_as_float(bw[e] << 16), __uint_as_float(bw[e] & 0xFFFF0000u));
                    }
                    warp_arrive(&sm->bfree[bstage], lane);
                }
                if (!fast) {
                    float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
                    for (int i = 4; i < 64; i += 4) {
                        m0 = fmaxf(m0, x[i]);
                        m1 = fmaxf(m1, x[i + 1]);
                        m2 = fmaxf(m2, x[i + 2]);
                        m3 = fmaxf(m3, x[i + 3]);
                    }
                    const float hm = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * ea;  // ea > 0: the max commutes with the scaling
                    const bool need = hm > m_ref + kThr2;
                    const uint32_t mine = (stats || __any_sync(0xffffffffu, need)) ? 1u : 0u;
                    volatile uint32_t* fl = &sm->flag[gx & 1u][X][quad][0];
                    if (lane == 0) fl[half] = mine;
                    pair_sync(pair_id);
                    if (mine | fl[half ^ 1]) {  // rare after the first tile of a unit: agree on a new reference for the rows that need one
                        sm->xch[X][half][r] = hm;
                        pair_sync(pair_id);
                        const float tm = fmaxf(hm, sm->xch[X][half ^ 1][r]);
                        m_true = fmaxf(m_true, tm);
                        if (tm > m_ref + kThr2) {
                            const float alpha = ex2(m_ref - tm);  // first tile: 2^-inf = 0 on a still-unwritten O
                            // S(j) is complete, so P.V(j-1) -- issued before it -- has retired: O is quiescent
                            if (j > 0 && oc1 > oc0) rescale_o(o_addr + oc0, oc1 - oc0, alpha);
                            l0 *= alpha;
                            l1 *= alpha;
                            m_ref = tm;
                        }
                    }
                }
                const float nm = -m_ref;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int i = 32 * h + 2 * e;
                        float a0, a1;
                        fma2(a0, a1, x[i], x[i + 1], ea, ea, nm, nm);
                        const float p0 = ex2(a0), p1 = ex2(a1);
                        add2(l0, l1, p0, p1);
                        pk[e] = pack_bf16(p0, p1);
                    }
                    BA_TMEM_ST16U(s_addr + 16 * h, pk);
                    if (h == 0 && X == 0 && gx == 0) warp_arrive(&sm->stag, lane);
                }
                tc_wait_st();
                tc_fence_before();
                warp_arrive(&sm->pfull[X], lane);
            }
            bcount += (uint32_t)(T * 2 * nact);
            // ---------------------------------------------------------------- epilogue: O / l for my half of the columns
            mbar_wait(&sm->pvdone[X], (gx - 1) & 1u);
            tc_fence_after();
            sm->xch[X][half][r] = l0 + l1;
            pair_sync(pair_id);
            const float l = (l0 + l1) + sm->xch[X][half ^ 1][r];
            const float inv_l = 1.0f / l;
            float* orow = a.O + ((int64_t)head * N + row) * d;
            for (int c = oc0; c < oc1; c += 16) {
                float o[16];
                BA_TMEM_LD16(o_addr + c, o, 0);
                tc_wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) o[i] *= inv_l;
                if (row < N) {
                    if (c + 8 <= d) stg_256(orow + c, o);
                    if (c + 16 <= d) stg_256(orow + c + 8, o + 8);
                }
            }
            tc_fence_before();
            if (stats && half == 0 && row < N) {
                if (a.row_max) a.row_max[(int64_t)head * N + row] = m_true * kLn2;
                if (a.row_sum) a.row_sum[(int64_t)head * N + row] = l * ex2(m_ref - m_true);
            }
            warp_arrive(&sm->ofree[X], lane);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 16) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

constexpr size_t kSmemMax2 = 227 * 1024;

inline size_t smem_bytes2(const Params2& p, int kpad) {
    return (size_t)p.vst * p.nbox * kVBox + (size_t)p.bst * kBSub + (size_t)p.qst * 2 * TM * kpad + (size_t)p.kst * TN * kpad +
           sizeof(Smem2);
}

template <int KPAD, int BIAS, bool DBG>
static int launch_variant2(const Params2& prm, const CUtensorMap& vmap, const CUtensorMap& bmap, cudaStream_t stream) {
    static bool configured[kMaxDevices] = {};
    const int dev = current_device();
    if (!configured[dev]) {
        const cudaError_t e = cudaFuncSetAttribute(attn_tc2_kernel<KPAD, BIAS, DBG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)kSmemMax2);
        if (e != cudaSuccess) return -(int)e;
        configured[dev] = true;
    }
    int grid = (int)std::min<long>(prm.units, sm_count());
    if (env_long("BA_GRID", 0) > 0) grid = (int)std::min<long>(prm.units, env_long("BA_GRID", 0));  // dev knob
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads2);
    cfg.dynamicSmemBytes = smem_bytes2(prm, KPAD);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // the prologue overlaps K1's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = env_long("BA_PDL", 1) ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_tc2_kernel<KPAD, BIAS, DBG>, prm, vmap, bmap);
    return e == cudaSuccess ? 1 : -(int)e;
}

template <int KPAD>
static int launch_kpad2(const Params2& prm, int bias_mode, const CUtensorMap& vmap, const CUtensorMap& bmap, cudaStream_t stream) {
    if (prm.dbg_S && bias_mode == 0) return launch_variant2<KPAD, 0, true>(prm, vmap, bmap, stream);
    if (bias_mode == 1) return launch_variant2<KPAD, 1, false>(prm, vmap, bmap, stream);
    return launch_variant2<KPAD, 0, false>(prm, vmap, bmap, stream);
}

}  // namespace tc2
}  // namespace ba
