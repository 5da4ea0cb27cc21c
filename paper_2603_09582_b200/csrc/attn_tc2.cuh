// attn_tc2.cuh -- K2, second generation: fused BinaryAttention forward for sm_100a with ONE CTA per SM that keeps two
// 128-row query tiles in flight and FOUR softmax warps on every scheduler.
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
//   unit        = (head, 256 query rows) = query tiles A and B; both use the same expanded K tile and the same V tile
//   key tiles   = 64 keys; every query tile has TWO S stages in tensor memory, and the S MMA of tile j+1 is issued before
//                 the P.V MMA of tile j, so a softmax warp never waits for the tensor core
//   softmax     = 16 warps: (tile A | B) x (key columns 0-31 | 32-63) x 4 lane quadrants; thread = one row x 32 keys;
//                 the fixed per-tile cost of one warp (barrier, TMEM load / store round trips) hides behind the
//                 exponentials of the three other warps of its scheduler
//   (a first version used 128-key tiles with one S stage per query tile and 64 keys per thread; the two query tiles then
//    ran in phase -- both waiting for the tensor core at the same time -- and the MUFU pipe stayed at 64%)
// 640 threads: warps 0-15 softmax (104 registers), 16 / 17 MMA issue for tile A / B (16 also allocates TMEM), 18 TMA producer,
// 19 the Relative2dBias tables.  Q and K tiles come pre-expanded from expand_qk_kernel (workspace planes) by bulk copy.
// TMEM (512 columns): tile X owns S stages [128 X + 64 s, +64) and O [256 + 128 X, +dvp); the bf16 weights overwrite the
// S columns their thread has just read: keys 0-31 -> columns [0,16), keys 32-63 -> columns [32,48) of the stage.
//
// Reference max.  The running max follows the lazy rule of the first kernel (O and l are rescaled only when a row max
// grows by more than 2^kThr2 over the reference used so far; O / l is unaffected).  The two threads of a row exchange a
// one-word "needs a new reference" flag per tile through shared memory and a 64-thread named barrier, and their half-row
// maxima only when the flag is up (always on the first tile of a unit).  Without a bias every logit is bounded a priori by
// |x| <= d*mu_q*mu_k/tau, so when that bound is below 2^32 the reference is the bound itself and the kernel computes no
// row max at all (FAST path; the row_max / row_sum outputs need the true max and take the general path).
//
// I8 mode (template parameter; quantize_pv = true, the reference's default arithmetic, attention.cpp:332-343, 361-363): the
// same pipeline with an integer P.V half -- u8 weights relative to the TRUE running max of every 64-key block as A operand in
// tensor memory, s8 value levels as MN-major B operand, tcgen05.mma.kind::i8 into a fresh s32 accumulator per tile that the
// softmax threads fold into an fp32 O (also in tensor memory) one tile later.  See the comment at the kernel.
#pragma once
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc2 {

using namespace ba::tc;  // PTX wrappers, descriptors, Ring, expand_store, rescale_o

constexpr int TM = 128;            // rows of one query tile (UMMA M)
constexpr int TN = 64;             // keys per tile (UMMA N of the S MMA)
constexpr int kThreads2 = 640;
constexpr int kColO2 = 256;        // first O column; tile X owns [256 + 128 X, +dvp)
constexpr int kVBox = 8192;        // one TMA box of V: 64 keys x 64 columns bf16, 128B swizzle
constexpr int kVBox8 = 4096;       // I8: one TMA box of the s8 value levels: 64 keys x 64 columns, 64B swizzle
constexpr int kOStage = 16 * 2048;  // epilogue staging: 16 warps x one 2 KB box ([32 rows][16 floats], 64B swizzle)
constexpr int kBSub = 16384;       // one bias tile: 128 rows x 64 columns bf16, 128B swizzle
#ifndef BA_PP_AT
#define BA_PP_AT -1  // (measured: no gain with mbarriers or named barriers; kept as a dev knob) exponent pair after which a warp hands the MUFU pipe to the other query tile's pair (-1: no ping-pong)
#endif
#ifndef BA_EXP_LA
#define BA_EXP_LA 0  // dev knob: software-pipeline depth (exponent pairs) of the MUFU loop; 0 = leave the schedule to ptxas
#endif
#ifndef BA_THR2
#define BA_THR2 16.0f
#endif
constexpr float kThr2 = BA_THR2;     // lazy-rescale threshold, log2 units
constexpr float kFastBound = 32.0f;  // FAST path when d * mu_q mu_k / tau * log2(e) <= this (weights stay >= 2^-64)
#ifndef BA_REGS_SOFTMAX
#define BA_REGS_SOFTMAX 104  // dev knobs (setmaxnreg targets); the defaults are the whole launch allocation
#endif
#ifndef BA_REGS_CTRL
#define BA_REGS_CTRL 64
#endif
constexpr int kRegsSoftmax2 = BA_REGS_SOFTMAX, kRegsCtrl2 = BA_REGS_CTRL;  // the pool is what the launch allocated: 640 x 96 = 512 x 104 + 128 x 64

struct Smem2 {
    uint64_t qfull[2], qfree[2];  // Q tiles of a unit expanded / every S MMA of the unit retired
    uint64_t kfull[4], kfree[4];  // K tile expanded / its S MMAs retired
    uint64_t vfull[4], vfree[4];  // V tile landed (TMA) / its P.V MMAs retired
    uint64_t bfull[8], bfree[8];  // bias tile landed (TMA) / read out by the eight softmax warps of its query tile
    uint64_t sfull[2][2];         // [query tile][stage] S ready in TMEM
    uint64_t pfull[2][2];         // [query tile][stage] P written by the eight softmax warps of the query tile
    uint64_t pvdone[2][2];        // [query tile][stage] P.V MMA retired
    uint64_t ofree[2];            // O of query tile X read out by the epilogue
    float xch[2][2][TM];          // (query tile, column half, row): half-row max / partial denominator for the other half
    uint32_t flag[2][2][4][2];    // (tile parity, query tile, lane quadrant, column half): "my warp needs a new reference max"
    float rel2[3][2][256];        // BIAS 4: row / col offset tables (2g-1 <= 255 entries) of the heads of three consecutive units
    float xch8[2][2][2][TM];      // I8: (tile parity, query tile, column half, row) block max of my half, every tile
    uint32_t tmem_base;
};

struct Params2 {
    FwdArgs a;
    int tiles;     // N / 64 key tiles
    int ublocks;   // ceil(N / 256) units per head
    int units;     // END (exclusive) of this call's unit range: BH * ublocks unless unit-sharded (ba_params.unit_begin / unit_end)
    int unit0;     // first unit of the range
    int dvp;       // d rounded up to 16
    int nbox;      // ceil(d / 64) TMA boxes per V tile
    int qst, kst, vst, bst;
    int o_stage;   // the epilogue goes through per-warp staging boxes and TMA stores (when 32 KB of shared memory are left)
    int g;         // BIAS 4: grid side sqrt(N) (a multiple of 32)
    int vbox;      // bytes of one V box in shared memory (kVBox, or kVBox8 in the I8 mode)
    const double* vscales;  // I8: [BH, d] per-channel value scales (quantize_values, quantize.cpp:57-74)
    int vcol0, dsl;         // I8: this launch computes O columns [vcol0, vcol0 + dsl) (dsl <= 64; wider heads take one pass per slice)
    int32_t* dbg_S;
    int dbg_head;
    long long* dbg_T;
};

__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1) {
    asm("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
        "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1));
}
// 1-D bulk copy global -> shared, completion counted in bytes on an mbarrier (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
// D[tmem] (s32) (+)= A[tmem] (u8, K-major: lane = row, one 32-bit column = four K elements) * B[smem] (s8)
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
// s32 accumulator word (arrived through a float register) -> float.  I2F runs on the conversion unit that shares the
// 16-per-clock pipe with ex2; the alternative that stays off it -- integer add into the mantissa of 1.5 * 2^23, then subtract
// it, exact below 2^22 -- costs two issue slots instead of one, and the I8 loop is bound by issue slots, not by that pipe
// (measured: I2F 2.5 % faster at N = 16384).  BA_I8_MAGIC selects the other one.
__device__ __forceinline__ float s32_to_float(float bits) {
#ifdef BA_I8_MAGIC
    return __int_as_float(__float_as_int(bits) + 0x4B400000) - 12582912.0f;
#else
    return (float)__float_as_int(bits);
#endif
}
#define BA_TMEM_ST8U(taddr, v)                                                                                  \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%8], {%0,%1,%2,%3,%4,%5,%6,%7};"                        \
                 ::"r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(taddr) \
                 : "memory")
// mbarrier test with the poll and the look at its result in different places: the predicate takes ~170 clk to land, and an
// in-order warp that reads it at once (mbar_test) stalls for all of it -- three mbar_test in a row cost ~500 clk.  PRED is a
// predicate register declared once at function scope (BA_DECLARE_PRED); MBAR_POLLs issued back to back share one round trip.
#define BA_DECLARE_PRED(PRED) asm volatile(".reg .pred " #PRED ";")
#define MBAR_POLL(PRED, bar, parity) \
    asm volatile("mbarrier.test_wait.parity.shared::cta.b64 " #PRED ", [%0], %1;" ::"r"(smem_u32(bar)), "r"(parity) : "memory")
#define MBAR_POLLED(PRED, out) asm volatile("selp.u32 %0, 1, 0, " #PRED ";" : "=r"(out)::"memory")
// Per-thread constants of the softmax loop (addresses derived from %tid) are passed through this so that they live in a
// register: left alone, the compiler re-derives them from %tid in every key tile (a dozen S2R + ~40 integer instructions
// per tile in a loop whose issue slots are the bound).
__device__ __forceinline__ uint32_t keep_u32(uint32_t v) {
    asm volatile("" : "+r"(v));
    return v;
}
__device__ __forceinline__ uint4 lds_128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u32_volatile(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32_volatile(uint32_t addr, uint32_t v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// BIAS: 0 = none, 1 = dense bf16 table staged by TMA, 4 = Relative2dBias generated from its two offset tables (see below).  Any N >= 128: the K plane is zero-padded to whole 64-key tiles, V and bias
// tiles are zero-filled past N by the TMA unit, and the last tile's surplus columns are masked to -inf before the row max.
#ifdef BA_DEV_TL_MMA  // dev builds only: extra stamps inside the elected S-issue block (scripts/timeline_tc2.py ... mma8)
#define BA_STAMP3() BA_STAMP2()
#else
#define BA_STAMP3() do { } while (0)
#endif
#ifdef BA_DEV_TL_EPI  // dev builds only: stamps around the epilogue's phases (scripts/timeline_units.py ... epi)
#define BA_STAMP4() BA_STAMP2()
#else
#define BA_STAMP4() do { } while (0)
#endif
#define BA_STAMP2()                                                      \
    do {                                                                 \
        if (TL && tl_buf && tl_n < kTlStamps) tl_buf[tl_n++] = clock64(); \
    } while (0)

// I8: the reference's integer P.V mode (quantize_pv = true, attention.cpp:332-343, 361-363) with block_cols = 64 = one key tile:
// per tile the TRUE running max (no lazy rescale: the u8 weight grid is relative to the running max after each block),
// P8 = round(255 * exp(S - m_new)) as u8 A operand in TMEM, s8 value levels (K1v) as MN-major B operand, tcgen05.mma.kind::i8 into
// a FRESH s32 accumulator per tile; the softmax threads fold it into an fp32 O kept in TMEM one tile later:
// O = O * rescale + acc.  TMEM per query tile X (256 columns): S stages [0,128), s32 accumulator [128,192), fp32 O [192,256)
// => d <= 64.  Epilogue: O / l / 255 * delta[c].
template <int KPAD, int BIAS, bool DBG, bool TL = false, bool RAGGED = false, bool I8 = false>
__global__ void __launch_bounds__(kThreads2, 1)
attn_tc2_kernel(const __grid_constant__ Params2 prm, const __grid_constant__ CUtensorMap vmap,
                const __grid_constant__ CUtensorMap bmap, const __grid_constant__ CUtensorMap omap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FwdArgs& a = prm.a;
    unsigned char* sV = smem_raw;                               // vst x nbox x 8 KB
    unsigned char* sB = sV + prm.vst * prm.nbox * prm.vbox;     // bst x 16 KB
    unsigned char* sQ = sB + prm.bst * kBSub;                   // qst x 256 x KPAD (tile A rows, then tile B rows)
    unsigned char* sO = sQ + prm.qst * 2 * TM * KPAD;           // o_stage x 16 x 2 KB: one [32 rows][16 floats] staging box per softmax warp
    unsigned char* sK = sO + prm.o_stage * kOStage;             // kst x 64 x KPAD
    Smem2* sm = reinterpret_cast<Smem2*>(sK + prm.kst * TN * KPAD);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = a.N, d = a.d, T = prm.tiles;
    const int G = gridDim.x;
    const int ub0 = prm.unit0 + (int)blockIdx.x;  // this CTA's first unit
    // dev timeline (TL builds): [cta][role 0 = softmax warp 0 (tile A), 1 = MMA warp, 2 = TMA lane, 3 = expander][kTlStamps]
    long long* tl_buf = nullptr;
    int tl_n = 0;
    (void)tl_n;
    if (TL && prm.dbg_T && (tid == 0 || tid == 512 || tid == 544 || tid == 608))
        tl_buf = prm.dbg_T + ((size_t)blockIdx.x * 4 + (tid == 0 ? 0 : tid == 512 ? 1 : tid == 544 ? 2 : 3)) * kTlStamps;

    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm->qfull[s], BIAS == 4 ? 2 : 1);  // the producer's expect_tx arrival (+ warp 19 with the BIAS 4 tables)
            mbar_init(&sm->qfree[s], 2);
            mbar_init(&sm->ofree[s], 8);
            for (int t = 0; t < 2; ++t) {
                mbar_init(&sm->sfull[s][t], 1);
                mbar_init(&sm->pfull[s][t], 8);
                mbar_init(&sm->pvdone[s][t], 1);
            }
        }
        for (int s = 0; s < 4; ++s) {
            mbar_init(&sm->kfull[s], 1);
            mbar_init(&sm->kfree[s], 2);
            mbar_init(&sm->vfull[s], 1);
            mbar_init(&sm->vfree[s], 2);
        }
        for (int s = 0; s < 8; ++s) {
            mbar_init(&sm->bfull[s], 1);
            mbar_init(&sm->bfree[s], 8);
        }
        fence_barrier_init();
    }
    if (warp == 16) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm->tmem_base)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 18 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        if (BIAS == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
        if (prm.o_stage) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&omap)) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm->tmem_base;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's packed words and scales are read from here on

    if (warp >= 16) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtrl2));
        if (warp <= 17) {
            // ======================================================== MMA issuers: warp 16 for query tile A, warp 17 for tile B
            // (whole warp, one elected lane issues).  One warp issuing for both tiles was the bottleneck of the first build of
            // this kernel: its serial chain of barrier polls (~250 clk each) and descriptor set-up took ~1900 clk per key tile
            // against 1024 clk of exponentials.  Each warp polls all barriers of an iteration up front (the predicates land
            // asynchronously) and only falls back to a blocking wait for the ones still open.
            const int X = warp - 16;
            const uint32_t idesc_s = (1u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
            // P.V: fp32 += bf16 x bf16 (B MN-major), or (I8) s32 = u8 x s8 (B MN-major)
            const uint32_t idesc_pv = (I8 ? (2u << 4) | (0u << 7) | (1u << 10) : (1u << 4) | (1u << 7) | (1u << 10)) | (1u << 16) |
                                      ((uint32_t)(prm.dvp >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
            const uint64_t q_desc = make_desc(smem_u32(sQ) + X * TM * KPAD, TM * 16, 128, 0);
            const uint64_t k_desc = make_desc(smem_u32(sK), TN * 16, 128, 0);
            const uint64_t v_desc = I8 ? make_desc(smem_u32(sV), kVBox8, 512, 4) : make_desc(smem_u32(sV), kVBox, 1024, 2);
            const uint32_t s_tmem = tmem + (I8 ? X * 256 : X * 128), o_tmem = I8 ? s_tmem + 128 : tmem + kColO2 + X * 128;
            // Issue order per key tile j: S(j), then P.V(j-1) once P(j-1) has arrived.  S(j) overwrites the stage that held
            // P(j-2), read by P.V(j-2) an iteration earlier (tcgen05.mma executes in issue order), and must not wait for P(j-1).
            // The barriers of an iteration are polled up front with test_wait (non-blocking; try_wait may sleep on an open
            // phase), blocking waits only for what is still open.  Variants measured and rejected (same box, 16384 x 64 /
            // 16384 x 128, ms): this order 1.30 / 1.51; "P.V(t), S(t+2)" with S two tiles ahead 1.45 / 1.72 -- every softmax
            // warp then finds its S ready, all sixteen run in lock-step and sit in their MUFU-free phases together.
            BA_DECLARE_PRED(ba_pk);
            BA_DECLARE_PRED(ba_pv);
            BA_DECLARE_PRED(ba_pp);
            Ring qr, kr, vr;
            uint32_t g = 0;   // key tiles of my query tile issued so far (S stage = g & 1); P.V runs one tile behind
            uint32_t up = 0;  // units of my query tile whose last P.V has been issued
            int pend = 0, pj = 0, pact = 0, pvs = 0;
            uint32_t pvph = 0;
            for (int u = ub0; u < prm.units; u += G) {
                const int ub = u % prm.ublocks;
                const int act = (X == 0 || ub * 2 * TM + TM < N) ? 1 : 0;  // tile B of a head's last unit may be empty: keep the rings moving
                mbar_wait(&sm->qfull[qr.stage], qr.phase);
                const uint64_t qd = q_desc + (uint64_t)((qr.stage * 2 * TM * KPAD) >> 4);
                for (int j = 0; j < T; ++j) {
                    const uint32_t pst = (g - 1) & 1u;  // stage of the pending tile (when there is one)
                    // the iteration's three barriers polled back to back (one ~170 clk round trip for all), looked at where needed
                    uint32_t k_ok, v_ok = 1, p_ok = 1;
                    MBAR_POLL(ba_pk, &sm->kfull[kr.stage], kr.phase);
                    if (pend) {
                        MBAR_POLL(ba_pv, &sm->vfull[pvs], pvph);
                        if (pact) MBAR_POLL(ba_pp, &sm->pfull[X][pst], ((g - 1) >> 1) & 1u);
                    }
                    MBAR_POLLED(ba_pk, k_ok);
                    if (!k_ok) mbar_wait(&sm->kfull[kr.stage], kr.phase);
                    BA_STAMP2();
                    if (act) {
                        tc_fence_after();
                        const uint64_t kd = k_desc + (uint64_t)((kr.stage * TN * KPAD) >> 4);
                        if (elect_one()) {
                            BA_STAMP3();
#pragma unroll
                            for (int ks = 0; ks < KPAD / 32; ++ks)
                                mma_f8(s_tmem + (g & 1u) * TN, qd + (uint64_t)(ks * ((2 * TM * 16) >> 4)),
                                       kd + (uint64_t)(ks * ((2 * TN * 16) >> 4)), idesc_s, ks > 0 ? 1u : 0u);
                            BA_STAMP3();
                            tc_commit(&sm->sfull[X][g & 1u]);
                            BA_STAMP3();
                            tc_commit(&sm->kfree[kr.stage]);
                            if (j == T - 1) tc_commit(&sm->qfree[qr.stage]);
                            BA_STAMP3();
                        }
                        __syncwarp();
                    } else if (lane == 0) {
                        mbar_arrive(&sm->kfree[kr.stage]);
                        if (j == T - 1) mbar_arrive(&sm->qfree[qr.stage]);
                    }
                    BA_STAMP2();
                    if (pend) {
                        MBAR_POLLED(ba_pv, v_ok);
                        if (!v_ok) mbar_wait(&sm->vfull[pvs], pvph);
                        if (pact) {
                            MBAR_POLLED(ba_pp, p_ok);
                            if (!p_ok) mbar_wait(&sm->pfull[X][pst], ((g - 1) >> 1) & 1u);
                            if (pj == 0 && up > 0) mbar_wait(&sm->ofree[X], (up - 1) & 1u);  // the epilogue has read the old O
                            BA_STAMP2();
                            tc_fence_after();
                            const uint64_t vd = v_desc + (uint64_t)((pvs * prm.nbox * prm.vbox) >> 4);
                            const uint32_t p_tmem = s_tmem + pst * TN;
                            if (elect_one()) {
                                if (I8) {  // two K = 32 steps; a fresh accumulator every tile; P8 of half h sits at column 32 h
#pragma unroll
                                    for (int ks = 0; ks < TN / 32; ++ks)
                                        mma_i8_ts(o_tmem, p_tmem + ks * 32, vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv, ks > 0 ? 1u : 0u);
                                } else {
#pragma unroll
                                    for (int ks = 0; ks < TN / 16; ++ks)
                                        mma_bf16_ts(o_tmem, p_tmem + (ks >> 1) * 32 + (ks & 1) * 8, vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv,
                                                    (pj > 0 || ks > 0) ? 1u : 0u);
                                }
                                tc_commit(&sm->pvdone[X][pst]);
                                tc_commit(&sm->vfree[pvs]);
                            }
                            __syncwarp();
                            BA_STAMP2();
                            if (pj == T - 1) ++up;
                        } else if (lane == 0) {
                            mbar_arrive(&sm->vfree[pvs]);
                        }
                    }
                    pend = 1;
                    pj = j;
                    pact = act;
                    pvs = vr.stage;
                    pvph = vr.phase;
                    vr.next(prm.vst);
                    kr.next(prm.kst);
                    if (act) ++g;
                }
                qr.next(prm.qst);
            }
            if (pend) {  // the last tile's P.V
                mbar_wait(&sm->vfull[pvs], pvph);
                if (pact) {
                    const uint32_t pst = (g - 1) & 1u;
                    mbar_wait(&sm->pfull[X][pst], ((g - 1) >> 1) & 1u);
                    if (pj == 0 && up > 0) mbar_wait(&sm->ofree[X], (up - 1) & 1u);
                    tc_fence_after();
                    const uint64_t vd = v_desc + (uint64_t)((pvs * prm.nbox * prm.vbox) >> 4);
                    const uint32_t p_tmem = s_tmem + pst * TN;
                    if (elect_one()) {
                        if (I8) {
#pragma unroll
                            for (int ks = 0; ks < TN / 32; ++ks)
                                mma_i8_ts(o_tmem, p_tmem + ks * 32, vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv, ks > 0 ? 1u : 0u);
                        } else {
#pragma unroll
                            for (int ks = 0; ks < TN / 16; ++ks)
                                mma_bf16_ts(o_tmem, p_tmem + (ks >> 1) * 32 + (ks & 1) * 8, vd + (uint64_t)(ks * (2048 >> 4)), idesc_pv,
                                            (pj > 0 || ks > 0) ? 1u : 0u);
                        }
                        tc_commit(&sm->pvdone[X][pst]);
                        tc_commit(&sm->vfree[pvs]);
                    }
                    __syncwarp();
                } else if (lane == 0) {
                    mbar_arrive(&sm->vfree[pvs]);
                }
            }
        } else if (warp == 18) {
            // ======================================================== TMA producer: bias tiles, V tiles
            if (lane == 0) {
                Ring vr, br, kr, qr;
                for (int u = ub0; u < prm.units; u += G) {
                    const int head = u / prm.ublocks;
                    const int ub = u - head * prm.ublocks;
                    const int nact = (ub * 2 * TM + TM < N) ? 2 : 1;
                    const int bh = (a.head0 + head) % a.H % a.bias_heads;
                    // the unit's two Q tiles, already expanded (expand_qk_kernel): one bulk copy
                    mbar_wait(&sm->qfree[qr.stage], qr.phase ^ 1u);
                    mbar_expect_tx(&sm->qfull[qr.stage], 2 * TM * KPAD);
                    bulk_load(sQ + qr.stage * 2 * TM * KPAD, a.q_exp + (int64_t)u * (2 * TM * KPAD), 2 * TM * KPAD, &sm->qfull[qr.stage]);
                    qr.next(prm.qst);
                    for (int j = 0; j < T; ++j) {
                        if (BIAS == 1) {
                            for (int X = 0; X < nact; ++X) {
                                mbar_wait(&sm->bfree[br.stage], br.phase ^ 1u);
                                mbar_expect_tx(&sm->bfull[br.stage], kBSub);
                                tma_load_3d(&bmap, &sm->bfull[br.stage], sB + br.stage * kBSub, j * TN, ub * 2 * TM + X * TM, bh);
                                br.next(prm.bst);
                            }
                        }
                        // K tile: 64 keys of e4m3 +-1.0 bytes, already in UMMA tile order (expand_k_kernel): one bulk copy
                        mbar_wait(&sm->kfree[kr.stage], kr.phase ^ 1u);
                        mbar_expect_tx(&sm->kfull[kr.stage], TN * KPAD);
                        bulk_load(sK + kr.stage * TN * KPAD, a.k_exp + ((int64_t)head * T + j) * (TN * KPAD), TN * KPAD, &sm->kfull[kr.stage]);
                        kr.next(prm.kst);
                        mbar_wait(&sm->vfree[vr.stage], vr.phase ^ 1u);
                        mbar_expect_tx(&sm->vfull[vr.stage], prm.nbox * prm.vbox);
                        for (int b = 0; b < prm.nbox; ++b)
                            tma_load_3d(&vmap, &sm->vfull[vr.stage], sV + (vr.stage * prm.nbox + b) * prm.vbox, (I8 ? prm.vcol0 : 0) + b * 64, j * TN, head);
                        vr.next(prm.vst);
                    }
                }
            }
        } else {
            // ======================================================== warp 19: Relative2dBias tables (BIAS 4); idle otherwise
            if (BIAS == 4) {
                Ring qr;
                int ui = 0;  // units of this CTA so far
                for (int u = ub0; u < prm.units; u += G, ++ui) {
                    const int head = u / prm.ublocks;
                    mbar_wait(&sm->qfree[qr.stage], qr.phase ^ 1u);
                    // tables of the unit's head (attention.hpp:22-26), published with the Q stage (qfull counts this warp too): the
                    // softmax warps read them after the first S of the unit (qfull -> MMA -> sfull orders the accesses).  Three
                    // slots: slot ui % 3 is rewritten for unit ui + 3, i.e. after every S MMA of unit ui + 1 has retired (qfree),
                    // by which time the softmax warps have long left unit ui (its last P precedes the next unit's third S).
                    const int len = 2 * prm.g - 1;
                    const int bh = (a.head0 + head) % a.H % a.bias_heads;
                    const char* tb = static_cast<const char*>(a.bias) + (size_t)bh * 2 * len * dtype_size(a.bias_dtype);
                    float* dst = &sm->rel2[ui % 3][0][0];
                    for (int i = lane; i < 2 * len; i += 32) dst[(i >= len ? 256 - len : 0) + i] = load_as_float(tb, a.bias_dtype, i);
                    warp_arrive(&sm->qfull[qr.stage], lane);
                    qr.next(prm.qst);
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax2));
        // ============================================================ softmax + epilogue: thread = (query row, 32 keys)
        const int X = warp >> 3, half = (warp >> 2) & 1, quad = warp & 3;
        const int r = quad * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const uint32_t s_base = keep_u32(lane_base + (I8 ? X * 256 : X * 128) + half * 32);  // + 64 * stage: my 32 S columns; P goes over the first 16 (I8: 8)
        // my row of a bias tile: 16-byte chunk (half*4 + c) ^ (r & 7) of row r = (this address) ^ (c << 4) (+ the stage offset;
        // the ring is 1024-byte aligned)
        const uint32_t b_thr = keep_u32(smem_u32(sB) + r * 128 + ((((uint32_t)half << 2) ^ (uint32_t)(r & 7)) << 4));
        const uint32_t fl_thr = keep_u32(smem_u32(&sm->flag[0][X][quad][0]));  // + (gx & 1) * sizeof(flag[0]); [half] = mine
        const uint32_t lane0 = keep_u32(lane == 0 ? 1u : 0u);
        const uint32_t o_addr = I8 ? lane_base + X * 256 + 128 : lane_base + kColO2 + X * 128;  // O (I8: the s32 accumulator; fp32 O at + 64)
        const int pair_id = 1 + X * 4 + quad;
        const int h16 = ((prm.dvp >> 1) + 15) & ~15;             // O columns [0,h16) belong to half 0, [h16,dvp) to half 1
        const int oc0 = half ? h16 : 0, oc1 = half ? prm.dvp : h16;
        const bool stats = a.row_max != nullptr || a.row_sum != nullptr;
        const int nlast = N - (T - 1) * TN;  // keys of the last tile (TN unless N is ragged)
        uint32_t gx = 0;  // key tiles this query tile has been through (stage = gx & 1, parity = (gx >> 1) & 1)
        int usm = -1;     // units of this CTA so far (slot of the BIAS 4 tables)
        // per-head scales are requested one unit ahead (a fresh global load costs this in-order thread ~700 clk per unit)
        float muq_n = 0.f, muk_n = 0.f;
        if (ub0 < prm.units) {
            muq_n = __ldg(a.mu_q + ub0 / prm.ublocks);
            muk_n = __ldg(a.mu_k + ub0 / prm.ublocks);
        }
        unsigned char* box = sO + warp * 2048;  // my warp's staging box (o_stage)
        uint32_t np = 0;  // tiles done in ping-pong with the other query tile
        Ring br;          // position of my query tile's next bias tile in the producer's ring
        if (BIAS == 1 && X == 1) br.next(prm.bst);
        for (int u = ub0; u < prm.units; u += G) {
            const int head = u / prm.ublocks;
            const int ub = u - head * prm.ublocks;
            const int nact = (ub * 2 * TM + TM < N) ? 2 : 1;
            ++usm;
            if (X >= nact) {  // tile B of the last unit of a head with an odd number of 128-row blocks: nothing to do
                if (BIAS == 1)
                    for (int j = 0; j < T; ++j) br.next(prm.bst);
                continue;
            }
            const bool pp = nact == 2 && BA_PP_AT >= 0;
            const int row = ub * 2 * TM + X * TM + r;
            const float sc = muq_n * muk_n * a.inv_tau;  // natural-log units per unit of dot
            if (u + G < prm.units) {
                muq_n = __ldg(a.mu_q + (u + G) / prm.ublocks);
                muk_n = __ldg(a.mu_k + (u + G) / prm.ublocks);
            }
            const float ea = (BIAS == 0) ? sc * kLog2e : kLog2e;  // BIAS 0 keeps x = raw dot and folds the scale into the exponent
            const bool fast = BIAS == 0 && !I8 && !stats && !DBG && sc * kLog2e * (float)d <= kFastBound;
            float m_ref = fast ? sc * kLog2e * (float)d : -INFINITY, m_true = -INFINITY;
            float l0 = 0.f, l1 = 0.f;
            const bool dump = DBG && prm.dbg_S && head == prm.dbg_head;
            // BIAS 4: my token's grid position and this unit's tables
            const int rg = BIAS == 4 ? row / prm.g : 0, cg = BIAS == 4 ? row - rg * prm.g : 0;
            const float* rowtab = &sm->rel2[usm % 3][0][0];
            const float* coltab = &sm->rel2[usm % 3][1][0];
            float x[32];
            float m_run = -INFINITY, rs_prev = 0.f;  // I8: running max (log2 units); rescale of the tile whose P.V is still to be folded into O
            for (int j = 0; j < T; ++j, ++gx) {
                const uint32_t st = gx & 1u, par = (gx >> 1) & 1u;
                const uint32_t s_addr = s_base + st * TN;
                BA_STAMP2();
                // (Requesting the next tile's scores before this tile's P is handed over -- the "rolling refill" of the first
                // kernel -- was tried here: no gain, and rare wrong rows under the run-to-run identity stress test that stayed
                // unexplained, so every tile waits for its own S.)
                mbar_wait(&sm->sfull[X][st], par);
                tc_fence_after();
                BA_TMEM_LD16(s_addr + 0, x, 0);
                BA_TMEM_LD16(s_addr + 16, x, 16);
                BA_STAMP2();
                if (BIAS == 1) mbar_wait(&sm->bfull[br.stage], br.phase);
                tc_wait_ld();
                BA_STAMP2();
                if (DBG && dump) {
                    int32_t* drow = prm.dbg_S + (int64_t)row * N + j * TN + half * 32;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (row < N && j * TN + half * 32 + i < N) drow[i] = (int)x[i];
                }
                if (BIAS == 1) {
                    const uint32_t brow = b_thr + br.stage * kBSub;  // row r of the 128 x 64 bf16 tile, my half's first chunk
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const uint4 b = lds_128(brow ^ (c << 4));
                        const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            fma2(x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], x[c * 8 + 2 * e], x[c * 8 + 2 * e + 1], sc, sc,
                                 __uint_as_float(bw[e] << 16), __uint_as_float(bw[e] & 0xFFFF0000u));
                    }
                    warp_arrive(&sm->bfree[br.stage], (int)(lane0 ^ 1u));
                    br.next(prm.bst);  // tile A and tile B alternate in the ring when both are active
                    if (nact == 2) br.next(prm.bst);
                }
                if (BIAS == 4) {
                    // b = row_offsets[ri - rj + g - 1] + col_offsets[ci - cj + g - 1] (attention.cpp:84-94).  g % 32 == 0, so my 32
                    // keys lie in one grid row: rj is one value, cj = cj0 + c.  fp32 sum first, then x = dot*sc + b, exactly what
                    // the dense path computes from the materialised table (bit-identical when the sums are bf16-representable).
                    const int kb = j * TN + half * 32;
                    const int rj = kb / prm.g, cj0 = kb - rj * prm.g;
                    const float rv = rowtab[rg - rj + prm.g - 1];
                    const float* cw = coltab + (cg - cj0 + prm.g - 1);  // element c reads cw[-c]: consecutive words across the warp
#pragma unroll
                    for (int c = 0; c < 32; ++c) x[c] = fmaf(x[c], sc, rv + cw[-c]);
                }
                if (RAGGED && j == T - 1) {  // ragged N (its own instantiation: the test and the masking loop cost the others 5-13%): keys at or past N get weight 0 (attention.cpp:285-287 stops the block there)
                    const int nk = nlast - half * 32;  // valid keys among my 32 columns
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i >= nk) x[i] = -INFINITY;
                }
                if (I8) {
                    // ---- block max, agreed between the two halves EVERY tile (attention.cpp:306-310)
                    float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
                    for (int i = 4; i < 32; i += 4) {
                        m0 = fmaxf(m0, x[i]);
                        m1 = fmaxf(m1, x[i + 1]);
                        m2 = fmaxf(m2, x[i + 2]);
                        m3 = fmaxf(m3, x[i + 3]);
                    }
                    const float hm = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * ea;
                    sm->xch8[gx & 1u][X][half][r] = hm;
                    pair_sync(pair_id);
                    const float m_new = fmaxf(m_run, fmaxf(hm, sm->xch8[gx & 1u][X][half ^ 1][r]));
                    const float rs = ex2(m_run - m_new);  // first block: 2^-inf = 0
                    // ---- fold the previous tile's integer P.V into the fp32 O: O = O * rescale(prev) + acc(prev)
                    if (j > 0) {
                        mbar_wait(&sm->pvdone[X][st ^ 1u], ((gx - 1) >> 1) & 1u);
                        tc_fence_after();
                        for (int c = oc0; c < oc1; c += 16) {
                            float acc[16], of[16];
                            BA_TMEM_LD16(o_addr + c, acc, 0);
                            if (j > 1) BA_TMEM_LD16(o_addr + 64 + c, of, 0);
                            tc_wait_ld();
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                of[i] = j > 1 ? fmaf(of[i], rs_prev, s32_to_float(acc[i])) : s32_to_float(acc[i]);
                            BA_TMEM_ST16(o_addr + 64 + c, of, 0);
                        }
                    }
                    rs_prev = rs;
                    m_run = m_new;
                    // ---- weights: P = 2^(x - m_new), l = l * rescale + sum P, P8 = round_half_away(255 P) (attention.cpp:312-337)
                    l0 *= rs;
                    l1 *= rs;
                    // round(255 P) without the conversion unit (it shares the 16-per-clock pipe with ex2): 255 P + 1.5 * 2^23 rounds
                    // to the nearest integer in the low mantissa bits.  Nearest-even there equals the reference's half-away
                    // rounding for every float P: a tie needs 255 P = k + 1/2, i.e. P = (2k+1)/510, which no binary float is.
                    uint32_t pk8[8];
                    const float nm8 = -m_new;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float a0, a1, a2, a3;
                        fma2(a0, a1, x[4 * e], x[4 * e + 1], ea, ea, nm8, nm8);
                        fma2(a2, a3, x[4 * e + 2], x[4 * e + 3], ea, ea, nm8, nm8);
                        const float p0 = ex2(a0), p1 = ex2(a1), p2 = ex2(a2), p3 = ex2(a3);
                        add2(l0, l1, p0, p1);
                        add2(l0, l1, p2, p3);
                        const uint32_t t0 = __float_as_uint(fmaf(p0, 255.0f, 12582912.0f)), t1 = __float_as_uint(fmaf(p1, 255.0f, 12582912.0f));
                        const uint32_t t2 = __float_as_uint(fmaf(p2, 255.0f, 12582912.0f)), t3 = __float_as_uint(fmaf(p3, 255.0f, 12582912.0f));
                        pk8[e] = __byte_perm(__byte_perm(t0, t1, 0x0040), __byte_perm(t2, t3, 0x0040), 0x5410);  // low bytes of t0..t3
                    }
                    BA_TMEM_ST8U(s_addr, pk8);
                    tc_wait_st();
                    tc_fence_before();
                    warp_arrive(&sm->pfull[X][st], (int)(lane0 ^ 1u));
                    continue;
                }
                if (!fast) {
                    float m0 = x[0], m1 = x[1], m2 = x[2], m3 = x[3];
#pragma unroll
                    for (int i = 4; i < 32; i += 4) {
                        m0 = fmaxf(m0, x[i]);
                        m1 = fmaxf(m1, x[i + 1]);
                        m2 = fmaxf(m2, x[i + 2]);
                        m3 = fmaxf(m3, x[i + 3]);
                    }
                    const float hm = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * ea;  // ea > 0: the max commutes with the scaling
                    const bool need = hm > m_ref + kThr2;
                    const uint32_t mine = (stats || __any_sync(0xffffffffu, need)) ? 1u : 0u;
                    const uint32_t fl = fl_thr + (gx & 1u) * (uint32_t)sizeof(sm->flag[0]);
                    if (lane0) sts_u32_volatile(fl + half * 4, mine);
                    pair_sync(pair_id);
                    if (mine | lds_u32_volatile(fl + (half ^ 1) * 4)) {  // rare after the first tile of a unit: agree on a new reference for the rows that need one
                        sm->xch[X][half][r] = hm;
                        pair_sync(pair_id);
                        const float tm = fmaxf(hm, sm->xch[X][half ^ 1][r]);
                        m_true = fmaxf(m_true, tm);
                        // (warp-uniform: the tcgen05.ld / st inside rescale_o are .sync.aligned -- rows that keep their reference
                        // multiply by 1)
                        const bool upd = tm > m_ref + kThr2;
                        if (__any_sync(0xffffffffu, upd)) {
                            const float alpha = upd ? ex2(m_ref - tm) : 1.0f;  // first tile: 2^-inf = 0 on a still-unwritten O
                            if (j > 0 && oc1 > oc0) {
                                // S(j) was issued BEFORE P.V(j-1): wait for that MMA before touching O.  Tile j-1 is this
                                // barrier's previous use and tile j-3 (the one before) retired before S(j) did, so the
                                // parity is unambiguous.
                                mbar_wait(&sm->pvdone[X][st ^ 1u], ((gx - 1) >> 1) & 1u);
                                rescale_o(o_addr + oc0, oc1 - oc0, alpha);
                            }
                            l0 *= alpha;
                            l1 *= alpha;
                            if (upd) m_ref = tm;
                        }
                    }
                }
                BA_STAMP2();
                // PING-PONG.  The four softmax warps of a scheduler share its MUFU pipe fairly, so warps that start a tile together
                // finish together and then all sit in their MUFU-free phases (hand-over, barrier and TMEM round trips, ~480 clk)
                // at the same time.  The two warps of tile A and the two of tile B on a scheduler therefore take turns: a pair
                // starts its exponentials when the other pair is three quarters through its own (two warps saturate the pipe,
                // pipe_bench.cu) and does everything else while the other pair owns the pipe.  One named barrier per lane quadrant
                // (ids 9..12, 128 threads): the pair that hands over does bar.arrive, the pair that takes over bar.sync; the
                // roles swap every phase.  (mbarriers cost ~200 clk per hand-over, as much as was to be gained.)
                if (pp && (X == 1 || np > 0)) asm volatile("bar.sync %0, 128;" ::"r"(9 + quad) : "memory");
                const float nm = -m_ref;
                uint32_t pk[16];
#if BA_EXP_LA > 0
                // exponentials issued BA_EXP_LA pairs ahead of their consumers (volatile: the order is the one written), in place
#pragma unroll
                for (int e = 0; e < 16; ++e) fma2(x[2 * e], x[2 * e + 1], x[2 * e], x[2 * e + 1], ea, ea, nm, nm);
#pragma unroll
                for (int e = 0; e < 16 + BA_EXP_LA; ++e) {
                    if (e < 16) {
                        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[2 * e]));
                        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[2 * e + 1]));
                    }
                    if (e >= BA_EXP_LA) {
                        const int c = e - BA_EXP_LA;
                        asm volatile("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rd, {%0, %1};\n\t"
                                     "add.rn.f32x2 rd, rd, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                                     : "+f"(l0), "+f"(l1)
                                     : "f"(x[2 * c]), "f"(x[2 * c + 1]));
                        pk[c] = pack_bf16(x[2 * c], x[2 * c + 1]);
                    }
                }
#else
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    float a0, a1;
                    fma2(a0, a1, x[2 * e], x[2 * e + 1], ea, ea, nm, nm);
                    const float p0 = ex2(a0), p1 = ex2(a1);
                    add2(l0, l1, p0, p1);
                    pk[e] = pack_bf16(p0, p1);
                    if (e == BA_PP_AT && pp) {
                        asm volatile("bar.arrive %0, 128;" ::"r"(9 + quad) : "memory");
                        ++np;
                    }
                }
#endif
                BA_TMEM_ST16U(s_addr, pk);
                BA_STAMP2();
                tc_wait_st();
                tc_fence_before();
                warp_arrive(&sm->pfull[X][st], (int)(lane0 ^ 1u));
            }
            // ---------------------------------------------------------------- epilogue: O / l for my half of the columns
            BA_STAMP4();
            mbar_wait(&sm->pvdone[X][(gx - 1) & 1u], ((gx - 1) >> 1) & 1u);
            BA_STAMP4();
            tc_fence_after();
            sm->xch[X][half][r] = l0 + l1;
            pair_sync(pair_id);
            const float l = (l0 + l1) + sm->xch[X][half ^ 1][r];
            BA_STAMP4();
            const float inv_l = I8 ? 1.0f / l / 255.0f : 1.0f / l;
            const int vc0 = I8 ? prm.vcol0 : 0, dcols = I8 ? prm.dsl : d;  // I8: this pass owns O columns [vc0, vc0 + dcols)
            float* orow = a.O + ((int64_t)head * N + row) * d + vc0;
            __nv_bfloat16* orow16 = reinterpret_cast<__nv_bfloat16*>(a.O) + ((int64_t)head * N + row) * d + vc0;  // (out_bf16)
            for (int c = oc0; c < oc1; c += 16) {
                float o[16], of[16];
                BA_TMEM_LD16(o_addr + c, o, 0);
                if (I8 && T > 1) BA_TMEM_LD16(o_addr + 64 + c, of, 0);
                if (prm.o_stage) {  // the box is free again once the TMA unit has READ the previous chunk out of it
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
                tc_wait_ld();
                if (I8) {  // O = (O * rescale(last) + acc(last)) / l / 255 * delta[c]  (attention.cpp:338-343, 361-363)
                    const double* dl = prm.vscales + (int64_t)head * d + vc0 + c;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float acc = s32_to_float(o[i]);
                        o[i] = (T > 1 ? fmaf(of[i], rs_prev, acc) : acc) * inv_l * (c + i < dcols ? (float)__ldg(dl + i) : 0.f);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] *= inv_l;
                }
                if (prm.o_stage) {
                    // Direct stores (32 lanes x 32 B to 32 different rows per instruction) keep the LSU busy for ~2000 clk per
                    // unit; a [32 rows][16 floats] box in shared memory (64B swizzle: 16-byte chunk q of row r sits at
                    // q ^ ((r >> 1) & 3)) goes out as ONE asynchronous TMA store, clipped at N and d by the hardware.
                    if (a.out_bf16) {  // [32 rows][16 bf16]: 32-byte rows, 32B swizzle (chunk q of row r sits at q ^ ((r >> 2) & 1))
#pragma unroll
                        for (int q = 0; q < 2; ++q)
                            *reinterpret_cast<uint4*>(box + lane * 32 + ((q ^ ((lane >> 2) & 1)) << 4)) =
                                make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                                           pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            *reinterpret_cast<float4*>(box + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
                                make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&omap, box, vc0 + c, row - lane, head);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else if (row < N) {
                    if (a.out_bf16) {
#pragma unroll
                        for (int q = 0; q < 2; ++q)
                            if (c + 8 * q + 8 <= dcols)
                                *reinterpret_cast<uint4*>(orow16 + c + 8 * q) =
                                    make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                                               pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
                    } else {
                        if (c + 8 <= dcols) stg_256(orow + c, o);
                        if (c + 16 <= dcols) stg_256(orow + c + 8, o + 8);
                    }
                }
            }
            BA_STAMP4();
            tc_fence_before();
            if (stats && half == 0 && row < N) {
                if (a.row_max) a.row_max[(int64_t)head * N + row] = (I8 ? m_run : m_true) * kLn2;
                if (a.row_sum) a.row_sum[(int64_t)head * N + row] = I8 ? l : l * ex2(m_ref - m_true);
            }
            warp_arrive(&sm->ofree[X], lane);
        }
        if (prm.o_stage && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory may be released
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 16) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// Sign planes -> e4m3 +-1.0 bytes in the order the S MMA reads them (K-major, no swizzle, 8 x 16 B core matrices), one launch
// for both operands (blockIdx.y = 0: K in 64-key tiles, 1: Q in 128-row tiles, two per 256-row unit):
// byte (row r, element kb) of tile t of a head lives at t*R*KPAD + (kb/16)*(R*16) + r*16 + kb%16 (R = 64 or 128); rows at or
// past N (ragged last tile / unit) and elements at or past d are 0.0.  One thread per 16-byte chunk; a warp writes 512
// consecutive bytes.  (Expanding in the attention kernel -- one or two warps, through a lookup table -- took longer per key
// tile than the tile's exponentials and ~5000 clk per unit for Q: it was what the kernel was really waiting for.)
template <int KPAD>
__global__ void __launch_bounds__(256) expand_qk_kernel(const uint64_t* __restrict__ q_words, const uint64_t* __restrict__ k_words,
                                                        unsigned char* __restrict__ q_out, unsigned char* __restrict__ k_out,
                                                        int64_t heads, int N, int ktiles, int qtiles, int w64, int d) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the attention kernel's prologue may start
    asm volatile("griddepcontrol.wait;" ::: "memory");               // K1's packed words are read from here on
    constexpr int C = KPAD / 16;
    const bool isq = blockIdx.y == 1;
    const int R = isq ? 128 : 64, sh = isq ? 7 : 6, tiles = isq ? qtiles : ktiles;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // = ((head * tiles + tile) * C + c) * R + r
    if (idx >= heads * tiles * C * R) return;
    const int r = (int)(idx & (R - 1));
    const int c = (int)((idx >> sh) % C);
    const int64_t ht = (idx >> sh) / C;  // head * tiles + tile
    const int64_t head = ht / tiles;
    const int row = (int)(ht - head * tiles) * R + r;
    const bool valid = row < N;
    const uint64_t* words = isq ? q_words : k_words;
    const uint64_t w = (valid && (c >> 2) < w64) ? __ldg(words + (head * N + row) * w64 + (c >> 2)) : 0ull;
    const uint32_t bits16 = (uint32_t)(w >> (16 * (c & 3))) & 0xFFFFu;
    const uint2 lo = (valid && 16 * c < d) ? expand_byte(bits16 & 0xFF) : make_uint2(0, 0);
    const uint2 hi = (valid && 16 * c + 8 < d) ? expand_byte(bits16 >> 8) : make_uint2(0, 0);
    reinterpret_cast<uint4*>(isq ? q_out : k_out)[idx] = make_uint4(lo.x, lo.y, hi.x, hi.y);
}

template <int KPAD>
static int launch_expand_qk(const FwdArgs& a, int ktiles, int ublocks, cudaStream_t stream) {
    const int64_t qchunks = (int64_t)a.BH * ublocks * 2 * (KPAD / 16) * 128;  // >= the K plane's chunk count
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((qchunks + 255) / 256), 2);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // launch latency hides behind K1 (which releases its
    attr[0].val.programmaticStreamSerializationAllowed = 1;           // dependents on entry); the data wait is in the kernel
    cfg.attrs = attr;
    cfg.numAttrs = env_long("BA_PDL", 1) ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, expand_qk_kernel<KPAD>, a.q_words, a.k_words, const_cast<unsigned char*>(a.q_exp),
                                             const_cast<unsigned char*>(a.k_exp), (int64_t)a.BH, a.N, ktiles, 2 * ublocks, a.W64, a.d);
    return e == cudaSuccess ? 1 : -(int)e;
}

constexpr size_t kSmemMax2 = 227 * 1024;

inline size_t smem_bytes2(const Params2& p, int kpad) {
    return (size_t)p.vst * p.nbox * p.vbox + (size_t)p.bst * kBSub + (size_t)p.qst * 2 * TM * kpad + (size_t)p.kst * TN * kpad +
           (size_t)p.o_stage * kOStage + sizeof(Smem2);
}

template <int KPAD, int BIAS, bool DBG, bool TL = false, bool RAGGED = false, bool I8 = false>
static int launch_variant2(const Params2& prm, const CUtensorMap& vmap, const CUtensorMap& bmap, const CUtensorMap& omap, cudaStream_t stream) {
    static bool configured[kMaxDevices] = {};
    const int dev = current_device();
    if (!configured[dev]) {
        const cudaError_t e = cudaFuncSetAttribute(attn_tc2_kernel<KPAD, BIAS, DBG, TL, RAGGED, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)kSmemMax2);
        if (e != cudaSuccess) return -(int)e;
        configured[dev] = true;
    }
    int grid = (int)std::min<long>(prm.units - prm.unit0, sm_count());
    if (env_long("BA_GRID", 0) > 0) grid = (int)std::min<long>(prm.units - prm.unit0, env_long("BA_GRID", 0));  // dev knob
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
    const cudaError_t e = cudaLaunchKernelEx(&cfg, attn_tc2_kernel<KPAD, BIAS, DBG, TL, RAGGED, I8>, prm, vmap, bmap, omap);
    return e == cudaSuccess ? 1 : -(int)e;
}

template <int KPAD>
static int launch_main2(const Params2& prm, int bias_mode, const CUtensorMap& vmap, const CUtensorMap& bmap, const CUtensorMap& omap, cudaStream_t stream);

template <int KPAD>
static int launch_kpad2(const Params2& prm, int bias_mode, const CUtensorMap& vmap, const CUtensorMap& bmap, const CUtensorMap& omap, cudaStream_t stream) {
    const int ne = launch_expand_qk<KPAD>(prm.a, prm.tiles, prm.ublocks, stream);
    if (ne < 0) return ne;
    const int nk = launch_main2<KPAD>(prm, bias_mode, vmap, bmap, omap, stream);
    return nk < 0 ? nk : ne + nk;
}

template <int KPAD>
static int launch_main2(const Params2& prm, int bias_mode, const CUtensorMap& vmap, const CUtensorMap& bmap, const CUtensorMap& omap, cudaStream_t stream) {
    if (prm.dbg_T && bias_mode == 0 && (KPAD == 64 || KPAD == 128)) {
        if (prm.a.N % TN != 0 && KPAD == 64) return launch_variant2<KPAD, 0, false, true, true>(prm, vmap, bmap, omap, stream);
        return launch_variant2<KPAD, 0, false, true>(prm, vmap, bmap, omap, stream);
    }
#ifdef BA_DEV_TL_BIAS  // dev builds only: clock64 timeline of the dense-bias variant (scripts/timeline_tc2.py)
    if (prm.dbg_T && bias_mode == 1 && KPAD == 128 && prm.a.N % TN == 0) return launch_variant2<KPAD, 1, false, true>(prm, vmap, bmap, omap, stream);
#endif
    if (prm.dbg_S && bias_mode == 0) return launch_variant2<KPAD, 0, true>(prm, vmap, bmap, omap, stream);
    if (bias_mode == 4) return launch_variant2<KPAD, 4, false>(prm, vmap, bmap, omap, stream);
    if (prm.a.N % TN != 0) {
        if (bias_mode == 1) return launch_variant2<KPAD, 1, false, false, true>(prm, vmap, bmap, omap, stream);
        return launch_variant2<KPAD, 0, false, false, true>(prm, vmap, bmap, omap, stream);
    }
    if (bias_mode == 1) return launch_variant2<KPAD, 1, false>(prm, vmap, bmap, omap, stream);
    return launch_variant2<KPAD, 0, false>(prm, vmap, bmap, omap, stream);
}

// I8 mode (quantize_pv = true on the tensor cores): bias none or the dense bf16 TMA table; one launch per 64-column slice of V
// (prm.vcol0 / prm.dsl), the plane expansion before the first one only.
template <int KPAD>
static int launch_i8(const Params2& prm, int bias_mode, const CUtensorMap& vmap, const CUtensorMap& bmap, const CUtensorMap& omap, cudaStream_t stream) {
    const int ne = prm.vcol0 == 0 ? launch_expand_qk<KPAD>(prm.a, prm.tiles, prm.ublocks, stream) : 0;
    if (ne < 0) return ne;
    int nk;
    if (prm.a.N % TN != 0)
        nk = bias_mode == 1 ? launch_variant2<KPAD, 1, false, false, true, true>(prm, vmap, bmap, omap, stream)
                            : launch_variant2<KPAD, 0, false, false, true, true>(prm, vmap, bmap, omap, stream);
    else
        nk = bias_mode == 1 ? launch_variant2<KPAD, 1, false, false, false, true>(prm, vmap, bmap, omap, stream)
                            : launch_variant2<KPAD, 0, false, false, false, true>(prm, vmap, bmap, omap, stream);
    return nk < 0 ? nk : ne + nk;
}

}  // namespace tc2
}  // namespace ba
