// pack_signs.cu -- K1: sign-pack + per-head mean-abs for Q and K (sm_100a).
//
// Replaces binattn::binary_quantize = mean|x| + pack_signs
//   (proj/src/quantize.cpp:16-23, proj/src/bitops.cpp:37-49; layout contract proj/include/binattn/tensor.hpp:57-94):
//   bit c of row i = 1 iff x[i,c] >= 0 (so +0 and -0 map to +1), LSB-first in u64 words, pad bits zero,
//   mu = sum|x| / (N*d) per head.
//
// HBM-bound streaming kernel: each lane owns one 16-byte vector (8 bf16 / 4 fp32) of a row, builds its
// 8 (4) sign bits locally, and an 8- (16-) lane shuffle butterfly ORs them into one u64 output word, so
// every global read is a coalesced 16-byte vector and every write a coalesced 8-byte word.  Rows are padded
// to whole u64 groups in the LANE mapping only (d=72 -> 9 active + 7 idle lanes per row), never in memory.
// The per-head |x| sum is reduced block-wide in a fixed order; the last CTA of a head (ticket counter)
// folds the per-CTA partials in index order, so mu is bit-reproducible run to run.
#include "ba_common.cuh"

namespace ba {

constexpr int kPackThreads = 128;  // (256 was 11% slower at N=197: the per-thread prologue / block-sum cost is amortised over twice the vectors)
constexpr int kPackRowsPerCta = 256;
constexpr int kPackUnroll = 16;

struct PackJob {
    const void* X;
    uint64_t* words;
    float* mu;         // [heads] or nullptr
    float* partials;   // [heads, chunks]
    unsigned int* tickets;  // [heads], zero on entry, zero on exit
};

struct PackJobs {
    PackJob job[2];
};

__device__ __forceinline__ uint4 ldg_nc_16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <typename T>
struct Vec16;

template <>
struct Vec16<__nv_bfloat16> {
    static constexpr int kElems = 8;
    static constexpr bool kIsBf16 = true;
    __device__ static void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(r[i] << 16);
            f[2 * i + 1] = __uint_as_float(r[i] & 0xFFFF0000u);
        }
    }
};

// bf16 fast path: 8 sign bits and sum |x| of one 16-byte vector without per-element compares.
// A bf16 is negative-and-nonzero (bit = 0) iff its sign bit is set and its magnitude bits are not all zero; for a pair
// packed in a u32, (mag + 0x7FFF7FFF) sets bit 15 / 31 exactly when that half's magnitude is nonzero (no carry crosses
// the halves because mag <= 0x7FFF), so neg = w & (mag + 0x7FFF7FFF) & 0x80008000.  -0.0 therefore maps to +1 like the
// reference's `x >= 0` (bitops.cpp:45).
__device__ __forceinline__ void bf16x8_signs_abs(const uint4& v, unsigned int& bits, float& sum_abs) {
    const uint32_t r[4] = {v.x, v.y, v.z, v.w};
    uint32_t neg[4];
    float sa = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t mag = r[i] & 0x7FFF7FFFu;
        // "negative and non-zero", or NaN of either sign (x >= 0.0 is false for NaN, bitops.cpp:45): a half is NaN when its
        // magnitude exceeds 0x7F80, i.e. when mag + 0x007F carries into bit 15 / 31 (mag <= 0x7FFF: no carry leaves the half)
        neg[i] = ((r[i] & (mag + 0x7FFF7FFFu)) | (mag + 0x007F007Fu)) & 0x80008000u;
        sa += __uint_as_float(mag << 16);          // |even element|
        sa += __uint_as_float(mag & 0xFFFF0000u);  // |odd element|
    }
    // bytes 1 and 3 of every word carry the flags in their top bit: gather the 8 flag bytes, then the 8 bits
    const uint32_t lo = __byte_perm(neg[0], neg[1], 0x7531);  // elements 0..3 -> bytes 0..3
    const uint32_t hi = __byte_perm(neg[2], neg[3], 0x7531);  // elements 4..7
    const uint32_t nlo = ((lo >> 7) * 0x01020408u) >> 24;     // bit k = flag of byte k (flags are the only bits set)
    const uint32_t nhi = ((hi >> 7) * 0x01020408u) >> 24;
    bits = ~(nlo | (nhi << 4)) & 0xFFu;
    sum_abs = sa;
}

template <>
struct Vec16<__half> {
    static constexpr int kElems = 8;
    static constexpr bool kIsBf16 = false;
    __device__ static void unpack(const uint4& v, float (&f)[8]) {
        const uint32_t r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __half2 h = *reinterpret_cast<const __half2*>(&r[i]);
            const float2 p = __half22float2(h);
            f[2 * i] = p.x;
            f[2 * i + 1] = p.y;
        }
    }
};

template <>
struct Vec16<float> {
    static constexpr int kElems = 4;
    static constexpr bool kIsBf16 = false;
    __device__ static void unpack(const uint4& v, float (&f)[4]) {
        f[0] = __uint_as_float(v.x);
        f[1] = __uint_as_float(v.y);
        f[2] = __uint_as_float(v.z);
        f[3] = __uint_as_float(v.w);
    }
};

// Block-wide sum in a fixed order (warp butterfly, then warp 0 over the warp partials); then the
// last-arriving CTA of the head folds all per-CTA partials in chunk order.
__device__ __forceinline__ void finish_head_sum(float acc, const PackJob& job, int head, int chunk, int chunks,
                                               double inv_count) {
    __shared__ float warp_sums[kPackThreads / 32];
    __shared__ int is_last;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_sums[warp] = acc;
    __syncthreads();
    if (chunks == 1) {  // the CTA saw the whole head: no cross-CTA fold, no fence, no ticket
        if (threadIdx.x == 0 && job.mu) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kPackThreads / 32; ++w) s += warp_sums[w];
            job.mu[head] = (float)((double)s * inv_count);
        }
        return;
    }
    if (threadIdx.x == 0) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kPackThreads / 32; ++w) s += warp_sums[w];
        job.partials[(int64_t)head * chunks + chunk] = s;
        __threadfence();
        const unsigned int t = atomicAdd(&job.tickets[head], 1u);
        is_last = (t == (unsigned int)(chunks - 1));
    }
    __syncthreads();
    if (is_last && warp == 0) {
        __threadfence();
        double s = 0.0;
        for (int c = lane; c < chunks; c += 32) s += (double)__ldcg(&job.partials[(int64_t)head * chunks + c]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) {
            if (job.mu) job.mu[head] = (float)(s * inv_count);
            job.tickets[head] = 0u;  // self-cleaning for the next call
        }
    }
}

// Fast path: (d * sizeof(T)) % 16 == 0 and X 16-byte aligned.
template <typename T>
__global__ void __launch_bounds__(kPackThreads) pack_signs_vec_kernel(const __grid_constant__ PackJobs jobs, int N, int d, int chunks) {
    asm volatile("griddepcontrol.launch_dependents;");  // see pack_signs_bf16_kernel
    constexpr int EPV = Vec16<T>::kElems;  // elements per 16-byte vector
    constexpr int LPG = 64 / EPV;          // lanes per u64 output word
    constexpr int HALF = LPG / 2;          // lanes per 32-bit half
    const PackJob& job = jobs.job[blockIdx.z];
    const int head = blockIdx.x, chunk = blockIdx.y;
    const int vpr = d / EPV;                      // vectors per row
    const int vprp = (vpr + LPG - 1) / LPG * LPG;  // lane slots per row (whole u64 groups)
    const int w64 = vprp / LPG;
    const int row0 = chunk * kPackRowsPerCta;
    const int rows = min(kPackRowsPerCta, N - row0);
    const int slots = rows * vprp;
    const int g = threadIdx.x % LPG;  // lane position inside its u64 group (invariant over the loop)
    const char* xbase = static_cast<const char*>(job.X) + ((int64_t)head * N + row0) * d * (int64_t)sizeof(T);
    uint64_t* wbase = job.words + ((int64_t)head * N + row0) * w64;

    // Lane slot s = pass * kPackThreads + tid  ->  (row, vector-in-row).  When the slots per row divide the CTA size
    // (d = 64, 72, 128, 256 ...: vprp is 8, 16 or 32) the vector index is the same in every pass and the row advances by
    // a constant, so the loop carries no division; other head dims take the general mapping.  (ncu on the first
    // version: 137 instructions per 16-byte vector, ALU pipe 75% busy -- index arithmetic, not HBM, was the limit.)
    const bool regular = (kPackThreads % vprp) == 0;
    const int vs_fix = threadIdx.x % vprp, row_fix = threadIdx.x / vprp, row_step = kPackThreads / vprp;
    const bool lane_act = vs_fix < vpr;
    float acc = 0.f;
    for (int s0 = 0; s0 < slots; s0 += kPackThreads * kPackUnroll) {
        uint4 v[kPackUnroll];
        int rowl[kPackUnroll], vs[kPackUnroll];
        bool act[kPackUnroll];
        const int pass0 = s0 / kPackThreads;
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
            if (regular) {
                rowl[u] = (pass0 + u) * row_step + row_fix;
                vs[u] = vs_fix;
                act[u] = lane_act && rowl[u] < rows;
            } else {
                const int s = s0 + u * kPackThreads + threadIdx.x;
                rowl[u] = s / vprp;
                vs[u] = s - rowl[u] * vprp;
                act[u] = (s < slots) && (vs[u] < vpr);
            }
            v[u] = make_uint4(0, 0, 0, 0);
            if (act[u]) v[u] = ldg_nc_16(xbase + (uint32_t)(rowl[u] * vpr + vs[u]) * 16u);
        }
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
            if (s0 + u * kPackThreads >= slots) break;  // block-uniform
            unsigned int m = 0;
            float sa = 0.f;
            if (sizeof(T) == 2 && Vec16<T>::kIsBf16) {
                bf16x8_signs_abs(v[u], m, sa);
            } else {
                float f[EPV];
                Vec16<T>::unpack(v[u], f);
#pragma unroll
                for (int e = 0; e < EPV; ++e) {
                    m |= (f[e] >= 0.0f ? 1u : 0u) << e;  // -0.0f >= 0 is true, NaN is false: the reference's rule
                    sa += fabsf(f[e]);
                }
            }
            if (!act[u]) m = 0;
            acc += sa;
            unsigned int w = m << (EPV * (g % HALF));
#pragma unroll
            for (int off = 1; off < HALF; off <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, off);
            const unsigned int hi = __shfl_down_sync(0xffffffffu, w, HALF);
            if (g == 0 && rowl[u] < rows) wbase[(uint32_t)(rowl[u] * w64 + vs[u] / LPG)] = ((uint64_t)hi << 32) | (uint64_t)w;
        }
    }
    finish_head_sum(acc, job, head, chunk, chunks, 1.0 / ((double)N * (double)d));
}

// bf16 fast path for the head dims that matter (d = 64: VPRP = 8 lane slots per row; 64 < d <= 128: VPRP = 16): the
// slot -> (row, vector) mapping is shifts and masks on compile-time constants, the loads are predicated instead of
// branched, and the word assembly uses the same butterfly.  ncu on the general kernel (C2): 106 instructions per
// 16-byte vector and 82% of the issue slots busy -- instruction issue, not HBM, was the limit.
__device__ __forceinline__ uint4 ldg_nc_16_pred(const void* p, bool pred) {
    uint4 r = make_uint4(0, 0, 0, 0);
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
        : "l"(p), "r"((int)pred));
    return r;
}

template <int VPRP>
__global__ void __launch_bounds__(kPackThreads) pack_signs_bf16_kernel(const __grid_constant__ PackJobs jobs, int N, int d, int chunks) {
    asm volatile("griddepcontrol.launch_dependents;");   // K2's CTAs may start their prologue as this grid drains (PDL)
    constexpr int W64 = VPRP / 8;                        // u64 words per row (one lane slot = 8 bf16 = one byte of signs)
    constexpr int ROWS_PER_PASS = kPackThreads / VPRP;   // rows one pass of the CTA covers
    const PackJob& job = jobs.job[blockIdx.z];
    const int head = blockIdx.x, chunk = blockIdx.y;
    const int vpr = d >> 3;                              // real vectors per row (<= VPRP)
    const int row0 = chunk * kPackRowsPerCta;
    const int rows = min(kPackRowsPerCta, N - row0);
    const int vs = threadIdx.x & (VPRP - 1), rbase = threadIdx.x / VPRP;
    const bool lane_act = vs < vpr;
    const char* xbase = static_cast<const char*>(job.X) + ((int64_t)head * N + row0) * d * 2 + (rbase * vpr + vs) * 16;
    unsigned char* wbytes = reinterpret_cast<unsigned char*>(job.words + ((int64_t)head * N + row0) * W64) + rbase * VPRP + vs;
    const int row_bytes = ROWS_PER_PASS * vpr * 16;      // byte stride between a lane's vectors of consecutive passes
    constexpr int PASSES = kPackRowsPerCta / ROWS_PER_PASS;  // 16 (VPRP 8) or 32 (VPRP 16); kPackUnroll of them are in flight at once
    // |x| is summed by the tensor core: the four words of magnitudes are the A fragment of an m16n8k16 bf16 MMA against a
    // B of ones, fp32 accumulate.  Which matrix position a value lands in does not matter -- every column of D holds the
    // row sums, so the sum of all D entries is 8x the sum of all inputs -- and one HMMA replaces 8 FADD + 8 unpack ops
    // per 16-byte vector in a kernel that is bound by instruction issue.  (bf16 x 1.0 products are exact; the fp32
    // accumulation is deterministic on a given GPU.)
    float dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int p0 = 0; p0 < PASSES; p0 += kPackUnroll) {
        if (p0 * ROWS_PER_PASS >= rows) break;           // block-uniform
        uint4 v[kPackUnroll];
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u)
            v[u] = ldg_nc_16_pred(xbase + (p0 + u) * row_bytes, lane_act && (p0 + u) * ROWS_PER_PASS + rbase < rows);
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
            if ((p0 + u) * ROWS_PER_PASS >= rows) break;  // block-uniform: passes past the last row do no work
            const uint32_t r[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
            uint32_t neg[4], mag[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                mag[i] = r[i] & 0x7FFF7FFFu;
                neg[i] = ((r[i] & (mag[i] + 0x7FFF7FFFu)) | (mag[i] + 0x007F007Fu)) & 0x80008000u;  // negative and non-zero, or NaN (see bf16x8_signs_abs)
            }
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%8}, {%0,%1,%2,%3};"
                : "+f"(dacc[0]), "+f"(dacc[1]), "+f"(dacc[2]), "+f"(dacc[3])
                : "r"(mag[0]), "r"(mag[1]), "r"(mag[2]), "r"(mag[3]), "r"(0x3F803F80u));
            const uint32_t lo = __byte_perm(neg[0], neg[1], 0x7531), hi = __byte_perm(neg[2], neg[3], 0x7531);
            const uint32_t nbits = (((lo >> 7) * 0x01020408u) >> 24) | ((((hi >> 7) * 0x01020408u) >> 24) << 4);
            // every lane slot owns one BYTE of the packed row (bits 8*vs .. 8*vs+7 of the little-endian u64 words): a warp
            // writes 32 consecutive bytes with one store, no shuffles.  Idle slots (pad) and predicated-off lanes, whose
            // zero vector would read as +0.0 -> bit 1, write zero: pad bits must be zero (tensor.hpp:57-94)
            const bool in_rows = (p0 + u) * ROWS_PER_PASS + rbase < rows;
            if (in_rows) wbytes[(p0 + u) * ROWS_PER_PASS * VPRP] = lane_act ? (unsigned char)(~nbits & 0xFFu) : (unsigned char)0;
        }
    }
    finish_head_sum(((dacc[0] + dacc[1]) + (dacc[2] + dacc[3])) * 0.125f, job, head, chunk, chunks, 1.0 / ((double)N * (double)d));
}

// bf16 rows whose vector count is not a power of two (VPR 16-byte vectors per row, 8 < VPR < 16: d = 72 has 9): the lane-slot
// mapping of pack_signs_bf16_kernel<16> leaves 7 of every 16 lanes idle there (K1 at 0.41-0.49 of HBM on the d = 72 configs).
// A chunk of rows is a CONTIGUOUS array of vectors, so here lane slot i simply loads vector i of the chunk; (row, vector) =
// (i / VPR, i % VPR) with a compile-time divisor.  Every lane owns one byte of the packed row; the lane of vector 8 writes
// bytes 8..15 of the row as one u64 (its byte, then the zero pad bits -- tensor.hpp:57-94).
template <int VPR>
__global__ void __launch_bounds__(kPackThreads) pack_signs_bf16_odd_kernel(const __grid_constant__ PackJobs jobs, int N, int d, int chunks) {
    static_assert(VPR == 9, "the pad store below assumes the last vector of a row sits at byte 8");
    asm volatile("griddepcontrol.launch_dependents;");   // see pack_signs_bf16_kernel
    constexpr int kU = 9;                                // loads in flight per lane; 2 x 9 x 128 slots = 256 rows x 9 vectors
    const PackJob& job = jobs.job[blockIdx.z];
    const int head = blockIdx.x, chunk = blockIdx.y;
    const int row0 = chunk * kPackRowsPerCta;
    const int rows = min(kPackRowsPerCta, N - row0);
    const int slots = rows * VPR;
    const char* xbase = static_cast<const char*>(job.X) + ((int64_t)head * N + row0) * d * 2;
    unsigned char* wbytes = reinterpret_cast<unsigned char*>(job.words + ((int64_t)head * N + row0) * 2);
    float dacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int p0 = 0; p0 < 2; ++p0) {
        if (p0 * kU * kPackThreads >= slots) break;      // block-uniform
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = (p0 * kU + u) * kPackThreads + threadIdx.x;
            v[u] = ldg_nc_16_pred(xbase + (uint32_t)i * 16u, i < slots);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = (p0 * kU + u) * kPackThreads + threadIdx.x;
            if ((p0 * kU + u) * kPackThreads >= slots) break;  // block-uniform
            const uint32_t r[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
            uint32_t neg[4], mag[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                mag[k] = r[k] & 0x7FFF7FFFu;
                neg[k] = ((r[k] & (mag[k] + 0x7FFF7FFFu)) | (mag[k] + 0x007F007Fu)) & 0x80008000u;  // see bf16x8_signs_abs
            }
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%8}, {%0,%1,%2,%3};"
                : "+f"(dacc[0]), "+f"(dacc[1]), "+f"(dacc[2]), "+f"(dacc[3])
                : "r"(mag[0]), "r"(mag[1]), "r"(mag[2]), "r"(mag[3]), "r"(0x3F803F80u));
            const uint32_t lo = __byte_perm(neg[0], neg[1], 0x7531), hi = __byte_perm(neg[2], neg[3], 0x7531);
            const uint32_t nbits = (((lo >> 7) * 0x01020408u) >> 24) | ((((hi >> 7) * 0x01020408u) >> 24) << 4);
            const uint32_t byte = ~nbits & 0xFFu;
            if (i < slots) {
                const int row = i / VPR, vs = i - row * VPR;
                if (vs == 8) *reinterpret_cast<uint64_t*>(wbytes + row * 16 + 8) = (uint64_t)byte;
                else wbytes[row * 16 + vs] = (unsigned char)byte;
            }
        }
    }
    finish_head_sum(((dacc[0] + dacc[1]) + (dacc[2] + dacc[3])) * 0.125f, job, head, chunk, chunks, 1.0 / ((double)N * (double)d));
}

// Generic path: any d, any alignment; one thread per (row, u64 word), scalar loads.
__global__ void __launch_bounds__(kPackThreads) pack_signs_generic_kernel(const __grid_constant__ PackJobs jobs, int N, int d, int dtype,
                                                                          int chunks) {
    asm volatile("griddepcontrol.launch_dependents;");  // see pack_signs_bf16_kernel
    const PackJob& job = jobs.job[blockIdx.z];
    const int head = blockIdx.x, chunk = blockIdx.y;
    const int w64 = (d + 63) / 64;
    const int row0 = chunk * kPackRowsPerCta;
    const int rows = min(kPackRowsPerCta, N - row0);
    float acc = 0.f;
    for (int s = threadIdx.x; s < rows * w64; s += kPackThreads) {
        const int rowl = s / w64, w = s - rowl * w64;
        const int64_t base = ((int64_t)head * N + row0 + rowl) * d;
        uint64_t bits = 0;
        const int c1 = min(d, (w + 1) * 64);
        for (int c = w * 64; c < c1; ++c) {
            const float x = load_as_float(job.X, dtype, base + c);
            if (x >= 0.0f) bits |= 1ull << (c & 63);
            acc += fabsf(x);
        }
        job.words[((int64_t)head * N + row0 + rowl) * w64 + w] = bits;
    }
    finish_head_sum(acc, job, head, chunk, chunks, 1.0 / ((double)N * (double)d));
}

int pack_partials_per_head(int N, int, int) { return (N + kPackRowsPerCta - 1) / kPackRowsPerCta; }

// Packs one matrix (words/mu) or, when X2 != nullptr via launch_pack_signs2, Q and K in one launch.
static int launch_pack_jobs(const PackJobs& jobs, int njobs, int in_dtype, int64_t heads, int N, int d,
                            cudaStream_t stream) {
    const int chunks = pack_partials_per_head(N, d, in_dtype);
    const dim3 grid((unsigned)heads, chunks, njobs);
    const int esz = dtype_size(in_dtype);
    bool vec = (d * esz) % 16 == 0;
    for (int j = 0; j < njobs; ++j) vec = vec && (reinterpret_cast<uintptr_t>(jobs.job[j].X) % 16 == 0);
    if (vec && in_dtype == BA_BF16 && d == 64)
        pack_signs_bf16_kernel<8><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else if (vec && in_dtype == BA_BF16 && d == 72 && !getenv("BA_PACK_NO_D72"))
        pack_signs_bf16_odd_kernel<9><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else if (vec && in_dtype == BA_BF16 && d > 64 && d <= 128)
        pack_signs_bf16_kernel<16><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else if (vec && in_dtype == BA_BF16)
        pack_signs_vec_kernel<__nv_bfloat16><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else if (vec && in_dtype == BA_F16)
        pack_signs_vec_kernel<__half><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else if (vec && in_dtype == BA_F32)
        pack_signs_vec_kernel<float><<<grid, kPackThreads, 0, stream>>>(jobs, N, d, chunks);
    else
        pack_signs_generic_kernel<<<grid, kPackThreads, 0, stream>>>(jobs, N, d, in_dtype, chunks);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

int launch_pack_signs(const void* X, int in_dtype, int64_t heads, int N, int d, uint64_t* words, float* mu,
                      float* partials, unsigned int* tickets, cudaStream_t stream) {
    PackJobs jobs{};
    jobs.job[0] = PackJob{X, words, mu, partials, tickets};
    return launch_pack_jobs(jobs, 1, in_dtype, heads, N, d, stream);
}

int launch_pack_signs_qk(const void* Q, const void* K, int in_dtype, int64_t heads, int N, int d, uint64_t* q_words,
                         uint64_t* k_words, float* mu_q, float* mu_k, float* partials, unsigned int* tickets,
                         cudaStream_t stream) {
    const int chunks = pack_partials_per_head(N, d, in_dtype);
    PackJobs jobs{};
    jobs.job[0] = PackJob{Q, q_words, mu_q, partials, tickets};
    jobs.job[1] = PackJob{K, k_words, mu_k, partials + heads * chunks, tickets + heads};
    return launch_pack_jobs(jobs, 2, in_dtype, heads, N, d, stream);
}

}  // namespace ba
