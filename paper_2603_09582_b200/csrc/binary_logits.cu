// binary_logits.cu -- K3: integer logits of one head, S[i,j] = d - 2*popc(q_i xor k_j).
//
// Verification kernel for binattn::binary_gemm (proj/src/bitops.cpp:96-131) / xnor_popcount_dot
// (bitops.cpp:59-67).  With canonical rows (pad bits zero in both operands, tensor.hpp:56) the
// reference's 2*popc(~(a^b) & tailmask) - d equals d - 2*popc(a^b) bit for bit.
// The fused kernels never materialise S; this exists so tests can compare int32 logits exactly.
#include "ba_common.cuh"

namespace ba {

constexpr int kLgTile = 32;

__global__ void __launch_bounds__(kLgTile* kLgTile) binary_logits_kernel(const uint64_t* __restrict__ qw,
                                                                         const uint64_t* __restrict__ kw, int N, int d,
                                                                         int w64, int32_t* __restrict__ S) {
    extern __shared__ uint64_t sm[];  // [2][kLgTile][w64]
    uint64_t* sq = sm;
    uint64_t* sk = sm + kLgTile * w64;
    const int i0 = blockIdx.y * kLgTile, j0 = blockIdx.x * kLgTile;
    const int tid = threadIdx.y * kLgTile + threadIdx.x;
    for (int t = tid; t < kLgTile * w64; t += kLgTile * kLgTile) {
        const int r = t / w64, w = t - r * w64;
        sq[t] = (i0 + r < N) ? qw[(int64_t)(i0 + r) * w64 + w] : 0ull;
        sk[t] = (j0 + r < N) ? kw[(int64_t)(j0 + r) * w64 + w] : 0ull;
    }
    __syncthreads();
    const int i = i0 + threadIdx.y, j = j0 + threadIdx.x;
    if (i >= N || j >= N) return;
    int diff = 0;
    for (int w = 0; w < w64; ++w) diff += __popcll(sq[threadIdx.y * w64 + w] ^ sk[threadIdx.x * w64 + w]);
    S[(int64_t)i * N + j] = d - 2 * diff;
}

int launch_binary_logits(const uint64_t* qw, const uint64_t* kw, int N, int d, int32_t* S, cudaStream_t stream) {
    const int w64 = (d + 63) / 64;
    const dim3 grid((N + kLgTile - 1) / kLgTile, (N + kLgTile - 1) / kLgTile);
    const dim3 block(kLgTile, kLgTile);
    const size_t smem = 2ull * kLgTile * w64 * sizeof(uint64_t);
    binary_logits_kernel<<<grid, block, smem, stream>>>(qw, kw, N, d, w64, S);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ba
