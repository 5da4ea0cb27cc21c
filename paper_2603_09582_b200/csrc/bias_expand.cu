// bias_expand.cu -- Relative2dBias -> dense table on the device (materialize_bias, proj/src/attention.cpp:78-96), for the
// shapes whose kernel does not generate the bias itself: table[h][i][j] = row[h][ri - rj + g - 1] + col[h][ci - cj + g - 1]
// with (ri, ci) = (i / g, i % g), tokens on a g x g grid.  fp32 sums of the (bf16 or fp32) offsets.
#include "ba_common.cuh"

namespace ba {

__global__ void __launch_bounds__(256) expand_rel2d_kernel(const void* __restrict__ tables, int dtype, int N, int g,
                                                           float* __restrict__ out) {
    const int h = blockIdx.z, i = blockIdx.y;
    const int len = 2 * g - 1;
    const char* row = static_cast<const char*>(tables) + (size_t)h * 2 * len * dtype_size(dtype);
    const char* col = row + (size_t)len * dtype_size(dtype);
    const int ri = i / g, ci = i % g;
    float* o = out + ((size_t)h * N + i) * N;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        const int rj = j / g, cj = j % g;
        o[j] = load_as_float(row, dtype, ri - rj + g - 1) + load_as_float(col, dtype, ci - cj + g - 1);
    }
}

int launch_expand_rel2d(const void* tables, int dtype, int heads, int N, int g, float* out, cudaStream_t stream) {
    dim3 grid((unsigned)std::min(64, (N + 255) / 256), (unsigned)N, (unsigned)heads);
    expand_rel2d_kernel<<<grid, 256, 0, stream>>>(tables, dtype, N, g, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

// Dense bf16 table whose rows are not 16-byte multiples (a contiguous [H,N,N] table with N % 8 != 0 -- the natural layout of the
// N = 197 ViT configs) -> the same table with rows padded to ld_out = 8-element multiples, which the TMA tile loads need.  The
// direct-load bias path the unpadded table would take is 2x slower at N = 197 (0.165 -> 0.335 ms) and costs the integer P.V
// mode its tensor-core kernel altogether (0.36 -> 3.05 ms); the copy is ~1 MB there.  One thread per 8 output elements.
__global__ void __launch_bounds__(256) pad_bias_rows_kernel(const uint16_t* __restrict__ in, int64_t ld_in, int N, int64_t ld_out,
                                                            uint16_t* __restrict__ out, int64_t rows) {
    const int cpr = (int)(ld_out / 8);  // 16-byte chunks per output row
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * cpr) return;
    const int64_t row = idx / cpr;
    const int c0 = (int)(idx - row * cpr) * 8;
    const uint16_t* src = in + row * ld_in + c0;
    uint16_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = c0 + i < N ? src[i] : (uint16_t)0;
    *reinterpret_cast<uint4*>(out + row * ld_out + c0) = *reinterpret_cast<const uint4*>(v);
}

// in: [heads, N, ld_in] bf16 (ld_in >= N), out: [heads, N, ld_out] with ld_out % 8 == 0; out must be 16-byte aligned.
int launch_pad_bias_rows(const void* in, int64_t ld_in, int heads, int N, int64_t ld_out, void* out, cudaStream_t stream) {
    const int64_t rows = (int64_t)heads * N, chunks = rows * (ld_out / 8);
    if (chunks == 0) return 0;
    pad_bias_rows_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, stream>>>(static_cast<const uint16_t*>(in), ld_in, N, ld_out,
                                                                            static_cast<uint16_t*>(out), rows);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 1 : -(int)e;
}

}  // namespace ba
