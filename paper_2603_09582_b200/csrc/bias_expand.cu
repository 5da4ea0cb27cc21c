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

}  // namespace ba
