// attn_tcgen05_k32.cu -- every attn_tc_kernel variant with head dims padded to 32 (see attn_tcgen05.cuh).
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc {

int launch_tc_k32(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline) {
    (void)timeline;
    return launch_kpad<32>(prm, bias_mode, m, stream);
}

}  // namespace tc
}  // namespace ba
