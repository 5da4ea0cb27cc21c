// attn_tcgen05_k128.cu -- every attn_tc_kernel variant with head dims padded to 128 (see attn_tcgen05.cuh).
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc {

int launch_tc_k128(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline) {
    if (timeline && bias_mode == 0 && prm.a.N % BN == 0) return launch_variant<128, 0, 2, false, true>(prm, m, stream);
    return launch_kpad<128>(prm, bias_mode, m, stream);
}

}  // namespace tc
}  // namespace ba
