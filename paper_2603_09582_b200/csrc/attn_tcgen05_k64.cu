// attn_tcgen05_k64.cu -- every attn_tc_kernel variant with head dims padded to 64 (see attn_tcgen05.cuh).
#include "attn_tcgen05.cuh"

namespace ba {
namespace tc {

int launch_tc_k64(const Params& prm, int bias_mode, const Maps& m, cudaStream_t stream, bool timeline) {
    if (timeline) {
        if (bias_mode == 1 && prm.fold) return launch_variant<64, 1, 1, false, true>(prm, m, stream);
        if (bias_mode == 0 && prm.fold) return launch_variant<64, 0, 1, false, true>(prm, m, stream);
        if (bias_mode == 0 && prm.a.N % BN == 0) return launch_variant<64, 0, 2, false, true>(prm, m, stream);
    }
    return launch_kpad<64>(prm, bias_mode, m, stream);
}

}  // namespace tc
}  // namespace ba
