// attn_tcgen05.cu -- K2 (tensor-core variant): placeholder until the tcgen05/TMEM/TMA kernel lands.
#include "ba_common.cuh"

namespace ba {

bool tcgen05_supported(const ba_params*, const char** why) {
    if (why) *why = "tcgen05 kernel not built in this revision";
    return false;
}

int launch_attn_tcgen05(const FwdArgs&, cudaStream_t) { return -(int)cudaErrorNotSupported; }

}  // namespace ba
