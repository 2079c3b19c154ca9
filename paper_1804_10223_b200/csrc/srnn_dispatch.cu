// Dispatch (NP, BT, G, precision) -> compiled instance of the persistent kernel.
#include <cuda_runtime.h>

#include "srnn_internal.h"

namespace srnn {
template <int NP, bool F16>
int launch_np(int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
              int* regs_out, int* max_blocks_out);

int launch_recurrent(int np, int bt, int g, int f16, const RecParams& p, int num_ctas, size_t smem_bytes,
                     void* stream, bool query_only, int* regs_out, int* max_blocks_per_sm_out) {
#define SRNN_NP(N)                                                                                          \
    case N:                                                                                                 \
        return f16 ? launch_np<N, true>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out,      \
                                        max_blocks_per_sm_out)                                              \
                   : launch_np<N, false>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out,     \
                                         max_blocks_per_sm_out);
    switch (np) {
        SRNN_NP(4)
        SRNN_NP(8)
        SRNN_NP(12)
        SRNN_NP(16)
        SRNN_NP(24)
        SRNN_NP(32)
        SRNN_NP(48)
        SRNN_NP(64)
        case 96:
            if (!f16) return static_cast<int>(cudaErrorInvalidValue);
            return launch_np<96, true>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out,
                                       max_blocks_per_sm_out);
        default:
            return static_cast<int>(cudaErrorInvalidValue);
    }
#undef SRNN_NP
}
}  // namespace srnn
