// Dispatch (NP, BT, G) -> compiled instance of the persistent kernel.
#include <cuda_runtime.h>

#include "srnn_internal.h"

namespace srnn {
template <int NP>
int launch_np(int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
              int* regs_out, int* max_blocks_out);

int launch_recurrent(int np, int bt, int g, int packed, const RecParams& p, int num_ctas, size_t smem_bytes,
                     void* stream, bool query_only, int* regs_out, int* max_blocks_per_sm_out) {
    if (packed) return static_cast<int>(cudaErrorNotSupported);
    switch (np) {
        case 4: return launch_np<4>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 8: return launch_np<8>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 12: return launch_np<12>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 16: return launch_np<16>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 24: return launch_np<24>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 32: return launch_np<32>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 48: return launch_np<48>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        case 64: return launch_np<64>(bt, g, p, num_ctas, smem_bytes, stream, query_only, regs_out, max_blocks_per_sm_out);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}
}  // namespace srnn
