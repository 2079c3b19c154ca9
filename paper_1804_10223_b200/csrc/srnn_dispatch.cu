#include <algorithm>
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
// Exchange re-initialisation from the host side (column-split plans, whose cluster launch does
// not use the kernel's grid-wide barrier): every exchanged 16/32-bit value of parity q gets
// the stale tag of the step that parity last held (pattern pat_q), i.e. "not yet written".
__global__ void xbuf_fill_kernel(uint32_t* buf, int64_t words_per_parity, uint32_t pat0, uint32_t pat1) {
    const int64_t n = 2 * words_per_parity;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        buf[i] = i < words_per_parity ? pat0 : pat1;
}

int launch_xbuf_fill(void* buf, int64_t bytes_per_parity, uint32_t pat0, uint32_t pat1, void* stream) {
    const int64_t w = bytes_per_parity / 4;
    const int blocks = static_cast<int>(std::min<int64_t>(1024, (2 * w + 255) / 256));
    xbuf_fill_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint32_t*>(buf), w, pat0, pat1);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace srnn
