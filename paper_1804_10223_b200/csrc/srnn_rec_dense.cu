// Instances of the dense tensor-core comparator (SRNN_FLAG_DENSE_TC, SURVEY.md
// Sec. 8(f)1): the persistent kernel with MT row tiles of 16 per CTA and NF
// register-resident mma A fragments per lane (fp16 only).
#include "srnn_recurrent.cuh"

namespace srnn {

template <int NF, int MT>
static int launch_dense_bt(int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream,
                           bool query_only, int* regs_out, int* max_blocks_out) {
#define SRNN_DCASE(BT_, G_)                                                                                \
    if (bt == BT_ && g == G_)                                                                              \
        return launch_one<NF, BT_, G_, true, MT>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    SRNN_DCASE(4, 1)
    SRNN_DCASE(8, 1)
    SRNN_DCASE(4, 4)
    SRNN_DCASE(8, 4)
#undef SRNN_DCASE
    return static_cast<int>(cudaErrorInvalidValue);
}

int launch_dense(int nf, int mt, int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream,
                 bool query_only, int* regs_out, int* max_blocks_out) {
    if (mt == 1 && nf == 8) return launch_dense_bt<8, 1>(bt, g, p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    if (mt == 1 && nf == 12) return launch_dense_bt<12, 1>(bt, g, p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    if (mt == 2 && nf == 8) return launch_dense_bt<8, 2>(bt, g, p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    if (mt == 2 && nf == 12) return launch_dense_bt<12, 2>(bt, g, p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace srnn
