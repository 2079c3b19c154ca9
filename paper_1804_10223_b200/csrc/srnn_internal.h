// srnn_internal.h -- shared between the host planner (srnn_api.cpp) and the
// CUDA kernels of the product path.  Never included by oracle/.
#pragma once
#include <cuda.h>

#include <cstdint>

#ifdef __CUDACC__
#define SRNN_HD __host__ __device__
#else
#define SRNN_HD
#endif

#ifndef SRNN_MAX_THREADS
#define SRNN_MAX_THREADS 1024
#endif

namespace srnn {

// Kernel arguments of the persistent recurrent kernel (one struct, passed by
// value through cudaLaunchCooperativeKernel).
struct RecParams {
    // b' tensor map (see bp_tma below): first member, so it sits at the 128-byte aligned start of
    // the kernel's parameter buffer (__grid_constant__: the TMA unit reads it from param space)
    alignas(128) CUtensorMap bp_map;
    // problem
    int32_t H;        // hidden units
    int32_t G;        // gates per unit (1 RNN, 4 LSTM)
    int32_t B;        // batch of this call (<= n_tiles*BT)
    int32_t T;        // timesteps of this call (>= 1)
    int32_t n_tiles;  // batch tiles of width BT processed per step
    int32_t act;      // srnn_act_t (RNN only)
    int32_t threads;  // threads per CTA
    int32_t lanes_per_row;  // L
    int32_t np_inst;  // register slots per lane (= template NP)
    int32_t smem_slots;  // shared-memory tier slots per lane (multiple of 4; image width = NP + smem_slots)
    int32_t units_max;      // max units of any CTA (smem sizing)
    uint32_t epoch;   // global step of h_0 for this call; h_s is global step epoch + s (1-bit tag: bit 1)
    uint32_t flags;   // SRNN_FLAG_* subset relevant on device
    // packed weights: [cta][slot][thread]
    const uint2* img_f32;      // fp32 mode: {hs byte offset, float bits}
    const uint32_t* img_f16;   // fp16 mode: (hs byte offset << 16) | half bits
    const int32_t* cta_unit0;  // [num_ctas + 1] first exchange position of each CTA
    const int32_t* unit_perm;  // [H] hidden unit at each exchange position (class balancing), or null = identity
    const int32_t* piece0;     // [cta][G*units_max + 1] first virtual row of each local row (split heavy rows), or null
    int32_t vrows_max;         // virtual rows of the largest CTA (zs rows)
    const int32_t* warp_slots; // [num_ctas][warps] slots used by each warp (warp-uniform)
    // staged instance (MT = -3): slots [0, warp_early) read only hs positions of the first
    // early_chunks exchange chunks; the rest read the others
    const int32_t* warp_early; // [num_ctas][warps], or null
    int32_t early_chunks;
    // data
    const float* bprime;  // [T][B][G*H]
    const float* h0;      // [B][H] or null
    const float* c0;      // [B][H] or null
    const float* bias_hn; // GRU: [H] recurrent bias of the n gate (inside r * (.)), or null
    float* y;             // element (t, b, unit) at b * y_bstride + t * y_tstride + unit, or null
    int64_t y_bstride;    // [T][B][H]: H;      batch-major [B][T][H]: T * H
    int64_t y_tstride;    // [T][B][H]: B * H;  batch-major: H
    float* hT;            // [B][H] or null
    float* cT;            // [B][H] or null
    unsigned char* xbuf;  // exchange images [2 global-step parities][xbuf_tiles][tile_bytes] (= the hs layout, tag in each LSB)
    int32_t xbuf_tiles;   // tile stride of xbuf (the plan's maximum, fixed across launches)
    int32_t tile_bytes;   // bytes of one (parity, tile) image: H * E rounded up to 16 (BT = 16: 2 planes of H * 16)
    int32_t reinit;       // host: the buffers' stale tags are not those of steps epoch - 2 / epoch - 1 (rewrite them)
    int32_t* xdirty;      // device: set by an aborted launch (buffers inconsistent), cleared by the next re-init
    int32_t* status;      // device status word (srnn_status_t)
    unsigned long long timeout_ns;
    uint32_t poll_backoff_ns;  // sleep between stale poll rounds (tuning knob, SRNN_POLL_BACKOFF_NS)
    int32_t loader_threads;    // threads that poll/stage h (0 = all; tuning knob, SRNN_LOADER_THREADS)
    long long* profile;   // SRNN_FLAG_PROFILE: [cta][T][n_tiles][8] clock64 stamps or null
    // host-pipelined forward (srnn_forward_host): b' arrives in chunks while the
    // kernel runs; y leaves in chunks while it runs
    const uint32_t* bp_ready;  // b' rows of steps <= *bp_ready - bp_ready_base are written (or null)
    uint32_t bp_ready_base;
    uint32_t* progress;        // +1 per CTA every progress_every steps (after y is stored), or null
    int32_t progress_every;
    int32_t k8;                // host-side instance choice: the 8-poll-slot instance (k8_compiled)
    // b' by TMA (one batch tile, resident b'): CUtensorMap in device memory over b' [T][B][G*H]
    // (3-D: units, samples, steps), box {bp_boxu, BT, kBpWin}; one thread loads the next window
    // of kBpWin steps per gate while the current window is consumed (double buffer, mbarriers)
    // column split (SRNN_FLAG_COLUMN_SPLIT): CTA pairs form 2-CTA clusters; both CTAs
    // of cluster q hold all rows of the cluster's units, CTA rank r only the columns of half r
    // ([0, hsplit) or [hsplit, H)), and stage only that half of h; partial row sums are added
    // across the pair through distributed shared memory.  cta_unit0 then lists the units each
    // CTA finalises and publishes (its half of the cluster's units), cta_vunit0 the cluster's
    // units (2 * first unit, +UQ, ...: UQ = the pair's unit count, the CTA's row count / G).
    int32_t csplit;
    int32_t hsplit;
    const int32_t* cta_vunit0;
    int32_t bp_tma;            // 1: b' by TMA windows through bp_map; 0: per-step cp.async of b'
    int32_t bp_boxu;           // units per box (bp_box_units(units_max))
    // SRNN_FLAG_DENSE_TC comparator (dense U_r as mma.sync A fragments)
    const uint4* img_dense;    // [cta][frag][thread] A fragments (4 x 2 fp16), frag = kk * MT + m
    int32_t dense_kpw;         // k-blocks (16 columns) per warp
    int32_t dense_nf;          // fragments per lane in the image (= MT * dense_kpw)
    int32_t hs_rows;           // staged h rows (>= H, = 16 warps * 16 * dense_kpw), 16 bytes each
};

struct GemmParams {
    int64_t M;   // rows of x (T*B)
    int32_t N;   // G*H
    int32_t K;   // I
    const float* A;      // [M][K] fp32
    const float* W;      // [N][K] fp32
    const float* bias;   // [N] or null
    float* C;            // [M][N]
};

// Launch helpers implemented in the .cu files. Return cudaError_t as int.  regs_out, if
// given, is int[2]: compiled registers per thread and local-memory (spill) bytes per thread.
int launch_recurrent(int np, int bt, int g, int f16, const RecParams& p, int num_ctas,
                     size_t smem_bytes, void* stream, bool query_only, int* regs_out,
                     int* max_blocks_per_sm_out);
// Dense tensor-core comparator (srnn_rec_dense.cu): nf = register fragments
// per lane (8 or 12), mt = 16-row tiles per CTA (1 or 2), bt = 4 or 8.
constexpr int kDenseThreads = 512;
int launch_dense(int nf, int mt, int bt, int g, const RecParams& p, int num_ctas, size_t smem_bytes, void* stream,
                 bool query_only, int* regs_out, int* max_blocks_per_sm_out);
int launch_gemm_f32(const GemmParams& p, void* stream);
// fp16 tensor-core input GEMM (srnn_gemm_tc.cu); maps are CUtensorMap*.
int launch_gemm_tc(const void* map_a, const void* map_b, const float* bias, float* C, int M, int N, int K,
                   void* stream, int m_off = 0, int bn = 0, int sms = 148, const void* map_b32 = nullptr,
                   const void* map_b48 = nullptr);  // W_x maps in 32 / 48-row boxes (multicast clusters)
// rows [m_off, m_off + M) of A and C; bn = tile width (0: pick from the grid size vs `sms`, the SMs it may use)
int launch_f32_to_f16(const float* in, void* out, int64_t n, void* stream);
// fp32 mode: 3xTF32 tcgen05 GEMM on tf32 hi/lo splits (maps: fp32 K-major, 32-element boxes)
int launch_gemm_tf32x3(const void* map_a_hi, const void* map_a_lo, const void* map_b_hi, const void* map_b_lo,
                       const float* bias, float* C, int M, int N, int K, void* stream, int m_off, int sms);
int launch_split_tf32(const float* in, float* hi, float* lo, int64_t rows, int cols, int ld_out, void* stream);
int launch_xbuf_fill(void* buf, int64_t bytes_per_parity, uint32_t pat0, uint32_t pat1, void* stream);
int preload_projection_kernels();
int preload_gemm_f32();
int launch_f32_to_f16_padded(const float* in, void* out, int64_t rows, int cols, int ld_out, void* stream);

// b' TMA window (steps per bulk tensor load) and the shared-memory bytes of its double buffer
// plus two mbarriers (must match the kernel's carve-up).
constexpr int kBpWin = 8;
// units per b' box: a CTA's units start at any column, the box at the 16-byte aligned column
// below it (TMA tile mode needs the innermost start coordinate 16-byte aligned): up to 3 more
SRNN_HD constexpr int bp_box_units(int units_max) { return (units_max + 3 + 3) / 4 * 4; }
SRNN_HD constexpr int64_t bp_tma_smem_bytes(int G, int bt, int units_max) {
    return 2LL * G * kBpWin * bt * bp_box_units(units_max) * 4 + 16 + 128;  // + alignment of the TMA window
}
// Poll slots (16-byte exchange chunks in flight per loader thread) of each compiled
// instance; the k8 instances (MT = -1 in srnn_recurrent.cuh) poll 8.  Measured on B200
// (DESIGN.md Sec. 4 "exchange protocol"); SRNN_LOADK_* override for A/B builds.
#ifndef SRNN_LOADK_BT4
#define SRNN_LOADK_BT4 3
#endif
#ifndef SRNN_LOADK_WIDE8
#define SRNN_LOADK_WIDE8 6
#endif
#ifndef SRNN_LOADK_F32
#define SRNN_LOADK_F32 5
#endif
SRNN_HD constexpr int poll_slots(int np, bool f16, int bt, bool k8) {
    return k8 ? 8
         : (f16 && bt == 4 && np <= 24) ? SRNN_LOADK_BT4
         : (f16 && bt >= 8)             ? SRNN_LOADK_WIDE8
         : !f16                         ? SRNN_LOADK_F32
         : (np <= 48 ? 8 : 4);
}
// Slots per operate group of the fp16 kernel (all gathers of a group issue before its FMAs).
SRNN_HD constexpr int operate_group_slots(bool f16, int bt) { return f16 ? (bt == 16 ? 2 : bt >= 4 ? 4 : 8) : (bt == 4 ? 4 : 8); }
// Staged instance (MT = -3, partial progress): the operate of the early exchange
// chunks overlaps the arrival of the late ones.  Compiled for fp16 tiles of 4 and 8 samples.
SRNN_HD constexpr bool staged_compiled(int np, bool f16, int bt) { return f16 && (bt == 4 || bt == 8) && np <= 48; }
// largest register instance compiled with the 16-sample tile (fp16, two hs planes)
constexpr int kMaxNP16 = 48;
// An 8-poll-slot instance exists for this (np, precision, tile)?  Must match launch_np.
SRNN_HD constexpr bool k8_compiled(int np, bool f16, int bt) {
    return f16 && ((bt == 4 && np <= 24) || bt == 8 || (bt == 16 && np <= kMaxNP16));
}
// Bytes of one exchange image (one parity, one batch tile): the staged hs layout,
// H units x E bytes (E = 2 BT fp16, 4 BT fp32), padded to whole 16-byte chunks.
SRNN_HD constexpr int64_t exchange_tile_bytes(int64_t H, bool f16, int bt) {
    return ((H * (f16 ? 2 : 4) * bt) + 15) / 16 * 16;
}

// Compiled register-slot instances (pairs per lane); 96 exists only for the
// fp16 mode (one register per pair).
constexpr int kNumNP = 9;
constexpr int kNPList[kNumNP] = {4, 8, 12, 16, 24, 32, 48, 64, 96};
inline int max_np(bool f16) { return f16 ? 96 : 64; }
inline int max_np(bool f16, int bt) { return bt == 16 ? kMaxNP16 : max_np(f16); }
// Must match MaxThreadsBT<NP, F16, BT> in srnn_recurrent.cuh.
inline int max_threads_for(int np, bool f16, int bt = 1) {
    if (f16 && bt == 16) return np <= 4 ? 640 : np <= 8 ? 512 : np <= 16 ? 384 : 256;
    if (f16) return np <= 12 ? 640 : np <= 32 ? 512 : np <= 64 ? 384 : 256;
    return np <= 4 ? 768 : np <= 12 ? 640 : np <= 32 ? 512 : np <= 48 ? 384 : 256;
}

}  // namespace srnn
