/*
 * srnn.h -- C ABI of the B200-native sparse persistent RNN hot path
 *           (arXiv 1804.10223, "sparse persistent RNNs").
 *
 * The library computes, for a pruned recurrent layer, the whole sequence
 *
 *     b'_t = W x_t + b                       (Eq. 2 hoist)
 *     h_t  = g(U_r h_{t-1} + b'_t)           (Eq. 2)
 *
 * or, for the LSTM case study (App. B), four gate rows per
 * hidden unit ([i; f; g; o], standard cell; reading R3).
 * U_r is unstructured-sparse.  The sparse weights are
 * packed once ("only has to happen when the network's sparsity
 * pattern changes") into a register-resident image and kept on-chip for the
 * whole sequence by one persistent cooperative kernel;
 * steps are ordered by timestep-tagged h words, not a grid barrier
 * (PAPER.md:102-107 Lamport timestamps, re-designed).
 *
 * Conventions for every entry point:
 *   - All pointers are plain host or device pointers as stated per argument.
 *     The caller owns every array it passes; the plan owns its packed weight
 *     image, exchange buffers and b' workspace (device) and frees them in
 *     srnn_destroy.  Nothing is retained after a call returns except what
 *     srnn_load_weights copies.
 *   - Layouts are row-major, fp32 unless stated: x [T][B][I], h0/c0/hT/cT
 *     [B][H], y [T][B][H], W_x [G*H][I], bias [G*H]; G = 1 (RNN), 4 (LSTM) or
 *     3 (GRU, whose bias has 4H entries: [b_r; b_z; b_n; b_hn]).  c0/cT are
 *     used by the LSTM only.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device work is enqueued asynchronously; errors of the
 *     asynchronous part surface through srnn_plan_status after the caller
 *     synchronises the stream.
 *   - A plan is not thread-safe: one call at a time per plan, one forward in
 *     flight per plan (its exchange buffers are reused).  Distinct plans are
 *     independent.
 *   - Return value: SRNN_OK or a negative srnn_status_t; on error no device
 *     work has been enqueued by that call.
 */
#ifndef SRNN_H_
#define SRNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct srnn_plan *srnn_plan_t;

typedef enum {
    SRNN_OK = 0,
    SRNN_ERR_INVALID_VALUE = -1, /* bad argument, size or NULL pointer            */
    SRNN_ERR_NOT_ON_CHIP = -2,   /* weights/activations exceed the on-chip budget */
    SRNN_ERR_BAD_WEIGHTS = -3,   /* malformed CSR (rowptr, col range, duplicates) */
    SRNN_ERR_STATE = -4,         /* call out of order (e.g. forward before load)  */
    SRNN_ERR_CUDA = -5,          /* a CUDA runtime call failed                    */
    SRNN_ERR_TIMEOUT = -6,       /* device watchdog: a tagged h word never arrived*/
    SRNN_ERR_UNSUPPORTED = -7    /* configuration not supported by this build     */
} srnn_status_t;

/* Cell type: vanilla RNN (Eq. 2), LSTM, or GRU (a cell extension
 * beyond the paper; reading R15: gate blocks
 * [r; z; n], n = tanh(W_n x + b_n + r * (U_n h + b_hn)), h' = (1 - z) n + z h). */
typedef enum { SRNN_CELL_RNN = 0, SRNN_CELL_LSTM = 1, SRNN_CELL_GRU = 2 } srnn_cell_t;

/* Activation g of Eq. 1/2 ("g is an elementwise activation
 * function"; unspecified by the paper -> a parameter, R1).
 * Ignored for LSTM (gates use sigmoid/tanh). */
typedef enum { SRNN_ACT_RELU = 0, SRNN_ACT_TANH = 1, SRNN_ACT_IDENTITY = 2 } srnn_act_t;

/* Precision mode.
 *   FP32:              fp32 weights and activations, exact fp32 SIMT input
 *                      GEMM (no TF32; SRNN_FLAG_FP32_TC_GEMM trades accuracy for
 *                      a 3xTF32 tensor-core GEMM), accurate transcendentals.
 *                      Tolerance vs oracle 1e-5.
 *   FP16W_FP32ACC:     W_h stored fp16 (RNE, "lower-precision data
 *                      type such as fp16 for the weights"), W_x and x rounded
 *                      to fp16 for a tensor-core input GEMM, all accumulation
 *                      and activations fp32.  Tolerance vs oracle 2e-2. */
typedef enum { SRNN_PREC_FP32 = 0, SRNN_PREC_FP16W_FP32ACC = 1 } srnn_prec_t;

/* Flag bits (srnn_config_t.flags): ablations and fallbacks. */
#define SRNN_FLAG_GRID_SYNC      (1u << 0) /* grid.sync() per step instead of tags   */
#define SRNN_FLAG_NAIVE_LAYOUT   (1u << 1) /* CSR-order lane-strided pairs, no bank-aware order     */
#define SRNN_FLAG_HOST_ONLY      (1u << 2) /* plan + pack on the host only; no device calls at all */
#define SRNN_FLAG_SIMT_GEMM      (1u << 3) /* fp16 mode: use the exact fp32 SIMT input GEMM instead of
                                              the fp16 tcgen05 GEMM (ablation)                   */
#define SRNN_FLAG_DEBUG_JITTER   (1u << 4) /* inject per-CTA __nanosleep delays (sync-protocol test)*/
#define SRNN_FLAG_FP32_STAGING   (1u << 5) /* fp16 mode: stage/exchange h in fp32 and keep fp32
                                              register pairs (ablation; default fp16 staging and
                                              one register per pair)        */
#define SRNN_FLAG_PROFILE        (1u << 6) /* record per-CTA phase timestamps (srnn_plan_debug_timeline);
                                              diagnostics build libsrnn_profile.so only, else
                                              srnn_plan_create returns SRNN_ERR_UNSUPPORTED */
#define SRNN_FLAG_RESERVE_SMS    (1u << 7) /* leave 4 SMs free so srnn_forward_host can pipeline: x
                                              chunks are copied and projected (GEMM on the free SMs)
                                              while the persistent kernel runs, y chunks are copied
                                              back as the kernel reports progress               */
#define SRNN_FLAG_DEBUG_DROP_PUBLISH (1u << 9) /* fault injection: CTA 0 never publishes h_2 (a lost
                                              exchange message); the device watchdog must end the
                                              kernel and srnn_plan_status report SRNN_ERR_TIMEOUT
                                              (timeout: env SRNN_TIMEOUT_MS, default 2000)       */
#define SRNN_FLAG_FP32_TC_GEMM   (1u << 10) /* fp32 mode, opt-in: input projection as a 3xTF32
                                              tcgen05 GEMM (x, W_x split into tf32 hi + lo, D +=
                                              hi*hi + hi*lo + lo*hi): 6.5x faster than the SIMT
                                              GEMM at C2, but the tensor cores' fp32 accumulation
                                              leaves ~1.5e-8 * K relative error in b' (4.9e-5 at
                                              K = 2304 vs 6e-6 for SIMT), above the 1e-5 parity
                                              bound of the fp32 mode -- not the default        */
#define SRNN_FLAG_Y_BATCH_MAJOR  (1u << 11) /* y is written batch-major, [B][T][H], instead of [T][B][H]:
                                              the shards of a batch-partitioned run (SURVEY.md
                                              Sec. 8(e)) are then contiguous blocks
                                              of the global [B][T][H] y, so an all-gather needs no
                                              re-layout.  srnn_forward / srnn_recurrence /
                                              srnn_forward_host (the latter unpipelined)         */
#define SRNN_FLAG_CLASS_BALANCE  (1u << 12) /* class-based load balancing: hidden units are
                                              bucketed into classes by their nonzero count and dealt
                                              over the CTAs so every CTA gets the same class mix and
                                              warps get rows of similar length; the exchange and hs
                                              use the resulting unit order (results unchanged up to
                                              fp reassociation)                                  */
#define SRNN_FLAG_COLUMN_SPLIT   (1u << 13) /* column split ("split one row among multiple
                                              blocks"): CTAs run as 2-CTA thread-block clusters; both
                                              CTAs of a pair hold every row of the pair's units, each
                                              only the nonzeros of one half of the columns, so each
                                              stages and fetches only half of h_{t-1} per step; the
                                              two partial row sums are added through distributed
                                              shared memory (fixed order: deterministic).  Halves the
                                              h staging and exchange ingress per SM: larger H on chip
                                              (the 16-bit staged offsets cover twice the columns) and
                                              a faster load phase at large H.  RNN / LSTM / GRU cells,
                                              batch tiles <= 8; not with CLASS_BALANCE / DENSE_TC  */
#define SRNN_FLAG_STAGED         (1u << 14) /* partial progress ("the load stage can make
                                              partial progress as values are marked complete, allowing
                                              the operate stage to proceed before all values are
                                              finished"): each warp's slots are packed in two stages,
                                              the pairs whose column lies in the exchange chunks the
                                              loaders fetch first, then the rest; the kernel stages the
                                              early chunks, operates on the early slots while the late
                                              chunks are still in flight, then completes the late stage.
                                              fp16 mode, batch tiles of 4 / 8, register-resident plans
                                              with one poll batch; ignored (plan_query staged = 0)
                                              where it does not apply.  Results are identical up to fp
                                              reassociation (a row's sum is taken in another order) */
#define SRNN_FLAG_DENSE_TC       (1u << 8) /* comparator: the DENSE persistent
                                              RNN of PAPER.md:51-71 (Sec. 3.2, Diamos et al.)
                                              re-done for sm_100a tensor cores.  U_r is densified
                                              (fp16 RNE, zeros kept) into mma.sync m16n8k16
                                              A fragments held in registers (overflow: shared
                                              memory); h_{t-1} is staged as [H][8] fp16 rows and
                                              read with ldmatrix.trans; the exchange, epilogue and
                                              LSTM gates are those of the sparse kernel.  FP16W
                                              mode only (else SRNN_ERR_UNSUPPORTED); batch tiles
                                              of 4 or 8; SRNN_ERR_NOT_ON_CHIP when the dense
                                              fragments do not fit registers + shared memory  */

typedef struct {
    int32_t hidden;     /* H >= 1, <= 65536 (u16 column index)                          */
    int32_t input;      /* I >= 1 (width of x_t)                                         */
    int32_t batch;      /* B_max >= 1: largest batch srnn_forward will be called with    */
    int32_t max_steps;  /* T_max >= 0: largest T srnn_forward will be called with        */
    float density;      /* expected density of U_r in [0,1], used for capacity planning  */
    int32_t cell;       /* srnn_cell_t                                                   */
    int32_t act;        /* srnn_act_t                                                    */
    int32_t prec;       /* srnn_prec_t                                                   */
    int32_t device;     /* CUDA device ordinal (ignored with SRNN_FLAG_HOST_ONLY)        */
    uint32_t flags;     /* SRNN_FLAG_* bits                                              */
    int32_t num_ctas;   /* 0 = planner's choice; else force this CTA count (<= SMs)     */
    int32_t lanes_per_row; /* 0 = planner's choice; else 1,2,4,8,16 or 32              */
    int32_t batch_tile; /* 0 = planner's choice; else 1, 2, 4 (fp32) or 1..16 (fp16) samples per h tile */
} srnn_config_t;

/* What the planner decided (srnn_plan_query). Fields marked (L) are final
 * only after srnn_load_weights (they depend on the actual sparsity pattern). */
typedef struct {
    int32_t sm_count;          /* SMs of the device (148 on B200; profile value in host-only mode) */
    int32_t num_ctas;          /* persistent CTAs, one per SM (L)                            */
    int32_t threads_per_cta;   /* (L)                                                        */
    int32_t lanes_per_row;     /* L: lanes cooperating on one row (L)                        */
    int32_t pairs_per_lane;    /* NP: register slots per lane = compiled instance (L)        */
    int32_t slots_used;        /* max slots actually used by any warp (<= NP) (L)            */
    int32_t batch_tile;        /* BT: samples staged per smem h tile (1, 2, 4; fp16 also 8, 16) */
    int32_t num_batch_tiles;   /* ceil(B_max / BT)                                           */
    int32_t units_per_cta_max; /* hidden units owned by the largest CTA (L)                  */
    int32_t regs_per_thread;   /* compiled register count of the chosen kernel instance (L)  */
    int32_t packed_registers;  /* 1: one u32 register per pair (decode per step), 0: two (L) */
    int32_t fits;              /* 1 if the layer runs fully on-chip with this plan           */
    int64_t nnz;               /* true nonzeros of U_r (L)                                   */
    int64_t slots_total;       /* pair slots incl. zero padding over all CTAs (L)            */
    int64_t smem_bytes_per_cta;/* dynamic shared memory per CTA                              */
    int64_t weight_image_bytes;/* packed image size in HBM (L)                               */
    int64_t wavefronts_per_step_max; /* packer's predicted smem wavefronts of the busiest CTA per batch tile (L) */
    int64_t wavefronts_per_step_ideal; /* same, if every phase were conflict-free and unpadded (L) */
    int64_t conflict_wavefronts;       /* extra wavefronts from bank conflicts in that CTA (L)        */
    int64_t smem_weight_bytes_per_cta; /* shared-memory weight tier (pairs beyond the register slots) (L) */
    int64_t image_slots_per_lane;      /* register + shared-memory slots per lane in the image (L)     */
    int64_t model_cycles_per_step;     /* planner's cost-model estimate of one timestep, SM cycles (L) */
    /* SRNN_FLAG_DENSE_TC plans only (zero otherwise) (L): */
    int32_t dense_m_tiles;     /* 16-row mma tiles per CTA                                   */
    int32_t dense_kblocks_per_warp; /* 16-column k-blocks of U_r per warp                      */
    int32_t dense_frags_reg;   /* A fragments per lane held in registers (compiled instance) */
    int32_t dense_frags_smem;  /* A fragments per lane held in shared memory                 */
    int32_t spill_bytes;       /* local memory (register spills / stack) per thread of the
                                  chosen compiled instance; 0 for a spill-free instance  (L) */
    int32_t column_split;      /* 1: SRNN_FLAG_COLUMN_SPLIT plan (2-CTA clusters)             */
    int32_t column_half;       /* column split: first column of the second half (units)      */
    int32_t staged;            /* 1: partial-progress plan (SRNN_FLAG_STAGED): each warp's slots
                                  are ordered early chunks first, late chunks second     (L) */
    int32_t early_chunks;      /* staged plans: 16-byte exchange chunks of the early stage   (L) */
} srnn_plan_info_t;

/* Create a plan for the layer described by *cfg.
 * Queries the device (SM count, shared-memory opt-in) unless
 * SRNN_FLAG_HOST_ONLY, then checks the on-chip budget for the expected density
 * (PAPER.md:151 capacity limits).  Allocates the plan's device buffers
 * (exchange words, b' workspace for B_max x T_max).
 * Errors: SRNN_ERR_INVALID_VALUE (bad sizes, NULL), SRNN_ERR_NOT_ON_CHIP
 * (the expected nonzeros or h staging cannot fit), SRNN_ERR_CUDA. */
srnn_status_t srnn_plan_create(const srnn_config_t *cfg, srnn_plan_t *out);

/* Fill *out with the plan's decisions (see srnn_plan_info_t). Host-only. */
srnn_status_t srnn_plan_query(srnn_plan_t plan, srnn_plan_info_t *out);

/* Load the layer's weights (host pointers; copied, caller may free after).
 *   wh_rowptr [G*H+1] int32, wh_col [nnz] int32 in [0,H), wh_val [nnz] fp32:
 *       U_r in CSR (rows = gate*H + unit for LSTM), no duplicate (row,col);
 *   wx [G*H][I] fp32 row-major (dense W), bias [G*H] fp32 or NULL
 *       (GRU: [4H] = [b_r; b_z; b_n; b_hn], the last block the n gate's recurrent bias).
 * Runs the packer (PAPER.md:91 zero padding, :99-100 + App. A Alg. 1
 * bank-aware order, re-targeted to sm_100a shared-memory phases; fp16 RNE
 * quantisation in FP16W mode) and uploads the image (skipped in host-only
 * mode).  May be called again to replace the weights.
 * Errors: SRNN_ERR_BAD_WEIGHTS (non-monotone rowptr, col out of range,
 * duplicate entry, nnz mismatch), SRNN_ERR_NOT_ON_CHIP (pattern does not fit
 * the register budget), SRNN_ERR_CUDA. */
srnn_status_t srnn_load_weights(srnn_plan_t plan, const int32_t *wh_rowptr, const int32_t *wh_col,
                                const float *wh_val, int64_t nnz, const float *wx, const float *bias);

/* Whole hot path on device buffers:
 * input projection GEMM into the plan's b' workspace, then the persistent
 * recurrent kernel.  x: device [T][B][I]; h0, c0: device [B][H] or NULL (=0;
 * c0 only for LSTM); y: device [T][B][H] ([B][T][H] with SRNN_FLAG_Y_BATCH_MAJOR;
 * may be NULL if hT is wanted only);
 * hT, cT: device [B][H] or NULL.  0 <= T <= T_max, 1 <= B <= B_max.
 * T == 0 copies h0 (or zeros) to hT.
 * Errors: SRNN_ERR_STATE (no weights loaded, or host-only plan),
 * SRNN_ERR_INVALID_VALUE, SRNN_ERR_CUDA. */
srnn_status_t srnn_forward(srnn_plan_t plan, int32_t T, int32_t B, const float *x, const float *h0,
                           const float *c0, float *y, float *hT, float *cT, void *stream);

/* Step a1 only: b'[T*B][G*H] = x W^T + b (Eq. 2 hoist) into the
 * caller's device buffer `bprime` (fp32). Same x layout/limits as srnn_forward. */
srnn_status_t srnn_input_projection(srnn_plan_t plan, int32_t T, int32_t B, const float *x,
                                    float *bprime, void *stream);

/* Steps a3-a9 only: the persistent recurrent kernel over a caller-supplied
 * device b' [T][B][G*H] fp32 (e.g. from srnn_input_projection).  Other
 * arguments as in srnn_forward. */
srnn_status_t srnn_recurrence(srnn_plan_t plan, int32_t T, int32_t B, const float *bprime,
                              const float *h0, const float *c0, float *y, float *hT, float *cT,
                              void *stream);

/* End-to-end call on HOST buffers (same layouts as srnn_forward): copies x
 * (and h0/c0) host->device, runs the input projection and the recurrence,
 * copies y (and hT/cT) back, and synchronises before returning.  Any output
 * pointer may be NULL.  Pageable or pinned host memory is accepted (pinned
 * overlaps).  If the plan leaves SMs free (SRNN_FLAG_RESERVE_SMS) the call is
 * pipelined: x arrives and is projected in chunks of steps while the
 * persistent kernel already runs (it waits per step for its b' rows), and y
 * leaves in chunks as the kernel reports progress (stream memory operations,
 * cuStreamWaitValue32 / cuStreamWriteValue32). */
srnn_status_t srnn_forward_host(srnn_plan_t plan, int32_t T, int32_t B, const float *x_host,
                                const float *h0_host, const float *c0_host, float *y_host,
                                float *hT_host, float *cT_host);

/* Device-side status of the last forward (watchdog / protocol errors); call
 * after synchronising the stream.  Resets the status word to SRNN_OK. */
srnn_status_t srnn_plan_status(srnn_plan_t plan);

/* Copy the packer's host-side layout for inspection/tests (works in
 * host-only mode).  Arrays are [num_ctas][image_slots_per_lane][threads_per_cta]:
 *   col_out  int32: U_r column of each slot (padding slots: a valid column)
 *   val_out  float: value (fp16-rounded in FP16W mode; 0 for padding)
 *   row_out  int32: global row (gate*H+unit) the slot's lane works on, -1 if idle
 * Any pointer may be NULL; `capacity` is the element capacity of each array.
 * Errors: SRNN_ERR_STATE before load, SRNN_ERR_INVALID_VALUE if too small. */
srnn_status_t srnn_plan_export_layout(srnn_plan_t plan, int32_t *col_out, float *val_out,
                                      int32_t *row_out, int64_t capacity);

/* Debug: with SRNN_FLAG_PROFILE, copy the stamps of the last forward to host
 * `out` as [num_ctas][T][num_tiles][16] int64.  Slots 0-7 and 10 are clock64
 * (SM cycle counter of that CTA's SM, thread 0): 0 step start, 1 h staged
 * (after the barrier), 2 after the second barrier, 3 h published, 4 operate
 * loop done, 5 butterfly done, 6 b' copies landed, 7 after the post-publish
 * barrier, 10 thread 0's first poll round returned.  8: poll rounds of
 * thread 0, 9: max poll rounds over the CTA's threads.  11 / 12: %globaltimer
 * (ns, comparable across CTAs) at 3 / 1.  13-15 unused.
 * `capacity` in elements; returns the element count via *count.
 * Errors: SRNN_ERR_STATE without the flag or before a forward. */
srnn_status_t srnn_plan_debug_timeline(srnn_plan_t plan, int64_t *out, int64_t capacity, int64_t *count);

/* Human-readable name of a status code (static storage). */
const char *srnn_status_string(srnn_status_t status);

/* Library version string, e.g. "srnn 0.1 sm_100a". */
const char *srnn_version(void);

/* Free the plan and all its device buffers. NULL is a no-op. */
srnn_status_t srnn_destroy(srnn_plan_t plan);

#ifdef __cplusplus
}
#endif
#endif /* SRNN_H_ */
