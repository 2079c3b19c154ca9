// srnn_api.cpp -- the C ABI declared in include/srnn.h: plan creation and
// capacity planning, weight loading through the packer
// (a2), and the forward entry points that enqueue the input-projection GEMM
// (a1) and the persistent recurrent kernel (a3-a9).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/srnn.h"
#include "srnn_internal.h"
#include "srnn_packer.h"

using namespace srnn;

struct srnn_plan {
    srnn_config_t cfg{};
    int G = 1;
    int sm_count = 148;
    int smem_optin = 232448;  // B200: 227 KB per block opt-in
    int BT = 4, n_tiles_max = 1;
    bool f16 = false;  // fp16 register pairs + fp16 h staging/exchange (fp16 mode default)
    int E = 16;        // bytes per staged h row
    bool host_only = false;
    bool loaded = false;
    // layout decisions
    Layout lay;
    int np_inst = 0;   // register slots per lane (compiled instance)
    double model_cost = 0;  // planner cost-model estimate of one timestep (SM cycles)
    int ns_slots = 0;  // shared-memory tier slots per lane
    int regs = 0;
    int spill_bytes = 0;  // local memory per thread of the compiled instance (0 = no spills)
    size_t smem_bytes = 0;
    int64_t nnz = 0;
    // device buffers
    void* d_img = nullptr;          // uint2 (fp32) or uint32 (fp16) image
    int32_t* d_unit0 = nullptr;
    int32_t* d_perm = nullptr;            // class balancing: unit of each exchange position
    int32_t* d_piece0 = nullptr;          // class balancing: pieces of heavy rows (Layout::piece0)
    std::vector<int32_t> unit_of_pos, pos_of_unit;  // chosen layout's permutation (empty = identity)
    int32_t* d_wslots = nullptr;
    // partial progress (SRNN_FLAG_STAGED): two-stage slot order, early-stage slots per warp
    bool staged = false;
    int early_chunks = 0;
    int32_t* d_wearly = nullptr;
    float* d_wx = nullptr;
    // fp16 mode tensor-core GEMM: W_x and x rounded to fp16, K padded to a multiple of 8
    bool tc_gemm = false;
    int k_pad = 0;
    void* d_wx16 = nullptr;
    void* d_x16 = nullptr;  // [T_max*B_max][k_pad]
    alignas(64) CUtensorMap map_x16;
    alignas(64) CUtensorMap map_wx16;
    alignas(64) CUtensorMap map_wx16_32;  // W_x in 32 / 48-row boxes (the 4-CTA multicast clusters' B slices)
    alignas(64) CUtensorMap map_wx16_48;
    // fp32 mode: 3xTF32 tensor-core GEMM on tf32 hi/lo splits of x and W_x, K padded to 4
    bool tf32x3 = false;
    int k_pad4 = 0;
    float *d_wx_hi = nullptr, *d_wx_lo = nullptr, *d_x_hi = nullptr, *d_x_lo = nullptr;
    alignas(64) CUtensorMap map_xhi;
    alignas(64) CUtensorMap map_xlo;
    alignas(64) CUtensorMap map_wxhi;
    alignas(64) CUtensorMap map_wxlo;
    float* d_bias = nullptr;
    float* d_bhn = nullptr;         // GRU: n-gate recurrent bias [H]
    float* d_bprime = nullptr;      // [T_max][B_max][G*H]
    unsigned char* d_xbuf = nullptr;  // exchange images [2][n_tiles_max][tile_bytes] (srnn_recurrent.cuh Fmt)
    int32_t* d_xdirty = nullptr;       // set on device by an aborted launch
    int32_t* d_status = nullptr;
    size_t xbuf_bytes = 0;
    int64_t tile_bytes = 0;
    int xbuf_valid_tiles = 0;          // tiles whose stale tags follow the global step sequence
    uint32_t epoch = 1;
    // host-call staging (srnn_forward_host)
    cudaStream_t stream = nullptr;
    float *d_x = nullptr, *d_h0 = nullptr, *d_c0 = nullptr, *d_y = nullptr, *d_hT = nullptr, *d_cT = nullptr;
    unsigned long long timeout_ns = 2000000000ull;
    long long* d_prof = nullptr;
    int64_t prof_elems = 0;
    // pipelined srnn_forward_host
    uint32_t* d_ready = nullptr;     // b' rows ready (monotone counter)
    uint32_t* d_progress = nullptr;  // per-CTA progress increments (monotone counter)
    uint32_t ready_cur = 0, progress_base = 0;  // ready_cur: value of *d_ready between calls
    cudaStream_t s_rec = nullptr, s_out = nullptr, s_copy = nullptr;
    cudaEvent_t ev_in = nullptr, ev_rec = nullptr;
    cudaEvent_t ev_chunk[10] = {};  // x chunk c resident (s_copy -> projection stream)
    int32_t* h_status = nullptr;     // pinned: status read back on s_out at the end of a call
    // SRNN_FLAG_DENSE_TC comparator: dense mma.sync A fragments of U_r
    bool dense = false;
    int dense_mt = 0, dense_kpw = 0, dense_nf = 0, dense_inst = 0, hs_rows = 0;
    std::vector<uint4> dense_img;  // host image [cta][frag][thread] (freed after upload)
    bool k8 = false;               // sparse fp16 tile-of-4 plan that needs 8 poll slots per thread
    // column split (SRNN_FLAG_COLUMN_SPLIT): 2-CTA clusters, each CTA one column half
    bool csplit = false;
    bool auto_split = false;   // the planner chose the split (load_weights falls back if it does not fit)
    int bt_unsplit = 0;        // tile width of the unsplit plan (0: the unsplit layer does not fit)
    int hsplit = 0;                       // first column of the second half (units, multiple of 8)
    std::vector<int32_t> unit0_real;      // [num_ctas + 1] units each CTA finalises / publishes
    int32_t* d_vunit0 = nullptr;          // lay.cta_unit0 (virtual: the pair's units per CTA)
    // b' by TMA windows (RecParams::bp_map, a kernel parameter): re-encoded when the call's
    // (b' pointer, T, B) differ from the last one
    alignas(64) CUtensorMap bp_map;
    const float* bpmap_ptr = nullptr;
    int32_t bpmap_T = 0, bpmap_B = 0;
    std::vector<std::pair<int, bool>> spill_cache;  // (instance key, spills?) of queried instances
};

namespace {

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int inst_for(int slots, bool f16, int bt) {
    for (int i = 0; i < kNumNP; ++i)
        if (kNPList[i] >= slots && kNPList[i] <= max_np(f16, bt)) return kNPList[i];
    return -1;
}

int elem_bytes(bool f16, int bt) { return f16 ? 2 * bt : 4 * bt; }

// b' can come by TMA windows: one batch tile, no unit permutation, 16-byte b' row pitch
bool bp_tma_ok(const srnn_plan* p, int n_tiles, int units_max) {
    // (the window buffer is capped at 8 KB of shared memory: at large H the weight tier needs it)
    return !p->dense && p->G == 1 && n_tiles == 1 && p->cfg.hidden % 4 == 0 && bp_box_units(units_max) <= 256 &&
           bp_tma_smem_bytes(p->G, p->BT, units_max) <= 8192 + 144 &&
           (p->cfg.flags & SRNN_FLAG_CLASS_BALANCE) == 0 && std::getenv("SRNN_NO_BP_TMA") == nullptr;
}

size_t smem_for(const srnn_plan* p, int units_max, int bt, int n_tiles, int vrows = 0) {
    const int hs_units = p->csplit ? p->hsplit : p->cfg.hidden;  // column split: one half of h staged
    size_t s = (static_cast<size_t>(hs_units) * elem_bytes(p->f16, bt) + 15) & ~static_cast<size_t>(15);
    if (p->csplit && vrows == 0) vrows = 2 * p->G * units_max;  // a CTA holds the rows of its pair's units
    const size_t zrows = std::max<size_t>(static_cast<size_t>(p->G) * units_max, vrows);  // zs: (virtual) rows
    s += (p->csplit ? 2 : 1) * zrows * bt * 4 + 2 * static_cast<size_t>(p->G) * units_max * bt * 4;  // zs + b'
    if (p->G >= 3) s += static_cast<size_t>(n_tiles) * units_max * bt * 4;  // LSTM c / GRU fp32 h
    if (bp_tma_ok(p, n_tiles, units_max)) s += static_cast<size_t>(bp_tma_smem_bytes(p->G, bt, units_max));  // TMA b' windows
    return s + 16;
}

// 3-D tensor map over b' [T][B][G*H] fp32: box {boxu units, bt samples, kBpWin steps}
bool encode_bprime_map(CUtensorMap* map, const float* bprime, int64_t GH, int B, int T, int boxu, int bt) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(GH), static_cast<cuuint64_t>(B), static_cast<cuuint64_t>(T)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(GH) * 4, static_cast<cuuint64_t>(GH) * 4 * B};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(boxu), static_cast<cuuint32_t>(bt), static_cast<cuuint32_t>(kBpWin)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(bprime), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void free_device(srnn_plan* p) {
    cudaFree(p->d_img);
    cudaFree(p->d_unit0);
    cudaFree(p->d_vunit0);
    cudaFree(p->d_perm);
    cudaFree(p->d_piece0);
    cudaFree(p->d_wslots);
    cudaFree(p->d_wearly);
    cudaFree(p->d_wx);
    cudaFree(p->d_wx16);
    cudaFree(p->d_x16);
    cudaFree(p->d_wx_hi);
    cudaFree(p->d_wx_lo);
    cudaFree(p->d_x_hi);
    cudaFree(p->d_x_lo);
    cudaFree(p->d_bias);
    cudaFree(p->d_bhn);
    cudaFree(p->d_bprime);
    cudaFree(p->d_xbuf);
    cudaFree(p->d_xdirty);
    cudaFree(p->d_status);
    cudaFree(p->d_x);
    cudaFree(p->d_h0);
    cudaFree(p->d_c0);
    cudaFree(p->d_y);
    cudaFree(p->d_hT);
    cudaFree(p->d_cT);
    cudaFree(p->d_prof);
    cudaFree(p->d_ready);
    cudaFree(p->d_progress);
    if (p->s_rec) cudaStreamDestroy(p->s_rec);
    if (p->s_out) cudaStreamDestroy(p->s_out);
    if (p->s_copy) cudaStreamDestroy(p->s_copy);
    if (p->h_status) cudaFreeHost(p->h_status);
    p->h_status = nullptr;
    for (cudaEvent_t& ev : p->ev_chunk)
        if (ev) cudaEventDestroy(ev);
    if (p->ev_in) cudaEventDestroy(p->ev_in);
    if (p->ev_rec) cudaEventDestroy(p->ev_rec);
    if (p->stream) cudaStreamDestroy(p->stream);
    p->d_img = nullptr;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
bool encode_fp16_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k_pad, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {k_pad, rows};
    cuuint64_t strides[1] = {k_pad * 2};
    cuuint32_t box[2] = {64, box_rows};  // 64 fp16 = one 128-byte swizzle row (srnn_gemm_tc.cu)
    cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 (tf32-split) operand map: 32 fp32 = one 128-byte swizzle row.
bool encode_f32_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k_pad, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {k_pad, rows};
    cuuint64_t strides[1] = {k_pad * 4};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Estimated cycles of one tile-step on the busiest CTA (planner cost model,
// DESIGN.md Sec. 5), calibrated on B200 at C2:
//   operate  = max(shared-memory wavefronts, issue over 4 SMSPs, the longest
//              warp's dependent LDS->FMA chain)
//   load     = poll rounds (one round trip each) + tagged-word ingress bytes
//   reduce   = xor-butterfly latency, epilogue per item round, exchange RTT.
double cost_model(const Layout& lay, int bt, int H, int n_tiles, bool f16, int inst) {
    const double wf = static_cast<double>(lay.wavefronts_max_cta) * (bt == 16 ? 2 : 1);
    const double instr_per_slot = f16 ? (3.0 + bt) : (2.0 + bt);
    const double issue = static_cast<double>(lay.issue_max_cta) * instr_per_slot / 4.0;
    const double chain = lay.slots_used * 11.0;
    int lg = 0;
    while ((1 << lg) < lay.lanes_per_row) ++lg;
    const double reduce = lg * (30.0 + 2.0 * bt);
    const double chunks = static_cast<double>(exchange_tile_bytes(H, f16, bt)) / 16.0;
    const double k = poll_slots(inst, f16, bt, false);
    const double groups = std::ceil(chunks / (lay.threads * k));
    const double load = groups * 900.0 + chunks * 16.0 / 48.0;
    int umax = 0;
    for (int c = 0; c < lay.num_ctas; ++c) umax = std::max(umax, lay.cta_unit0[c + 1] - lay.cta_unit0[c]);
    const double epi = std::ceil(static_cast<double>(umax) * bt / lay.threads) * 300.0;
    const double sync = lay.num_ctas > 1 ? 1200.0 : 600.0;
    if (std::getenv("SRNN_PLAN_LOG") != nullptr)
        std::fprintf(stderr, "srnn cost: C=%d L=%d threads=%d inst=%d wf=%.0f issue=%.0f chain=%.0f groups=%.0f "
                     "chunks=%.0f reduce=%.0f epi=%.0f sync=%.0f tiles=%d\n", lay.num_ctas, lay.lanes_per_row,
                     lay.threads, inst, wf, issue, chain, groups, chunks, reduce, epi, sync, n_tiles);
    return n_tiles * (std::max(std::max(wf, issue), chain) + load + reduce + epi + sync);
}

}  // namespace

// Exchange images, status words, b' buffer and the plan stream (sparse and dense plans).
srnn_status_t alloc_exchange(srnn_plan* p) {
    const srnn_config_t& c = p->cfg;
    p->tile_bytes = exchange_tile_bytes(c.hidden, p->f16 || p->dense, p->BT);
    p->xbuf_bytes = 2 * static_cast<size_t>(p->n_tiles_max) * p->tile_bytes;
    p->xbuf_valid_tiles = 0;  // the first launch writes the stale tags (kernel re-init)
    const size_t bp_elems = static_cast<size_t>(std::max(1, c.max_steps)) * c.batch * p->G * c.hidden;
    if (cudaMalloc(&p->d_xbuf, p->xbuf_bytes) != cudaSuccess ||
        cudaMalloc(&p->d_xdirty, sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p->d_status, sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p->d_bprime, bp_elems * sizeof(float)) != cudaSuccess ||
        cudaMemset(p->d_xbuf, 0, p->xbuf_bytes) != cudaSuccess ||
        cudaMemset(p->d_xdirty, 0, sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(p->d_status, 0, sizeof(int32_t)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)  // memsets complete before any non-blocking stream
        return SRNN_ERR_CUDA;
    return SRNN_OK;
}

// ---------------------------------------------------------------------------
// SRNN_FLAG_DENSE_TC: the dense persistent RNN comparator (SURVEY.md Sec.
// 8(f)1).  Same exchange, b' staging and epilogue as the
// sparse plan; U_r densified into mma.sync m16n8k16 A fragments.
// ---------------------------------------------------------------------------
size_t dense_smem(const srnn_plan* p, int umax) {
    size_t s = static_cast<size_t>(p->hs_rows) * 16;
    s += 3 * static_cast<size_t>(p->G) * umax * p->BT * 4;
    if (p->G == 4) s += static_cast<size_t>(p->n_tiles_max) * umax * p->BT * 4;
    s += 16 + 16;  // abort flag, alignment of the fragment tier
    s += static_cast<size_t>(std::max(0, p->dense_nf - p->dense_inst)) * kDenseThreads * 16;
    s += static_cast<size_t>(kDenseThreads / 32) * p->dense_mt * 16 * 8 * 4;  // partial tiles
    return s;
}

srnn_status_t create_dense(srnn_plan* p, srnn_plan_t* out) {
    const srnn_config_t& c = p->cfg;
    if (!p->f16 || p->G == 3) {
        delete p;
        return SRNN_ERR_UNSUPPORTED;  // fp16 fragments and fp16 h staging only; RNN and LSTM cells
    }
    int bt = c.batch > 4 ? 8 : 4;
    if (c.batch_tile == 4 || c.batch_tile == 8) bt = c.batch_tile;
    p->BT = bt;
    p->E = 16;
    p->n_tiles_max = (c.batch + bt - 1) / bt;
    const int kpw = ((c.hidden + 15) / 16 + 15) / 16;
    p->dense_kpw = kpw;
    p->hs_rows = 256 * kpw;
    if (!p->host_only) {
        DeviceGuard g(c.device);
        if (alloc_exchange(p) != SRNN_OK) {
            free_device(p);
            delete p;
            return SRNN_ERR_CUDA;
        }
    }
    *out = p;
    return SRNN_OK;
}

// Units -> CTAs, row tiles, fragment tiers, and the fragment image.
// Fragment f of warp w covers k-block kb = w * kpw + f / MT and row tile
// m = f % MT; lane (gid = lane / 4, tig = lane % 4) holds, as in the PTX ISA
// m16n8k16 A layout, {A[gid][2tig..+1], A[gid+8][2tig..+1], A[gid][2tig+8..+9],
// A[gid+8][2tig+8..+9]} (low half = lower column).
srnn_status_t pack_dense(srnn_plan* p, const int32_t* rowptr, const int32_t* col, const float* qval) {
    const int H = p->cfg.hidden, G = p->G;
    int reserve = 0;
    if (p->cfg.flags & SRNN_FLAG_RESERVE_SMS) {
        reserve = 4;
        if (const char* r = std::getenv("SRNN_RESERVE_SMS")) reserve = std::max(1, std::min(p->sm_count / 2, std::atoi(r)));
    }
    const int C = p->cfg.num_ctas > 0 ? p->cfg.num_ctas : std::max(1, std::min(p->sm_count - reserve, H));
    Layout lay;
    lay.num_ctas = C;
    lay.threads = kDenseThreads;
    lay.warps = kDenseThreads / 32;
    lay.lanes_per_row = 0;
    lay.cta_unit0.resize(C + 1);
    int umax = 0;
    for (int c = 0; c <= C; ++c) lay.cta_unit0[c] = static_cast<int>((static_cast<int64_t>(c) * H) / C);
    for (int c = 0; c < C; ++c) umax = std::max(umax, lay.cta_unit0[c + 1] - lay.cta_unit0[c]);
    const int mt = (G * umax + 15) / 16;
    if (mt > 2) return SRNN_ERR_NOT_ON_CHIP;  // > 32 rows per CTA: compiled for 1 or 2 row tiles
    const int kpw = p->dense_kpw, nf = mt * kpw;
    p->dense_mt = mt;
    p->dense_nf = nf;
    p->dense_inst = nf <= 8 ? 8 : 12;
    if (dense_smem(p, umax) > static_cast<size_t>(p->smem_optin)) return SRNN_ERR_NOT_ON_CHIP;
    const int W = lay.warps, NT = kDenseThreads;
    p->dense_img.assign(static_cast<size_t>(C) * nf * NT, make_uint4(0u, 0u, 0u, 0u));
    std::vector<uint16_t> blk;  // dense rows of one CTA: [G*U][kcols] fp16 bits (zero padded)
    const int kcols = p->hs_rows;
    for (int c = 0; c < C; ++c) {
        const int u0 = lay.cta_unit0[c], U = lay.cta_unit0[c + 1] - u0;
        blk.assign(static_cast<size_t>(mt) * 16 * kcols, 0);
        for (int q = 0; q < G; ++q)
            for (int u = 0; u < U; ++u) {
                const int r = q * U + u, grow = q * H + u0 + u;
                for (int i = rowptr[grow]; i < rowptr[grow + 1]; ++i)
                    blk[static_cast<size_t>(r) * kcols + col[i]] = float_to_half_rne(qval[i]);
            }
        auto pair = [&](int r, int k) -> uint32_t {
            return static_cast<uint32_t>(blk[static_cast<size_t>(r) * kcols + k]) |
                   (static_cast<uint32_t>(blk[static_cast<size_t>(r) * kcols + k + 1]) << 16);
        };
        for (int f = 0; f < nf; ++f)
            for (int w = 0; w < W; ++w)
                for (int lane = 0; lane < 32; ++lane) {
                    const int m = f % mt, kb = w * kpw + f / mt, gid = lane >> 2, tig = lane & 3;
                    const int r0 = m * 16 + gid, k0 = kb * 16 + 2 * tig;
                    uint4 a;
                    a.x = pair(r0, k0);
                    a.y = pair(r0 + 8, k0);
                    a.z = pair(r0, k0 + 8);
                    a.w = pair(r0 + 8, k0 + 8);
                    p->dense_img[(static_cast<size_t>(c) * nf + f) * NT + w * 32 + lane] = a;
                }
    }
    p->smem_bytes = dense_smem(p, umax);
    p->np_inst = 0;
    p->ns_slots = 0;
    p->model_cost = 0;
    p->regs = 128;  // host-only estimate; replaced by the compiled count
    p->lay = std::move(lay);
    return SRNN_OK;
}

extern "C" {

const char* srnn_status_string(srnn_status_t s) {
    switch (s) {
        case SRNN_OK: return "SRNN_OK";
        case SRNN_ERR_INVALID_VALUE: return "SRNN_ERR_INVALID_VALUE";
        case SRNN_ERR_NOT_ON_CHIP: return "SRNN_ERR_NOT_ON_CHIP";
        case SRNN_ERR_BAD_WEIGHTS: return "SRNN_ERR_BAD_WEIGHTS";
        case SRNN_ERR_STATE: return "SRNN_ERR_STATE";
        case SRNN_ERR_CUDA: return "SRNN_ERR_CUDA";
        case SRNN_ERR_TIMEOUT: return "SRNN_ERR_TIMEOUT";
        case SRNN_ERR_UNSUPPORTED: return "SRNN_ERR_UNSUPPORTED";
    }
    return "SRNN_ERR_UNKNOWN";
}

const char* srnn_version(void) { return "srnn 0.1 sm_100a"; }

srnn_status_t srnn_plan_create(const srnn_config_t* cfg, srnn_plan_t* out) {
    if (cfg == nullptr || out == nullptr) return SRNN_ERR_INVALID_VALUE;
    *out = nullptr;
    const srnn_config_t& c = *cfg;
    if (c.hidden < 1 || c.hidden > 65536 || c.input < 1 || c.batch < 1 || c.max_steps < 0) return SRNN_ERR_INVALID_VALUE;
    if (!(c.density >= 0.0f && c.density <= 1.0f)) return SRNN_ERR_INVALID_VALUE;
    if (c.cell != SRNN_CELL_RNN && c.cell != SRNN_CELL_LSTM && c.cell != SRNN_CELL_GRU) return SRNN_ERR_INVALID_VALUE;
    if (c.act < SRNN_ACT_RELU || c.act > SRNN_ACT_IDENTITY) return SRNN_ERR_INVALID_VALUE;
    if (c.prec != SRNN_PREC_FP32 && c.prec != SRNN_PREC_FP16W_FP32ACC) return SRNN_ERR_INVALID_VALUE;
    if (c.lanes_per_row != 0 &&
        (c.lanes_per_row < 1 || c.lanes_per_row > 32 || (c.lanes_per_row & (c.lanes_per_row - 1)) != 0))
        return SRNN_ERR_INVALID_VALUE;
    if (c.num_ctas < 0) return SRNN_ERR_INVALID_VALUE;
    if (c.batch_tile != 0 && c.batch_tile != 1 && c.batch_tile != 2 && c.batch_tile != 4 && c.batch_tile != 8 &&
        c.batch_tile != 16)
        return SRNN_ERR_INVALID_VALUE;

#ifndef SRNN_PROFILE
    if (c.flags & SRNN_FLAG_PROFILE) return SRNN_ERR_UNSUPPORTED;  // timestamps exist only in libsrnn_profile.so
#endif
    srnn_plan* p = new (std::nothrow) srnn_plan();
    if (!p) return SRNN_ERR_INVALID_VALUE;
    p->cfg = c;
    p->G = c.cell == SRNN_CELL_LSTM ? 4 : c.cell == SRNN_CELL_GRU ? 3 : 1;
    p->host_only = (c.flags & SRNN_FLAG_HOST_ONLY) != 0;
    if (const char* t = std::getenv("SRNN_TIMEOUT_MS")) p->timeout_ns = std::strtoull(t, nullptr, 10) * 1000000ull;
    // test hook: start the timestep tags near the u32 wrap so the wrap path (buffer clear +
    // epoch restart) is exercised in a few calls
    if (const char* t = std::getenv("SRNN_DEBUG_EPOCH0")) p->epoch = static_cast<uint32_t>(std::strtoull(t, nullptr, 10));
    if (!p->host_only) {
        DeviceGuard g(c.device);
        if (!g.ok) {
            delete p;
            return SRNN_ERR_CUDA;
        }
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, c.device) != cudaSuccess) {
            delete p;
            return SRNN_ERR_CUDA;
        }
        p->sm_count = prop.multiProcessorCount;
        p->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
        if (!prop.cooperativeLaunch) {
            delete p;
            return SRNN_ERR_UNSUPPORTED;
        }
    }
    if (c.num_ctas > p->sm_count) {
        delete p;
        return SRNN_ERR_INVALID_VALUE;
    }
    p->f16 = c.prec == SRNN_PREC_FP16W_FP32ACC && (c.flags & SRNN_FLAG_FP32_STAGING) == 0;
    p->dense = (c.flags & SRNN_FLAG_DENSE_TC) != 0;
    if (p->dense) return create_dense(p, out);
    // Batch tile: the paper's wide load interleaves 4 samples.  tile_for(split) is
    // the widest tile that fits (h staging in shared memory; 16-bit staged offsets for fp16 tiles
    // <= 4 and fp32: hs <= 64 KB, the staged half under the column split), 0 if none does.
    const int umax_guess = (c.hidden + p->sm_count - 1) / p->sm_count;
    const int hsplit = ((c.hidden + 1) / 2 + 7) & ~7;  // column split: the half boundary on a 16-byte chunk
    auto tile_for = [&](bool split) -> int {
        p->csplit = split;
        p->hsplit = split ? hsplit : 0;
        int bt = c.batch >= 4 ? 4 : (c.batch >= 2 ? 2 : 1);
        if (p->f16 && c.batch >= 8) bt = 8;    // fp16: 8 samples per LDS.128 (one exchange round for B = 8)
        if (p->f16 && c.batch >= 16) bt = 16;  // fp16: two planes of 8 (every extra tile costs a whole exchange)
        if (c.batch_tile == 1 || c.batch_tile == 2 || c.batch_tile == 4 ||
            ((c.batch_tile == 8 || c.batch_tile == 16) && p->f16))
            bt = c.batch_tile;
        if (const char* e = std::getenv("SRNN_BT")) {  // experiment override: batch tile width
            const int v = std::atoi(e);
            if (v == 1 || v == 2 || v == 4 || ((v == 8 || v == 16) && p->f16)) bt = v;
        }
        while (bt > 1 && bt > c.batch) bt /= 2;
        if (split && bt > 8) bt = 8;  // the column split stages one plane of h
        while (bt > 1 && smem_for(p, umax_guess, bt, (c.batch + bt - 1) / bt) > static_cast<size_t>(p->smem_optin)) bt /= 2;
        const int64_t hs_units = split ? hsplit : c.hidden;
        while (bt > 1 && (!p->f16 || bt < 8) && hs_units * elem_bytes(p->f16, bt) > 65536) bt /= 2;
        if ((!p->f16 || bt < 8) && hs_units * elem_bytes(p->f16, bt) > 65536) return 0;
        return bt;
    };
    // Column split (SRNN_FLAG_COLUMN_SPLIT, or automatically when the unsplit layer needs more batch
    // tiles -- each a whole exchange round per step -- or does not fit the offset format at all)
    const bool split_ok = !(c.flags & (SRNN_FLAG_CLASS_BALANCE | SRNN_FLAG_GRID_SYNC)) && hsplit < c.hidden &&
                          p->sm_count >= 2 && !(c.num_ctas != 0 && (c.num_ctas & 1));
    bool split = (c.flags & SRNN_FLAG_COLUMN_SPLIT) != 0;
    if (split && !split_ok) {
        delete p;
        return SRNN_ERR_UNSUPPORTED;
    }
    if (!split && split_ok && c.hidden >= 2 * p->sm_count && std::getenv("SRNN_NO_AUTO_SPLIT") == nullptr) {
        const int b0 = tile_for(false), b1 = tile_for(true);
        split = b1 > 0 && (b0 == 0 || (c.batch + b1 - 1) / b1 < (c.batch + b0 - 1) / b0);
        p->auto_split = split;
        p->bt_unsplit = b0;
    }
    int bt = tile_for(split);
    // Register budget for the expected pairs: two registers per pair in the hoisted
    // format, at most ~75% of each SM's 64K registers.  Checked before the offset-format
    // limit below: a layer that cannot be on-chip at all is NOT_ON_CHIP, not UNSUPPORTED.
    const double exp_pairs = static_cast<double>(c.density) * p->G * c.hidden * static_cast<double>(c.hidden);
    // plus the shared-memory weight tier (up to ~60% of shared memory)
    const double reg_capacity_pairs =
        (0.75 * 65536.0 / (p->f16 ? 1.0 : 2.0) + 0.6 * p->smem_optin / (p->f16 ? 4.0 : 8.0)) * p->sm_count;
    if (exp_pairs > reg_capacity_pairs) {
        delete p;
        return SRNN_ERR_NOT_ON_CHIP;
    }
    if (bt == 0) {  // the staged h does not fit the 16-bit offsets of the register pairs
        delete p;
        return SRNN_ERR_UNSUPPORTED;
    }
    p->BT = bt;
    p->E = elem_bytes(p->f16, bt);
    p->n_tiles_max = (c.batch + bt - 1) / bt;
    if (smem_for(p, umax_guess, bt, p->n_tiles_max) > static_cast<size_t>(p->smem_optin)) {
        delete p;
        return SRNN_ERR_NOT_ON_CHIP;  // h staging alone exceeds shared memory
    }
    if (!p->host_only) {
        DeviceGuard g(c.device);
        if (alloc_exchange(p) != SRNN_OK) {
            free_device(p);
            delete p;
            return SRNN_ERR_CUDA;
        }
    }
    *out = p;
    return SRNN_OK;
}

srnn_status_t srnn_plan_query(srnn_plan_t p, srnn_plan_info_t* out) {
    if (!p || !out) return SRNN_ERR_INVALID_VALUE;
    std::memset(out, 0, sizeof(*out));
    out->sm_count = p->sm_count;
    out->batch_tile = p->BT;
    out->num_batch_tiles = p->n_tiles_max;
    out->fits = 1;
    out->column_split = p->csplit ? 1 : 0;
    out->column_half = p->csplit ? p->hsplit : 0;
    out->staged = p->staged ? 1 : 0;
    out->early_chunks = p->staged ? p->early_chunks : 0;
    if (p->loaded) {
        const Layout& l = p->lay;
        out->num_ctas = l.num_ctas;
        out->threads_per_cta = l.threads;
        out->lanes_per_row = l.lanes_per_row;
        out->pairs_per_lane = p->np_inst;
        out->slots_used = l.slots_used;
        const std::vector<int32_t>& u0 = p->csplit ? p->unit0_real : l.cta_unit0;  // units a CTA publishes
        int umax = 0;
        for (int c = 0; c < l.num_ctas; ++c) umax = std::max(umax, u0[c + 1] - u0[c]);
        out->units_per_cta_max = umax;
        out->regs_per_thread = p->regs;
        out->spill_bytes = p->spill_bytes;
        out->packed_registers = p->f16 ? 1 : 0;
        out->nnz = p->nnz;
        out->slots_total = l.slots_total;
        out->smem_bytes_per_cta = static_cast<int64_t>(p->smem_bytes);
        out->smem_weight_bytes_per_cta = static_cast<int64_t>(p->ns_slots) * l.threads * (p->f16 ? 4 : 8);
        out->image_slots_per_lane = p->np_inst + p->ns_slots;
        out->model_cycles_per_step = static_cast<int64_t>(p->model_cost);
        out->weight_image_bytes = static_cast<int64_t>(l.num_ctas) * (p->np_inst + p->ns_slots) * l.threads *
                                  (p->f16 ? 4 : 8);
        if (p->dense) {
            out->packed_registers = 0;
            out->dense_m_tiles = p->dense_mt;
            out->dense_kblocks_per_warp = p->dense_kpw;
            out->dense_frags_reg = std::min(p->dense_inst, p->dense_nf);
            out->dense_frags_smem = std::max(0, p->dense_nf - p->dense_inst);
            out->weight_image_bytes = static_cast<int64_t>(l.num_ctas) * p->dense_nf * l.threads * 16;
            out->smem_weight_bytes_per_cta = static_cast<int64_t>(out->dense_frags_smem) * l.threads * 16;
            out->image_slots_per_lane = 0;
        }
        const int planes = p->BT == 16 ? 2 : 1;  // two LDS.128 per pair at BT = 16
        out->wavefronts_per_step_max = l.wavefronts_max_cta * planes;
        out->wavefronts_per_step_ideal = l.wavefronts_ideal_cta * planes;
        out->conflict_wavefronts = l.conflicts_max_cta * planes;
    }
    return SRNN_OK;
}

srnn_status_t srnn_load_weights(srnn_plan_t p, const int32_t* rowptr, const int32_t* col, const float* val,
                                int64_t nnz, const float* wx, const float* bias) {
    if (!p || !rowptr || (nnz > 0 && (!col || !val)) || !wx || nnz < 0) return SRNN_ERR_INVALID_VALUE;
    const int H = p->cfg.hidden, G = p->G, R = G * H;
    // ---- validate CSR (S:125 duplicates; rowptr monotone; col range) ----
    if (rowptr[0] != 0 || rowptr[R] != nnz) return SRNN_ERR_BAD_WEIGHTS;
    // every row range inside [0, nnz] before any column is read
    for (int r = 0; r < R; ++r)
        if (rowptr[r + 1] < rowptr[r] || rowptr[r + 1] > nnz) return SRNN_ERR_BAD_WEIGHTS;
    for (int r = 0; r < R; ++r) {
        std::vector<int32_t> cs(col + rowptr[r], col + rowptr[r + 1]);
        for (int32_t v : cs)
            if (v < 0 || v >= H) return SRNN_ERR_BAD_WEIGHTS;
        std::sort(cs.begin(), cs.end());
        for (size_t i = 1; i < cs.size(); ++i)
            if (cs[i] == cs[i - 1]) return SRNN_ERR_BAD_WEIGHTS;
    }
    const bool fp16 = p->cfg.prec == SRNN_PREC_FP16W_FP32ACC;
    // fp16 mode: RNE-quantise the values once.
    std::vector<float> qval(val, val + nnz);
    if (fp16)
        for (auto& v : qval) v = half_to_float(float_to_half_rne(v));
    PackInput in;
    in.H = H;
    in.G = G;
    in.rowptr = rowptr;
    in.col = col;
    in.val = qval.data();
    in.BT = p->BT;
    in.E = p->BT == 16 ? 16 : p->E;  // BT = 16 gathers two 16-byte planes: the bank model of BT = 8, twice
    in.naive = (p->cfg.flags & SRNN_FLAG_NAIVE_LAYOUT) != 0;

    if (p->dense) {
        const srnn_status_t st = pack_dense(p, rowptr, col, qval.data());
        if (st != SRNN_OK) return st;
        p->nnz = nnz;
    } else {
    // ---- search (num_ctas, lanes_per_row, slot budget) ----
    bool spill_strict = true;
search_again:
    std::vector<int> cands_c;
    if (p->cfg.num_ctas > 0) {
        cands_c.push_back(std::min(p->cfg.num_ctas, H));  // every CTA owns >= 1 unit (its publish writes the pad word)
    } else {
        int reserve = 0;
        if (p->cfg.flags & SRNN_FLAG_RESERVE_SMS) {
            reserve = 4;
            if (const char* r = std::getenv("SRNN_RESERVE_SMS")) reserve = std::max(1, std::min(p->sm_count / 2, std::atoi(r)));
        }
        const int cmax = std::max(1, std::min(p->sm_count - reserve, H));
        cands_c.push_back(cmax);
        for (int cc = cmax / 2; cc >= 1; cc /= 2) cands_c.push_back(cc);
    }
    // Column split: one even CTA count (pairs = clusters); the packer sees a virtual matrix whose
    // units are (pair unit, column half): CTA 2q + r holds the rows of pair q's units restricted
    // to the columns of half r, renumbered from the half's first column (its hs position).
    std::vector<int32_t> v_rowptr, v_col, v_unit0;
    std::vector<float> v_val;
    if (p->csplit) {
        int C = cands_c[0] & ~1;
        if (C < 2 || H < C) return SRNN_ERR_UNSUPPORTED;
        cands_c.assign(1, C);
        const int NQ = C / 2, Hc = p->hsplit;
        v_unit0.assign(C + 1, 0);
        p->unit0_real.assign(C + 1, 0);
        std::vector<int32_t> vreal(2 * static_cast<size_t>(H)), vhalf(2 * static_cast<size_t>(H));
        for (int q = 0; q < NQ; ++q) {
            const int q0 = static_cast<int>(static_cast<int64_t>(q) * H / NQ);
            const int q1 = static_cast<int>(static_cast<int64_t>(q + 1) * H / NQ), UQ = q1 - q0;
            v_unit0[2 * q] = 2 * q0;
            v_unit0[2 * q + 1] = 2 * q0 + UQ;
            p->unit0_real[2 * q] = q0;
            p->unit0_real[2 * q + 1] = q0 + UQ / 2;
            for (int r = 0; r < 2; ++r)
                for (int i = 0; i < UQ; ++i) {
                    vreal[2 * q0 + r * UQ + i] = q0 + i;
                    vhalf[2 * q0 + r * UQ + i] = r;
                }
        }
        v_unit0[C] = 2 * H;
        p->unit0_real[C] = H;
        v_rowptr.assign(static_cast<size_t>(G) * 2 * H + 1, 0);
        v_col.reserve(nnz);
        v_val.reserve(nnz);
        for (int g = 0; g < G; ++g)
            for (int v = 0; v < 2 * H; ++v) {
                const int32_t rr = g * H + vreal[v], hf = vhalf[v];
                for (int32_t i = rowptr[rr]; i < rowptr[rr + 1]; ++i) {
                    const int32_t cc = col[i];
                    if ((cc >= Hc) == (hf == 1)) {
                        v_col.push_back(cc - hf * Hc);
                        v_val.push_back(qval[i]);
                    }
                }
                v_rowptr[static_cast<size_t>(g) * 2 * H + v + 1] = static_cast<int32_t>(v_col.size());
            }
        in.H = 2 * H;
        in.rowptr = v_rowptr.data();
        in.col = v_col.data();
        in.val = v_val.data();
        in.cta_unit0 = v_unit0.data();
    }
    std::vector<int> cands_l;
    if (p->cfg.lanes_per_row > 0)
        cands_l.push_back(p->cfg.lanes_per_row);
    else
        cands_l = {32, 16, 8, 4, 2, 1};
    double best_cost = 1e300;
    Layout best;
    int best_inst = 0, best_ns = 0;
    bool any = false;
    const int pair_bytes = p->f16 ? 4 : 8;
    const int P = p->E >= 4 ? 128 / p->E : 32;  // lanes per shared-memory phase
    const bool plan_log = std::getenv("SRNN_PLAN_LOG") != nullptr;  // diagnostics: every candidate to stderr
    // Evaluate one (CTAs, lanes per row, slot budget) candidate.
    const bool class_balance = (p->cfg.flags & SRNN_FLAG_CLASS_BALANCE) != 0 && !in.naive;
    if (class_balance) {  // heavy rows (> 1.25 x the mean length) are handled as several pieces
        const double mean = static_cast<double>(nnz) / std::max(1, R);
        in.piece_cap = std::max(32, static_cast<int>(std::ceil(1.25 * mean)));
    }
    std::vector<std::vector<int32_t>> perm_uop, perm_pou;  // per candidate CTA count
    std::vector<int> perm_c;
    auto use_perm = [&](int C) {
        if (!class_balance) return;
        size_t i = 0;
        while (i < perm_c.size() && perm_c[i] != C) ++i;
        if (i == perm_c.size()) {
            perm_c.push_back(C);
            perm_uop.emplace_back();
            perm_pou.emplace_back();
            class_balanced_units(in, C, 8, &perm_uop.back(), &perm_pou.back());
        }
        in.unit_of_pos = perm_uop[i].data();
        in.pos_of_unit = perm_pou[i].data();
    };
    int best_perm_c = -1;
    // Compiled instances whose registers spill are avoided (SURVEY Sec. 8 d-vi: 0 spill bytes):
    // the search takes the next wider register instance that fits, and only if no spill-free
    // plan exists at all does it accept a spilling one (second pass).
    auto spills = [&](int inst, bool k8, bool staged = false) -> bool {
        if (p->host_only) return false;
        const int key = inst * 256 + p->BT * 4 + (k8 ? 2 : 0) + (p->f16 ? 1 : 0) + (p->csplit ? 64 : 0) + (staged ? 128 : 0);
        for (auto& kv : p->spill_cache)
            if (kv.first == key) return kv.second;
        RecParams q{};
        q.threads = 32;
        q.k8 = k8 ? 1 : 0;
        q.csplit = p->csplit ? 1 : 0;
        static const int32_t dummy_early = 0;  // selects the staged instance (query only, never read)
        q.warp_early = staged ? &dummy_early : nullptr;
        int regs[2] = {0, 0};
        const bool sp = launch_recurrent(inst, p->BT, G, p->f16 ? 1 : 0, q, 1, 0, nullptr, true, regs, nullptr) == 0 &&
                        regs[1] > 0;
        p->spill_cache.emplace_back(key, sp);
        return sp;
    };
    auto try_layout = [&](int C, int L, int np, int reg_cap, int64_t ns_cap) {
        Layout lay;
        use_perm(C);
        if (!pack_layout(in, C, L, np, &lay)) return;
        if (lay.threads > 1024) return;
        const int su = std::max(1, lay.slots_used);
        int inst = inst_for(su, p->f16, p->BT);
        int ns = 0;
        if (inst < 0 || inst > reg_cap) {  // registers + shared-memory tier
            inst = reg_cap;
            ns = ((su - reg_cap) + 3) & ~3;
            if (ns > ns_cap) return;
        }
        if (spill_strict && spills(inst, false)) {  // next wider spill-free instance under the thread cap
            int alt = -1;
            for (int i = 0; i < kNumNP; ++i)
                if (kNPList[i] > inst && kNPList[i] <= reg_cap && !spills(kNPList[i], false)) {
                    alt = kNPList[i];
                    break;
                }
            if (alt < 0) return;
            inst = alt;
            ns = su > inst ? ((su - inst) + 3) & ~3 : 0;
        }
        if (lay.vrows_max > G * ((H + C - 1) / C)) {  // pieces: more zs rows (and maybe threads)
            int um = 0;
            for (int c = 0; c < C; ++c) um = std::max(um, lay.cta_unit0[c + 1] - lay.cta_unit0[c]);
            if (lay.threads > max_threads_for(inst, p->f16, p->BT) ||
                smem_for(p, um, p->BT, p->n_tiles_max, lay.vrows_max) + 16 +
                        static_cast<size_t>(ns) * lay.threads * (p->f16 ? 4 : 8) >
                    static_cast<size_t>(p->smem_optin))
                return;
        }
        double cst = cost_model(lay, p->BT, p->csplit ? p->hsplit : H, p->n_tiles_max, p->f16, inst);
        if (ns > 0) cst += static_cast<double>(ns) * lay.warps * 2.0;  // weight LDS + issue per smem slot
        cst += 2.0 * inst;  // tie-break toward the smaller register instance (code size)
        if (plan_log)
            std::fprintf(stderr, "srnn plan: C=%d L=%d np=%d slots=%d inst=%d ns=%d threads=%d wf=%lld issue=%lld cost=%.0f\n",
                         C, L, np, su, inst, ns, lay.threads, static_cast<long long>(lay.wavefronts_max_cta),
                         static_cast<long long>(lay.issue_max_cta), cst);
        if (cst < best_cost) {
            best_cost = cst;
            best = std::move(lay);
            best_inst = inst;
            best_ns = ns;
            best_perm_c = C;
            any = true;
        }
    };
    struct Cand { int C, L, np0, reg_cap; int64_t ns_cap; };
    std::vector<Cand> feasible;
    // phase 1: the minimum slot budget of every (CTAs, lanes per row)
    for (int C : cands_c) {
        const int umax = (H + C - 1) / C;
        const size_t smem_base = smem_for(p, umax, p->BT, p->n_tiles_max);
        if (smem_base > static_cast<size_t>(p->smem_optin)) continue;
        // lower bound: ideal wavefronts of the busiest CTA (every phase full, no conflicts)
        int64_t pairs_max = 0;
        for (int c = 0; c < C; ++c) {
            const int ua = static_cast<int>((static_cast<int64_t>(c) * H) / C);
            const int ub = static_cast<int>((static_cast<int64_t>(c + 1) * H) / C);
            int64_t pc = 0;
            for (int g = 0; g < G; ++g) pc += rowptr[g * H + ub] - rowptr[g * H + ua];
            pairs_max = std::max(pairs_max, pc);
        }
        if (any && static_cast<double>(pairs_max) / P * p->n_tiles_max > best_cost) continue;
        for (int L : cands_l) {
            const int rows_max = (p->csplit ? 2 : 1) * G * umax;  // column split: the pair's rows
            const int threads = ((rows_max * L + 31) / 32) * 32;
            if (threads > 1024) continue;
            int reg_cap = -1;  // largest register instance whose thread cap admits this CTA size
            for (int i = 0; i < kNumNP; ++i)
                if (kNPList[i] <= max_np(p->f16, p->BT) && threads <= max_threads_for(kNPList[i], p->f16, p->BT)) reg_cap = kNPList[i];
            if (reg_cap < 0) continue;
            if (std::getenv("SRNN_FORCE_SMEM_TIER") != nullptr) reg_cap = kNPList[0];  // test hook
            const int64_t ns_cap =
                (static_cast<int64_t>(p->smem_optin) - static_cast<int64_t>(smem_base) - 16) / (threads * pair_bytes);
            const int np0 = std::max(1, min_np(in, L));
            if (np0 > reg_cap + ns_cap) continue;
            if (any && np0 * 11.0 * p->n_tiles_max > best_cost) continue;  // dependent slot chain bound
            feasible.push_back({C, L, np0, reg_cap, ns_cap});
            try_layout(C, L, np0, reg_cap, ns_cap);
        }
    }
    // phase 2: looser slot budgets (bank-aware slack) for the best (CTAs, lanes per row)
    if (any && !in.naive) {
        const int bc = best.num_ctas, bl = best.lanes_per_row;
        for (const Cand& f : feasible) {
            if (f.C != bc || f.L != bl) continue;
            for (int extra : {1, 2, 4, std::max(1, f.np0 / 8), std::max(2, f.np0 / 4)})
                try_layout(f.C, f.L, f.np0 + extra, f.reg_cap, f.ns_cap);
        }
    }
    if (!any && p->f16 && p->BT == 16 && p->cfg.batch_tile != 16) {
        // the 16-sample tile's h staging left no room for the weights: 8-sample tiles
        p->BT = 8;
        p->E = elem_bytes(true, 8);
        p->n_tiles_max = (p->cfg.batch + 7) / 8;  // exchange bytes: ceil(B/8)*16H <= ceil(B/16)*32H, xbuf fits
        p->tile_bytes = exchange_tile_bytes(H, true, 8);
        p->xbuf_valid_tiles = 0;
        in.BT = 8;
        in.E = 16;
        goto search_again;
    }
    if (!any && spill_strict && !p->host_only) {  // only spilling instances fit: accept them
        spill_strict = false;
        goto search_again;
    }
    if (!any && p->csplit && p->auto_split && p->bt_unsplit > 0) {
        // the automatic column split doubles each CTA's rows: if its lanes cannot hold the half
        // rows, plan the unsplit layer (more batch tiles) instead
        p->csplit = p->auto_split = false;
        p->hsplit = 0;
        p->unit0_real.clear();
        p->BT = p->bt_unsplit;
        p->E = elem_bytes(p->f16, p->BT);
        p->n_tiles_max = (p->cfg.batch + p->BT - 1) / p->BT;
        p->tile_bytes = exchange_tile_bytes(H, p->f16, p->BT);
        p->xbuf_valid_tiles = 0;
        if (!p->host_only) {
            DeviceGuard g(p->cfg.device);
            cudaFree(p->d_xbuf);
            p->d_xbuf = nullptr;
            p->xbuf_bytes = 2 * static_cast<size_t>(p->n_tiles_max) * p->tile_bytes;
            if (cudaMalloc(&p->d_xbuf, p->xbuf_bytes) != cudaSuccess ||
                cudaMemset(p->d_xbuf, 0, p->xbuf_bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
                return SRNN_ERR_CUDA;
        }
        in.H = H;
        in.rowptr = rowptr;
        in.col = col;
        in.val = qval.data();
        in.cta_unit0 = nullptr;
        in.BT = p->BT;
        in.E = p->BT == 16 ? 16 : p->E;
        spill_strict = true;
        goto search_again;
    }
    if (!any) return SRNN_ERR_NOT_ON_CHIP;
    // Partial progress (SRNN_FLAG_STAGED): re-pack the chosen (CTAs, lanes per row)
    // with each warp's slots in two stages -- the pairs whose column lies in the first
    // early_chunks exchange chunks (the chunks every loader thread fetches first, j = 0), then
    // the rest -- at the smallest slot budget that fits a compiled staged instance.
    p->staged = false;
    p->early_chunks = 0;
    {
        bool want = (p->cfg.flags & SRNN_FLAG_STAGED) != 0;
        if (const char* es = std::getenv("SRNN_STAGED")) want = std::atoi(es) != 0;  // A/B override
        const int64_t chunks = exchange_tile_bytes(H, p->f16, p->BT) / 16;
        if (plan_log && want)
            std::fprintf(stderr, "srnn plan staged: f16=%d BT=%d ns=%d csplit=%d chunks=%lld K=%d threads=%d\n", p->f16,
                         p->BT, best_ns, p->csplit, static_cast<long long>(chunks), poll_slots(best_inst, true, p->BT, false),
                         best.threads);
        if (want && p->f16 && (p->BT == 4 || p->BT == 8) && best_ns == 0 && !p->csplit && !in.naive &&
            chunks <= static_cast<int64_t>(poll_slots(best_inst, true, p->BT, false)) * best.threads) {
            int64_t ec = std::min<int64_t>(best.threads, chunks / 2);
            if (const char* e = std::getenv("SRNN_EARLY_CHUNKS")) ec = std::atoi(e);
            if (ec > 0 && ec < chunks) {
                use_perm(best_perm_c);
                PackInput si = in;
                si.early_pos = static_cast<int32_t>(ec * 16 / p->E);
                si.early_align = operate_group_slots(true, p->BT);
                for (int np = best.np_budget; np <= best.np_budget + 12; ++np) {
                    Layout sl;
                    if (!pack_layout(si, best.num_ctas, best.lanes_per_row, np, &sl)) continue;
                    const int inst = inst_for(std::max(1, sl.slots_used), true, p->BT);
                    if (plan_log)
                        std::fprintf(stderr, "srnn plan staged: np=%d slots=%d inst=%d wf=%lld\n", np, sl.slots_used, inst,
                                     static_cast<long long>(sl.wavefronts_max_cta));
                    if (inst < 0 || !staged_compiled(inst, true, p->BT) ||
                        sl.threads > max_threads_for(inst, true, p->BT) || (spill_strict && spills(inst, false, true)))
                        break;
                    best = std::move(sl);
                    best_inst = inst;
                    p->staged = true;
                    p->early_chunks = static_cast<int>(ec);
                    break;
                }
            }
        }
    }
    // Re-pack at the chosen instance width so the image has np_inst slots.
    Layout fin;
    {
        // pack with the same budget, then widen the image to np_inst slots (padding)
        fin = best;
        const int width = best_inst + best_ns;
        if (best.np_budget != width) {
            Layout w = best;
            w.np_budget = width;
            const size_t n = static_cast<size_t>(w.num_ctas) * width * w.threads;
            w.col.assign(n, 0);
            w.val.assign(n, 0.0f);
            w.row.assign(n, -1);
            const int nslot = std::min(best.np_budget, width);
            for (int c = 0; c < w.num_ctas; ++c)
                for (int i = 0; i < nslot; ++i)
                    for (int t = 0; t < w.threads; ++t) {
                        w.col[w.idx(c, i, t)] = best.col[best.idx(c, i, t)];
                        w.val[w.idx(c, i, t)] = best.val[best.idx(c, i, t)];
                        w.row[w.idx(c, i, t)] = best.row[best.idx(c, i, t)];
                    }
            fin = std::move(w);
        }
    }
    int umax = 0;
    {
        const std::vector<int32_t>& u0 = p->csplit ? p->unit0_real : fin.cta_unit0;
        for (int c = 0; c < fin.num_ctas; ++c) umax = std::max(umax, u0[c + 1] - u0[c]);
    }
    p->smem_bytes = smem_for(p, umax, p->BT, p->n_tiles_max, fin.vrows_max) + 16 +
                    static_cast<size_t>(best_ns) * fin.threads * pair_bytes;
    p->np_inst = best_inst;
    // A plan whose threads own more exchange chunks than the default instance polls at once
    // (poll_slots) takes the 8-slot instance of the same width, where one is compiled,
    // instead of paying another poll round trip per step.
    {
        const int ksmall = poll_slots(best_inst, p->f16, p->BT, false);
        const int64_t chunks = exchange_tile_bytes(H, p->f16, p->BT) / 16;  // 16-byte chunks per tile
        const int64_t c = (chunks + best.threads - 1) / best.threads;       // per thread
        p->k8 = !p->csplit && !p->staged && k8_compiled(best_inst, p->f16, p->BT) && ksmall < 8 &&
                (c + 7) / 8 < (c + ksmall - 1) / ksmall;
        if (p->k8 && spills(best_inst, true) && !spills(best_inst, false)) p->k8 = false;  // spill-free first
    }
    p->unit_of_pos.clear();
    p->pos_of_unit.clear();
    if (class_balance) {
        for (size_t i = 0; i < perm_c.size(); ++i)
            if (perm_c[i] == best_perm_c) {
                p->unit_of_pos = perm_uop[i];
                p->pos_of_unit = perm_pou[i];
            }
    }
    p->model_cost = best_cost;
    p->ns_slots = best_ns;
    p->lay = std::move(fin);
    p->nnz = nnz;
    p->regs = (p->f16 ? 1 : 2) * best_inst + 60;  // host-only estimate; replaced by the compiled count below
    }  // sparse search

    if (!p->host_only) {
        DeviceGuard g(p->cfg.device);
        const Layout& l = p->lay;
        const size_t n = static_cast<size_t>(l.num_ctas) * (p->np_inst + p->ns_slots) * l.threads;
        cudaFree(p->d_img);
        cudaFree(p->d_unit0);
        cudaFree(p->d_wslots);
        cudaFree(p->d_wx);
        cudaFree(p->d_bias);
        p->d_img = nullptr;
        cudaFree(p->d_wearly);
        p->d_unit0 = p->d_wslots = p->d_wearly = nullptr;
        p->d_wx = p->d_bias = nullptr;
        cudaError_t e = cudaSuccess;
        if (p->dense) {
            const size_t nb = p->dense_img.size() * sizeof(uint4);
            e = cudaMalloc(&p->d_img, nb);
            if (e == cudaSuccess) e = cudaMemcpy(p->d_img, p->dense_img.data(), nb, cudaMemcpyHostToDevice);
            std::vector<uint4>().swap(p->dense_img);
        } else if (p->f16) {
            std::vector<uint32_t> img(n);
            const bool perm = !p->pos_of_unit.empty();
            for (size_t i = 0; i < n; ++i) {
                const int32_t pos = perm ? p->pos_of_unit[l.col[i]] : l.col[i];  // hs position of the column
                img[i] = (static_cast<uint32_t>(p->BT >= 8 ? pos : pos * p->E) << 16) | float_to_half_rne(l.val[i]);
            }
            e = cudaMalloc(&p->d_img, n * 4);
            if (e == cudaSuccess) e = cudaMemcpy(p->d_img, img.data(), n * 4, cudaMemcpyHostToDevice);
        } else {
            std::vector<uint2> img(n);
            const bool perm = !p->pos_of_unit.empty();
            for (size_t i = 0; i < n; ++i) {
                uint32_t b;
                std::memcpy(&b, &l.val[i], 4);
                const int32_t pos = perm ? p->pos_of_unit[l.col[i]] : l.col[i];
                img[i] = make_uint2(static_cast<uint32_t>(pos * p->E), b);
            }
            e = cudaMalloc(&p->d_img, n * 8);
            if (e == cudaSuccess) e = cudaMemcpy(p->d_img, img.data(), n * 8, cudaMemcpyHostToDevice);
        }
        const size_t wx_n = static_cast<size_t>(R) * p->cfg.input;
        cudaFree(p->d_perm);
        cudaFree(p->d_piece0);
        p->d_perm = nullptr;
        p->d_piece0 = nullptr;
        if (e == cudaSuccess && !l.piece0.empty()) {
            e = cudaMalloc(&p->d_piece0, l.piece0.size() * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(p->d_piece0, l.piece0.data(), l.piece0.size() * 4, cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess && !p->unit_of_pos.empty()) {
            e = cudaMalloc(&p->d_perm, p->unit_of_pos.size() * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(p->d_perm, p->unit_of_pos.data(), p->unit_of_pos.size() * 4, cudaMemcpyHostToDevice);
        }
        // units each CTA finalises and publishes (column split: its half of the pair's units; the
        // packed layout's ranges are then the virtual (pair unit, half) ones)
        const std::vector<int32_t>& u0v = p->csplit ? p->unit0_real : l.cta_unit0;
        if (e == cudaSuccess) e = cudaMalloc(&p->d_unit0, u0v.size() * 4);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_unit0, u0v.data(), u0v.size() * 4, cudaMemcpyHostToDevice);
        cudaFree(p->d_vunit0);
        p->d_vunit0 = nullptr;
        if (e == cudaSuccess && p->csplit) e = cudaMalloc(&p->d_vunit0, l.cta_unit0.size() * 4);
        if (e == cudaSuccess && p->csplit)
            e = cudaMemcpy(p->d_vunit0, l.cta_unit0.data(), l.cta_unit0.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_wslots, l.warp_slots.size() * 4);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_wslots, l.warp_slots.data(), l.warp_slots.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess && p->staged) {
            e = cudaMalloc(&p->d_wearly, l.warp_early.size() * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(p->d_wearly, l.warp_early.data(), l.warp_early.size() * 4, cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess) e = cudaMalloc(&p->d_wx, wx_n * 4);
        if (e == cudaSuccess) e = cudaMemcpy(p->d_wx, wx, wx_n * 4, cudaMemcpyHostToDevice);
        cudaFree(p->d_wx16);
        cudaFree(p->d_x16);
        p->d_wx16 = p->d_x16 = nullptr;
        cudaFree(p->d_wx_hi);
        cudaFree(p->d_wx_lo);
        cudaFree(p->d_x_hi);
        cudaFree(p->d_x_lo);
        p->d_wx_hi = p->d_wx_lo = p->d_x_hi = p->d_x_lo = nullptr;
        // fp32 mode, opt-in (SRNN_FLAG_FP32_TC_GEMM): the 3xTF32 tensor-core projection
        p->tf32x3 = !fp16 && (p->cfg.flags & SRNN_FLAG_FP32_TC_GEMM) != 0;
        if (e == cudaSuccess && p->tf32x3) {
            const int I = p->cfg.input;
            p->k_pad4 = (I + 3) & ~3;
            const size_t xrows = static_cast<size_t>(std::max(1, p->cfg.max_steps)) * p->cfg.batch;
            const size_t wn = static_cast<size_t>(R) * p->k_pad4, xn = xrows * p->k_pad4;
            e = cudaMalloc(&p->d_wx_hi, wn * 4);
            if (e == cudaSuccess) e = cudaMalloc(&p->d_wx_lo, wn * 4);
            if (e == cudaSuccess) e = cudaMalloc(&p->d_x_hi, xn * 4);
            if (e == cudaSuccess) e = cudaMalloc(&p->d_x_lo, xn * 4);
            if (e == cudaSuccess &&
                launch_split_tf32(p->d_wx, p->d_wx_hi, p->d_wx_lo, R, I, p->k_pad4, nullptr) != 0)
                e = cudaErrorUnknown;
            if (e == cudaSuccess && (!encode_f32_kmajor(&p->map_wxhi, p->d_wx_hi, R, p->k_pad4, 64) ||
                                     !encode_f32_kmajor(&p->map_wxlo, p->d_wx_lo, R, p->k_pad4, 64) ||
                                     !encode_f32_kmajor(&p->map_xhi, p->d_x_hi, xrows, p->k_pad4, 128) ||
                                     !encode_f32_kmajor(&p->map_xlo, p->d_x_lo, xrows, p->k_pad4, 128)))
                return SRNN_ERR_CUDA;
        }
        p->tc_gemm = fp16 && (p->cfg.flags & SRNN_FLAG_SIMT_GEMM) == 0;
        if (e == cudaSuccess && p->tc_gemm) {
            // W_x and x rounded to fp16 (RNE) for the tensor-core input GEMM (srnn_gemm_tc.cu)
            const int I = p->cfg.input;
            p->k_pad = (I + 7) & ~7;
            std::vector<uint16_t> w16(static_cast<size_t>(R) * p->k_pad, 0);
            for (int r = 0; r < R; ++r)
                for (int i = 0; i < I; ++i)
                    w16[static_cast<size_t>(r) * p->k_pad + i] = float_to_half_rne(wx[static_cast<size_t>(r) * I + i]);
            const size_t xrows = static_cast<size_t>(std::max(1, p->cfg.max_steps)) * p->cfg.batch;
            e = cudaMalloc(&p->d_wx16, w16.size() * 2);
            if (e == cudaSuccess) e = cudaMemcpy(p->d_wx16, w16.data(), w16.size() * 2, cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = cudaMalloc(&p->d_x16, xrows * p->k_pad * 2);
            // A (x) in 128-row boxes, B (W_x) in 64-row boxes (tile widths 128 / 192 / 256)
            if (e == cudaSuccess && (!encode_fp16_kmajor(&p->map_wx16, p->d_wx16, R, p->k_pad, 64) ||
                                     !encode_fp16_kmajor(&p->map_wx16_32, p->d_wx16, R, p->k_pad, 32) ||
                                     !encode_fp16_kmajor(&p->map_wx16_48, p->d_wx16, R, p->k_pad, 48) ||
                                     !encode_fp16_kmajor(&p->map_x16, p->d_x16, xrows, p->k_pad, 128)))
                return SRNN_ERR_CUDA;
        }
        if (e == cudaSuccess) e = cudaMalloc(&p->d_bias, static_cast<size_t>(R) * 4);
        if (e == cudaSuccess) {
            if (bias)
                e = cudaMemcpy(p->d_bias, bias, static_cast<size_t>(R) * 4, cudaMemcpyHostToDevice);
            else
                e = cudaMemset(p->d_bias, 0, static_cast<size_t>(R) * 4);
        }
        cudaFree(p->d_bhn);
        p->d_bhn = nullptr;
        if (e == cudaSuccess && G == 3 && bias) {  // GRU: bias[3H .. 4H) = b_hn
            e = cudaMalloc(&p->d_bhn, static_cast<size_t>(H) * 4);
            if (e == cudaSuccess) e = cudaMemcpy(p->d_bhn, bias + R, static_cast<size_t>(H) * 4, cudaMemcpyHostToDevice);
        }
        if (e != cudaSuccess) return SRNN_ERR_CUDA;
        // Compiled register count and co-residency check for the instance.
        RecParams rp{};
        rp.threads = l.threads;
        rp.k8 = p->k8 ? 1 : 0;
        rp.warp_early = p->staged ? p->d_wearly : nullptr;  // the staged instance's registers
        rp.csplit = p->csplit ? 1 : 0;  // cluster co-residency check
        int regs[2] = {0, 0}, maxb = 0;
        int le = p->dense ? launch_dense(p->dense_inst, p->dense_mt, p->BT, G, rp, l.num_ctas, p->smem_bytes, nullptr,
                                         true, regs, &maxb)
                          : launch_recurrent(p->np_inst, p->BT, G, p->f16 ? 1 : 0, rp, l.num_ctas, p->smem_bytes,
                                             nullptr, true, regs, &maxb);
        if (le != 0) return SRNN_ERR_CUDA;
        p->regs = regs[0];
        p->spill_bytes = regs[1];
        if (maxb < 1) return SRNN_ERR_NOT_ON_CHIP;
        if (preload_projection_kernels() != 0 || preload_gemm_f32() != 0) return SRNN_ERR_CUDA;
        if (cudaDeviceSynchronize() != cudaSuccess) return SRNN_ERR_CUDA;  // uploads visible to every stream
    }
    p->loaded = true;
    return SRNN_OK;
}

// b' rows [r0, r0 + M) from x rows [r0, r0 + M) (x, bprime: full device buffers).
// `sms`: SMs the projection can use (all of them, or the few the pipelined forward leaves free)
static srnn_status_t project_rows(srnn_plan_t p, int64_t r0, int64_t M, const float* x, float* bprime, void* stream,
                                  int sms) {
    const int I = p->cfg.input, N = p->G * p->cfg.hidden;
    if (M <= 0) return SRNN_OK;
    if (p->tc_gemm) {
        void* x16 = static_cast<char*>(p->d_x16) + static_cast<size_t>(r0) * p->k_pad * 2;
        int e = I == p->k_pad ? launch_f32_to_f16(x + r0 * I, x16, M * I, stream)
                              : launch_f32_to_f16_padded(x + r0 * I, x16, M, I, p->k_pad, stream);
        if (e == 0)
            e = launch_gemm_tc(&p->map_x16, &p->map_wx16, p->d_bias, bprime, static_cast<int>(M), N, p->k_pad, stream,
                               static_cast<int>(r0), 0, sms, &p->map_wx16_32, &p->map_wx16_48);
        return e == 0 ? SRNN_OK : SRNN_ERR_CUDA;
    }
    if (p->tf32x3) {
        float* xh = p->d_x_hi + static_cast<size_t>(r0) * p->k_pad4;
        float* xl = p->d_x_lo + static_cast<size_t>(r0) * p->k_pad4;
        int e = launch_split_tf32(x + r0 * I, xh, xl, M, I, p->k_pad4, stream);
        if (e == 0)
            e = launch_gemm_tf32x3(&p->map_xhi, &p->map_xlo, &p->map_wxhi, &p->map_wxlo, p->d_bias, bprime,
                                   static_cast<int>(M), N, p->k_pad4, stream, static_cast<int>(r0), sms);
        return e == 0 ? SRNN_OK : SRNN_ERR_CUDA;
    }
    GemmParams gp;
    gp.M = M;
    gp.N = N;
    gp.K = I;
    gp.A = x + r0 * I;
    gp.W = p->d_wx;
    gp.bias = p->d_bias;
    gp.C = bprime + r0 * N;
    return launch_gemm_f32(gp, stream) == 0 ? SRNN_OK : SRNN_ERR_CUDA;
}

srnn_status_t srnn_input_projection(srnn_plan_t p, int32_t T, int32_t B, const float* x, float* bprime, void* stream) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (!p->loaded || p->host_only) return SRNN_ERR_STATE;
    if (T < 0 || T > p->cfg.max_steps || B < 1 || B > p->cfg.batch || (T > 0 && (!x || !bprime)))
        return SRNN_ERR_INVALID_VALUE;
    if (T == 0) return SRNN_OK;
    DeviceGuard g(p->cfg.device);
    return project_rows(p, 0, static_cast<int64_t>(T) * B, x, bprime, stream, p->sm_count);
}

struct PipeArgs {
    const uint32_t* bp_ready = nullptr;
    uint32_t bp_ready_base = 0;
    uint32_t* progress = nullptr;
    int every = 0;
};
static srnn_status_t recurrence_impl(srnn_plan_t p, int32_t T, int32_t B, const float* bprime, const float* h0,
                                     const float* c0, float* y, float* hT, float* cT, void* stream,
                                     const PipeArgs& pa);

srnn_status_t srnn_recurrence(srnn_plan_t p, int32_t T, int32_t B, const float* bprime, const float* h0,
                              const float* c0, float* y, float* hT, float* cT, void* stream) {
    return recurrence_impl(p, T, B, bprime, h0, c0, y, hT, cT, stream, PipeArgs());
}

}  // extern "C"

static srnn_status_t recurrence_impl(srnn_plan_t p, int32_t T, int32_t B, const float* bprime, const float* h0,
                                     const float* c0, float* y, float* hT, float* cT, void* stream,
                                     const PipeArgs& pa) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (!p->loaded || p->host_only) return SRNN_ERR_STATE;
    if (T < 0 || T > p->cfg.max_steps || B < 1 || B > p->cfg.batch || (T > 0 && !bprime)) return SRNN_ERR_INVALID_VALUE;
    DeviceGuard g(p->cfg.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t hb = static_cast<size_t>(B) * p->cfg.hidden * sizeof(float);
    if (T == 0) {  // T = 0 returns h0 unchanged
        cudaError_t e = cudaSuccess;
        if (hT) e = h0 ? cudaMemcpyAsync(hT, h0, hb, cudaMemcpyDeviceToDevice, st) : cudaMemsetAsync(hT, 0, hb, st);
        if (e == cudaSuccess && cT && p->G == 4)
            e = c0 ? cudaMemcpyAsync(cT, c0, hb, cudaMemcpyDeviceToDevice, st) : cudaMemsetAsync(cT, 0, hb, st);
        return e == cudaSuccess ? SRNN_OK : SRNN_ERR_CUDA;
    }
    RecParams rp{};
    rp.H = p->cfg.hidden;
    rp.G = p->G;
    rp.B = B;
    rp.T = T;
    rp.n_tiles = (B + p->BT - 1) / p->BT;
    rp.act = p->cfg.act;
    rp.threads = p->lay.threads;
    rp.lanes_per_row = p->lay.lanes_per_row;
    rp.np_inst = p->np_inst;
    rp.smem_slots = p->ns_slots;
    int umax = 0;
    {
        const std::vector<int32_t>& u0 = p->csplit ? p->unit0_real : p->lay.cta_unit0;
        for (int c = 0; c < p->lay.num_ctas; ++c) umax = std::max(umax, u0[c + 1] - u0[c]);
    }
    rp.units_max = umax;
    rp.csplit = p->csplit ? 1 : 0;
    rp.hsplit = p->hsplit;
    rp.cta_vunit0 = p->d_vunit0;
    rp.epoch = p->epoch;
    rp.flags = p->cfg.flags;
    rp.k8 = p->k8 ? 1 : 0;
    if (p->f16)
        rp.img_f16 = static_cast<const uint32_t*>(p->d_img);
    else
        rp.img_f32 = static_cast<const uint2*>(p->d_img);
    rp.cta_unit0 = p->d_unit0;
    rp.unit_perm = p->dense ? nullptr : p->d_perm;
    rp.piece0 = p->dense ? nullptr : p->d_piece0;
    rp.vrows_max = p->lay.vrows_max;
    rp.warp_slots = p->d_wslots;
    rp.warp_early = p->staged && !p->dense ? p->d_wearly : nullptr;
    rp.early_chunks = p->early_chunks;
    rp.bprime = bprime;
    rp.h0 = h0;
    rp.c0 = p->G == 4 ? c0 : nullptr;
    rp.bias_hn = p->G == 3 ? p->d_bhn : nullptr;
    rp.y = y;
    const bool batch_major = (p->cfg.flags & SRNN_FLAG_Y_BATCH_MAJOR) != 0;
    rp.y_bstride = batch_major ? static_cast<int64_t>(T) * p->cfg.hidden : p->cfg.hidden;
    rp.y_tstride = batch_major ? p->cfg.hidden : static_cast<int64_t>(B) * p->cfg.hidden;
    rp.hT = hT;
    rp.cT = p->G == 4 ? cT : nullptr;
    rp.xbuf = p->d_xbuf;
    rp.tile_bytes = static_cast<int32_t>(p->tile_bytes);
    rp.xbuf_tiles = p->n_tiles_max;
    rp.xdirty = p->d_xdirty;
    // 1-bit tags follow the global step (epoch + s, continuous across launches and
    // across the u32 wrap); tiles idle in the previous launch hold older steps
    rp.reinit = rp.n_tiles > p->xbuf_valid_tiles ? 1 : 0;
    if (p->csplit) {
        // the cluster launch has no grid-wide barrier for the in-kernel re-initialisation: the
        // host fills both parities with the stale tags (cheap: 2 x tiles x H x E bytes) every call
        auto pat = [&](uint32_t q) {
            const uint32_t g = p->epoch + q, stale = ((g - 2u) >> 1) & 1u;  // tag of step g - 2
            return p->f16 ? (stale | (stale << 16)) : stale;
        };
        const int64_t per = static_cast<int64_t>(p->n_tiles_max) * p->tile_bytes;
        // parity of global step epoch is epoch & 1: buffer (epoch & 1) holds pattern q = 0
        const uint32_t pa = (p->epoch & 1u) ? pat(1) : pat(0), pb = (p->epoch & 1u) ? pat(0) : pat(1);
        if (launch_xbuf_fill(p->d_xbuf, per, pa, pb, stream) != 0) return SRNN_ERR_CUDA;
        rp.reinit = 0;
    }
    rp.status = p->d_status;
    rp.timeout_ns = p->timeout_ns;
    if (const char* d = std::getenv("SRNN_POLL_BACKOFF_NS")) rp.poll_backoff_ns = static_cast<uint32_t>(std::atoi(d));
    if (const char* d = std::getenv("SRNN_LOADER_THREADS")) rp.loader_threads = std::atoi(d);
    if (p->cfg.flags & SRNN_FLAG_PROFILE) {
        const int64_t need = static_cast<int64_t>(p->lay.num_ctas) * T * rp.n_tiles * 16;
        if (need > p->prof_elems) {
            cudaFree(p->d_prof);
            p->d_prof = nullptr;
            if (cudaMalloc(&p->d_prof, need * 8) != cudaSuccess) return SRNN_ERR_CUDA;
        }
        if (cudaMemsetAsync(p->d_prof, 0, need * 8, static_cast<cudaStream_t>(stream)) != cudaSuccess) return SRNN_ERR_CUDA;
        p->prof_elems = need;
        rp.profile = p->d_prof;
    }
    rp.bp_ready = pa.bp_ready;
    rp.bp_ready_base = pa.bp_ready_base;
    // b' by TMA windows when the plan reserved them and b' is resident (not the pipelined host forward)
    if (!p->dense && pa.bp_ready == nullptr && rp.n_tiles == 1 && bp_tma_ok(p, p->n_tiles_max, umax) &&
        (reinterpret_cast<uintptr_t>(bprime) & 15) == 0) {
        const int boxu = bp_box_units(umax);
        if (p->bpmap_ptr != bprime || p->bpmap_T != T || p->bpmap_B != B) {
            if (!encode_bprime_map(&p->bp_map, bprime, static_cast<int64_t>(p->G) * p->cfg.hidden, B, T, boxu, p->BT))
                return SRNN_ERR_CUDA;
            p->bpmap_ptr = bprime;
            p->bpmap_T = T;
            p->bpmap_B = B;
        }
        rp.bp_map = p->bp_map;
        rp.bp_tma = 1;
        rp.bp_boxu = boxu;
    }
    rp.progress = pa.progress;
    rp.progress_every = pa.every > 0 ? pa.every : 1;
    int e;
    if (p->dense) {
        rp.img_dense = static_cast<const uint4*>(p->d_img);
        rp.img_f16 = nullptr;
        rp.dense_kpw = p->dense_kpw;
        rp.dense_nf = p->dense_nf;
        rp.hs_rows = p->hs_rows;
        e = launch_dense(p->dense_inst, p->dense_mt, p->BT, p->G, rp, p->lay.num_ctas, p->smem_bytes, stream, false,
                         nullptr, nullptr);
    } else {
        e = launch_recurrent(p->np_inst, p->BT, p->G, p->f16 ? 1 : 0, rp, p->lay.num_ctas, p->smem_bytes, stream,
                             false, nullptr, nullptr);
    }
    if (e != 0) return SRNN_ERR_CUDA;
    p->epoch += static_cast<uint32_t>(T) + 1;
    p->xbuf_valid_tiles = rp.n_tiles;
    return SRNN_OK;
}

extern "C" {

srnn_status_t srnn_forward(srnn_plan_t p, int32_t T, int32_t B, const float* x, const float* h0, const float* c0,
                           float* y, float* hT, float* cT, void* stream) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (!p->loaded || p->host_only) return SRNN_ERR_STATE;
    if (T < 0 || T > p->cfg.max_steps || B < 1 || B > p->cfg.batch || (T > 0 && !x)) return SRNN_ERR_INVALID_VALUE;
    if (T > 0) {
        srnn_status_t s = srnn_input_projection(p, T, B, x, p->d_bprime, stream);
        if (s != SRNN_OK) return s;
    }
    return srnn_recurrence(p, T, B, p->d_bprime, h0, c0, y, hT, cT, stream);
}

// Driver stream-memory operations (cuStreamWaitValue32 / cuStreamWriteValue32)
// through the runtime's driver entry point (no -lcuda).
namespace {
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_wait32 g_wait32 = nullptr;
PFN_write32 g_write32 = nullptr;
bool stream_mem_ops() {
    if (g_wait32 && g_write32) return true;
    void* f1 = nullptr;
    void* f2 = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f1, cudaEnableDefault, &q) != cudaSuccess || !f1) return false;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f2, cudaEnableDefault, &q) != cudaSuccess || !f2) return false;
    g_wait32 = reinterpret_cast<PFN_wait32>(f1);
    g_write32 = reinterpret_cast<PFN_write32>(f2);
    return true;
}
}  // namespace

srnn_status_t srnn_forward_host(srnn_plan_t p, int32_t T, int32_t B, const float* x_host, const float* h0_host,
                                const float* c0_host, float* y_host, float* hT_host, float* cT_host) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (!p->loaded || p->host_only) return SRNN_ERR_STATE;
    if (T < 0 || T > p->cfg.max_steps || B < 1 || B > p->cfg.batch || (T > 0 && !x_host)) return SRNN_ERR_INVALID_VALUE;
    DeviceGuard g(p->cfg.device);
    const int H = p->cfg.hidden, I = p->cfg.input, GH = p->G * H;
    const size_t xs = static_cast<size_t>(std::max(1, p->cfg.max_steps)) * p->cfg.batch * I * 4;
    const size_t ys = static_cast<size_t>(std::max(1, p->cfg.max_steps)) * p->cfg.batch * H * 4;
    const size_t hs = static_cast<size_t>(p->cfg.batch) * H * 4;
    if (!p->d_x) {
        if (cudaMalloc(&p->d_x, xs) != cudaSuccess || cudaMalloc(&p->d_y, ys) != cudaSuccess ||
            cudaMalloc(&p->d_h0, hs) != cudaSuccess || cudaMalloc(&p->d_c0, hs) != cudaSuccess ||
            cudaMalloc(&p->d_hT, hs) != cudaSuccess || cudaMalloc(&p->d_cT, hs) != cudaSuccess ||
            cudaMalloc(&p->d_ready, 4) != cudaSuccess || cudaMalloc(&p->d_progress, 4) != cudaSuccess ||
            cudaMemset(p->d_ready, 0, 4) != cudaSuccess || cudaMemset(p->d_progress, 0, 4) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p->s_rec, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_rec, cudaEventDisableTiming) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p->s_copy, cudaStreamNonBlocking) != cudaSuccess ||
            cudaMallocHost(&p->h_status, sizeof(int32_t)) != cudaSuccess)
            return SRNN_ERR_CUDA;
        for (cudaEvent_t& ev : p->ev_chunk)
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return SRNN_ERR_CUDA;
        // the memsets above run on the legacy stream; the non-blocking streams below must see them
        if (cudaDeviceSynchronize() != cudaSuccess) return SRNN_ERR_CUDA;
    }
    cudaStream_t st = p->stream;
    const size_t hb = static_cast<size_t>(B) * H * 4;
    cudaError_t e = cudaSuccess;
    // the pipelined path returns y in chunks of steps: [T][B][H] only
    const bool pipelined = T >= 2 && p->lay.num_ctas < p->sm_count && stream_mem_ops() &&
                           (p->cfg.flags & SRNN_FLAG_Y_BATCH_MAJOR) == 0;
    if (!pipelined) {  // plain: H2D, forward, D2H on one stream
        const size_t xb = static_cast<size_t>(T) * B * I * 4, yb = static_cast<size_t>(T) * B * H * 4;
        if (T > 0) e = cudaMemcpyAsync(p->d_x, x_host, xb, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && h0_host) e = cudaMemcpyAsync(p->d_h0, h0_host, hb, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && c0_host && p->G == 4) e = cudaMemcpyAsync(p->d_c0, c0_host, hb, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return SRNN_ERR_CUDA;
        srnn_status_t s = srnn_forward(p, T, B, p->d_x, h0_host ? p->d_h0 : nullptr, c0_host ? p->d_c0 : nullptr,
                                       y_host ? p->d_y : nullptr, p->d_hT, p->G == 4 ? p->d_cT : nullptr, st);
        if (s != SRNN_OK) return s;
        if (y_host && T > 0) e = cudaMemcpyAsync(y_host, p->d_y, yb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && hT_host) e = cudaMemcpyAsync(hT_host, p->d_hT, hb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && cT_host && p->G == 4) e = cudaMemcpyAsync(cT_host, p->d_cT, hb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return SRNN_ERR_CUDA;
        return srnn_plan_status(p);
    }
    // ---- pipelined: stream `st` copies + projects x chunk by chunk on the free SMs and
    // bumps d_ready; s_rec runs the persistent kernel, which waits per step for its b'
    // rows; s_out copies y chunks back as the kernel's progress counter passes them ----
    // input chunks: up to 8, each a whole number of 128-row GEMM tiles where the
    // batch allows (a partial tile costs the projection as much as a full one)
    int in_b[10] = {0};
    int n_chunks = 0;
    static const int max_in = std::max(1, std::min(8, std::getenv("SRNN_PIPE_IN_CHUNKS") ? std::atoi(std::getenv("SRNN_PIPE_IN_CHUNKS")) : 8));
    static const int max_out = std::max(1, std::getenv("SRNN_PIPE_OUT_CHUNKS") ? std::atoi(std::getenv("SRNN_PIPE_OUT_CHUNKS")) : 16);
    // the persistent kernel is enqueued on `st` right behind chunk 0's projection (same-stream
    // order, no cross-stream event on the critical path); later chunks are projected on s_rec
    static const bool k_on_st = !(std::getenv("SRNN_PIPE_KERNEL_ON_ST") && std::atoi(std::getenv("SRNN_PIPE_KERNEL_ON_ST")) == 0);
    cudaStream_t kst = k_on_st ? st : p->s_rec;
    cudaStream_t pst = k_on_st ? p->s_rec : st;
    {
        const int q = std::max(1, 128 / B);  // steps per 128 rows
        int per = (T + max_in - 1) / max_in;
        per = ((per + q - 1) / q) * q;
        for (int s0 = 0; s0 < T && n_chunks < max_in; s0 += per) in_b[++n_chunks] = std::min(T, s0 + per);
        in_b[n_chunks] = T;
    }
    // output chunks: 16 even ones (the last one's copy is the exposed tail)
    const int every = (T + std::min(max_out, T) - 1) / std::min(max_out, T);
    const int n_out = (T + every - 1) / every;
    const uint32_t prog_base = p->progress_base;
    if (h0_host) e = cudaMemcpyAsync(p->d_h0, h0_host, hb, cudaMemcpyHostToDevice, kst);
    if (e == cudaSuccess && c0_host && p->G == 4) e = cudaMemcpyAsync(p->d_c0, c0_host, hb, cudaMemcpyHostToDevice, kst);
    if (e != cudaSuccess) return SRNN_ERR_CUDA;
    // SRNN_PIPE_TRACE: timing events at every stage, printed to stderr (diagnostics)
    static const bool trace = std::getenv("SRNN_PIPE_TRACE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> tr;
    const auto host_t0 = std::chrono::steady_clock::now();
    std::vector<std::pair<std::string, double>> host_tr;  // host enqueue times (trace only)
    auto mark = [&](const std::string& label, cudaStream_t where) {
        if (!trace) return;
        host_tr.emplace_back(label, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count());
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, where);
        tr.emplace_back(label, ev);
    };
    mark("start", p->s_copy);
    // x chunks stream in on their own copy stream (one event each), so the copy
    // engine runs ahead of the projections instead of alternating with them.
    // Chunk 0 is enqueued first: the host's enqueue time is on the critical path.
    auto copy_chunk = [&](int c) -> srnn_status_t {
        const int s0 = in_b[c], s1 = in_b[c + 1];
        const int64_t r0 = static_cast<int64_t>(s0) * B, nr = static_cast<int64_t>(s1 - s0) * B;
        if (cudaMemcpyAsync(p->d_x + r0 * I, x_host + r0 * I, static_cast<size_t>(nr) * I * 4, cudaMemcpyHostToDevice,
                            p->s_copy) != cudaSuccess ||
            cudaEventRecord(p->ev_chunk[c], p->s_copy) != cudaSuccess)
            return SRNN_ERR_CUDA;
        mark("x" + std::to_string(c) + " in", p->s_copy);
        return SRNN_OK;
    };
    // The kernel treats steps <= *d_ready - ready_base as projected.  Chunk 0 is projected on
    // the kernel's own stream before it starts, so the base is chosen to cover it without a
    // stream memory op on the critical path; chunk c >= 1 then writes ready_base + its last step.
    const uint32_t ready_base = p->ready_cur - static_cast<uint32_t>(in_b[1]);
    // chunk c: projection once its x rows are resident, then d_ready = base + (its last step + 1)
    auto feed_chunk = [&](int c, int sms, cudaStream_t fst) -> srnn_status_t {
        const int s0 = in_b[c], s1 = in_b[c + 1];
        const int64_t r0 = static_cast<int64_t>(s0) * B, nr = static_cast<int64_t>(s1 - s0) * B;
        if (cudaStreamWaitEvent(fst, p->ev_chunk[c], 0) != cudaSuccess) return SRNN_ERR_CUDA;
        srnn_status_t fs = project_rows(p, r0, nr, p->d_x, p->d_bprime, fst, sms);
        if (fs != SRNN_OK) return fs;
        mark("b'" + std::to_string(c) + " ready", fst);
        if (c == 0) return SRNN_OK;  // covered by ready_base
        if (g_write32(fst, reinterpret_cast<CUdeviceptr>(p->d_ready), ready_base + static_cast<uint32_t>(s1),
                      CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return SRNN_ERR_CUDA;
        return SRNN_OK;
    };
    // The first chunk is projected on every SM before the persistent kernel
    // starts; the others on the SMs it leaves free, while it runs.
    srnn_status_t s = copy_chunk(0);
    if (s == SRNN_OK) s = feed_chunk(0, p->sm_count, kst);
    if (s != SRNN_OK) return s;
    PipeArgs pa;
    pa.bp_ready = p->d_ready;
    pa.bp_ready_base = ready_base;
    pa.progress = y_host ? p->d_progress : nullptr;
    pa.every = every;
    mark("kernel launch", kst);
    s = recurrence_impl(p, T, B, p->d_bprime, h0_host ? p->d_h0 : nullptr, c0_host ? p->d_c0 : nullptr,
                        y_host ? p->d_y : nullptr, p->d_hT, p->G == 4 ? p->d_cT : nullptr, kst, pa);
    if (s != SRNN_OK) return s;
    mark("kernel done", kst);
    if (cudaEventRecord(p->ev_rec, kst) != cudaSuccess) return SRNN_ERR_CUDA;
    for (int c = 1; c < n_chunks; ++c) {
        s = copy_chunk(c);
        if (s != SRNN_OK) return s;
    }
    for (int c = 1; c < n_chunks; ++c) {
        s = feed_chunk(c, p->sm_count - p->lay.num_ctas, pst);
        if (s != SRNN_OK) return s;
    }
    (void)GH;
    if (y_host) {
        const uint32_t C = static_cast<uint32_t>(p->lay.num_ctas);
        for (int c = 0; c < n_out; ++c) {
            const int s0 = c * every, s1 = std::min(T, s0 + every);
            if (g_wait32(p->s_out, reinterpret_cast<CUdeviceptr>(p->d_progress), prog_base + C * static_cast<uint32_t>(c + 1),
                         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                return SRNN_ERR_CUDA;
            const size_t r0 = static_cast<size_t>(s0) * B, nr = static_cast<size_t>(s1 - s0) * B;
            e = cudaMemcpyAsync(y_host + r0 * H, p->d_y + r0 * H, nr * H * 4, cudaMemcpyDeviceToHost, p->s_out);
            if (e != cudaSuccess) return SRNN_ERR_CUDA;
            mark("y" + std::to_string(c) + " out", p->s_out);
        }
        p->progress_base = prog_base + C * static_cast<uint32_t>(n_out);
    }
    if (n_chunks > 1) p->ready_cur = ready_base + static_cast<uint32_t>(T);
    e = cudaStreamWaitEvent(p->s_out, p->ev_rec, 0);
    if (e == cudaSuccess && hT_host) e = cudaMemcpyAsync(hT_host, p->d_hT, hb, cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess && cT_host && p->G == 4) e = cudaMemcpyAsync(cT_host, p->d_cT, hb, cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->h_status, p->d_status, 4, cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_rec);
    if (e != cudaSuccess) return SRNN_ERR_CUDA;
    mark("end", p->s_out);
    if (trace) {
        cudaDeviceSynchronize();
        for (auto& t : tr) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, tr[0].second, t.second);
            std::fprintf(stderr, "srnn pipe: %8.1f us  %s\n", 1000.0 * ms, t.first.c_str());
        }
        for (auto& h : host_tr) std::fprintf(stderr, "srnn pipe host: %8.1f us  %s enqueued\n", h.second, h.first.c_str());
        for (auto& t : tr) cudaEventDestroy(t.second);
    }
    if (*p->h_status != 0) {
        // the aborted kernel bumped the progress counter past every wait: resynchronise
        uint32_t v = 0;
        if (cudaMemcpy(&v, p->d_progress, 4, cudaMemcpyDeviceToHost) == cudaSuccess) p->progress_base = v;
        return srnn_plan_status(p);  // reads and clears it
    }
    return SRNN_OK;
}

srnn_status_t srnn_plan_status(srnn_plan_t p) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (p->host_only) return SRNN_OK;
    DeviceGuard g(p->cfg.device);
    int32_t s = 0;
    if (cudaMemcpy(&s, p->d_status, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return SRNN_ERR_CUDA;
    if (s != 0 && cudaMemset(p->d_status, 0, 4) != cudaSuccess) return SRNN_ERR_CUDA;
    return static_cast<srnn_status_t>(s);
}

srnn_status_t srnn_plan_export_layout(srnn_plan_t p, int32_t* col_out, float* val_out, int32_t* row_out,
                                      int64_t capacity) {
    if (!p) return SRNN_ERR_INVALID_VALUE;
    if (!p->loaded) return SRNN_ERR_STATE;
    const int64_t n = static_cast<int64_t>(p->lay.col.size());
    if (capacity < n) return SRNN_ERR_INVALID_VALUE;
    if (col_out) std::memcpy(col_out, p->lay.col.data(), n * 4);
    if (val_out) std::memcpy(val_out, p->lay.val.data(), n * 4);
    if (row_out) std::memcpy(row_out, p->lay.row.data(), n * 4);
    return SRNN_OK;
}

srnn_status_t srnn_plan_debug_timeline(srnn_plan_t p, int64_t* out, int64_t capacity, int64_t* count) {
    if (!p || !count) return SRNN_ERR_INVALID_VALUE;
    if (!(p->cfg.flags & SRNN_FLAG_PROFILE) || !p->d_prof) return SRNN_ERR_STATE;
    *count = p->prof_elems;
    if (!out) return SRNN_OK;
    if (capacity < p->prof_elems) return SRNN_ERR_INVALID_VALUE;
    DeviceGuard g(p->cfg.device);
    return cudaMemcpy(out, p->d_prof, p->prof_elems * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? SRNN_OK
                                                                                                : SRNN_ERR_CUDA;
}

srnn_status_t srnn_destroy(srnn_plan_t p) {
    if (!p) return SRNN_OK;
    if (!p->host_only) {
        DeviceGuard g(p->cfg.device);
        free_device(p);
    }
    delete p;
    return SRNN_OK;
}

}  // extern "C"
