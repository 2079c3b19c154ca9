// srnn_gemm_tc.cu -- step a1 in fp16 mode on the 5th-generation tensor cores.
//
// The input projection for all timesteps at once (Eq. 2: "W x_t
// ... has no dependency, so it can be processed in parallel and added to b,
// becoming b'"):
//
//     b'[m][n] = bias[n] + sum_k x16[m][k] * Wx16[n][k]     (fp16 in, fp32 accumulate)
//
// x (fp32, [T*B][I]) is first rounded to fp16 (RNE) by a small kernel; W_x is
// rounded once at srnn_load_weights.  One CTA computes a 128 x BN output
// tile (BN = 128 or 256) with tcgen05.mma (cta_group::1, kind::f16, M=128
// N=BN K=16) from shared-memory operands staged by TMA (cp.async.bulk.tensor,
// 128-byte swizzle, mbarrier ring of 192 KB: 6 stages at BN = 128, 4 at 256);
// the accumulator lives in TMEM and is read back by four epilogue warps with
// tcgen05.ld, + bias, stored as fp32.  The kernel is persistent over tiles
// (grid = min(tiles, SMs it may use)) with two TMEM accumulators, so the
// epilogue of one tile overlaps the loads and MMAs of the next.  BN = 256 halves the re-reads of the x tile and carries 1.5x
// the bytes in flight per SM: it is used when the 128 x 128 grid would not fill
// the SMs anyway (e.g. the per-chunk projections of the pipelined
// srnn_forward_host, which run on the few SMs the persistent kernel leaves free).
//
//   warp 0: TMA producer (one elected lane)    warp 1: TMEM alloc + MMA issuer
//   warps 2-5: epilogue (TMEM lane quarter = warp % 4)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "srnn_internal.h"

namespace srnn {
namespace {

constexpr int TC_BM = 128, TC_BK = 64, TC_STAGES = 4, TC_THREADS = 192;
constexpr uint32_t TC_TILE_BYTES = TC_BM * TC_BK * 2;  // 16 KB: one 128-row operand box

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nLAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// The same, multicast to every CTA of the cluster in cta_mask (same shared-memory offsets; each
// destination's mbarrier at that offset receives the complete_tx bytes).
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t cta_mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
        "%4}], [%2], %5;" ::"r"(su32(dst)),
        "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "h"(cta_mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
    const uint64_t addr = su32(p);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) /* LBO (unused for SW128 K-major) */ |
           ((1024ull >> 4) << 32) /* SBO */ | (1ull << 46) /* sm100 descriptor version */ |
           (2ull << 61) /* SWIZZLE_128B */;
}
// Instruction descriptor, kind::f16: D f32, A/B f16, both K-major, M = 128, N = BN.
// X3 (fp32 mode, "3xTF32"): kind::tf32, A/B format TF32 (2) -- see gemm_tc_f16_kernel.
template <int BN, bool X3 = false>
__host__ __device__ constexpr uint32_t idesc_f16() {
    return (1u << 4) | ((X3 ? 2u : 0u) << 7) | ((X3 ? 2u : 0u) << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
           (static_cast<uint32_t>(TC_BM >> 4) << 24);
}

// One K-block is one 128-byte swizzle row per operand row: 64 fp16, or 32 fp32
// (tf32) elements.  X3 stages four operand tiles per K-block: A_hi, A_lo, B_hi, B_lo.
template <int BN, bool X3 = false>
struct TcCfg {
    static constexpr uint32_t B_BYTES = BN * TC_BK * 2;  // BN/64 boxes of 64 rows, 8-row groups 1 KB apart
    static constexpr uint32_t STAGE_BYTES = (X3 ? 2 : 1) * (TC_TILE_BYTES + B_BYTES);
    static constexpr int STAGES = static_cast<int>((200u * 1024u) / STAGE_BYTES);  // ~200 KB in flight
    static constexpr uint32_t TMEM_COLS = BN == 128 ? 256 : 512;  // two accumulators (power-of-2 allocation)
    static constexpr uint32_t ACC_STRIDE = BN <= 128 ? 128 : 256;  // TMEM column of accumulator 1
    static constexpr size_t SMEM = STAGES * STAGE_BYTES + 1024 /* align */ + 256 /* barriers */;
};

// Persistent over output tiles: CTA b takes tiles b, b + gridDim.x, ... (n-fastest).
// The producer and the MMA issuer run ahead into the next tile while the
// epilogue warps drain the other TMEM accumulator.
//
// X3 = the fp32 mode's exact-enough projection on tensor cores ("3xTF32", the
// split named in SURVEY.md Sec. 7 hard part 7): x and W_x are split on the host
// side of the MMA into tf32 hi + lo parts (a = a_hi + a_lo, |a_lo| <= 2^-11 |a|),
// and D += A_hi B_hi + A_hi B_lo + A_lo B_hi, dropping only A_lo B_lo (~2^-22 of
// each product) -- fp32-level accuracy for the 1e-5 parity bound, with K in
// steps of 8 tf32 elements (32 bytes, the same descriptor advance as fp16 K=16).
//
// CM > 1: thread-block clusters of CM CTAs along M share the W_x tile of their common n0: the
// B operand of every K-block is fetched once per cluster and multicast into all CM CTAs'
// shared memory (CTA rank r loads B slices r, r + CM, ... of SLICE rows), cutting the L2 -> SM
// operand traffic that bounds the projection at M = T*B = 1024.  A stage is
// refilled only when all CM CTAs' MMAs have read it: every MMA commit arrives on the empty
// barrier of each CTA of the cluster (empty counts CM arrivals).
template <int BN, bool X3 = false, int CM = 1>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_f16_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       const float* __restrict__ bias, float* __restrict__ C, int M, int N, int K, int m_off,
                       const __grid_constant__ CUtensorMap map_a_lo, const __grid_constant__ CUtensorMap map_b_lo,
                       const __grid_constant__ CUtensorMap map_b32) {
    using Cfg = TcCfg<BN, X3>;
    static_assert(CM == 1 || !X3, "multicast clusters: fp16 operands only");
    // B slices: 64-row boxes (map_b); with clusters, CM slices of BN / CM rows (map_b32: 32-row
    // boxes for BN = 128, CM = 4) or, for BN = 144, three 48-row slices (map_b32 then holds
    // 48-row boxes; rank 3 loads none)
    constexpr int SLICE = BN == 144 ? 48 : BN / (CM > BN / 64 ? CM : BN / 64);
    constexpr int NSL = BN / SLICE;
    static_assert(BN % SLICE == 0 && (CM == 1 || NSL <= CM || NSL % CM == 0), "B slices");
    constexpr uint16_t kMask = static_cast<uint16_t>((1u << CM) - 1u);
    uint32_t crank = 0;
    if constexpr (CM > 1) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    constexpr int STAGES = Cfg::STAGES;
    constexpr uint32_t kIdesc = idesc_f16<BN, X3>();
    constexpr int KB_ELEMS = X3 ? TC_BK / 2 : TC_BK;  // elements of K per 128-byte row
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B-swizzled operand tiles
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // per stage: A [, A_lo] then B [, B_lo]
    unsigned char* sA = smem;
    unsigned char* sB = smem + STAGES * TC_TILE_BYTES * (X3 ? 2 : 1);
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES * (X3 ? 2 : 1));
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2] accumulator ready for the epilogue
    uint64_t* tempty = tfull + 2;      // [2] accumulator drained by the 4 epilogue warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (K + KB_ELEMS - 1) / KB_ELEMS;
    const int tiles_n = (N + BN - 1) / BN;
    // (cluster) tiles: CM vertically adjacent 128-row tiles with one n0; CTA rank r takes row
    // tile group * CM + r (rows past M are zero-filled by TMA and never stored)
    const int n_tiles = tiles_n * (((M + TC_BM - 1) / TC_BM + CM - 1) / CM);
    const int t0 = static_cast<int>(blockIdx.x) / CM, t_step = static_cast<int>(gridDim.x) / CM;
    auto tile_m0 = [&](int t) { return ((t / tiles_n) * CM + static_cast<int>(crank)) * TC_BM; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CM);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
        if (X3) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a_lo) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b_lo) : "memory");
        }
    }
    if (warp == 1) {  // TMEM allocation (whole warp)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(Cfg::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (CM > 1) cluster_sync_all();  // every CTA's barriers exist before any multicast
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        int it = 0;
        for (int t = t0; t < n_tiles; t += t_step) {
            const int m0 = tile_m0(t), n0 = (t % tiles_n) * BN;
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
                const int a_stride = TC_TILE_BYTES * (X3 ? 2 : 1), b_stride = Cfg::B_BYTES * (X3 ? 2 : 1);
                tma_load_2d(sA + s * a_stride, &map_a, &full[s], kb * KB_ELEMS, m_off + m0);
                if (X3) tma_load_2d(sA + s * a_stride + TC_TILE_BYTES, &map_a_lo, &full[s], kb * KB_ELEMS, m_off + m0);
                if constexpr (CM > 1) {  // this rank's B slices, multicast to the whole cluster
#pragma unroll
                    for (int j = 0; j < NSL; ++j)
                        if (j % CM == static_cast<int>(crank))
                            tma_load_2d_mc(sB + s * b_stride + j * SLICE * 128, SLICE == 64 ? &map_b : &map_b32,
                                           &full[s], kb * KB_ELEMS, n0 + SLICE * j, kMask);
                    continue;
                }
#pragma unroll
                for (int j = 0; j < BN / 64; ++j) {  // rows past N are zero-filled by TMA
                    tma_load_2d(sB + s * b_stride + j * (TC_TILE_BYTES / 2), &map_b, &full[s], kb * KB_ELEMS,
                                n0 + 64 * j);
                    if (X3)
                        tma_load_2d(sB + s * b_stride + Cfg::B_BYTES + j * (TC_TILE_BYTES / 2), &map_b_lo, &full[s],
                                    kb * KB_ELEMS, n0 + 64 * j);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: D[tmem acc] (+)= A[smem] * B[smem]^T ----
        int it = 0, lt = 0;
        for (int t = t0; t < n_tiles; t += t_step, ++lt) {
            const int acc = lt & 1;
            if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc) * Cfg::ACC_STRIDE;
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % STAGES;
                mbar_wait(&full[s], (it / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t da = smem_desc_sw128(sA + s * TC_TILE_BYTES * (X3 ? 2 : 1));
                const uint64_t db = smem_desc_sw128(sB + s * Cfg::B_BYTES * (X3 ? 2 : 1));
#pragma unroll
                for (int k = 0; k < TC_BK / 16; ++k) {
                    const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
                    // advance 16 fp16 / 8 tf32 (32 bytes) along K inside the swizzled row: +2 in the >>4 address field
                    if (X3) {
                        const uint64_t dal = da + (TC_TILE_BYTES >> 4), dbl = db + (Cfg::B_BYTES >> 4);
                        asm volatile(
                            "{\n.reg .pred p, q;\nsetp.ne.b32 p, %6, 0;\nsetp.eq.b32 q, %6, %6;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %5, p;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %3, %2, %5, q;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %4, %5, q;\n}\n" ::"r"(d_tmem),
                            "l"(da + 2ull * k), "l"(db + 2ull * k), "l"(dal + 2ull * k), "l"(dbl + 2ull * k),
                            "r"(kIdesc), "r"(accum)
                            : "memory");
                    } else {
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
                            "l"(da + 2ull * k), "l"(db + 2ull * k), "r"(kIdesc), "r"(accum)
                            : "memory");
                    }
                }
                // free the smem stage once these MMAs have read it (CM > 1: in every CTA of the
                // cluster, whose producers multicast into this stage)
                if constexpr (CM > 1)
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                        "%1;" ::"r"(su32(&empty[s])),
                        "h"(kMask)
                        : "memory");
                else
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     su32(&empty[s]))
                                 : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&tfull[acc]))
                         : "memory");
        }
    } else if (warp >= 2) {
        // ---- epilogue: TMEM -> registers -> + bias -> global ----
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
        int lt = 0;
        for (int t = t0; t < n_tiles; t += t_step, ++lt) {
            const int acc = lt & 1;
            const int m0 = tile_m0(t), n0 = (t % tiles_n) * BN;
            const int row = m0 + quarter * 32 + lane;
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                const uint32_t taddr =
                    tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc) * Cfg::ACC_STRIDE +
                    static_cast<uint32_t>(c);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c + 32 >= BN) {  // last chunk read: hand the accumulator back to the MMA issuer
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[acc])) : "memory");
                }
                if (row < M) {
                    float* crow = C + static_cast<size_t>(m_off + row) * N + n0 + c;
                    const int nvalid = min(min(32, BN - c), N - (n0 + c));  // BN = 144: a 16-column last chunk
                    if (nvalid == 32 && (N & 3) == 0) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            float4 o;
                            o.x = __uint_as_float(v[j + 0]) + (bias ? __ldg(bias + n0 + c + j + 0) : 0.0f);
                            o.y = __uint_as_float(v[j + 1]) + (bias ? __ldg(bias + n0 + c + j + 1) : 0.0f);
                            o.z = __uint_as_float(v[j + 2]) + (bias ? __ldg(bias + n0 + c + j + 2) : 0.0f);
                            o.w = __uint_as_float(v[j + 3]) + (bias ? __ldg(bias + n0 + c + j + 3) : 0.0f);
                            *reinterpret_cast<float4*>(crow + j) = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j < nvalid) crow[j] = __uint_as_float(v[j]) + (bias ? __ldg(bias + n0 + c + j) : 0.0f);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // no CTA leaves while a peer's last MMA commit may still arrive on its barriers
    if constexpr (CM > 1) cluster_sync_all();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS)
                     : "memory");
    }
}

// fp32 -> fp16 (RNE), 8 elements per thread (two 16-byte loads, one 16-byte store) where aligned.
__global__ void f32_to_f16_kernel(const float* __restrict__ in, __half* __restrict__ out, int64_t n) {
    const int64_t i8 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
    if (i8 + 7 < n) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(in + i8));
        const float4 w = __ldcs(reinterpret_cast<const float4*>(in + i8 + 4));
        __half2 h[4] = {__floats2half2_rn(v.x, v.y), __floats2half2_rn(v.z, v.w), __floats2half2_rn(w.x, w.y),
                        __floats2half2_rn(w.z, w.w)};
        *reinterpret_cast<uint4*>(out + i8) = *reinterpret_cast<const uint4*>(h);
    } else {
        for (int64_t i = i8; i < n; ++i) out[i] = __float2half_rn(in[i]);
    }
}

// fp32 [rows][cols] -> fp16 [rows][ld_out] (RNE), zero padding in columns [cols, ld_out).
__global__ void f32_to_f16_padded_kernel(const float* __restrict__ in, __half* __restrict__ out, int64_t rows,
                                         int cols, int ld_out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * ld_out) return;
    const int64_t r = i / ld_out;
    const int c = static_cast<int>(i - r * ld_out);
    out[i] = c < cols ? __float2half_rn(in[r * cols + c]) : __float2half_rn(0.0f);
}

}  // namespace

int launch_f32_to_f16_padded(const float* in, void* out, int64_t rows, int cols, int ld_out, void* stream) {
    const int64_t n = rows * ld_out;
    if (n <= 0) return 0;
    f32_to_f16_padded_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        in, static_cast<__half*>(out), rows, cols, ld_out);
    return static_cast<int>(cudaGetLastError());
}

// x -> (tf32(x), tf32(x - tf32(x))) stored as fp32 bit patterns, [rows][cols] -> [rows][ld_out]
// (zero padding in columns [cols, ld_out)).  cvt.rna = round to nearest, ties away (tf32).
__global__ void split_tf32_kernel(const float* __restrict__ in, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t rows, int cols, int ld_out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * ld_out) return;
    const int64_t r = i / ld_out;
    const int c = static_cast<int>(i - r * ld_out);
    const float v = c < cols ? in[r * cols + c] : 0.0f;
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float rem = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(rem));
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(l);
}

// Force module loading of the projection kernels (CUDA lazy loading would
// otherwise load them at first launch, which can stall behind a running
// persistent kernel that is waiting for their output).
static int fit_clusters_144x4();
int preload_projection_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<128>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<192>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<256>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<128, false, 2>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<128, false, 4>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<144, false, 4>);
    if (e == cudaSuccess) (void)fit_clusters_144x4();  // occupancy query once, outside any stream capture
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_tc_f16_kernel<128, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, split_tf32_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, f32_to_f16_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, f32_to_f16_padded_kernel);
    return static_cast<int>(e);
}

int launch_f32_to_f16(const float* in, void* out, int64_t n, void* stream) {
    if (n <= 0) return 0;
    const int64_t threads = (n + 7) / 8;
    const int blocks = static_cast<int>((threads + 255) / 256);
    f32_to_f16_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(in, static_cast<__half*>(out), n);
    return static_cast<int>(cudaGetLastError());
}

template <int BN, bool X3 = false, int CM = 1>
static int launch_gemm_tc_bn(const void* map_a, const void* map_b, const float* bias, float* C, int M, int N, int K,
                             cudaStream_t stream, int m_off, int sms, const void* map_a_lo = nullptr,
                             const void* map_b_lo = nullptr, const void* map_b32 = nullptr) {
    // The shared-memory opt-in is a per-device function attribute: set it on every launch
    // (cheap, thread-safe; a process may drive plans on several devices).
    const size_t smem = TcCfg<BN, X3>::SMEM;
    auto fn = gemm_tc_f16_kernel<BN, X3, CM>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    const int64_t tiles = static_cast<int64_t>((N + BN - 1) / BN) * (((M + TC_BM - 1) / TC_BM + CM - 1) / CM);
    const CUtensorMap& ma = *static_cast<const CUtensorMap*>(map_a);
    const CUtensorMap& mb = *static_cast<const CUtensorMap*>(map_b);
    const CUtensorMap& ma_lo = X3 ? *static_cast<const CUtensorMap*>(map_a_lo) : ma;
    const CUtensorMap& mb_lo = X3 ? *static_cast<const CUtensorMap*>(map_b_lo) : mb;
    const CUtensorMap& mb32 = map_b32 ? *static_cast<const CUtensorMap*>(map_b32) : mb;
    if constexpr (CM == 1) {
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
        fn<<<grid, TC_THREADS, smem, stream>>>(ma, mb, bias, C, M, N, K, m_off, ma_lo, mb_lo, mb32);
        return static_cast<int>(cudaGetLastError());
    } else {
        // clusters of CM CTAs; the persistent grid holds at most as many clusters as fit at once
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CM;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.blockDim = dim3(TC_THREADS);
        lc.dynamicSmemBytes = smem;
        lc.stream = stream;
        lc.attrs = at;
        lc.numAttrs = 1;
        lc.gridDim = dim3(static_cast<unsigned>(CM * std::max(1, sms / CM)));
        int fit = 0;
        e = cudaOccupancyMaxActiveClusters(&fit, fn, &lc);
        if (e != cudaSuccess) return static_cast<int>(e);
        const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>({tiles, static_cast<int64_t>(sms / CM),
                                                                    static_cast<int64_t>(std::max(1, fit))}));
        lc.gridDim = dim3(static_cast<unsigned>(CM * ncl));
        e = cudaLaunchKernelEx(&lc, fn, ma, mb, bias, C, M, N, K, m_off, ma_lo, mb_lo, mb32);
        return static_cast<int>(e);
    }
}

// fp32 mode: 3xTF32 tcgen05 GEMM on pre-split operands (tf32 hi / lo as fp32 arrays).
int launch_gemm_tf32x3(const void* map_a_hi, const void* map_a_lo, const void* map_b_hi, const void* map_b_lo,
                       const float* bias, float* C, int M, int N, int K, void* stream, int m_off, int sms) {
    if (M <= 0 || N <= 0) return 0;
    return launch_gemm_tc_bn<128, true>(map_a_hi, map_b_hi, bias, C, M, N, K, static_cast<cudaStream_t>(stream),
                                        m_off, std::max(1, sms), map_a_lo, map_b_lo);
}

int launch_split_tf32(const float* in, float* hi, float* lo, int64_t rows, int cols, int ld_out, void* stream) {
    const int64_t n = rows * ld_out;
    if (n <= 0) return 0;
    split_tf32_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        in, hi, lo, rows, cols, ld_out);
    return static_cast<int>(cudaGetLastError());
}

// bn = 128, 192 or 256; 0 picks the width that minimises the operand bytes of
// the busiest CTA: ceil(tiles / sms) x (128 + bn) rows of K -- 128 when the
// 128-wide grid fits in one wave, wider when the launch has few SMs (the
// pipelined projections on the SMs the persistent kernel leaves free).
// Clusters of 4 CTAs of the BN = 144 multicast instance that fit on the device at once (per
// device, cached; a benign race writes the same value).
static int fit_clusters_144x4() {
    static int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    if (cache[dev] > 0) return cache[dev];
    auto fn = gemm_tc_f16_kernel<144, false, 4>;
    const size_t smem = TcCfg<144>::SMEM;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.gridDim = dim3(4);
    lc.blockDim = dim3(TC_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.attrs = at;
    lc.numAttrs = 1;
    int fit = 0;
    if (cudaOccupancyMaxActiveClusters(&fit, fn, &lc) != cudaSuccess) return 0;
    cache[dev] = fit;
    return fit;
}

int launch_gemm_tc(const void* map_a, const void* map_b, const float* bias, float* C, int M, int N, int K,
                   void* stream, int m_off, int bn, int sms, const void* map_b32, const void* map_b48) {
    if (M <= 0 || N <= 0) return 0;
    if (const char* e = std::getenv("SRNN_GEMM_SMS")) sms = std::atoi(e);  // experiment: cap the grid
    sms = std::max(1, sms);
    const char* env_cm = std::getenv("SRNN_GEMM_CM");
    const char* env_bn = std::getenv("SRNN_GEMM_BN");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // Opt-in (SRNN_GEMM_CM=4): 144-wide tiles in 4-CTA clusters along M that multicast their W_x
    // tile, when all cluster tiles fit in one wave (C2: 2 x 16 = 32 <= 33 clusters).  Per CTA,
    // A 128 x K + a quarter of B 144 x K instead of 128 x K + 128 x K.  Measured on B200 (C2,
    // ncu): 26.4 us vs 21.8 us for the unclustered 128-wide kernel although the L2 sectors fall
    // 117 -> 82 MB -- L2 already merges the unicast reads of CTAs that fetch the same W_x tile
    // at the same time (B300_MICROARCH: multicast ~ unicast at cluster size <= 4) and the
    // cluster-wide stage release couples the four CTAs' pipelines.
    if (bn == 0 && map_b48 != nullptr && sms >= 128 && !env_bn && env_cm && std::atoi(env_cm) == 4) {
        const int64_t ctiles = static_cast<int64_t>((M + 4 * TC_BM - 1) / (4 * TC_BM)) * ((N + 143) / 144);
        const int fit = fit_clusters_144x4();
        if (ctiles >= 8 && ctiles <= std::min(fit, sms / 4))
            return launch_gemm_tc_bn<144, false, 4>(map_a, map_b, bias, C, M, N, K, st, m_off, sms, nullptr, nullptr,
                                                    map_b48);
    }
    if (env_bn && std::atoi(env_bn) == 144 && map_b48 != nullptr)  // forced (tests)
        return launch_gemm_tc_bn<144, false, 4>(map_a, map_b, bias, C, M, N, K, st, m_off, sms, nullptr, nullptr,
                                                map_b48);
    if (bn == 0) {
        const int64_t tm = (M + TC_BM - 1) / TC_BM;
        int64_t best = -1;
        for (int w : {128, 192, 256}) {
            const int64_t tiles = tm * ((N + w - 1) / w);
            const int64_t cost = ((tiles + sms - 1) / sms) * (128 + w);
            if (best < 0 || cost < best) {
                best = cost;
                bn = w;
            }
        }
        if (const char* e = std::getenv("SRNN_GEMM_BN")) bn = std::atoi(e);
    }
    // 128-wide tiles in clusters of 2 / 4 along M (experiments / tests only: at C2 the 128-wide
    // cluster tiles do not fit in one wave, measured slower than CM = 1)
    const int cm = env_cm ? std::atoi(env_cm) : 1;
    if (bn == 128 && cm == 2) return launch_gemm_tc_bn<128, false, 2>(map_a, map_b, bias, C, M, N, K, st, m_off, sms);
    if (bn == 128 && cm == 4 && map_b32 != nullptr)
        return launch_gemm_tc_bn<128, false, 4>(map_a, map_b, bias, C, M, N, K, st, m_off, sms, nullptr, nullptr, map_b32);
    switch (bn) {
        case 192: return launch_gemm_tc_bn<192>(map_a, map_b, bias, C, M, N, K, st, m_off, sms);
        case 256: return launch_gemm_tc_bn<256>(map_a, map_b, bias, C, M, N, K, st, m_off, sms);
        default: return launch_gemm_tc_bn<128>(map_a, map_b, bias, C, M, N, K, st, m_off, sms);
    }
}

}  // namespace srnn
