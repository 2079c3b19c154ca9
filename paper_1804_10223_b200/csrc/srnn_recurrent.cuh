// srnn_recurrent.cuh -- the persistent sparse recurrent kernel (sm_100a).
//
// One cooperative launch runs all T timesteps ("The number of
// thread blocks is set to the number of SMs", :74 sparse variant).  Per CTA:
//
//   prologue   packed <index,value> pairs -> registers, decoded
//              once (fp16 -> fp32 value, column -> shared-memory byte offset);
//              h_0 published as tagged words with tag `epoch`.
//   per step s = 1..T, per batch tile k (BT samples, interleaved [j][b] so one
//   LDS.{32,64,128} fetches all BT activations of column j -- PAPER.md:97
//   "wide memory loads"):
//     load     spin on the 64-bit tagged words {fp32 h, u32 tag} of h_{s-1},
//              tile k, until every tag == epoch + s - 1 (single-copy atomic
//              words: value and validity arrive together, no fence --
//              the re-designed Lamport scheme of PAPER.md:102-105), stage the
//              values in shared memory hs[H][BT]   ("Load")
//     operate  acc[b] += value[i] * hs[index[i]][b] over the lane's slots
//              ("Operate")
//     reduce   xor-butterfly over the L lanes of a row ("Reduce",
//              warp shuffles instead of shared memory, fixed order)
//     epilogue z + b'_s, g(.) or the LSTM gates, write y and
//              the tagged h_s word ("Synchronize")
//
// Exchange buffers are double-buffered by step parity; reuse is safe because
// a CTA only overwrites parity p at step s after it has read h_{s-1} from
// every CTA, which each CTA wrote only after it had read h_{s-2} (DESIGN.md
// Sec. 4 "exchange protocol").
#pragma once
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "srnn_internal.h"

namespace srnn {

namespace cg = cooperative_groups;

// Flag bits mirrored from include/srnn.h (device side only needs these).
constexpr uint32_t kFlagGridSync = 1u << 0;
constexpr uint32_t kFlagJitter = 1u << 4;
constexpr uint32_t kFlagProfile = 1u << 6;
#ifndef SRNN_POLL_BACKOFF_NS
#define SRNN_POLL_BACKOFF_NS 64
#endif
constexpr uint32_t kPollBackoffNs = SRNN_POLL_BACKOFF_NS;

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long pack_tagged(float v, uint32_t tag) {
    return (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v);
}
__device__ __forceinline__ uint32_t tag_of(unsigned long long w) { return static_cast<uint32_t>(w >> 32); }
__device__ __forceinline__ float val_of(unsigned long long w) {
    return __uint_as_float(static_cast<uint32_t>(w));
}

// g(.) of Eq. 1/2. Accurate libdevice transcendentals (no
// fast-math: the fp32 parity bound is 1e-5).
__device__ __forceinline__ float activation(int act, float z) {
    if (act == 0) return fmaxf(z, 0.0f);
    if (act == 1) return tanhf(z);
    return z;
}
__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

// Spin-wait bookkeeping of one loader thread.
struct Watchdog {
    unsigned long long t0;
    uint32_t spins;
};

// Returns true when the wait must be abandoned (timeout here or elsewhere).
__device__ __forceinline__ bool watchdog_tick(Watchdog& wd, int32_t* status, unsigned long long timeout_ns) {
    if ((++wd.spins & 15u) != 0u) return false;
    unsigned long long now = globaltimer_ns();
    if (wd.t0 == 0) wd.t0 = now;
    if (*reinterpret_cast<volatile int32_t*>(status) != 0) return true;
    if (now - wd.t0 > timeout_ns) {
        atomicCAS(status, 0, -6 /* SRNN_ERR_TIMEOUT */);
        return true;
    }
    return false;
}

// ---------------------------------------------------------------------------
// Exchange / staging formats.
//   F32: word = {fp32 h, u32 tag}, one word per (unit, sample); hs[H][BT] fp32.
//   F16: word = {fp16 h(b), fp16 h(b+1), u32 tag}, ceil(BT/2) words per unit;
//        hs[H][BT] fp16 ("a lower-precision data type for the
//        activations would remove the shared memory bandwidth and storage
//        burden").  A 16-byte chunk (two words) always maps onto a contiguous
//        piece of hs, so the loader is a pure copy with a tag check.
// ---------------------------------------------------------------------------
template <bool F16, int BT>
struct Fmt {
    static constexpr int WPR = F16 ? (BT == 4 ? 2 : 1) : BT;   // words per unit
    static constexpr int E = F16 ? 2 * BT : 4 * BT;            // hs bytes per unit
    static constexpr int CHUNK_HS = (F16 && BT == 1) ? 4 : 8;  // hs bytes per 16-byte chunk

    // store chunk `idx` (words w0, w1; w1 valid iff has1) into hs
    __device__ __forceinline__ static void store(unsigned char* hs, int idx, unsigned long long w0,
                                                 unsigned long long w1, bool has1) {
        if (F16 && BT == 1) {
            const uint32_t lo = static_cast<uint32_t>(w0) & 0xffffu;
            if (has1)
                *reinterpret_cast<uint32_t*>(hs + 4 * idx) = lo | (static_cast<uint32_t>(w1) << 16);
            else
                *reinterpret_cast<unsigned short*>(hs + 4 * idx) = static_cast<unsigned short>(lo);
        } else {
            if (has1)
                *reinterpret_cast<uint2*>(hs + 8 * idx) = make_uint2(static_cast<uint32_t>(w0), static_cast<uint32_t>(w1));
            else
                *reinterpret_cast<uint32_t*>(hs + 8 * idx) = static_cast<uint32_t>(w0);
        }
    }
};

// Stage h_{s-1} (one batch tile) into shared memory.  Every thread owns up
// to K 16-byte chunks per group; all of them are in flight at once, and
// chunks whose tags are stale are re-polled together (one round trip per
// round, not per chunk).  Tag mode spins; grid-sync mode checks once.
template <bool F16, int BT, int K>
__device__ __forceinline__ bool load_tile(const ulonglong2* __restrict__ src, unsigned char* hs, int n_words,
                                          uint32_t want, bool spin, int32_t* status,
                                          unsigned long long timeout_ns, int first = 0) {
    const int n_chunks = (n_words + 1) >> 1;
    const int nt = blockDim.x;
    Watchdog wd{0ull, 0u};
    bool ok = true;
    for (int base = threadIdx.x + first; base < n_chunks; base += K * nt) {
        ulonglong2 v[K];
        uint32_t pend = 0u;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int idx = base + j * nt;
            if (idx < n_chunks) {
                v[j] = ld_relaxed_v2(src + idx);
                pend |= 1u << j;
            }
        }
        while (true) {
#pragma unroll
            for (int j = 0; j < K; ++j) {
                if (pend & (1u << j)) {
                    const int idx = base + j * nt;
                    const bool has1 = 2 * idx + 1 < n_words;
                    if (tag_of(v[j].x) == want && (!has1 || tag_of(v[j].y) == want)) {
                        Fmt<F16, BT>::store(hs, idx, v[j].x, v[j].y, has1);
                        pend &= ~(1u << j);
                    }
                }
            }
            if (pend == 0u) break;
            if (!spin) {
                atomicCAS(status, 0, -4 /* protocol violation -> SRNN_ERR_STATE */);
                break;
            }
            if (watchdog_tick(wd, status, timeout_ns)) {
                ok = false;
                break;
            }
            __nanosleep(kPollBackoffNs);
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (pend & (1u << j)) v[j] = ld_relaxed_v2(src + base + j * nt);
        }
        if (!ok) break;
    }
    return ok;
}

// Register prefetch of the first KP chunks per thread of a tile: issued one
// tile-phase early (while the current tile computes), validated when the
// tile is due.  Chunks beyond KP*nt go through load_tile synchronously.
template <bool F16, int BT, int KP>
struct Prefetch {
    ulonglong2 v[KP];
    __device__ __forceinline__ void issue(const ulonglong2* __restrict__ src, int n_words) {
        const int n_chunks = (n_words + 1) >> 1;
#pragma unroll
        for (int j = 0; j < KP; ++j) {
            const int idx = threadIdx.x + j * blockDim.x;
            if (idx < n_chunks) v[j] = ld_relaxed_v2(src + idx);
        }
    }
    __device__ __forceinline__ bool finish(const ulonglong2* __restrict__ src, unsigned char* hs, int n_words,
                                           uint32_t want, bool spin, int32_t* status,
                                           unsigned long long timeout_ns) {
        const int n_chunks = (n_words + 1) >> 1;
        const int nt = blockDim.x;
        uint32_t pend = 0u;
#pragma unroll
        for (int j = 0; j < KP; ++j)
            if (threadIdx.x + j * nt < n_chunks) pend |= 1u << j;
        Watchdog wd{0ull, 0u};
        bool ok = true;
        while (true) {
#pragma unroll
            for (int j = 0; j < KP; ++j) {
                if (pend & (1u << j)) {
                    const int idx = threadIdx.x + j * nt;
                    const bool has1 = 2 * idx + 1 < n_words;
                    if (tag_of(v[j].x) == want && (!has1 || tag_of(v[j].y) == want)) {
                        Fmt<F16, BT>::store(hs, idx, v[j].x, v[j].y, has1);
                        pend &= ~(1u << j);
                    }
                }
            }
            if (pend == 0u) break;
            if (!spin) {
                atomicCAS(status, 0, -4);
                break;
            }
            if (watchdog_tick(wd, status, timeout_ns)) {
                ok = false;
                break;
            }
            __nanosleep(kPollBackoffNs);  // stale: back off instead of flooding the LSU
#pragma unroll
            for (int j = 0; j < KP; ++j)
                if (pend & (1u << j)) v[j] = ld_relaxed_v2(src + threadIdx.x + j * nt);
        }
        if (ok && n_chunks > KP * nt)
            ok = load_tile<F16, BT, 4>(src, hs, n_words, want, spin, status, timeout_ns, KP * nt);
        return ok;
    }
};

// ---------------------------------------------------------------------------
// TMA staging of the tagged h words (sm_90+/sm_100 bulk async copy).
// One elected thread moves a whole tile (or a segment of it) of tagged words
// global -> shared memory with cp.async.bulk, completion on an mbarrier; all
// threads then validate tags in shared memory and compact the values into hs.
// No registers are held while the copy is in flight, so the next tile's copy
// can be issued before the current tile computes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst before async writes
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Validate one staged segment (chunks [c0, c1)) and compact it into hs.
// Returns true if any chunk of this thread is stale.
template <bool F16, int BT>
__device__ __forceinline__ bool stage_pass(const ulonglong2* staging, unsigned char* hs, int c0, int c1, int n_words,
                                           uint32_t want) {
    bool stale = false;
    for (int c = c0 + static_cast<int>(threadIdx.x); c < c1; c += blockDim.x) {
        const ulonglong2 v = staging[c - c0];
        const bool has1 = 2 * c + 1 < n_words;
        stale |= !(tag_of(v.x) == want && (!has1 || tag_of(v.y) == want));
        Fmt<F16, BT>::store(hs, c, v.x, v.y, has1);
    }
    return stale;
}

// ---------------------------------------------------------------------------
// Register-resident weights and the operate stage.
//   F32: two registers per pair, {hs byte offset, fp32 value}, FFMA.
//   F16: one register per pair, (hs byte offset << 16) | fp16 value, and the
//        sm_100 mixed-precision FMA d.f32 = a.f16 * b.f16 + c.f32 (FHFMA), so
//        nothing is decoded per step ("two column indices can be
//        compressed into a 32-bit register ... fp16 for the weights").
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fma_f16f16f32(uint32_t a_lo_half, uint32_t b_half_bits, float c) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;"
        : "=f"(d)
        : "h"(static_cast<unsigned short>(a_lo_half)), "h"(static_cast<unsigned short>(b_half_bits)), "f"(c));
    return d;
}

template <int NP, int BT, bool F16>
struct Weights;

// The operate loop runs in groups of GS slots: all GS shared-memory loads of
// a group are issued before its FMAs (memory-level parallelism), and the
// warp-uniform slot count n_w is checked once per group.  Slots between n_w
// and the end of a group hold zero weights reading column 0 (a broadcast),
// exactly like the paper's <index, 0> padding pairs.
template <int NP, int BT>
struct Weights<NP, BT, false> {
    static constexpr int GS = BT == 4 ? 4 : 8;
    uint32_t off[NP];
    float w[NP];
    __device__ __forceinline__ void load(const RecParams& p, size_t img0, int n_w) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            off[i] = 0u;
            w[i] = 0.0f;
            if (i < n_w) {
                const uint2 e = p.img_f32[img0 + static_cast<size_t>(i) * p.threads];
                off[i] = e.x;
                w[i] = __uint_as_float(e.y);
            }
        }
    }
    __device__ __forceinline__ void operate(float (&acc)[BT], const unsigned char* hs, int n_w) const {
#pragma unroll
        for (int i0 = 0; i0 < NP; i0 += GS) {
            if (i0 < n_w) {
                if (BT == 4) {
                    float4 h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float4*>(hs + off[i0 + j]);
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            const float wv = w[i0 + j];
                            acc[0] = fmaf(wv, h[j].x, acc[0]);
                            acc[1 % BT] = fmaf(wv, h[j].y, acc[1 % BT]);
                            acc[2 % BT] = fmaf(wv, h[j].z, acc[2 % BT]);
                            acc[3 % BT] = fmaf(wv, h[j].w, acc[3 % BT]);
                        }
                    }
                } else if (BT == 2) {
                    float2 h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float2*>(hs + off[i0 + j]);
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            acc[0] = fmaf(w[i0 + j], h[j].x, acc[0]);
                            acc[1 % BT] = fmaf(w[i0 + j], h[j].y, acc[1 % BT]);
                        }
                    }
                } else {
                    float h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float*>(hs + off[i0 + j]);
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) acc[0] = fmaf(w[i0 + j], h[j], acc[0]);
                }
            }
        }
    }
};

template <int NP, int BT>
struct Weights<NP, BT, true> {
    static constexpr int GS = BT == 4 ? 4 : 8;
    uint32_t pw[NP];
    __device__ __forceinline__ void load(const RecParams& p, size_t img0, int n_w) {
#pragma unroll
        for (int i = 0; i < NP; ++i) pw[i] = i < n_w ? p.img_f16[img0 + static_cast<size_t>(i) * p.threads] : 0u;
    }
    __device__ __forceinline__ void operate(float (&acc)[BT], const unsigned char* hs, int n_w) const {
#pragma unroll
        for (int i0 = 0; i0 < NP; i0 += GS) {
            if (i0 < n_w) {
                if (BT == 4) {
                    uint2 h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const uint2*>(hs + (pw[i0 + j] >> 16));
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            const uint32_t wv = pw[i0 + j];
                            acc[0] = fma_f16f16f32(wv, h[j].x, acc[0]);
                            acc[1 % BT] = fma_f16f16f32(wv, h[j].x >> 16, acc[1 % BT]);
                            acc[2 % BT] = fma_f16f16f32(wv, h[j].y, acc[2 % BT]);
                            acc[3 % BT] = fma_f16f16f32(wv, h[j].y >> 16, acc[3 % BT]);
                        }
                    }
                } else if (BT == 2) {
                    uint32_t h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const uint32_t*>(hs + (pw[i0 + j] >> 16));
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            acc[0] = fma_f16f16f32(pw[i0 + j], h[j], acc[0]);
                            acc[1 % BT] = fma_f16f16f32(pw[i0 + j], h[j] >> 16, acc[1 % BT]);
                        }
                    }
                } else {
                    uint32_t h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const unsigned short*>(hs + (pw[i0 + j] >> 16));
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) acc[0] = fma_f16f16f32(pw[i0 + j], h[j], acc[0]);
                }
            }
        }
    }
};

// Max threads per CTA of each instance.  The register file is split over
// the 4 SM sub-partitions (16K registers each), so with W warps a thread may
// hold at most 512 / ceil(W/4) registers: 256 threads -> 255, 384 -> 168,
// 512 -> 128, 640 -> 96, 768 -> 80.  Each instance gets the largest thread
// count whose budget still holds its register-resident pairs.
template <int NP, bool F16>
struct MaxThreads {
    static constexpr int value = F16 ? (NP <= 12 ? 640 : NP <= 32 ? 512 : NP <= 48 ? 384 : 256)
                                     : (NP <= 4 ? 768 : NP <= 12 ? 640 : NP <= 32 ? 512 : NP <= 48 ? 384 : 256);
};
template <int NP, bool F16>
struct LoadK {
    static constexpr int value = F16 ? (NP <= 48 ? 8 : 4) : 4;
};

__device__ __forceinline__ void cp_async_f32(float* dst_smem, const float* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NP, int BT, int G, bool F16>
__global__ void __launch_bounds__(MaxThreads<NP, F16>::value, 1) srnn_persistent_kernel(const RecParams p) {
    using F = Fmt<F16, BT>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = p.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cta = blockIdx.x;
    const int u0 = p.cta_unit0[cta];
    const int U = p.cta_unit0[cta + 1] - u0;
    // shared memory: hs[2] (double-buffered h_{s-1} tile, E bytes per unit),
    // then the LSTM cell state of every (tile, unit, sample)
    const size_t hs_bytes = (static_cast<size_t>(H) * F::E + 15) & ~static_cast<size_t>(15);
    ulonglong2* staging = reinterpret_cast<ulonglong2*>(smem + 2 * hs_bytes);  // [stage_chunks] tagged words
    float* cs = reinterpret_cast<float*>(smem + 2 * hs_bytes + static_cast<size_t>(p.stage_chunks) * 16);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(cs + (G == 4 ? p.n_tiles * p.units_max * BT : 0)) + 7) & ~static_cast<uintptr_t>(7));
    int* s_abort = reinterpret_cast<int*>(mbar + 1);

    const int L = p.lanes_per_row;
    const int n_w = p.warp_slots[cta * (p.threads >> 5) + warp];
    const int n_words = H * F::WPR;
    const int tile_stride = (n_words + 1) & ~1;
    const int GH = G * H;

    // ---- prologue: weights HBM -> registers (once per forward) ----
    Weights<NP, BT, F16> W;
    W.load(p, static_cast<size_t>(cta) * NP * p.threads + tid, n_w);

    // Row of this lane: local row k = unit_local * G + gate (srnn_packer.cpp).
    const int krow = warp * (32 / L) + lane / L;
    const bool row_valid = krow < G * U;
    const bool row_leader = (lane % L) == 0 && row_valid;
    const int ul = krow / G, gate = krow % G;      // local unit, gate of this row
    const int unit = u0 + ul;
    const bool unit_leader = row_leader && gate == 0;  // owns h (and c) of its unit
    if (tid == 0) {
        *s_abort = 0;
        mbar_init(mbar, 1);
    }
    __syncthreads();

    // Per-lane bases hoisted out of the time loop.
    unsigned long long* const xb_unit = p.xbuf + unit * F::WPR;
    const float* const bp_row = p.bprime + gate * H + unit;
    float* const y_unit = p.y != nullptr ? p.y + unit : nullptr;
    const size_t bp_step = static_cast<size_t>(p.B) * GH, y_step = static_cast<size_t>(p.B) * H;
    const int act = p.act;

    // Publish the BT values of unit `unit`, (step s, tile k) as tagged words.
    auto publish = [&](int s, int k, const float (&h)[BT]) {
        unsigned long long* dst = xb_unit + static_cast<size_t>((s & 1) * p.n_tiles + k) * tile_stride - unit * F::WPR;
        const uint64_t tag = static_cast<uint64_t>(p.epoch + static_cast<uint32_t>(s)) << 32;
        if (!F16) {
#pragma unroll
            for (int b = 0; b < BT; ++b) st_relaxed_u64(dst + unit * BT + b, tag | __float_as_uint(h[b]));
        } else {
#pragma unroll
            for (int w = 0; w < F::WPR; ++w) {
                uint32_t lo = __half_as_ushort(__float2half_rn(h[2 * w]));
                if (2 * w + 1 < BT) lo |= static_cast<uint32_t>(__half_as_ushort(__float2half_rn(h[(2 * w + 1) % BT]))) << 16;
                st_relaxed_u64(dst + unit * F::WPR + w, tag | lo);
            }
        }
    };

    // ---- publish h_0 (tag = epoch) and initialise c ----
    if (unit_leader) {
        for (int k = 0; k < p.n_tiles; ++k) {
            float h[BT];
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                const int bg = k * BT + b;
                h[b] = (p.h0 != nullptr && bg < p.B) ? p.h0[static_cast<size_t>(bg) * H + unit] : 0.0f;
                if (G == 4)
                    cs[(k * p.units_max + ul) * BT + b] =
                        (p.c0 != nullptr && bg < p.B) ? p.c0[static_cast<size_t>(bg) * H + unit] : 0.0f;
            }
            publish(0, k, h);
        }
    }
    const bool grid_sync = (p.flags & kFlagGridSync) != 0u;
    if (grid_sync) cg::this_grid().sync();

    // Register prefetch of tile (s, k)'s h_{s-1} tagged words.  With >= 2
    // batch tiles the next tile's input was published one tile-phase ago and
    // its loads are issued right after this tile's operate, landing while the
    // epilogue runs ("as we process iteration n, we can load the
    // states for iteration n+1").
    const bool early = p.n_tiles > 1 && !grid_sync;
    const int n_chunks = (n_words + 1) >> 1;
    const int stage_chunks = p.stage_chunks;
    auto tile_src = [&](int s, int k) {
        return reinterpret_cast<const ulonglong2*>(p.xbuf +
                                                   static_cast<size_t>(((s - 1) & 1) * p.n_tiles + k) * tile_stride);
    };
    uint32_t mbar_phase = 0;
    auto issue_seg = [&](const ulonglong2* src, int c0) {  // thread 0 only
        const int c1 = min(n_chunks, c0 + stage_chunks);
        tma_load_1d(staging, src + c0, static_cast<uint32_t>(c1 - c0) * 16u, mbar);
    };
    if (early && tid == 0) issue_seg(tile_src(1, 0), 0);
    int parity = 0;

    for (int s = 1; s <= p.T; ++s) {
        for (int k = 0; k < p.n_tiles; ++k) {
            long long* prof = (p.flags & kFlagProfile) && p.profile != nullptr && tid == 0
                                  ? p.profile + ((static_cast<size_t>(cta) * p.T + (s - 1)) * p.n_tiles + k) * 4
                                  : nullptr;
            if (prof) prof[0] = clock64();
            // b'_s of this lane's row for the BT samples (lands during operate)
            float bp[BT];
            const float* bps = bp_row + static_cast<size_t>(s - 1) * bp_step + static_cast<size_t>(k * BT) * GH;
            float* ys = y_unit != nullptr ? y_unit + static_cast<size_t>(s - 1) * y_step + static_cast<size_t>(k * BT) * H
                                          : nullptr;
            const int nb = min(BT, p.B - k * BT);  // real samples in this tile
#pragma unroll
            for (int b = 0; b < BT; ++b) bp[b] = (row_leader && b < nb) ? __ldg(bps + b * GH) : 0.0f;
            // ---- load: h_{s-1} tile k -> hs[parity] ----
            // TMA-stage the tagged words (segment by segment), validate the
            // tags in shared memory, compact the values into hs; a stale
            // segment is re-fetched whole after a short backoff.
            unsigned char* hs = smem + parity * hs_bytes;
            {
                const uint32_t want = p.epoch + static_cast<uint32_t>(s - 1);
                const ulonglong2* src = tile_src(s, k);
                Watchdog wd{0ull, 0u};
                for (int c0 = 0; c0 < n_chunks; c0 += stage_chunks) {
                    bool prefetched = early && c0 == 0;
                    while (true) {
                        if (!prefetched && tid == 0) issue_seg(src, c0);
                        prefetched = false;
                        mbar_wait(mbar, mbar_phase);
                        mbar_phase ^= 1u;
                        const bool stale =
                            stage_pass<F16, BT>(staging, hs, c0, min(n_chunks, c0 + stage_chunks), n_words, want);
                        if (!__syncthreads_or(stale)) break;
                        if (tid == 0) {
                            if (grid_sync)
                                atomicCAS(p.status, 0, -4 /* protocol violation */);
                            else if (watchdog_tick(wd, p.status, p.timeout_ns))
                                *s_abort = 1;
                        }
                        __syncthreads();
                        if (*s_abort || grid_sync) break;
                        __nanosleep(kPollBackoffNs);
                    }
                    if (*s_abort) break;
                }
            }
            if (prof) prof[1] = clock64();
            if (*s_abort) goto done;
            const int ns = k + 1 < p.n_tiles ? s : s + 1, nk = k + 1 < p.n_tiles ? k + 1 : 0;

            // ---- operate + reduce ----
            float acc[BT];
#pragma unroll
            for (int b = 0; b < BT; ++b) acc[b] = 0.0f;
            W.operate(acc, hs, n_w);
            // next tile's input was published one tile-phase ago: stage it now
            if (early && ns <= p.T && tid == 0) issue_seg(tile_src(ns, nk), 0);
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                if (m < L) {
#pragma unroll
                    for (int b = 0; b < BT; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], m);
                }
            }
            if (prof) prof[2] = clock64();

            // ---- epilogue in the row-leader lanes: z = acc + b'; g / gates; publish ----
            float z[BT];
#pragma unroll
            for (int b = 0; b < BT; ++b) z[b] = acc[b] + bp[b];
            if (G == 4) {
                // gates i, f, g, o of a unit are rows 4u..4u+3: lanes +0, +L, +2L, +3L
                float zf[BT], zg[BT], zo[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) {
                    zf[b] = __shfl_down_sync(0xffffffffu, z[b], L);
                    zg[b] = __shfl_down_sync(0xffffffffu, z[b], 2 * L);
                    zo[b] = __shfl_down_sync(0xffffffffu, z[b], 3 * L);
                }
                if (unit_leader) {
                    float h[BT];
#pragma unroll
                    for (int b = 0; b < BT; ++b) {
                        float* cp = &cs[(k * p.units_max + ul) * BT + b];
                        const float c = sigmoidf_acc(zf[b]) * (*cp) + sigmoidf_acc(z[b]) * tanhf(zg[b]);
                        *cp = c;
                        h[b] = sigmoidf_acc(zo[b]) * tanhf(c);
                        if (b < nb) {
                            if (ys != nullptr) ys[b * H] = h[b];
                            if (s == p.T) {
                                const int bg = k * BT + b;
                                if (p.hT != nullptr) p.hT[static_cast<size_t>(bg) * H + unit] = h[b];
                                if (p.cT != nullptr) p.cT[static_cast<size_t>(bg) * H + unit] = c;
                            }
                        }
                    }
                    publish(s, k, h);
                }
            } else if (unit_leader) {
                float h[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) h[b] = activation(act, z[b]);
#pragma unroll
                for (int b = 0; b < BT; ++b) {
                    if (b < nb) {
                        if (ys != nullptr) ys[b * H] = h[b];
                        if (s == p.T && p.hT != nullptr) p.hT[static_cast<size_t>(k * BT + b) * H + unit] = h[b];
                    }
                }
                if ((p.flags & kFlagJitter) != 0u) {
                    const uint32_t r = (static_cast<uint32_t>(cta) * 2654435761u) ^ (static_cast<uint32_t>(s * 40503 + k));
                    __nanosleep((r >> 7) & 2047u);
                }
                publish(s, k, h);
            }
            if (prof) prof[3] = clock64();
            if (grid_sync) cg::this_grid().sync();
            parity ^= 1;
        }
    }
done:
    return;
}

template <int NP, int BT, int G, bool F16>
static int launch_one(const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
                      int* regs_out, int* max_blocks_out) {
    auto fn = srnn_persistent_kernel<NP, BT, G, F16>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (regs_out != nullptr || max_blocks_out != nullptr) {
        cudaFuncAttributes attr;
        e = cudaFuncGetAttributes(&attr, fn);
        if (e != cudaSuccess) return static_cast<int>(e);
        if (regs_out) *regs_out = attr.numRegs;
        if (max_blocks_out) {
            int nb = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, p.threads, smem);
            if (e != cudaSuccess) return static_cast<int>(e);
            *max_blocks_out = p.threads > MaxThreads<NP, F16>::value ? 0 : nb;
        }
    }
    if (query_only) return 0;
    void* args[] = {const_cast<RecParams*>(&p)};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(num_ctas), dim3(p.threads), args, smem,
                                    static_cast<cudaStream_t>(stream));
    return static_cast<int>(e);
}

template <int NP, bool F16>
int launch_np(int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
              int* regs_out, int* max_blocks_out) {
#define SRNN_CASE(BT_, G_)                                                                                    \
    if (bt == BT_ && g == G_)                                                                                 \
        return launch_one<NP, BT_, G_, F16>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
    SRNN_CASE(1, 1)
    SRNN_CASE(2, 1)
    SRNN_CASE(4, 1)
    SRNN_CASE(1, 4)
    SRNN_CASE(2, 4)
    SRNN_CASE(4, 4)
#undef SRNN_CASE
    return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace srnn
