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

// Phase timestamps (SRNN_FLAG_PROFILE) exist only in profile builds (-DSRNN_PROFILE):
// the production kernel carries no per-step instrumentation branches.
#ifdef SRNN_PROFILE
#define SRNN_STAMP(i, v)            \
    do {                            \
        if (prof) prof[i] = (v);    \
    } while (0)
#else
#define SRNN_STAMP(i, v) \
    do {                 \
    } while (0)
#endif

// Flag bits mirrored from include/srnn.h (device side only needs these).
constexpr uint32_t kFlagGridSync = 1u << 0;
constexpr uint32_t kFlagJitter = 1u << 4;
constexpr uint32_t kFlagProfile = 1u << 6;
constexpr uint32_t kFlagDropPublish = 1u << 9;

__device__ __forceinline__ void st_relaxed_u16(void* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b16 [%0], %1;" ::"l"(p), "h"(static_cast<unsigned short>(v)) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(void* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// g(.) of Eq. 1/2. Accurate libdevice transcendentals (no
// fast-math: the fp32 parity bound is 1e-5).
// Transcendentals.  FAST (the fp16-staged path) uses the SFU's tanh.approx.f32
// (relative error ~2^-11, the same order as the fp16 rounding every h goes
// through before the exchange) and sigma(z) = 0.5 + 0.5 tanh(z / 2); the fp32
// path keeps the accurate libm forms (reading R14).
__device__ __forceinline__ float tanh_approx(float z) {
    float r;
    asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(z));
    return r;
}
template <bool FAST>
__device__ __forceinline__ float tanh_g(float z) {
    return FAST ? tanh_approx(z) : tanhf(z);
}
template <bool FAST>
__device__ __forceinline__ float sigmoid_g(float z) {
    return FAST ? fmaf(0.5f, tanh_approx(0.5f * z), 0.5f) : 1.0f / (1.0f + expf(-z));
}
template <bool FAST>
__device__ __forceinline__ float activation(int act, float z) {
    if (act == 0) return fmaxf(z, 0.0f);
    if (act == 1) return tanh_g<FAST>(z);
    return z;
}

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
// Exchange format (reading R16).  The exchange image of one
// (step parity, batch tile) is byte for byte the staged layout hs: fp32 [H][BT],
// fp16 [H][BT] for BT <= 8 and two planes [2][H][8] for BT = 16 (so every
// gather stays one aligned LDS), padded to whole 16-byte chunks.  Validity
// travels inside the values: every exchanged value of global step g carries
// the 1-bit tag (g >> 1) & 1 in its mantissa LSB (PAPER.md:102-105 Lamport
// scheme re-designed: the "not yet written" test is a tag mismatch instead of
// the -0.0 sentinel).  Buffers alternate by step parity, so a consumer waiting
// for step g finds either g (fresh) or g - 2 (stale, opposite tag); every
// value is its own single-copy-atomic access (16 / 32 bits), so a 16-byte
// chunk is valid iff all its tags match and may be copied to hs unchanged.
// The producer rounds h (RNE) to one significand bit less than the exchange
// type -- 10 bits for fp16, 23 for fp32, LSB zero -- and ORs the tag in; the
// consumer clears it while staging.  So the staged value is the producer's
// rounded h exactly (error <= 1 ulp of the exchange type, 0 for values with a
// shorter significand, e.g. small integers), Inf and NaN survive, and y, c and
// the accumulation are unaffected.
// ---------------------------------------------------------------------------
template <bool F16, int BT>
struct Fmt {
    static constexpr int VB = F16 ? 2 : 4;  // bytes per exchanged value
    static constexpr int E = VB * BT;       // hs bytes per unit (per plane for BT = 16)
    static constexpr unsigned long long TAGMASK = F16 ? 0x0001000100010001ull : 0x0000000100000001ull;
    // byte offset of item (unit, sample b) inside a tile image / hs
    __device__ __forceinline__ static int offset(int H, int unit, int b) {
        if (F16 && BT == 16) return (b >> 3) * H * 16 + unit * 16 + (b & 7) * 2;
        return (unit * BT + b) * VB;
    }
    // the exchanged value of h: rounded to an even LSB (RNE), carrying `tag` in the LSB
    __device__ __forceinline__ static uint32_t encode(float h, uint32_t tag) {
        uint32_t b = __float_as_uint(h);
        const bool nan = (b & 0x7fffffffu) > 0x7f800000u;
        if (F16) {
            if (!nan) b = (b + 0x1fffu + ((b >> 14) & 1u)) & ~0x3fffu;  // RNE to 9 stored bits (exact in fp16)
            return (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(__uint_as_float(b)))) & ~1u) | tag;
        }
        if (!nan) b += (b >> 1) & 1u;  // RNE to 22 stored bits (the low bit is cleared below)
        return (b & ~1u) | tag;
    }
};

// Stage h_{s-1} (one batch tile) into shared memory, in two parts so the
// first poll round is in flight while the caller does its other per-step
// bookkeeping (the b' prefetch): issue() sends the loads of a thread's first
// batch of K 16-byte chunks (chunk c = thread + j * nt); complete() checks
// them, re-polls the stale ones together (one round trip per round, not per
// chunk), stages them into hs and then handles any further batches.  Tag mode
// spins; grid-sync mode checks once.  ROW16 (dense tensor-core comparator):
// every unit gets a 16-byte hs row (ldmatrix rows); with BT = 4 a chunk holds
// two units.
template <bool F16, int BT, int K, bool ROW16 = false>
struct Poller {
    static constexpr unsigned long long M = Fmt<F16, BT>::TAGMASK;
    ulonglong2 v[K];
    uint32_t pend;

    __device__ __forceinline__ void issue(const ulonglong2* __restrict__ src, int base, int n_chunks, int nt) {
        pend = 0u;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (base + j * nt < n_chunks) {
                v[j] = ld_relaxed_v2(src + base + j * nt);
                pend |= 1u << j;
            }
        }
    }

    // sel: the chunks j of the (single) batch to complete now (the staged instance completes the
    // early chunks, operates on them, then completes the rest); ~0 = all
    // The first poll round from hoisted addresses (chunk j at ptr + j * js bytes, valid j in
    // jmask): nothing but the loads between the post-publish barrier and the round trip.
    __device__ __forceinline__ void issue_at(const unsigned char* ptr, uint32_t jmask, uint32_t js) {
        pend = jmask;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if ((jmask >> j) & 1u) v[j] = ld_relaxed_v2(reinterpret_cast<const ulonglong2*>(ptr + j * js));
    }

    __device__ __forceinline__ bool complete(const ulonglong2* __restrict__ src, unsigned char* hs, int n_chunks,
                                             uint32_t tag, bool spin, int32_t* status, unsigned long long timeout_ns,
                                             uint32_t backoff_ns, int nt, int* rounds, long long* t_first,
                                             uint32_t sel = ~0u) {
        const unsigned long long want = tag ? M : 0ull;
        Watchdog wd{0ull, 0u};
        for (int base = threadIdx.x; base < n_chunks; base += K * nt) {
            if (base != static_cast<int>(threadIdx.x)) issue(src, base, n_chunks, nt);
            while (true) {
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    if ((pend >> j) & 1u) {
                        if ((((v[j].x & M) ^ want) | ((v[j].y & M) ^ want)) == 0ull) {
                            const int c = base + j * nt;
                            v[j].x &= ~M;  // strip the tags: the producer's rounded values
                            v[j].y &= ~M;
                            if (ROW16 && BT == 4) {
                                *reinterpret_cast<unsigned long long*>(hs + 32 * c) = v[j].x;
                                *reinterpret_cast<unsigned long long*>(hs + 32 * c + 16) = v[j].y;
                            } else {
                                *reinterpret_cast<ulonglong2*>(hs + 16 * c) = v[j];
                            }
                            pend &= ~(1u << j);
                        }
                    }
                }
                if (rounds) {
                    if (*rounds == 0 && t_first) *t_first = clock64();
                    ++*rounds;
                }
                if ((pend & sel) == 0u) {
                    // the selected chunks are staged; the other still-stale ones go out again
                    // now so they are in flight during the caller's next work (staged instance)
                    if (pend != 0u) {
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            if ((pend >> j) & 1u) v[j] = ld_relaxed_v2(src + base + j * nt);
                    }
                    break;
                }
                if (!spin) {
                    atomicCAS(status, 0, -4 /* protocol violation -> SRNN_ERR_STATE */);
                    return true;
                }
                if (watchdog_tick(wd, status, timeout_ns)) return false;
                if (backoff_ns) __nanosleep(backoff_ns);
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if ((pend >> j) & 1u) v[j] = ld_relaxed_v2(src + base + j * nt);
            }
        }
        return true;
    }
};

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

// hs byte offset of a slot, extracted from its packed register at every use.  volatile: the
// compiler would otherwise hoist all NP extractions out of the time loop and hold NP more
// registers live (one shift per gather is free on the idle ALU pipe; the registers are not).
#ifndef SRNN_HOIST_OFFSETS
__device__ __forceinline__ uint32_t xoff_hi16(uint32_t w) {
    uint32_t o;
    asm volatile("shr.b32 %0, %1, 16;" : "=r"(o) : "r"(w));
    return o;
}
__device__ __forceinline__ uint32_t xoff_lo16(uint32_t w) {
    uint32_t o;
    asm volatile("and.b32 %0, %1, 65535;" : "=r"(o) : "r"(w));
    return o;
}
__device__ __forceinline__ uint32_t xoff_u16(uint32_t w) {  // 16-byte units in the high half -> bytes
    uint32_t o;
    asm volatile("{\n.reg .b32 t;\nshr.b32 t, %1, 12;\nand.b32 %0, t, 1048560;\n}" : "=r"(o) : "r"(w));
    return o;
}
#else
__device__ __forceinline__ uint32_t xoff_hi16(uint32_t w) { return w >> 16; }
__device__ __forceinline__ uint32_t xoff_lo16(uint32_t w) { return w & 0xffffu; }
__device__ __forceinline__ uint32_t xoff_u16(uint32_t w) { return (w >> 12) & 0xffff0u; }
#endif

// Gathers by 32-bit shared-window addresses (base + offset, one LEA per slot): the generic
// pointer form made the compiler re-derive the shared window base (S2UR CgaCtaId + ULEA) in
// every operate group, a serialising dependency at the head of each group (ncu source view).
// volatile: per-use address (no hoisted NP-register offset arrays), order kept vs the barriers.
#ifndef SRNN_GENERIC_GATHER
#define SRNN_SHARED_GATHER 1
#endif
__device__ __forceinline__ uint32_t xaddr_hi16(uint32_t w, uint32_t base) {  // base + byte offset (high half)
    uint32_t a;
    asm volatile("{\n.reg .b32 t;\nshr.b32 t, %1, 16;\nadd.u32 %0, t, %2;\n}" : "=r"(a) : "r"(w), "r"(base));
    return a;
}
__device__ __forceinline__ uint32_t xaddr_u16(uint32_t w, uint32_t base) {  // base + 16-byte units (high half)
    uint32_t a;
    asm volatile("{\n.reg .b32 t;\nshr.b32 t, %1, 12;\nand.b32 t, t, 1048560;\nadd.u32 %0, t, %2;\n}"
                 : "=r"(a)
                 : "r"(w), "r"(base));
    return a;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short r;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}

// The operate loop runs in groups of GS slots: all GS shared-memory loads of
// a group are issued before its FMAs (memory-level parallelism), and the
// warp-uniform slot count n_w is checked once per group.  Slots between n_w
// and the end of a group hold zero weights reading column 0 (a broadcast),
// exactly like the paper's <index, 0> padding pairs.
#ifndef SRNN_GS_F32_BT4
#define SRNN_GS_F32_BT4 4
#endif
#ifndef SRNN_GS_F32
#define SRNN_GS_F32 8
#endif
template <int NP, int BT>
struct Weights<NP, BT, false> {
    static constexpr int GS = BT == 4 ? SRNN_GS_F32_BT4 : SRNN_GS_F32;
    // fp32 values, and the hs byte offsets of two slots per register (hs <= 64 KB in fp32
    // mode, host-checked): 1.5 registers per pair instead of 2, the difference between a
    // spill-free and a spilling instance at 128 registers (e.g. NP = 24, the C2 fp32 plan)
#ifndef SRNN_F32_UNPACKED
    uint32_t offp[(NP + 1) / 2];
    __device__ __forceinline__ uint32_t off(int i) const {
        return (i & 1) ? xoff_hi16(offp[i >> 1]) : xoff_lo16(offp[i >> 1]);
    }
#else  // A/B: one offset register per pair
    uint32_t offp[NP];
    __device__ __forceinline__ uint32_t off(int i) const { return offp[i]; }
#endif
    float w[NP];
    __device__ __forceinline__ void load(const RecParams& p, size_t img0, int n_w) {
#pragma unroll
        for (int i = 0; i < static_cast<int>(sizeof(offp) / 4); ++i) offp[i] = 0u;
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            w[i] = 0.0f;
            if (i < n_w) {
                const uint2 e = p.img_f32[img0 + static_cast<size_t>(i) * p.threads];
#ifndef SRNN_F32_UNPACKED
                offp[i >> 1] |= e.x << (16 * (i & 1));
#else
                offp[i] = e.x;
#endif
                w[i] = __uint_as_float(e.y);
            }
        }
    }
    __device__ __forceinline__ void operate(float (&acc)[BT], const unsigned char* hs, int n_w,
                                            const unsigned char* = nullptr, uint32_t = 0u) const {
#pragma unroll
        for (int i0 = 0; i0 < NP; i0 += GS) {
            if (i0 < n_w) {
                if (BT == 4) {
                    float4 h[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float4*>(hs + off(i0 + j));
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
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float2*>(hs + off(i0 + j));
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
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const float*>(hs + off(i0 + j));
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) acc[0] = fmaf(w[i0 + j], h[j], acc[0]);
                }
            }
        }
    }
};

// F16 register pair: high 16 bits = hs offset of the column, low 16 bits = fp16
// weight.  The offset is in bytes for BT <= 4 (E <= 8, H * E <= 64 KB) and in
// 16-byte units for BT = 8 (E = 16: the column index itself, any H <= 65536).
template <int NP, int BT>
struct Weights<NP, BT, true> {
    static constexpr int GS = operate_group_slots(true, BT);
    uint32_t pw[NP];
    __device__ __forceinline__ void load(const RecParams& p, size_t img0, int n_w) {
#pragma unroll
        for (int i = 0; i < NP; ++i) pw[i] = i < n_w ? p.img_f16[img0 + static_cast<size_t>(i) * p.threads] : 0u;
    }
    // hs2: the second sample plane (BT = 16 only).  A warp whose slots are all used (the common
    // case of a balanced layout) runs the groups without the per-group slot-count checks, so the
    // compiler may issue the next group's gathers under the current group's FMAs.
    // hb: shared-window address of hs (kept in a register for the whole launch)
    __device__ __forceinline__ void operate(float (&acc)[BT], const unsigned char* hs, int n_w,
                                            const unsigned char* hs2 = nullptr, uint32_t hb = 0u) const {
#ifdef SRNN_OPERATE_NOGUARD
        if (n_w >= NP)
            operate_groups<false>(acc, hs, 0, n_w, hs2, hb);
        else
#endif
            operate_groups<true>(acc, hs, 0, n_w, hs2, hb);
    }
    // Slots [lo, hi) only (the staged instance: lo and hi are multiples of GS, warp-uniform).
    __device__ __forceinline__ void operate_span(float (&acc)[BT], const unsigned char* hs, int lo, int hi,
                                                 const unsigned char* hs2 = nullptr, uint32_t hb = 0u) const {
        operate_groups<true>(acc, hs, lo, hi, hs2, hb);
    }
    template <bool GUARD>
    __device__ __forceinline__ void operate_groups(float (&acc)[BT], const unsigned char* hs, int lo, int n_w,
                                                   const unsigned char* hs2, uint32_t hb) const {
#pragma unroll
        for (int i0 = 0; i0 < NP; i0 += GS) {
            if (!GUARD || (i0 >= lo && i0 < n_w)) {
                if (BT == 16) {
                    uint4 ha[GS], hb[GS];
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            const uint32_t o = xoff_u16(pw[i0 + j]);
                            ha[j] = *reinterpret_cast<const uint4*>(hs + o);
                            hb[j] = *reinterpret_cast<const uint4*>(hs2 + o);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            const uint32_t wv = pw[i0 + j];
                            const uint32_t hv[8] = {ha[j].x, ha[j].y, ha[j].z, ha[j].w, hb[j].x, hb[j].y, hb[j].z, hb[j].w};
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                acc[(2 * q) % BT] = fma_f16f16f32(wv, hv[q], acc[(2 * q) % BT]);
                                acc[(2 * q + 1) % BT] = fma_f16f16f32(wv, hv[q] >> 16, acc[(2 * q + 1) % BT]);
                            }
                        }
                    }
                } else if (BT == 8) {
                    uint4 h[GS];
#ifdef SRNN_SHARED_GATHER
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = lds_v4(xaddr_u16(pw[i0 + j], hb));
#else
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const uint4*>(hs + (xoff_u16(pw[i0 + j])));
#endif
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        if (i0 + j < NP) {
                            const uint32_t wv = pw[i0 + j];
                            acc[0] = fma_f16f16f32(wv, h[j].x, acc[0]);
                            acc[1 % BT] = fma_f16f16f32(wv, h[j].x >> 16, acc[1 % BT]);
                            acc[2 % BT] = fma_f16f16f32(wv, h[j].y, acc[2 % BT]);
                            acc[3 % BT] = fma_f16f16f32(wv, h[j].y >> 16, acc[3 % BT]);
                            acc[4 % BT] = fma_f16f16f32(wv, h[j].z, acc[4 % BT]);
                            acc[5 % BT] = fma_f16f16f32(wv, h[j].z >> 16, acc[5 % BT]);
                            acc[6 % BT] = fma_f16f16f32(wv, h[j].w, acc[6 % BT]);
                            acc[7 % BT] = fma_f16f16f32(wv, h[j].w >> 16, acc[7 % BT]);
                        }
                    }
                } else if (BT == 4) {
                    uint2 h[GS];
#ifdef SRNN_SHARED_GATHER
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = lds_v2(xaddr_hi16(pw[i0 + j], hb));
#else
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const uint2*>(hs + xoff_hi16(pw[i0 + j]));
#endif
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
#ifdef SRNN_SHARED_GATHER
                        if (i0 + j < NP) h[j] = lds_u32(xaddr_hi16(pw[i0 + j], hb));
#else
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const uint32_t*>(hs + xoff_hi16(pw[i0 + j]));
#endif
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
#ifdef SRNN_SHARED_GATHER
                        if (i0 + j < NP) h[j] = lds_u16(xaddr_hi16(pw[i0 + j], hb));
#else
                        if (i0 + j < NP) h[j] = *reinterpret_cast<const unsigned short*>(hs + xoff_hi16(pw[i0 + j]));
#endif
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (i0 + j < NP) acc[0] = fma_f16f16f32(pw[i0 + j], h[j], acc[0]);
                }
            }
        }
    }
};

// Shared-memory weight tier (capacity planner): slots
// [NP, n_w) of a lane live in shared memory as [slot][thread] words (a
// conflict-free LDS.32/.64 per slot) instead of registers; the gather and the
// FMAs are the same as for register slots.  Used only when a layer's pairs do
// not fit the register file ("larger layer sizes").
template <int BT, bool F16>
__device__ __forceinline__ void operate_smem_tier(float (&acc)[BT], const unsigned char* hs, const void* ws,
                                                  int np_reg, int n_w, int nt, const unsigned char* hs2 = nullptr) {
    // (generic gathers here: the shared-window form measured slower for the C5 tier, 43.8 -> 45.2 us/step)
    for (int i0 = np_reg; i0 < n_w; i0 += 4) {
        if (F16) {
            const uint32_t* w32 = static_cast<const uint32_t*>(ws) + static_cast<size_t>(i0 - np_reg) * nt + threadIdx.x;
            uint32_t wv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = w32[j * nt];
            if (BT == 16) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t o = (wv[j] >> 12) & 0xffff0u;
                    const uint4 ha = *reinterpret_cast<const uint4*>(hs + o);
                    const uint4 hb = *reinterpret_cast<const uint4*>(hs2 + o);
                    const uint32_t hv[8] = {ha.x, ha.y, ha.z, ha.w, hb.x, hb.y, hb.z, hb.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        acc[(2 * q) % BT] = fma_f16f16f32(wv[j], hv[q], acc[(2 * q) % BT]);
                        acc[(2 * q + 1) % BT] = fma_f16f16f32(wv[j], hv[q] >> 16, acc[(2 * q + 1) % BT]);
                    }
                }
            } else if (BT == 8) {
                uint4 h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) h[j] = *reinterpret_cast<const uint4*>(hs + ((wv[j] >> 12) & 0xffff0u));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[0] = fma_f16f16f32(wv[j], h[j].x, acc[0]);
                    acc[1 % BT] = fma_f16f16f32(wv[j], h[j].x >> 16, acc[1 % BT]);
                    acc[2 % BT] = fma_f16f16f32(wv[j], h[j].y, acc[2 % BT]);
                    acc[3 % BT] = fma_f16f16f32(wv[j], h[j].y >> 16, acc[3 % BT]);
                    acc[4 % BT] = fma_f16f16f32(wv[j], h[j].z, acc[4 % BT]);
                    acc[5 % BT] = fma_f16f16f32(wv[j], h[j].z >> 16, acc[5 % BT]);
                    acc[6 % BT] = fma_f16f16f32(wv[j], h[j].w, acc[6 % BT]);
                    acc[7 % BT] = fma_f16f16f32(wv[j], h[j].w >> 16, acc[7 % BT]);
                }
            } else if (BT == 4) {
                uint2 h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) h[j] = *reinterpret_cast<const uint2*>(hs + (wv[j] >> 16));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[0] = fma_f16f16f32(wv[j], h[j].x, acc[0]);
                    acc[1 % BT] = fma_f16f16f32(wv[j], h[j].x >> 16, acc[1 % BT]);
                    acc[2 % BT] = fma_f16f16f32(wv[j], h[j].y, acc[2 % BT]);
                    acc[3 % BT] = fma_f16f16f32(wv[j], h[j].y >> 16, acc[3 % BT]);
                }
            } else if (BT == 2) {
                uint32_t h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) h[j] = *reinterpret_cast<const uint32_t*>(hs + (wv[j] >> 16));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[0] = fma_f16f16f32(wv[j], h[j], acc[0]);
                    acc[1 % BT] = fma_f16f16f32(wv[j], h[j] >> 16, acc[1 % BT]);
                }
            } else {
                uint32_t h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) h[j] = *reinterpret_cast<const unsigned short*>(hs + (wv[j] >> 16));
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[0] = fma_f16f16f32(wv[j], h[j], acc[0]);
            }
        } else {
            const uint2* w64 = static_cast<const uint2*>(ws) + static_cast<size_t>(i0 - np_reg) * nt + threadIdx.x;
            uint2 wv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) wv[j] = w64[j * nt];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float w = __uint_as_float(wv[j].y);
                if (BT == 4) {
                    const float4 h = *reinterpret_cast<const float4*>(hs + wv[j].x);
                    acc[0] = fmaf(w, h.x, acc[0]);
                    acc[1 % BT] = fmaf(w, h.y, acc[1 % BT]);
                    acc[2 % BT] = fmaf(w, h.z, acc[2 % BT]);
                    acc[3 % BT] = fmaf(w, h.w, acc[3 % BT]);
                } else if (BT == 2) {
                    const float2 h = *reinterpret_cast<const float2*>(hs + wv[j].x);
                    acc[0] = fmaf(w, h.x, acc[0]);
                    acc[1 % BT] = fmaf(w, h.y, acc[1 % BT]);
                } else {
                    acc[0] = fmaf(w, *reinterpret_cast<const float*>(hs + wv[j].x), acc[0]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Dense tensor-core comparator (the
// dense persistent RNN of Sec. 3.2, whose V100 version keeps U_r in registers
// and runs on CUDA cores).  Here a CTA owns MT tiles of 16 rows and the 16
// warps split the H columns into k-blocks of 16: warp w multiplies its
// k-blocks with mma.sync.m16n8k16 (A = U_r fragment from registers or shared
// memory, B = 16 staged h rows via ldmatrix.trans, N = 8 samples), the warps'
// partial 16x8 tiles are summed in shared memory in a fixed order (no
// atomics: deterministic), and the result lands in zs like the sparse
// butterfly's.  A per-CTA tile is 16 x 8 x H: far below tcgen05's 128-row
// minimum, so the warp-level MMA is the fitting unit here.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldmatrix_x2_trans(uint32_t& b0, uint32_t& b1, const void* row_addr) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(row_addr));
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(a));
}
__device__ __forceinline__ void mma_16816(float& d0, float& d1, float& d2, float& d3, const uint4& a, uint32_t b0,
                                          uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

template <int NF, int MT>
struct DenseFrags {
    uint4 a[NF];  // fragment f = kk * MT + m (k-block kk of this warp, row tile m)
    __device__ __forceinline__ void load(const RecParams& p, size_t img0, int nf_reg) {
#pragma unroll
        for (int f = 0; f < NF; ++f)
            a[f] = f < nf_reg ? p.img_dense[img0 + static_cast<size_t>(f) * p.threads] : make_uint4(0u, 0u, 0u, 0u);
    }
    // red: [warps][MT][16][8] fp32 partial tiles; hs: [hs_rows][16 B]
    __device__ __forceinline__ void operate(const unsigned char* hs, const uint4* ws, float* red, int kpw, int nf_reg,
                                            int nt) const {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        // two accumulator sets (even / odd k-blocks) halve the dependent mma chain
        float e0[MT], e1[MT], e2[MT], e3[MT], o0[MT], o1[MT], o2[MT], o3[MT];
#pragma unroll
        for (int m = 0; m < MT; ++m) e0[m] = e1[m] = e2[m] = e3[m] = o0[m] = o1[m] = o2[m] = o3[m] = 0.0f;
        const unsigned char* hw = hs + (static_cast<size_t>(warp) * kpw * 16 + (lane & 15)) * 16;
#pragma unroll
        for (int f = 0; f < NF; f += MT) {
            if (f < nf_reg) {  // warp-uniform
                uint32_t b0, b1;
                ldmatrix_x2_trans(b0, b1, hw + (f / MT) * 256);
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    if ((f / MT) & 1)
                        mma_16816(o0[m], o1[m], o2[m], o3[m], a[f + m], b0, b1);
                    else
                        mma_16816(e0[m], e1[m], e2[m], e3[m], a[f + m], b0, b1);
                }
            }
        }
        const int nf = MT * kpw;
        for (int f = nf_reg; f < nf; f += MT) {  // shared-memory fragments
            uint32_t b0, b1;
            ldmatrix_x2_trans(b0, b1, hw + (f / MT) * 256);
#pragma unroll
            for (int m = 0; m < MT; ++m)
                mma_16816(e0[m], e1[m], e2[m], e3[m], ws[static_cast<size_t>(f + m - nf_reg) * nt + threadIdx.x], b0, b1);
        }
        const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            float* r = red + ((warp * MT + m) * 16 + gid) * 8 + 2 * tig;
            *reinterpret_cast<float2*>(r) = make_float2(e0[m] + o0[m], e1[m] + o1[m]);
            *reinterpret_cast<float2*>(r + 64) = make_float2(e2[m] + o2[m], e3[m] + o3[m]);
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
    static constexpr int value = F16 ? (NP <= 12 ? 640 : NP <= 32 ? 512 : NP <= 64 ? 384 : 256)
                                     : (NP <= 4 ? 768 : NP <= 12 ? 640 : NP <= 32 ? 512 : NP <= 48 ? 384 : 256);
};
// BT = 16 (fp16) holds 16 accumulators and two 16-byte gathers per slot: one
// register tier more than the other tiles.  Must match max_threads_for().
template <int NP, bool F16, int BT>
struct MaxThreadsBT {
    static constexpr int value =
        (F16 && BT == 16) ? (NP <= 4 ? 640 : NP <= 8 ? 512 : NP <= 16 ? 384 : 256) : MaxThreads<NP, F16>::value;
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

// MT = 0: the sparse kernel (NP register slots per lane); MT = -1: the same with 8 poll
// slots per thread (plans whose threads own more chunks than poll_slots); MT = -2: the sparse
// kernel of a column-split plan (2-CTA clusters; compiled separately so the other instances
// carry none of its code).  MT >= 1: the dense
// tensor-core comparator (NP register A fragments per lane, MT row tiles).
template <int NP, int BT, int G, bool F16, int MT = 0>
__global__ void __launch_bounds__(MT > 0 ? kDenseThreads : MaxThreadsBT<NP, F16, BT>::value, 1)
    srnn_persistent_kernel(const __grid_constant__ RecParams p) {
    using F = Fmt<F16, BT>;
    constexpr bool DENSE = MT > 0;
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = p.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    const int cta = blockIdx.x;
    const int u0 = p.cta_unit0[cta];
    const int U = p.cta_unit0[cta + 1] - u0;
    const int n_items = U * BT;                       // epilogue items (unit, sample) of one tile
    const int item_rounds = (n_items + nt - 1) / nt;  // uniform within the CTA
    const int umax_bt = p.units_max * BT;
    // shared memory: hs [H][BT] at offset 0 (E bytes per unit), then fp32 areas
    unsigned char* hs = smem;
    // (column split: only this CTA's column half is staged, hsplit units; must match smem_for)
    const size_t hs_bytes = DENSE ? static_cast<size_t>(p.hs_rows) * 16
                                  : static_cast<size_t>(p.csplit != 0 ? p.hsplit : H) * F::E;
    float* zs = reinterpret_cast<float*>(smem + ((hs_bytes + 15) & ~static_cast<size_t>(15)));
    // zs: one BT-row of reduced sums per (virtual) row -- heavy rows split into pieces
    // (class balancing) have several, summed in the epilogue
    const int zrows = max(G * p.units_max, p.vrows_max);
    constexpr bool CS = MT == -2;  // column split over a 2-CTA cluster (p.csplit)
    const int crank = cta & 1;                // rank in the cluster (column half) when CS
    if (CS) {  // the column split needs the 2-CTA cluster launch (srnn_api.cpp / launch_one)
        uint32_t ncl, rk;
        asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rk));
        if (ncl != 2u || rk != static_cast<uint32_t>(crank)) {
            if (threadIdx.x == 0) atomicCAS(p.status, 0, -4 /* SRNN_ERR_STATE */);
            return;
        }
    }
    const int zbuf = zrows * BT;                             // floats of one zs buffer (two when CS: step parity)
    float* bpsb = zs + (CS ? 2 : 1) * zbuf;                  // b' double buffer: [2][item][G]
    float* cs = bpsb + 2 * G * umax_bt;                      // LSTM c / GRU fp32 h_{t-1}: [n_tiles][item]
    // b' TMA windows [2][G][kBpWin][BT][boxu] + two mbarriers (only when the host passed a map)
#ifdef SRNN_ABL_NO_BP_TMA
    constexpr bool bp_tma = false;
#else
    const bool bp_tma = G == 1 && p.bp_tma != 0;  // RNN cells only (the gate cells keep cp.async: registers)
#endif
    const int boxu = p.bp_boxu;
#ifndef SRNN_GENERIC_SMEM_PTRS
    // carve-up by byte offsets from the shared array (aligned in the shared window), so every
    // pointer below stays in the shared state space: LDS / STS, not generic loads, in the
    // epilogue's b' read and the abort-flag read after the staging barrier
    const uint32_t sm_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t cs_end = static_cast<uint32_t>(
        reinterpret_cast<unsigned char*>(cs + (G >= 3 ? p.n_tiles * umax_bt : 0)) - smem);
    const uint32_t bp_al = bp_tma ? 127u : 0u;  // TMA destination: 128-byte aligned
    float* bpw = reinterpret_cast<float*>(smem + (((sm_base + cs_end + bp_al) & ~bp_al) - sm_base));
    uint64_t* bp_mbar = reinterpret_cast<uint64_t*>(bpw + (bp_tma ? 2 * G * kBpWin * BT * boxu : 0));
    int* s_abort = reinterpret_cast<int*>(bp_mbar + (bp_tma ? 2 : 0));
    const uint32_t ab_end = static_cast<uint32_t>(reinterpret_cast<unsigned char*>(s_abort + 1) - smem);
    unsigned char* ws = smem + (((sm_base + ab_end + 15u) & ~15u) - sm_base);  // smem weight tier
#else
    float* bpw = reinterpret_cast<float*>(  // TMA destination: 128-byte aligned
        (reinterpret_cast<uintptr_t>(cs + (G >= 3 ? p.n_tiles * umax_bt : 0)) + (bp_tma ? 127 : 0)) &
        ~static_cast<uintptr_t>(bp_tma ? 127 : 0));
    uint64_t* bp_mbar = reinterpret_cast<uint64_t*>(bpw + (bp_tma ? 2 * G * kBpWin * BT * boxu : 0));
    int* s_abort = reinterpret_cast<int*>(bp_mbar + (bp_tma ? 2 : 0));
    unsigned char* ws = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(s_abort + 1) + 15) & ~static_cast<uintptr_t>(15));  // smem weight tier
#endif

    const int L = DENSE ? 32 : p.lanes_per_row;
    const int n_w = DENSE ? 0 : p.warp_slots[cta * (p.threads >> 5) + warp];
    const int n_chunks = p.tile_bytes >> 4;     // 16-byte chunks of one exchange image
    const int c_lo = CS && crank ? (p.hsplit * F::E) >> 4 : 0;             // first chunk this CTA stages
    const int n_ch = CS ? (crank ? n_chunks - c_lo : (p.hsplit * F::E) >> 4) : n_chunks;
    const unsigned char* hs2 = hs + H * 16;     // BT = 16: second hs plane
    // shared-window address of hs, from an opaque cvta so the compiler keeps it in a register
    // instead of re-deriving the window base in every operate group
    uint32_t hs_sb;
    asm volatile("{\n.reg .u64 t;\ncvta.to.shared.u64 t, %1;\ncvt.u32.u64 %0, t;\n}" : "=r"(hs_sb) : "l"(hs));
    const int GH = G * H;
    // values after the last unit that pad the image to whole chunks (written by the last CTA)
    const int n_pad = (cta == static_cast<int>(gridDim.x) - 1 && !(F16 && BT == 16))
                          ? (p.tile_bytes - H * F::E) / F::VB : 0;

    // ---- prologue: weights HBM -> registers (once per forward) ----
    Weights<NP, BT, F16> W;
    DenseFrags<DENSE ? NP : 1, DENSE ? MT : 1> DW;
    const int ns = p.smem_slots;  // shared-memory tier slots per lane (multiple of 4)
    const size_t img_cta = static_cast<size_t>(cta) * (NP + ns) * p.threads;
    const int dense_nf_reg = DENSE ? min(NP, p.dense_nf) : 0;
    float* red = nullptr;  // dense: [warps][MT][16][8] partial tiles, after the fragment tier
    if constexpr (DENSE) {
        const size_t img_d = static_cast<size_t>(cta) * p.dense_nf * p.threads;
        DW.load(p, img_d + tid, dense_nf_reg);
        const size_t n = static_cast<size_t>(p.dense_nf - dense_nf_reg) * p.threads;
        const uint4* src = p.img_dense + img_d + static_cast<size_t>(dense_nf_reg) * p.threads;
        for (size_t i = tid; i < n; i += nt) reinterpret_cast<uint4*>(ws)[i] = src[i];
        red = reinterpret_cast<float*>(ws + n * 16);
        // staged h rows: zero once (rows >= H and, for BT = 4, the upper 8 bytes are never written)
        for (size_t i = tid; i < hs_bytes / 16; i += nt) reinterpret_cast<uint4*>(hs)[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
        W.load(p, img_cta + tid, n_w);
    }
    if (!DENSE && ns > 0) {
        const size_t n = static_cast<size_t>(ns) * p.threads;
        if (F16) {
            const uint32_t* src = p.img_f16 + img_cta + static_cast<size_t>(NP) * p.threads;
            for (size_t i = tid; i < n; i += nt) reinterpret_cast<uint32_t*>(ws)[i] = src[i];
        } else {
            const uint2* src = p.img_f32 + img_cta + static_cast<size_t>(NP) * p.threads;
            for (size_t i = tid; i < n; i += nt) reinterpret_cast<uint2*>(ws)[i] = src[i];
        }
    }

    const int act = p.act;
    const int lg_l = __ffs(L) - 1;  // L is a power of two: shifts, no per-step integer division
    const int krow = (warp << (5 - lg_l)) + (lane >> lg_l);  // local row of this lane
    // lane of the row that stores sample sbase (L >= BT), hoisted out of the time loop
    const int* pc = p.piece0 != nullptr ? p.piece0 + cta * (G * p.units_max + 1) : nullptr;
    // column split: this CTA's rows are all G * UQ rows of its cluster's units (its column half)
    const int UQ = CS ? p.cta_vunit0[cta + 1] - p.cta_vunit0[cta] : U;
    const int lu_off = CS && crank ? UQ - U : 0;  // cluster-local index of this CTA's first own unit
    const int n_vrows = CS ? G * UQ : pc != nullptr ? __ldg(pc + G * U) : G * U;  // (virtual) rows of this CTA
    const bool zs_writer = (lane & (L - 1)) < BT && krow < n_vrows;
    // reduced sum of local row k (gate * U + unit), sample b: the sum of its pieces
    float* zsp = zs;  // this step's zs buffer (column split: alternates with the step parity)
    auto zval = [&](int k, int b) -> float {
        if (CS) {  // own partial + the peer's (DSMEM), always in the order half 0 + half 1
            const int g = G == 1 ? 0 : k / U, u = G == 1 ? k : k - g * U;
            const float* a = zsp + (g * UQ + lu_off + u) * BT + b;
            const uint32_t la = static_cast<uint32_t>(__cvta_generic_to_shared(a));
            uint32_t ra;
            float peer;
#ifdef SRNN_DBG_CS_NODSMEM
            peer = 0.0f; (void)la; (void)ra;
#else
            // (no memory clobber: the cluster barrier before the epilogue orders these reads)
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(crank ^ 1));
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(peer) : "r"(ra));
#endif
            const float mine = *a;
            return crank == 0 ? mine + peer : peer + mine;
        }
        if (pc == nullptr) return zs[k * BT + b];
        const int v1 = __ldg(pc + k + 1);
        float z = 0.0f;
        for (int v = __ldg(pc + k); v < v1; ++v) z += zs[v * BT + b];
        return z;
    };
    // epilogue fast path (one item per thread): item e1 = tid -> (unit, sample)
    // exchange positions vs hidden units: the same unless the plan balances classes (unit_perm)
    auto real_unit = [&](int pos) { return p.unit_perm != nullptr ? __ldg(p.unit_perm + pos) : pos; };
    const int e1 = tid, e1_b = tid % BT;
    const bool e1_ok = tid < n_items;
    const int e1_unit = e1_ok ? real_unit(u0 + e1 / BT) : 0;
    const float* zs_e1 = zs + e1;
    float* const y_e1 = (p.y != nullptr && e1_ok) ? p.y + e1_b * p.y_bstride + e1_unit : nullptr;
    const float* const bp_e1 = p.bprime + static_cast<size_t>(e1_b) * GH + e1_unit;
    const int xo_e1 = e1_ok ? F::offset(H, u0 + e1 / BT, e1_b) : 0;  // exchange offset of item e1 in a tile image
    const bool row_leader = (lane & (L - 1)) == 0 && krow < n_vrows;
    if (tid == 0) *s_abort = 0;

    // Publish item e's h of (step s, tile k) into the exchange image of parity
    // s & 1 (one relaxed 16/32-bit store per item, tag (global step >> 1) & 1
    // in the LSB, reading R16); `ok` masks items.  The first item round also
    // writes the tagged pad values of the last CTA.
    auto store_tagged = [&](unsigned char* img, int off, float h, uint32_t tag) {
        if (F16)
            st_relaxed_u16(img + off, F::encode(h, tag));
        else
            st_relaxed_u32(img + off, F::encode(h, tag));
    };
    const bool drop_cta = (p.flags & kFlagDropPublish) && cta == 0;  // test hook: lost exchange message
    const bool jitter0 = (p.flags & kFlagJitter) && tid == 0;          // test hook: per-CTA delays
    auto publish = [&](int s, int k, int e, bool ok, float h) {
        if (drop_cta && s == 2) return;  // fault injection (CTA-uniform)
        const uint32_t g = p.epoch + static_cast<uint32_t>(s);  // global step: parity g & 1, tag (g >> 1) & 1
        unsigned char* dst = p.xbuf + static_cast<size_t>((g & 1u) * p.xbuf_tiles + k) * p.tile_bytes;
        const uint32_t tag = (g >> 1) & 1u;
#ifdef SRNN_PUB32
        if (F16 && BT >= 2 && BT <= 8) {  // A/B: two samples per 32-bit store
            const uint32_t v = F::encode(h, tag);
            const uint32_t nb = __shfl_down_sync(0xffffffffu, v, 1);
            if (ok && ((e % BT) & 1) == 0) st_relaxed_u32(dst + F::offset(H, u0 + e / BT, e % BT), v | (nb << 16));
        } else
#endif
        if (ok) store_tagged(dst, F::offset(H, u0 + e / BT, e % BT), h, tag);
        if (e < n_pad) store_tagged(dst, H * F::E + e * F::VB, 0.0f, tag);
    };

    // ---- exchange re-initialisation: the stale values of both parities must carry the
    // tags of global steps epoch - 2 / epoch - 1 (the host asks for it when the buffers
    // are fresh or were idle for some tiles; an aborted launch marks them dirty) ----
    if (!CS && (p.reinit || *reinterpret_cast<volatile int32_t*>(p.xdirty) != 0)) {  // CS: the host re-fills
        for (int q = 0; q < 2; ++q) {
            const uint32_t g = p.epoch + static_cast<uint32_t>(q);  // first step of this launch in parity g & 1
            const uint32_t stale = ((g - 2u) >> 1) & 1u;
            for (int k = 0; k < p.n_tiles; ++k) {
                unsigned char* dst = p.xbuf + static_cast<size_t>((g & 1u) * p.xbuf_tiles + k) * p.tile_bytes;
                for (int e = tid; e < n_items; e += nt) store_tagged(dst, F::offset(H, u0 + e / BT, e % BT), 0.0f, stale);
                if (tid < n_pad) store_tagged(dst, H * F::E + tid * F::VB, 0.0f, stale);
            }
        }
        cg::this_grid().sync();
        if (cta == 0 && tid == 0) *p.xdirty = 0;  // every CTA read the flag before the grid barrier
    }

    // ---- publish h_0 (tag = epoch) and initialise c ----
    for (int k = 0; k < p.n_tiles; ++k) {
        for (int j = 0; j < item_rounds; ++j) {
            const int e = tid + j * nt;
            const bool ok = e < n_items;
            const int unit = ok ? real_unit(u0 + e / BT) : 0, bg = k * BT + e % BT;
            float h = 0.0f;
            if (ok) {
                h = (p.h0 != nullptr && bg < p.B) ? p.h0[static_cast<size_t>(bg) * H + unit] : 0.0f;
                if (G == 4)
                    cs[k * umax_bt + e] = (p.c0 != nullptr && bg < p.B) ? p.c0[static_cast<size_t>(bg) * H + unit] : 0.0f;
                if (G == 3) cs[k * umax_bt + e] = h;  // GRU keeps its own fp32 h_{t-1} (the exchange carries fp16 in fp16 mode)
            }
            publish(0, k, e, ok, h);
        }
    }
    // b' windows by TMA: window w (steps w*kBpWin + 1 ..) lands in slot w & 1; phase (w >> 1) & 1
    auto bp_issue = [&](int w) {
        const int slot = w & 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // slot's previous generic reads
        const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(bp_mbar + slot));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"(static_cast<uint32_t>(G * kBpWin * BT * boxu * 4))
                     : "memory");
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const uint32_t dst = static_cast<uint32_t>(
                __cvta_generic_to_shared(bpw + static_cast<size_t>(slot * G + q) * kBpWin * BT * boxu));
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(dst), "l"(&p.bp_map), "r"(q * H + (u0 & ~3)), "r"(0), "r"(w * kBpWin), "r"(mb)
                : "memory");
        }
    };
    if (bp_tma && tid == 0) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bp_mbar + i)))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&p.bp_map) : "memory");
        bp_issue(0);
    }
    const bool grid_sync = (p.flags & kFlagGridSync) != 0u;
    if (grid_sync) cg::this_grid().sync();
    // launch-constant switches of the time loop in one register (as single flags the compiler
    // re-loaded them from the parameter bank every step, on the step's critical path)
    constexpr uint32_t kCtlJitter = 1u, kCtlBpTma = 2u;
    uint32_t kctl = (jitter0 ? kCtlJitter : 0u) | (bp_tma ? kCtlBpTma : 0u);
    // opaque: kept in a register -- RNN tiles <= 4 with a 128-register budget only (same-box
    // A/B: C2 2.165 -> 2.115 us/step, B = 8 2.86 -> 2.83; the 96-register instances lost: 1152 @
    // 10% 1.71 -> 1.87)
    constexpr bool kPinCtl = G == 1 && BT <= 4 && MaxThreadsBT<NP, F16, BT>::value <= 512;
    if constexpr (kPinCtl) asm volatile("" : "+r"(kctl));
    // shared-window address of this lane's zs slot (fast path: L >= BT, one writer per sample)
    int sbase0 = 0;
    for (int lvl = 0, half = BT / 2; half >= 1; ++lvl, half /= 2)
        if (lane & (1 << lvl)) sbase0 += half;
    uint32_t zs_wa = static_cast<uint32_t>(__cvta_generic_to_shared(zs)) +
                     static_cast<uint32_t>(krow * BT + sbase0) * 4u;
    if constexpr (kPinCtl) asm volatile("" : "+r"(zs_wa));
    __syncthreads();

    // pipelined host forward: b' arrives in chunks of steps and the ready counter only
    // grows, so each thread re-polls (acquire) only when its last observed value is behind
    uint32_t bp_seen = p.bp_ready_base;
    bool bp_failed = false;  // the b' readiness wait timed out: abort at the next barrier
    const bool bp_pipelined = p.bp_ready != nullptr;
    // one item per thread (the common case): b' source of item e1 = tid hoisted out of the time loop
    auto issue_bprime = [&](int s, int k, int b) {
        if (kPinCtl ? (kctl & kCtlBpTma) != 0u : bp_tma) {  // one thread loads window w + 1 during the first step of window w (s = that step + 1)
            if (tid == 0 && (s - 2) % kBpWin == 0 && (s - 2 + kBpWin) < p.T) bp_issue((s - 2) / kBpWin + 1);
            return;
        }
        float* dstb = bpsb + b * G * umax_bt;
        if (bp_pipelined && tid < n_items && static_cast<int32_t>(bp_seen - p.bp_ready_base) < s) {
            Watchdog wdb{0ull, 0u};
            while (static_cast<int32_t>((bp_seen = ld_acquire_u32(p.bp_ready)) - p.bp_ready_base) < s)
                if (watchdog_tick(wdb, p.status, p.timeout_ns)) {
                    bp_failed = true;
                    return;
                }
        }
        if (item_rounds == 1) {
            if (e1_ok) {
                float* d = dstb + e1 * G;
                if (k * BT + e1_b < p.B) {
                    const float* src = bp_e1 + (static_cast<size_t>(s - 1) * p.B + k * BT) * GH;
#pragma unroll
                    for (int q = 0; q < G; ++q) cp_async_f32(d + q, src + q * H);
                } else {
#pragma unroll
                    for (int q = 0; q < G; ++q) d[q] = 0.0f;
                }
            }
            return;
        }
        for (int j = 0; j < item_rounds; ++j) {
            const int e = tid + j * nt;
            if (e < n_items) {
                const int unit = real_unit(u0 + e / BT), bg = k * BT + e % BT;
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    if (bg < p.B)
                        cp_async_f32(&dstb[e * G + q], p.bprime + (static_cast<size_t>(s - 1) * p.B + bg) * GH + q * H + unit);
                    else
                        dstb[e * G + q] = 0.0f;
                }
            }
        }
    };
    int buf = 0;
    if (p.T >= 1) issue_bprime(1, 0, 0);
    cp_async_commit();
#ifdef SRNN_PROFILE
    const bool prof_on = (p.flags & kFlagProfile) && p.profile != nullptr;
#endif
    const int n_loaders = p.loader_threads > 0 ? min(p.loader_threads, nt) : nt;
    Poller<F16, BT, poll_slots(NP, F16, BT, MT == -1), DENSE> poll;
    // The first poll round's addresses, the exchange store address, the global step and the y
    // pointer hoisted out of the time loop: fp16 RNN tiles of 4 (instances of <= 512 threads).
    // Same-box A/B with the shared-window gathers: C2 2.204 -> 2.164 us/step, 1152 @ 10% and
    // 2304 @ 10% within noise; tiles of 8 slower (2.85 -> 3.10) and the gate cells slower
    // (C4 LSTM 2.06 -> 2.09), so they keep the per-step form.  -DSRNN_HOIST_POLL=0 / 1 forces.
#ifndef SRNN_HOIST_POLL
    constexpr bool kHoistPoll = F16 && BT == 4 && G == 1 && MaxThreadsBT<NP, F16, BT>::value <= 512 && MT <= 0;
#else
    constexpr bool kHoistPoll = SRNN_HOIST_POLL != 0 && G == 1 && MaxThreadsBT<NP, F16, BT>::value <= 512 && MT <= 0;
#endif
    const unsigned char* poll0 = p.xbuf + (static_cast<size_t>(c_lo) + tid) * 16;
    uint32_t poll_par = static_cast<uint32_t>(p.xbuf_tiles) * static_cast<uint32_t>(p.tile_bytes);
    const uint32_t poll_js = static_cast<uint32_t>(n_loaders) * 16u;
    unsigned char* pub0 = p.xbuf + xo_e1;  // this thread's exchange value of tile 0, parity 0 (RNN fast path)
    uint32_t poll_jmask = 0u;
#pragma unroll
    for (int j = 0; j < poll_slots(NP, F16, BT, MT == -1); ++j)
        if (tid + j * n_loaders < n_ch) poll_jmask |= 1u << j;
    // staged instance (partial progress): this thread's early chunks (chunk
    // tid + j * n_loaders < early_chunks; one poll batch, host-checked) and its warp's
    // early slots [0, n_we)
    constexpr bool STAGED = MT == -3;
    uint32_t sel_early = 0u;
    int n_we = 0;
    if constexpr (STAGED) {
#pragma unroll
        for (int j = 0; j < poll_slots(NP, F16, BT, false); ++j)
            if (tid + j * n_loaders < p.early_chunks) sel_early |= 1u << j;
        n_we = p.warp_early[cta * (p.threads >> 5) + warp];
    }

    // RNN fast-path epilogue state in two registers instead of per-step parameter / special
    // register reloads (the compiler rematerialised them at 128 registers): bit 0 this thread
    // owns an item, 1 the lost-message test hook, 2 its warp has items or pad values to publish,
    // 3 y is written; the running global step of h_{s-1}; y of step s for tile 0
    constexpr uint32_t kEpiItem = 1u, kEpiDrop = 2u, kEpiWarp = 4u, kEpiY = 8u;
    uint32_t epi_ctl = (e1_ok ? kEpiItem : 0u) | (drop_cta ? kEpiDrop : 0u) |
                       ((warp * 32 < max(n_items, n_pad)) ? kEpiWarp : 0u) | (y_e1 != nullptr ? kEpiY : 0u);
#ifndef SRNN_NO_PIN_EPI
    if constexpr (kHoistPoll) {  // pinned (else rematerialised from CTAID / parameter reloads every step)
        asm volatile("" : "+r"(epi_ctl));
        asm volatile("" : "+r"(poll_par));
        asm volatile("" : "+l"(pub0));
    }
#endif
    uint32_t g_run = p.epoch;
    float* y_run = y_e1;
    for (int s = 1; s <= p.T; ++s) {
        for (int k = 0; k < p.n_tiles; ++k) {
#ifdef SRNN_PROFILE
            long long* prof_all = prof_on
                                      ? p.profile + ((static_cast<size_t>(cta) * p.T + (s - 1)) * p.n_tiles + k) * 16
                                      : nullptr;
            long long* prof = tid == 0 ? prof_all : nullptr;
            int rounds = 0;
#endif
            SRNN_STAMP(0, clock64());
            // ---- load: h_{s-1} tile k -> hs; the first poll round goes out first ----
            // global step of h_{s-1}
            const uint32_t g_prev = kHoistPoll ? g_run : p.epoch + static_cast<uint32_t>(s - 1);
            // column split: only the chunks of this CTA's column half [c_lo, c_lo + n_ch)
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(
                p.xbuf + static_cast<size_t>((g_prev & 1u) * p.xbuf_tiles + k) * p.tile_bytes) + c_lo;
            // fp16 tiles of <= 4 samples send the first poll round before the b' prefetch (the
            // round trip hides the prefetch's address work); wider / fp32 tiles hold more chunks
            // per thread, whose registers would stay live across it (measured: slower), so they
            // poll after it
            constexpr bool kEarlyPoll = F16 && BT <= 4;
            if (kEarlyPoll && tid < n_loaders) {
                if constexpr (kHoistPoll)
                    poll.issue_at(poll0 + ((g_prev & 1u) ? poll_par : 0u) + static_cast<uint32_t>(k) * p.tile_bytes,
                                  poll_jmask, poll_js);
                else
                    poll.issue(src, tid, n_ch, n_loaders);
            }
            // b' of the NEXT tile -> shared memory (cp.async, double-buffered) while the
            // poll loads are in flight; it lands during this whole tile (this tile's b'
            // was issued one tile earlier)
            {
                const int ns = k + 1 < p.n_tiles ? s : s + 1, nk = k + 1 < p.n_tiles ? k + 1 : 0;
#ifndef SRNN_ABL_NO_BP
                if (ns <= p.T) issue_bprime(ns, nk, buf ^ 1);
#endif
                cp_async_commit();
            }

            if (!kEarlyPoll && tid < n_loaders) {
                if constexpr (kHoistPoll)
                    poll.issue_at(poll0 + ((g_prev & 1u) ? poll_par : 0u) + static_cast<uint32_t>(k) * p.tile_bytes,
                                  poll_jmask, poll_js);
                else
                    poll.issue(src, tid, n_ch, n_loaders);
            }
            bool failed = bp_failed;
            float acc_early[BT];  // staged instance: the early slots' partial sums
#pragma unroll
            for (int b = 0; b < BT; ++b) acc_early[b] = 0.0f;
            if constexpr (STAGED) {
                // early chunks -> hs, barrier, operate on the early slots while the late chunks
                // (issued in the same poll batch) are still arriving, then complete those
                if (tid < n_loaders && !poll.complete(src, hs, n_ch, (g_prev >> 1) & 1u, !grid_sync, p.status,
                                                      p.timeout_ns, p.poll_backoff_ns, n_loaders, nullptr, nullptr,
                                                      sel_early))
                    failed = true;
                __syncthreads();
                SRNN_STAMP(13, clock64());
#ifndef SRNN_ABL_NO_OP
                W.operate_span(acc_early, hs, 0, n_we, nullptr, hs_sb);
#endif
                SRNN_STAMP(14, clock64());
            }
            if (tid < n_loaders &&
                !poll.complete(src, hs, n_ch, (g_prev >> 1) & 1u, !grid_sync, p.status, p.timeout_ns,
                               p.poll_backoff_ns, n_loaders,
#ifdef SRNN_PROFILE
                               prof_all ? &rounds : nullptr, prof ? prof + 10 : nullptr,
#else
                               nullptr, nullptr,
#endif
                               STAGED ? ~sel_early : ~0u))
                failed = true;
#ifdef SRNN_PROFILE
            if (prof_all) atomicMax(reinterpret_cast<unsigned long long*>(prof_all + 9), static_cast<unsigned long long>(rounds));
#endif
            if (failed) *s_abort = 1;
            __syncthreads();
            SRNN_STAMP(1, clock64());
            SRNN_STAMP(8, rounds);
            SRNN_STAMP(12, static_cast<long long>(globaltimer_ns()));
            // abort check: the flag is read here, the branch is taken after the operate (its
            // latency hides behind it; an aborted step computes on stale hs but never publishes)
            const int aborted = *reinterpret_cast<volatile int*>(s_abort);

#ifdef SRNN_ABL_EARLY_ABORT
            if (aborted) goto done;
#endif

            if (CS) zsp = zs + (s & 1) * zbuf;
            // ---- operate + reduce ----
            if constexpr (DENSE) {
                DW.operate(hs, reinterpret_cast<const uint4*>(ws), red, p.dense_kpw, dense_nf_reg, nt);
                SRNN_STAMP(4, clock64());
                __syncthreads();
                // fixed-order sum of the 16 warps' partial tiles -> zs[local row][sample]
                for (int e = tid; e < G * U * BT; e += nt) {
                    const int r = e / BT, b = e % BT;
                    const float* q = red + r * 8 + b;
                    float v[kDenseThreads / 32];  // all loads in flight, then a fixed-order sum
#pragma unroll
                    for (int w = 0; w < kDenseThreads / 32; ++w) v[w] = q[w * MT * 128];
                    float z = 0.0f;
#pragma unroll
                    for (int w = 0; w < kDenseThreads / 32; ++w) z += v[w];
                    zs[e] = z;
                }
                SRNN_STAMP(5, clock64());
            } else {
                float acc[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) acc[b] = acc_early[b];
#ifndef SRNN_ABL_NO_OP  // A/B ablation builds only (scripts/abl.sh): phase costs
                if constexpr (STAGED) {
                    W.operate_span(acc, hs, n_we, n_w, nullptr, hs_sb);  // the late slots (no smem tier: host-checked)
                } else {
                    W.operate(acc, hs, n_w, hs2, hs_sb);
                    if (n_w > NP) operate_smem_tier<BT, F16>(acc, hs, ws, NP, n_w, nt, hs2);
                }
#endif
                SRNN_STAMP(4, clock64());
                // ---- reduce over the row's L lanes, fixed order ----
                // L >= BT: log2(BT) halving levels (each lane keeps half of its
                // samples and receives the partner's sums for them: BT-1
                // shuffles instead of BT*log2(BT)), then plain levels; lane j of
                // the row then holds the sum of sample bitrev(j mod BT).
                // L < BT: plain xor butterfly, the row leader holds all samples.
                int sbase = 0;
#ifdef SRNN_ABL_NO_BFLY
                if (false) {
#else
                if (L >= BT) {
#endif
#pragma unroll
                    for (int lvl = 0, half = BT / 2; half >= 1; ++lvl, half /= 2) {
                        const int m = 1 << lvl;
                        const bool upper = (lane & m) != 0;
#pragma unroll
                        for (int i = 0; i < half; ++i) {
                            const float keep = upper ? acc[(i + half) % BT] : acc[i];
                            const float send = upper ? acc[i] : acc[(i + half) % BT];
                            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                        }
                        if (upper) sbase += half;
                    }
#pragma unroll
                    for (int m = BT; m <= 16; m <<= 1)
                        if (m < L) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], m);
                } else
#ifdef SRNN_ABL_NO_BFLY
                if (false)
#endif
                {
#pragma unroll
                    for (int m = 16; m >= 1; m >>= 1) {
                        if (m < L) {  // warp-uniform
#pragma unroll
                            for (int b = 0; b < BT; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], m);
                        }
                    }
                }
                SRNN_STAMP(5, clock64());
                if (L >= BT) {
                    if (CS || !kPinCtl) {
                        if (zs_writer) zsp[krow * BT + sbase] = acc[0];
                    } else if (zs_writer) {  // (sbase == sbase0: the same lane bits)
                        asm volatile("st.shared.f32 [%0], %1;" ::"r"(zs_wa), "f"(acc[0]) : "memory");
                    }
                } else if (row_leader) {
#pragma unroll
                    for (int b = 0; b < BT; ++b) zsp[krow * BT + b] = acc[b];
                }
            }
            if (!CS && aborted) goto done;
            if ((kPinCtl ? (kctl & kCtlBpTma) != 0u : bp_tma) && (s - 1) % kBpWin == 0) {  // first step of a b' window: wait for its TMA load
                const int w = (s - 1) / kBpWin;
                const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(bp_mbar + (w & 1)));
                Watchdog wdb{0ull, 0u};
                uint32_t done_ = 0;
                while (true) {
                    asm volatile(
                        "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}"
                        : "=r"(done_)
                        : "r"(mb), "r"(static_cast<uint32_t>((w >> 1) & 1))
                        : "memory");
                    if (done_) break;
                    if (watchdog_tick(wdb, p.status, p.timeout_ns)) break;  // the next poll aborts the launch
                }
            }
            if (!kPinCtl || !(kctl & kCtlBpTma))  // (b' by TMA: no cp.async in flight)
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's b' (the newest group may pend)
            SRNN_STAMP(6, clock64());
            // fast path with b' by TMA: this item's b' is in shared memory once the window's
            // mbarrier wait above has passed, so the epilogue warps read it before the barrier
            // (off the chain zs -> g -> publish that follows it)
            float bp_pre = 0.0f;
            if constexpr (kHoistPoll) {
                if ((kctl & kCtlBpTma) && item_rounds == 1 && (epi_ctl & kEpiItem))
                    bp_pre = bpw[static_cast<size_t>(((s - 1) & (2 * kBpWin - 1)) * BT * boxu) + (e1 % BT) * boxu +
                                 (u0 & 3) + e1 / BT];
            }
            if (CS) {
                // both CTAs' partial sums are complete (release / acquire across the cluster); the
                // pair takes the same abort decision (own flag or the peer's) so neither waits alone
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
                const uint32_t la = static_cast<uint32_t>(__cvta_generic_to_shared(s_abort));
                uint32_t ra;
                int peer_ab;
#ifdef SRNN_DBG_CS_NODSMEM
                peer_ab = 0; (void)la; (void)ra;
#else
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(crank ^ 1));
                asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(peer_ab) : "r"(ra) : "memory");
#endif
                if (aborted | peer_ab) goto done;
            } else {
                __syncthreads();
            }
            SRNN_STAMP(2, clock64());

            // ---- epilogue: activation / gates, y, tagged publish of h_s ----
            // b' of this (step, tile): bps[e * G + q] (cp.async double buffer), or the TMA window
            // element (q, j, b, unit) at bpt[q * kBpWin * BT * boxu + b * boxu + (u0 & 3) + unit] (the box
            // starts at the 16-byte aligned column u0 & ~3)
            const float* bps = bpsb + buf * G * umax_bt;
            const float* bpt = bpw + static_cast<size_t>((((s - 1) / kBpWin) & 1) * G * kBpWin + (s - 1) % kBpWin) * BT * boxu;
            auto bpv = [&](int e, int q) -> float {
                return bp_tma ? bpt[q * kBpWin * BT * boxu + (e % BT) * boxu + (u0 & 3) + e / BT] : bps[e * G + q];
            };
            if (kPinCtl ? (kctl & kCtlJitter) != 0u : jitter0) {
                const uint32_t r = (static_cast<uint32_t>(cta) * 2654435761u) ^ (static_cast<uint32_t>(s * 40503 + k));
                __nanosleep((r >> 7) & 2047u);
            }
            if (G == 1 && item_rounds == 1) {
                // fast path (one item per thread, RNN): hoisted offsets; the exchange store goes
                // out first (it is the step's critical path), y / h_T after it
              if constexpr (kHoistPoll) {
              if (epi_ctl & kEpiWarp) {  // warps without items go straight to the barrier
                float h = 0.0f;
                const uint32_t g = g_prev + 1u;  // parity g & 1, tag (g >> 1) & 1
                if (epi_ctl & kEpiItem)
                    h = activation<F16>(act, (pc == nullptr && !CS ? zs_e1[0] : zval(e1 / BT, e1_b)) +
                                                 ((kctl & kCtlBpTma) ? bp_pre : bpv(e1, 0)));
                if ((epi_ctl & kEpiItem) && !((epi_ctl & kEpiDrop) && s == 2))
                    store_tagged(pub0 + ((g & 1u) ? poll_par : 0u) + static_cast<uint32_t>(k) * p.tile_bytes, 0, h,
                                 (g >> 1) & 1u);
                publish(s, k, e1, false, 0.0f);  // only the pad values of the last chunk (last CTA)
                if ((epi_ctl & kEpiItem) && k * BT + e1_b < p.B) {
#ifndef SRNN_ABL_NO_Y
                    if (epi_ctl & kEpiY) y_run[k * BT * p.y_bstride] = h;
#endif
                    if (s == p.T && p.hT != nullptr) p.hT[static_cast<size_t>(k * BT + e1_b) * H + e1_unit] = h;
                }
                if ((epi_ctl & kEpiY) && k == p.n_tiles - 1) y_run += p.y_tstride;  // (only this block uses y_run)
              }
              } else {
                float h = 0.0f;
                const uint32_t g = p.epoch + static_cast<uint32_t>(s);  // parity g & 1, tag (g >> 1) & 1
                if (e1_ok) h = activation<F16>(act, (pc == nullptr && !CS ? zs_e1[0] : zval(e1 / BT, e1_b)) + bpv(e1, 0));
#ifdef SRNN_ABL_Y_FIRST
                if (y_e1 != nullptr && k * BT + e1_b < p.B) y_e1[(s - 1) * p.y_tstride + k * BT * p.y_bstride] = h;
#endif
                if (e1_ok && !(drop_cta && s == 2))
                    store_tagged(p.xbuf + static_cast<size_t>((g & 1u) * p.xbuf_tiles + k) * p.tile_bytes, xo_e1, h,
                                 (g >> 1) & 1u);
                publish(s, k, e1, false, 0.0f);  // only the pad values of the last chunk (last CTA)
                if (e1_ok && k * BT + e1_b < p.B) {
#if !defined(SRNN_ABL_NO_Y) && !defined(SRNN_ABL_Y_FIRST)
                    if (y_e1 != nullptr) y_e1[(s - 1) * p.y_tstride + k * BT * p.y_bstride] = h;
#endif
                    if (s == p.T && p.hT != nullptr) p.hT[static_cast<size_t>(k * BT + e1_b) * H + e1_unit] = h;
                }
              }
            } else
            for (int j = 0; j < item_rounds; ++j) {
                const int e = tid + j * nt;
                const bool ok = e < n_items;
                float h = 0.0f;
                if (ok) {
                    const int unit = real_unit(u0 + e / BT), bg = k * BT + e % BT;
                    if (G == 1) {
                        h = activation<F16>(p.act, zval(e / BT, e % BT) + bpv(e, 0));
                    } else if (G == 3) {
                        // GRU (R15): r, z from the product; the reset gate scales the
                        // n-gate product + b_hn; the previous h of this item stays in fp32 in cs
                        const float r = sigmoid_g<F16>(zval(0 * U + e / BT, e % BT) + bpv(e, 0));
                        const float u = sigmoid_g<F16>(zval(1 * U + e / BT, e % BT) + bpv(e, 1 % G));
                        const float bhn = p.bias_hn != nullptr ? p.bias_hn[unit] : 0.0f;
                        const float n = tanh_g<F16>(fmaf(r, zval(2 * U + e / BT, e % BT) + bhn, bpv(e, 2 % G)));
                        float* hp = &cs[k * umax_bt + e];
                        h = fmaf(u, *hp - n, n);  // (1 - u) n + u h_prev
                        *hp = h;
                    } else {
                        const float zi = zval(0 * U + e / BT, e % BT) + bpv(e, 0);
                        const float zf = zval(1 * U + e / BT, e % BT) + bpv(e, 1 % G);
                        const float zg = zval(2 * U + e / BT, e % BT) + bpv(e, 2 % G);
                        const float zo = zval(3 * U + e / BT, e % BT) + bpv(e, 3 % G);
                        float* cp = &cs[k * umax_bt + e];
                        const float c = sigmoid_g<F16>(zf) * (*cp) + sigmoid_g<F16>(zi) * tanh_g<F16>(zg);
                        *cp = c;
                        h = sigmoid_g<F16>(zo) * tanh_g<F16>(c);
                        if (s == p.T && p.cT != nullptr && bg < p.B) p.cT[static_cast<size_t>(bg) * H + unit] = c;
                    }
                    if (bg < p.B) {
                        if (p.y != nullptr) p.y[bg * p.y_bstride + (s - 1) * p.y_tstride + unit] = h;
                        if (s == p.T && p.hT != nullptr) p.hT[static_cast<size_t>(bg) * H + unit] = h;
                    }
                }
                publish(s, k, e, ok, h);
            }
            SRNN_STAMP(3, clock64());
            SRNN_STAMP(11, static_cast<long long>(globaltimer_ns()));
            if (grid_sync) cg::this_grid().sync();
#ifndef SRNN_ABL_NO_BAR3
            // Start polling for the next tile only once this CTA has published:
            // early pollers only add stale round trips and contend with the
            // epilogue warps for the LSU (measured: -6..10% step time).
            __syncthreads();
#endif
            SRNN_STAMP(7, clock64());
            if (kHoistPoll && k == p.n_tiles - 1) ++g_run;
            buf ^= 1;
            if (p.progress != nullptr && tid == 0 && k == p.n_tiles - 1 &&
                (s % p.progress_every == 0 || s == p.T)) {
                __threadfence();  // this CTA's y of steps <= s (ordered by the barrier above) before the count
                atomicAdd(p.progress, 1u);
            }
        }
    }
done:
    // column split: the pair leaves together (the peer may still read this CTA's zs / flag)
    if (CS) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // An aborted launch (watchdog / lost message) still releases the host pipeline's
    // y-copy waits on the progress counter (the host re-reads the counter on error).
    if (*s_abort && tid == 0) {
        atomicExch(p.xdirty, 1);  // the exchange buffers are inconsistent: the next launch re-initialises them
        if (p.progress != nullptr) atomicAdd(p.progress, 1u << 20);
    }
    return;
}

template <int NP, int BT, int G, bool F16, int MT = 0>
static int launch_one(const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
                      int* regs_out, int* max_blocks_out) {
    auto fn = srnn_persistent_kernel<NP, BT, G, F16, MT>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (regs_out != nullptr || max_blocks_out != nullptr) {
        cudaFuncAttributes attr;
        e = cudaFuncGetAttributes(&attr, fn);
        if (e != cudaSuccess) return static_cast<int>(e);
        if (regs_out) {  // int[2]: registers per thread, local-memory (spill/stack) bytes per thread
            regs_out[0] = attr.numRegs;
            regs_out[1] = static_cast<int>(attr.localSizeBytes);
        }
        if (max_blocks_out) {
            int nb = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, p.threads, smem);
            if (e != cudaSuccess) return static_cast<int>(e);
            *max_blocks_out = p.threads > (MT > 0 ? kDenseThreads : MaxThreadsBT<NP, F16, BT>::value) ? 0 : nb;
        }
    }
    if (p.csplit) {  // column split: 2-CTA clusters, all co-resident (cooperative)
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(num_ctas);
        lc.blockDim = dim3(p.threads);
        lc.dynamicSmemBytes = smem;
        lc.stream = static_cast<cudaStream_t>(stream);
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 2;
        if (max_blocks_out != nullptr && *max_blocks_out > 0) {
            int ncl = 0;
            lc.attrs = at;
            lc.numAttrs = 1;
            e = cudaOccupancyMaxActiveClusters(&ncl, fn, &lc);
            if (e != cudaSuccess) return static_cast<int>(e);
            if (2 * ncl < num_ctas) *max_blocks_out = 0;  // the pairs do not all fit at once
            lc.numAttrs = 2;
        }
        if (query_only) return 0;
        e = cudaLaunchKernelEx(&lc, fn, p);
        return static_cast<int>(e);
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
    if (p.csplit) {  // column split (MT = -2): tiles of <= 8 samples
#define SRNN_CS(BT_)                                                                                          \
    if (bt == BT_) {                                                                                          \
        if (g == 1) return launch_one<NP, BT_, 1, F16, -2>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 3) return launch_one<NP, BT_, 3, F16, -2>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 4) return launch_one<NP, BT_, 4, F16, -2>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
    }
        SRNN_CS(1)
        SRNN_CS(2)
        SRNN_CS(4)
        if constexpr (F16) { SRNN_CS(8) }
#undef SRNN_CS
        return static_cast<int>(cudaErrorInvalidValue);
    }
    if constexpr (staged_compiled(NP, F16, 4)) {  // staged plans (partial progress): MT = -3
        if (p.warp_early != nullptr) {
#define SRNN_ST(BT_)                                                                                          \
    if (bt == BT_) {                                                                                          \
        if (g == 1) return launch_one<NP, BT_, 1, F16, -3>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 3) return launch_one<NP, BT_, 3, F16, -3>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 4) return launch_one<NP, BT_, 4, F16, -3>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
    }
            SRNN_ST(4)
            SRNN_ST(8)
#undef SRNN_ST
            return static_cast<int>(cudaErrorInvalidValue);
        }
    }
    if constexpr (F16) {  // plans whose threads own more chunks than the default slots: 8 poll slots
        if (p.k8) {
#define SRNN_K8(BT_)                                                                                          \
    if (bt == BT_) {                                                                                          \
        if (g == 1) return launch_one<NP, BT_, 1, F16, -1>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 3) return launch_one<NP, BT_, 3, F16, -1>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
        if (g == 4) return launch_one<NP, BT_, 4, F16, -1>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out); \
    }
            if constexpr (NP <= 24) { SRNN_K8(4) }
            SRNN_K8(8)
            if constexpr (NP <= kMaxNP16) { SRNN_K8(16) }
#undef SRNN_K8
        }
    }
    SRNN_CASE(1, 1)
    SRNN_CASE(2, 1)
    SRNN_CASE(4, 1)
    SRNN_CASE(1, 4)
    SRNN_CASE(2, 4)
    SRNN_CASE(4, 4)
    SRNN_CASE(1, 3)
    SRNN_CASE(2, 3)
    SRNN_CASE(4, 3)
    if constexpr (F16) {
        SRNN_CASE(8, 1)
        SRNN_CASE(8, 4)
        SRNN_CASE(8, 3)
        if constexpr (NP <= kMaxNP16) {
            SRNN_CASE(16, 1)
            SRNN_CASE(16, 4)
            SRNN_CASE(16, 3)
        }
    }
#undef SRNN_CASE
    return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace srnn
