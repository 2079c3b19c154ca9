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

// Spin-wait bookkeeping shared by all loaders of a CTA.
struct Watchdog {
    unsigned long long t0;
    uint32_t spins;
};

// Returns true when the wait must be abandoned (timeout here or elsewhere).
__device__ __forceinline__ bool watchdog_tick(Watchdog& wd, int32_t* status, unsigned long long timeout_ns) {
    if ((++wd.spins & 255u) != 0u) return false;
    unsigned long long now = globaltimer_ns();
    if (wd.t0 == 0) wd.t0 = now;
    if (*reinterpret_cast<volatile int32_t*>(status) != 0) return true;
    if (now - wd.t0 > timeout_ns) {
        atomicCAS(status, 0, -6 /* SRNN_ERR_TIMEOUT */);
        return true;
    }
    return false;
}

// Stage h_{s-1} (tile k) into shared memory: spin on tags (tag mode) or
// check them once (grid-sync mode).  Returns false on abort.
__device__ __forceinline__ bool load_tile(const unsigned long long* __restrict__ src, float* hs,
                                          int n_words, uint32_t want, bool spin,
                                          int32_t* status, unsigned long long timeout_ns) {
    constexpr int K = 4;
    const int n2 = n_words >> 1;
    const ulonglong2* src2 = reinterpret_cast<const ulonglong2*>(src);
    Watchdog wd{0ull, 0u};
    bool ok = true;
    const int nt = blockDim.x;
    for (int base = threadIdx.x; base < n2; base += K * nt) {
        ulonglong2 v[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int idx = base + j * nt;
            if (idx < n2) v[j] = ld_relaxed_v2(src2 + idx);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int idx = base + j * nt;
            ulonglong2 x = v[j];
            if (idx < n2) {
                bool ready = tag_of(x.x) == want && tag_of(x.y) == want;
                if (!ready && !spin) {
                    atomicCAS(status, 0, -4 /* protocol violation -> SRNN_ERR_STATE */);
                    ready = true;
                }
                while (!ready && ok) {
                    ok = !watchdog_tick(wd, status, timeout_ns);
                    x = ld_relaxed_v2(src2 + idx);
                    ready = tag_of(x.x) == want && tag_of(x.y) == want;
                }
                *reinterpret_cast<float2*>(hs + 2 * idx) = make_float2(val_of(x.x), val_of(x.y));
            }
        }
    }
    if ((n_words & 1) && threadIdx.x == 0) {
        unsigned long long x = ld_relaxed_u64(src + n_words - 1);
        bool ready = tag_of(x) == want;
        if (!ready && !spin) {
            atomicCAS(status, 0, -4);
            ready = true;
        }
        while (!ready && ok) {
            ok = !watchdog_tick(wd, status, timeout_ns);
            x = ld_relaxed_u64(src + n_words - 1);
            ready = tag_of(x) == want;
        }
        hs[n_words - 1] = val_of(x);
    }
    return ok;
}

template <int BT>
struct HVec;
template <>
struct HVec<1> {
    __device__ __forceinline__ static void fma(float (&acc)[1], float w, const unsigned char* base, uint32_t off) {
        const float h = *reinterpret_cast<const float*>(base + off);
        acc[0] = fmaf(w, h, acc[0]);
    }
};
template <>
struct HVec<2> {
    __device__ __forceinline__ static void fma(float (&acc)[2], float w, const unsigned char* base, uint32_t off) {
        const float2 h = *reinterpret_cast<const float2*>(base + off);
        acc[0] = fmaf(w, h.x, acc[0]);
        acc[1] = fmaf(w, h.y, acc[1]);
    }
};
template <>
struct HVec<4> {
    __device__ __forceinline__ static void fma(float (&acc)[4], float w, const unsigned char* base, uint32_t off) {
        const float4 h = *reinterpret_cast<const float4*>(base + off);
        acc[0] = fmaf(w, h.x, acc[0]);
        acc[1] = fmaf(w, h.y, acc[1]);
        acc[2] = fmaf(w, h.z, acc[2]);
        acc[3] = fmaf(w, h.w, acc[3]);
    }
};

// Max threads per CTA of each register-slot instance (caps ptxas' register
// budget at 65536 / MAXT while leaving room for the 2*NP hoisted registers).
template <int NP>
struct MaxThreads {
    static constexpr int value = NP <= 8 ? 1024 : NP <= 16 ? 768 : NP <= 32 ? 512 : NP <= 48 ? 352 : 320;
};

template <int NP, int BT, int G>
__global__ void __launch_bounds__(MaxThreads<NP>::value, 1) srnn_persistent_kernel(const RecParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = p.H;
    float* hs = reinterpret_cast<float*>(smem);        // [H][BT]   h_{s-1} tile (offset 0)
    float* zs = hs + H * BT;                           // [G*Umax][BT] reduced rows
    float* cs = zs + G * p.units_max * BT;             // LSTM cell state [n_tiles][Umax][BT]
    int* s_abort = reinterpret_cast<int*>(cs + (G == 4 ? p.n_tiles * p.units_max * BT : 0));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cta = blockIdx.x;
    const int u0 = p.cta_unit0[cta];
    const int U = p.cta_unit0[cta + 1] - u0;
    const int L = p.lanes_per_row;
    const int n_w = p.warp_slots[cta * (p.threads >> 5) + warp];
    const int tile_stride = (H * BT + 1) & ~1;

    // ---- prologue: weights HBM -> registers (once per forward) ----
    uint32_t off[NP];
    float w[NP];
    const size_t img0 = static_cast<size_t>(cta) * NP * p.threads + tid;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        off[i] = 0u;
        w[i] = 0.0f;
        if (i < n_w) {
            const size_t at = img0 + static_cast<size_t>(i) * p.threads;
            if (p.img_f32 != nullptr) {
                const uint2 e = p.img_f32[at];
                off[i] = e.x * (BT * 4);
                w[i] = __uint_as_float(e.y);
            } else {
                const uint32_t e = p.img_f16[at];
                off[i] = (e >> 16) * (BT * 4);
                w[i] = __half2float(__ushort_as_half(static_cast<unsigned short>(e & 0xffffu)));
            }
        }
    }

    // Epilogue role: thread e < U*BT owns (unit eu, sample eb) of every tile.
    const bool epi = tid < U * BT;
    const int eb = epi ? tid / U : 0;
    const int eu = epi ? tid - eb * U : 0;
    const int unit = u0 + eu;
    const int krow = warp * (32 / L) + lane / L;  // local row of this lane
    const bool row_leader = (lane % L) == 0 && krow < G * U;

    if (tid == 0) {
        *s_abort = 0;
        if (U * BT > p.threads) atomicCAS(p.status, 0, -7 /* SRNN_ERR_UNSUPPORTED: planner bug */);
    }
    // ---- publish h_0 (tag = epoch) and initialise c ----
    if (epi) {
        for (int k = 0; k < p.n_tiles; ++k) {
            const int bg = k * BT + eb;
            const float h = (p.h0 != nullptr && bg < p.B) ? p.h0[static_cast<size_t>(bg) * H + unit] : 0.0f;
            st_relaxed_u64(p.xbuf + static_cast<size_t>(k) * tile_stride + unit * BT + eb, pack_tagged(h, p.epoch));
            if (G == 4) {
                cs[(k * p.units_max + eu) * BT + eb] =
                    (p.c0 != nullptr && bg < p.B) ? p.c0[static_cast<size_t>(bg) * H + unit] : 0.0f;
            }
        }
    }
    const bool grid_sync = (p.flags & kFlagGridSync) != 0u;
    if (grid_sync) cg::this_grid().sync();
    __syncthreads();

    const int GH = G * H;
    for (int s = 1; s <= p.T; ++s) {
        for (int k = 0; k < p.n_tiles; ++k) {
            const int bg = k * BT + eb;
            // b'_s prefetch for the epilogue (in flight while we spin).
            float bp[G];
            if (epi) {
#pragma unroll
                for (int q = 0; q < G; ++q)
                    bp[q] = bg < p.B ? __ldg(p.bprime + (static_cast<size_t>(s - 1) * p.B + bg) * GH + q * H + unit) : 0.0f;
            }
            // ---- load: h_{s-1} tile k -> hs ----
            const unsigned long long* src =
                p.xbuf + static_cast<size_t>(((s - 1) & 1) * p.n_tiles + k) * tile_stride;
            if (!load_tile(src, hs, H * BT, p.epoch + static_cast<uint32_t>(s - 1), !grid_sync, p.status, p.timeout_ns))
                *s_abort = 1;
            __syncthreads();
            if (*s_abort) goto done;

            // ---- operate ----
            {
                float acc[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) acc[b] = 0.0f;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    if (i < n_w) HVec<BT>::fma(acc, w[i], smem, off[i]);
                }
                // ---- reduce over the row's L lanes (fixed butterfly order) ----
                for (int m = L >> 1; m >= 1; m >>= 1) {
#pragma unroll
                    for (int b = 0; b < BT; ++b) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], m);
                }
                if (row_leader) {
#pragma unroll
                    for (int b = 0; b < BT; ++b) zs[krow * BT + b] = acc[b];
                }
            }
            __syncthreads();

            // ---- epilogue: activation / gates, y, tagged publish of h_s ----
            if (epi) {
                float h;
                if (G == 1) {
                    h = activation(p.act, zs[eu * BT + eb] + bp[0]);
                } else {
                    const float zi = zs[(0 * U + eu) * BT + eb] + bp[0];
                    const float zf = zs[(1 * U + eu) * BT + eb] + bp[1 % G];
                    const float zg = zs[(2 * U + eu) * BT + eb] + bp[2 % G];
                    const float zo = zs[(3 * U + eu) * BT + eb] + bp[3 % G];
                    float* cp = &cs[(k * p.units_max + eu) * BT + eb];
                    const float c = sigmoidf_acc(zf) * (*cp) + sigmoidf_acc(zi) * tanhf(zg);
                    *cp = c;
                    h = sigmoidf_acc(zo) * tanhf(c);
                    if (s == p.T && p.cT != nullptr && bg < p.B) p.cT[static_cast<size_t>(bg) * H + unit] = c;
                }
                if (bg < p.B) {
                    if (p.y != nullptr) p.y[(static_cast<size_t>(s - 1) * p.B + bg) * H + unit] = h;
                    if (s == p.T && p.hT != nullptr) p.hT[static_cast<size_t>(bg) * H + unit] = h;
                }
                if (p.flags & kFlagJitter) {
                    const uint32_t r = (static_cast<uint32_t>(cta) * 2654435761u) ^ (static_cast<uint32_t>(s * 40503 + k));
                    __nanosleep((r >> 7) & 2047u);
                }
                st_relaxed_u64(p.xbuf + static_cast<size_t>((s & 1) * p.n_tiles + k) * tile_stride + unit * BT + eb,
                               pack_tagged(h, p.epoch + static_cast<uint32_t>(s)));
            }
            if (grid_sync) cg::this_grid().sync();
        }
    }
done:
    return;
}

template <int NP, int BT, int G>
static int launch_one(const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
                      int* regs_out, int* max_blocks_out) {
    auto fn = srnn_persistent_kernel<NP, BT, G>;
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
            *max_blocks_out = p.threads > MaxThreads<NP>::value ? 0 : nb;
        }
    }
    if (query_only) return 0;
    void* args[] = {const_cast<RecParams*>(&p)};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(num_ctas), dim3(p.threads), args, smem,
                                    static_cast<cudaStream_t>(stream));
    return static_cast<int>(e);
}

template <int NP>
int launch_np(int bt, int g, const RecParams& p, int num_ctas, size_t smem, void* stream, bool query_only,
              int* regs_out, int* max_blocks_out) {
#define SRNN_CASE(BT_, G_)                                                                                    \
    if (bt == BT_ && g == G_)                                                                                 \
        return launch_one<NP, BT_, G_>(p, num_ctas, smem, stream, query_only, regs_out, max_blocks_out);
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
