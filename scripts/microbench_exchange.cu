// microbench_exchange.cu -- B200 floors for the per-step inter-CTA exchange
// (SURVEY.md Sec. 7 step 3): what one timestep costs with NO compute, for the
// synchronisation schemes the recurrent kernel can use.
//
//   pingpong      2 CTAs bounce a tagged word through L2: one-way latency
//   gridsync      cooperative-groups grid.sync() per step
//   a2a_flag      every CTA publishes one tagged word, polls all 148
//   a2a_bulk      every CTA publishes its slice of tagged words (fp16 pairs +
//                 tag, the kernel's format) and polls the whole h (batch poll)
//   a2a_sent      poll one sentinel word per producer, then one bulk read
//   a2a_relacq    raw data + st.release flag per producer; ld.acquire flag,
//                 then plain bulk read of the raw data (half the bytes)
//   a2a_cluster<CS>  thread-block clusters of CS CTAs: each CTA polls 1/CS of
//                 the chunks from L2 and forwards them into every cluster
//                 peer's shared memory (DSMEM, double-buffered), then one
//                 cluster barrier -- L2 polling traffic / CS
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_exchange.cu
// run:   ./mb [units_per_cta=16] [words_per_unit=2] [steps=2000]
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned r;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ uint4 ld_cg_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.relaxed.gpu.global.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}

struct Args {
    int steps, upc, wpu;  // units per CTA, tagged words per unit
    unsigned long long* words;  // [2][ncta*upc*wpu]
    unsigned* flags;            // [ncta]
    uint2* raw;                 // [2][ncta*upc] raw fp16x4 data
    long long* out;
    unsigned delay_ns;
    unsigned long long* pflags;  // [consumer][producer] step words
};

__global__ void k_pingpong(Args a) {
    if (threadIdx.x != 0 || blockIdx.x > 1) return;
    unsigned long long* w = a.words;
    long long t0 = clock64();
    for (int s = 1; s <= a.steps; ++s) {
        if (blockIdx.x == (s & 1)) {
            while (ld_relaxed(w) != static_cast<unsigned long long>(s - 1)) {
            }
            st_relaxed(w, s);
        }
    }
    if (blockIdx.x == 0) a.out[0] = clock64() - t0;
}

__global__ void k_gridsync(Args a) {
    cg::grid_group g = cg::this_grid();
    for (int s = 0; s < a.steps; ++s) g.sync();
}

__global__ void k_a2a_flag(Args a) {
    const int n = gridDim.x;
    for (int s = 1; s <= a.steps; ++s) {
        if (threadIdx.x == 0) st_relaxed(a.words + blockIdx.x, s);
        if (threadIdx.x < n)
            while (ld_relaxed(a.words + threadIdx.x) < static_cast<unsigned long long>(s)) {
            }
        __syncthreads();
    }
}

// tagged bulk: word = (tag << 32) | payload
__global__ void k_a2a_bulk(Args a) {
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* dst = a.words + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x)
            st_relaxed(dst + blockIdx.x * per + i, (static_cast<unsigned long long>(s) << 32) | i);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        // batch poll, <= 8 chunks per thread in flight
        for (int base = threadIdx.x; base < chunks; base += 8 * blockDim.x) {
            ulonglong2 v[8];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int idx = base + j * blockDim.x;
                if (idx < chunks) {
                    v[j] = ld_relaxed_v2(src + idx);
                    pend |= 1u << j;
                }
            }
            while (pend) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (v[j].x >> 32) == static_cast<unsigned long long>(s) &&
                        (v[j].y >> 32) == static_cast<unsigned long long>(s))
                        pend &= ~(1u << j);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            }
        }
        __syncthreads();
    }
}

// The product's exchange (srnn_recurrent.cuh, R16): every CTA publishes its
// units' values as 16-bit words carrying the 1-bit step tag in the LSB (one relaxed store
// per value), then a CTA barrier, then every thread polls K 16-byte chunks of the whole
// image at once, re-polling stale ones, and stages them into shared memory; a second
// barrier ends the step.  vals = units_per_cta * BT values per CTA.
template <int K>
__global__ void k_a2a_lsb(Args a) {
    extern __shared__ __align__(16) unsigned char hs[];
    const int n = gridDim.x;
    const int vals = a.upc * a.wpu;  // wpu reused as values per unit (BT)
    const int total = n * vals;      // 16-bit values per image
    const int chunks = (total * 2 + 15) / 16;
    unsigned short* img = reinterpret_cast<unsigned short*>(a.words);
    for (int s = 1; s <= a.steps; ++s) {
        unsigned short* dst = img + static_cast<size_t>(s & 1) * (chunks * 8);
        const unsigned tag = (s >> 1) & 1u;
        for (int i = threadIdx.x; i < vals; i += blockDim.x) {
            const unsigned short v = static_cast<unsigned short>((0x3c00u + i) & ~1u) | tag;
            asm volatile("st.relaxed.gpu.global.b16 [%0], %1;" ::"l"(dst + blockIdx.x * vals + i), "h"(v) : "memory");
        }
        if (blockIdx.x == n - 1)  // pad values of the last chunk
            for (int i = total + threadIdx.x; i < chunks * 8; i += blockDim.x)
                asm volatile("st.relaxed.gpu.global.b16 [%0], %1;" ::"l"(dst + i), "h"(static_cast<unsigned short>(tag)) : "memory");
        __syncthreads();
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        const unsigned long long M = 0x0001000100010001ull, want = tag ? M : 0ull;
        for (int base = threadIdx.x; base < chunks; base += K * blockDim.x) {
            ulonglong2 v[K];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (base + j * static_cast<int>(blockDim.x) < chunks) {
                    v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
                    pend |= 1u << j;
                }
            while (pend) {
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if ((pend >> j & 1) && ((((v[j].x & M) ^ want) | ((v[j].y & M) ^ want)) == 0ull)) {
                        *reinterpret_cast<ulonglong2*>(hs + 16 * (base + j * blockDim.x)) = v[j];
                        pend &= ~(1u << j);
                    }
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (pend >> j & 1) v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            }
        }
        __syncthreads();
    }
}

// replicated bulk: producers write their slice into R copies, consumer c polls copy c % R
// (tests whether 148 SMs polling the same L2 lines -- hot-line serialisation -- is the cost).
// DELAY: __nanosleep before the first poll round (is the first, early round wasted?)
template <int R>
__global__ void k_a2a_rep(Args a) {
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* buf = a.words + static_cast<size_t>(s & 1) * total * R;
        for (int i = threadIdx.x; i < per; i += blockDim.x) {
            const unsigned long long w = (static_cast<unsigned long long>(s) << 32) | i;
#pragma unroll
            for (int r = 0; r < R; ++r) st_relaxed(buf + static_cast<size_t>(r) * total + blockIdx.x * per + i, w);
        }
        if (a.delay_ns) __nanosleep(a.delay_ns);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(buf + static_cast<size_t>(blockIdx.x % R) * total);
        for (int base = threadIdx.x; base < chunks; base += 8 * blockDim.x) {
            ulonglong2 v[8];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int idx = base + j * blockDim.x;
                if (idx < chunks) {
                    v[j] = ld_relaxed_v2(src + idx);
                    pend |= 1u << j;
                }
            }
            while (pend) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (v[j].x >> 32) == static_cast<unsigned long long>(s) &&
                        (v[j].y >> 32) == static_cast<unsigned long long>(s))
                        pend &= ~(1u << j);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            }
        }
        __syncthreads();
    }
}

// overlapped polling: two register sets of the same chunks, the second round issued GAP ns
// after the first, then each stale set is re-issued as soon as it has been checked, so two
// rounds are always in flight and the L2 is sampled every ~RTT/2 instead of every RTT.
__global__ void k_a2a_ov(Args a) {
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* dst = a.words + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x)
            st_relaxed(dst + blockIdx.x * per + i, (static_cast<unsigned long long>(s) << 32) | i);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        const unsigned long long want = static_cast<unsigned long long>(s);
        for (int base = threadIdx.x; base < chunks; base += 8 * blockDim.x) {
            ulonglong2 va[8], vb[8];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (base + j * blockDim.x < chunks) {
                    va[j] = ld_relaxed_v2(src + base + j * blockDim.x);
                    pend |= 1u << j;
                }
            if (a.delay_ns) __nanosleep(a.delay_ns);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (pend >> j & 1) vb[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            while (true) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (va[j].x >> 32) == want && (va[j].y >> 32) == want) pend &= ~(1u << j);
                if (!pend) break;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) va[j] = ld_relaxed_v2(src + base + j * blockDim.x);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (vb[j].x >> 32) == want && (vb[j].y >> 32) == want) pend &= ~(1u << j);
                if (!pend) break;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) vb[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            }
        }
        __syncthreads();
    }
}

// per-consumer flag arrays: producer p writes word [c][p] = step for EVERY consumer c (148
// relaxed stores into 148 different lines), consumer c polls only its own 148-word array
// (no line is polled by more than one SM), then reads the tagged data once (stale chunks
// re-polled: the flags are only a hint, the tags stay the correctness check -- no fences).
__global__ void k_a2a_pflag(Args a) {
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* dst = a.words + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x)
            st_relaxed(dst + blockIdx.x * per + i, (static_cast<unsigned long long>(s) << 32) | i);
        if (a.delay_ns == 0) __syncthreads();  // data stores issued before the flags (not ordered: a hint)
        for (int c = threadIdx.x; c < n; c += blockDim.x)
            st_relaxed(a.pflags + static_cast<size_t>(c) * n + blockIdx.x, static_cast<unsigned long long>(s));
        for (int p = threadIdx.x; p < n; p += blockDim.x)
            while (ld_relaxed(a.pflags + static_cast<size_t>(blockIdx.x) * n + p) < static_cast<unsigned long long>(s)) {
            }
        __syncthreads();
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        const unsigned long long want = static_cast<unsigned long long>(s);
        for (int base = threadIdx.x; base < chunks; base += 8 * blockDim.x) {
            ulonglong2 v[8];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (base + j * blockDim.x < chunks) {
                    v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
                    pend |= 1u << j;
                }
            while (pend) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (v[j].x >> 32) == want && (v[j].y >> 32) == want) pend &= ~(1u << j);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) v[j] = ld_relaxed_v2(src + base + j * blockDim.x);
            }
        }
        __syncthreads();
    }
}

// sentinel: poll the last word of each producer's slice, then one bulk read
__global__ void k_a2a_sent(Args a) {
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    __shared__ unsigned long long sink;
    unsigned long long acc = 0;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* dst = a.words + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x)
            st_relaxed(dst + blockIdx.x * per + i, (static_cast<unsigned long long>(s) << 32) | i);
        if (threadIdx.x < n)
            while ((ld_relaxed(dst + threadIdx.x * per + per - 1) >> 32) != static_cast<unsigned long long>(s)) {
            }
        __syncthreads();
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        for (int idx = threadIdx.x; idx < chunks; idx += blockDim.x) {
            ulonglong2 v = ld_relaxed_v2(src + idx);
            while ((v.x >> 32) != static_cast<unsigned long long>(s) || (v.y >> 32) != static_cast<unsigned long long>(s))
                v = ld_relaxed_v2(src + idx);
            acc += v.x;
        }
        __syncthreads();
    }
    if (acc == 12345) sink = acc;
}

// release/acquire: raw fp16x4 per unit (8 B), one flag per producer
__global__ void k_a2a_relacq(Args a) {
    const int n = gridDim.x;
    const int per = a.upc;  // units
    const int total = n * per;
    __shared__ unsigned long long sink;
    unsigned acc = 0;
    for (int s = 1; s <= a.steps; ++s) {
        uint2* dst = a.raw + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x) dst[blockIdx.x * per + i] = make_uint2(s, i);
        __syncthreads();
        if (threadIdx.x == 0) st_release(a.flags + blockIdx.x, s);
        if (threadIdx.x < n)
            while (ld_acquire(a.flags + threadIdx.x) < static_cast<unsigned>(s)) {
            }
        __syncthreads();
        const uint4* src = reinterpret_cast<const uint4*>(dst);
        for (int idx = threadIdx.x; idx < total / 2; idx += blockDim.x) {
            uint4 v = ld_cg_v4(src + idx);
            acc += v.x + v.z;
        }
        __syncthreads();
    }
    if (acc == 12345) sink = acc;
}

// cluster forwarding: CTA r of a CS-cluster polls chunks c with c % CS == r, writes each fresh
// chunk into hs[(s & 1)] of all CS CTAs (DSMEM), then barrier.cluster (release/acquire).
template <int CS>
__global__ void k_a2a_cluster(Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int n = gridDim.x;
    const int per = a.upc * a.wpu;
    const int total = n * per;
    const int chunks = total / 2;
    ulonglong2* hs0 = reinterpret_cast<ulonglong2*>(smem);
    ulonglong2* peer[CS];
    for (int r = 0; r < CS; ++r) peer[r] = cl.map_shared_rank(hs0, r);
    unsigned long long acc = 0;
    for (int s = 1; s <= a.steps; ++s) {
        unsigned long long* dst = a.words + static_cast<size_t>(s & 1) * total;
        for (int i = threadIdx.x; i < per; i += blockDim.x)
            st_relaxed(dst + blockIdx.x * per + i, (static_cast<unsigned long long>(s) << 32) | i);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(dst);
        const int boff = (s & 1) * chunks;
        const int mine = (chunks - rank + CS - 1) / CS;  // chunks rank, rank + CS, ...
        for (int base = threadIdx.x; base < mine; base += 8 * blockDim.x) {
            ulonglong2 v[8];
            unsigned pend = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int idx = base + j * blockDim.x;
                if (idx < mine) {
                    v[j] = ld_relaxed_v2(src + idx * CS + rank);
                    pend |= 1u << j;
                }
            }
            while (pend) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((pend >> j & 1) && (v[j].x >> 32) == static_cast<unsigned long long>(s) &&
                        (v[j].y >> 32) == static_cast<unsigned long long>(s)) {
                        const int c = (base + j * blockDim.x) * CS + rank;
#pragma unroll
                        for (int r = 0; r < CS; ++r) peer[r][boff + c] = v[j];
                        pend &= ~(1u << j);
                    }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (pend >> j & 1) v[j] = ld_relaxed_v2(src + (base + j * blockDim.x) * CS + rank);
            }
        }
        cl.sync();
        acc += hs0[boff + threadIdx.x].x;
    }
    if (acc == 12345) a.out[1] = acc;
}

static float run_cluster(void* fn, Args a, int grid, int block, int cs, size_t smem) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (cs > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
    if (ncl * cs < grid) {
        printf(", \"cluster%d_max_active_clusters\": %d", cs, ncl);
        return -1.0f;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    void* args[] = {&a};
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(a.words, 0, static_cast<size_t>(2) * 148 * 64 * 8 * 8);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelExC(&cfg, fn, args);
        cudaEventRecord(e1);
        if (err == cudaSuccess) err = cudaDeviceSynchronize();
        if (err != cudaSuccess) {
            printf(", \"cluster%d_error\": \"%s\"", cs, cudaGetErrorString(err));
            return -1.0f;
        }
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.0f / a.steps;
}

static float run(void* fn, Args a, int grid, int block) {
    void* args[] = {&a};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemset(a.words, 0, static_cast<size_t>(2) * 148 * 64 * 8 * 8);
    cudaMemset(a.flags, 0, 148 * 4 * 4);
    cudaMemset(a.pflags, 0, static_cast<size_t>(148) * 148 * 8);
    cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);  // warm
    cudaDeviceSynchronize();
    cudaMemset(a.words, 0, static_cast<size_t>(2) * 148 * 64 * 8 * 8);
    cudaMemset(a.flags, 0, 148 * 4 * 4);
    cudaMemset(a.pflags, 0, static_cast<size_t>(148) * 148 * 8);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(err));
        exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.0f / a.steps;
}

static float run_smem(void* fn, Args a, int grid, int block, size_t smem) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    void* args[] = {&a};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, nullptr);  // warm-up
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) return -1.f;
    return 1000.f * ms / a.steps;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "--floor") {
        // bench.py: the product-format exchange floor for H units x BT fp16 values on 148 CTAs
        Args a;
        const int H = argc > 2 ? atoi(argv[2]) : 2304, bt = argc > 3 ? atoi(argv[3]) : 4;
        const int ncta = argc > 4 ? atoi(argv[4]) : 148, threads = argc > 5 ? atoi(argv[5]) : 512;
        a.upc = (H + ncta - 1) / ncta;
        a.wpu = bt;
        a.steps = 4000;
        a.delay_ns = 0;
        const size_t img = static_cast<size_t>(ncta) * a.upc * bt * 2 + 16;
        cudaMalloc(&a.words, 2 * img + 64);
        cudaMemset(a.words, 0, 2 * img + 64);
        cudaMalloc(&a.out, 64);
        const float us = run_smem(reinterpret_cast<void*>(k_a2a_lsb<3>), a, ncta, threads, img + 64);
        printf("{\"a2a_lsb_us_per_step\": %.4f, \"units_per_cta\": %d, \"bt\": %d, \"ctas\": %d, \"threads\": %d, "
               "\"bytes_per_cta\": %zu}\n", us, a.upc, bt, ncta, threads, img - 16);
        return us > 0 ? 0 : 1;
    }
    Args a;
    a.upc = argc > 1 ? atoi(argv[1]) : 16;
    a.wpu = argc > 2 ? atoi(argv[2]) : 2;
    a.steps = argc > 3 ? atoi(argv[3]) : 2000;
    a.delay_ns = 0;
    cudaMalloc(&a.pflags, static_cast<size_t>(148) * 148 * 8);
    int ncta = 148;
    cudaMalloc(&a.words, static_cast<size_t>(2) * 148 * 64 * 8 * 8);
    cudaMalloc(&a.flags, 148 * 4 * 4);
    cudaMalloc(&a.raw, static_cast<size_t>(2) * 148 * 64 * 8);
    cudaMalloc(&a.out, 64);
    cudaMemset(a.words, 0, static_cast<size_t>(2) * 148 * 64 * 8 * 8);
    printf("{\"units_per_cta\": %d, \"words_per_unit\": %d, \"steps\": %d", a.upc, a.wpu, a.steps);
    float pp = run(reinterpret_cast<void*>(k_pingpong), a, 2, 32);
    long long cyc;
    cudaMemcpy(&cyc, a.out, 8, cudaMemcpyDeviceToHost);
    printf(", \"pingpong_us_per_hop\": %.4f, \"pingpong_cycles_per_hop\": %.1f", pp, static_cast<double>(cyc) / a.steps);
    for (int blk : {512}) {
        printf(", \"gridsync_us\": %.4f", run(reinterpret_cast<void*>(k_gridsync), a, ncta, blk));
        printf(", \"a2a_flag_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_flag), a, ncta, blk));
        printf(", \"a2a_bulk_tagged_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_bulk), a, ncta, blk));
        printf(", \"a2a_sentinel_then_bulk_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_sent), a, ncta, blk));
        printf(", \"a2a_release_acquire_raw_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_relacq), a, ncta, blk));
        printf(", \"a2a_rep1_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_rep<1>), a, ncta, blk));
        printf(", \"a2a_rep2_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_rep<2>), a, ncta, blk));
        printf(", \"a2a_rep4_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_rep<4>), a, ncta, blk));
        printf(", \"a2a_rep8_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_rep<8>), a, ncta, blk));
        for (unsigned d : {200u, 400u, 800u}) {
            Args b = a;
            b.delay_ns = d;
            printf(", \"a2a_rep1_delay%u_us\": %.4f", d, run(reinterpret_cast<void*>(k_a2a_rep<1>), b, ncta, blk));
        }
    }
    {
        const size_t smem = static_cast<size_t>(2) * ncta * a.upc * a.wpu * 8;
        for (int cs : {2, 4, 8}) {
            const int grid = (ncta / cs) * cs;
            void* fn = cs == 2 ? reinterpret_cast<void*>(k_a2a_cluster<2>)
                     : cs == 4 ? reinterpret_cast<void*>(k_a2a_cluster<4>) : reinterpret_cast<void*>(k_a2a_cluster<8>);
            Args b = a;
            b.upc = a.upc * ncta / grid + (a.upc * ncta % grid ? 1 : 0);  // same h size on fewer CTAs
            printf(", \"a2a_cluster%d_ctas\": %d, \"a2a_cluster%d_us\": %.4f", cs, grid, cs,
                   run_cluster(fn, b, grid, 512, cs, smem + 4096));
        }
    }
    printf(", \"a2a_pflag_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_pflag), a, ncta, 512));
    {
        Args b = a;
        b.delay_ns = 1;  // no barrier between the data and the flag stores
        printf(", \"a2a_pflag_nobar_us\": %.4f", run(reinterpret_cast<void*>(k_a2a_pflag), b, ncta, 512));
    }
    for (unsigned d : {0u, 100u, 200u, 300u, 500u}) {
        Args b = a;
        b.delay_ns = d;
        printf(", \"a2a_overlap_gap%u_us\": %.4f", d, run(reinterpret_cast<void*>(k_a2a_ov), b, ncta, 512));
    }
    // scaling of the replicated-bulk all-to-all (R = 1) with the CTA count (same h bytes) and block size
    for (int g : {16, 37, 74, 148}) {
        for (int blk : {256, 512, 1024}) {
            Args b = a;
            b.upc = a.upc * ncta / g;
            printf(", \"a2a_ctas%d_thr%d_us\": %.4f", g, blk, run(reinterpret_cast<void*>(k_a2a_rep<1>), b, g, blk));
        }
    }
    printf(", \"bytes_tagged_per_cta\": %d, \"bytes_raw_per_cta\": %d}\n", ncta * a.upc * a.wpu * 8, ncta * a.upc * 8);
    return 0;
}
