// microbench_fetch.cu -- how long does one SM take to pull an N-byte block of
// already-valid data from L2 into shared memory while all 148 SMs do the same
// (the per-step h fetch of the persistent kernel without any waiting)?
//
//   mode 0  ld.relaxed.gpu.v2.b64 (LDG.128.STRONG.GPU) K chunks in flight / thread, STS
//   mode 1  cp.async.cg 16 B per chunk (LDGSTS), wait_all
//   mode 2  cp.async.bulk (TMA 1-D) in pieces of `piece` bytes, one mbarrier
//   mode 3  ld.global.cg (weak, L2 only) v4, STS
//   mode 4/5/6  as mode 0, but every CTA first rewrites its own 1/ctas slice of the block
//           (st.relaxed.gpu b16 / b32 / v2.b64 per thread), then a CTA barrier, then the fetch:
//           the per-step exchange pattern without the wait for other CTAs
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbf scripts/microbench_fetch.cu
// run:   ./mbf bytes mode [piece=4096] [iters=200] [ctas=148] [threads=512]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
}

template <int K>
__global__ void __launch_bounds__(1024, 1) k_fetch(const unsigned char* __restrict__ src, int nbytes, int mode, int piece,
                                                   int iters, long long* out, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mbar;
    const int nch = nbytes / 16;
    const int tid = threadIdx.x, nt = blockDim.x;
    unsigned long long acc = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned phase = 0;
    long long tsum = 0;
    for (int it = 0; it < iters; ++it) {
        if (mode >= 4) {
            // rewrite this CTA's slice (same bytes, so later fetches stay identical)
            const int sl = nbytes / gridDim.x / 16 * 16, off = blockIdx.x * sl;
            const int w = mode == 4 ? 2 : mode == 5 ? 4 : 16;
            for (int o = tid * w; o < sl; o += nt * w) {
                unsigned char* d = const_cast<unsigned char*>(src) + off + o;
                if (w == 2) asm volatile("st.relaxed.gpu.global.b16 [%0], %1;" ::"l"(d), "h"((unsigned short)0x0101) : "memory");
                else if (w == 4) asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(d), "r"(0x01010101u) : "memory");
                else asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %1};" ::"l"(d), "l"(0x0101010101010101ull) : "memory");
            }
        }
        __syncthreads();
        long long t0 = clock64();
        if (mode == 0 || mode >= 4) {
            for (int base = tid; base < nch; base += K * nt) {
                ulonglong2 v[K];
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j * nt < nch) v[j] = ld_relaxed_v2(reinterpret_cast<const ulonglong2*>(src) + base + j * nt);
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j * nt < nch) *reinterpret_cast<ulonglong2*>(sm + 16 * (base + j * nt)) = v[j];
            }
        } else if (mode == 3) {
            for (int base = tid; base < nch; base += K * nt) {
                uint4 v[K];
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j * nt < nch) v[j] = ld_cg(reinterpret_cast<const uint4*>(src) + base + j * nt);
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j * nt < nch) *reinterpret_cast<uint4*>(sm + 16 * (base + j * nt)) = v[j];
            }
        } else if (mode == 1) {
            for (int c = tid; c < nch; c += nt) {
                unsigned d = (unsigned)__cvta_generic_to_shared(sm + 16 * c);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 16 * c) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
        } else {
            const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
            if (tid == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(nbytes) : "memory");
                for (int o = 0; o < nbytes; o += piece) {
                    const int n = min(piece, nbytes - o);
                    unsigned d = (unsigned)__cvta_generic_to_shared(sm + o);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(d), "l"(src + o), "r"(n), "r"(mb) : "memory");
                }
            }
            // wait for the phase
            asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(mb), "r"(phase) : "memory");
            phase ^= 1;
        }
        __syncthreads();
        long long t1 = clock64();
        tsum += t1 - t0;
        acc += sm[(tid * 16 + it) % nbytes];
    }
    if (tid == 0) out[blockIdx.x] = tsum / iters;
    if (acc == 0x123456789ull) *sink = acc;
}

int main(int argc, char** argv) {
    int nbytes = argc > 1 ? atoi(argv[1]) : 18432;
    int mode = argc > 2 ? atoi(argv[2]) : 0;
    int piece = argc > 3 ? atoi(argv[3]) : 4096;
    int iters = argc > 4 ? atoi(argv[4]) : 200;
    int ctas = argc > 5 ? atoi(argv[5]) : 148;
    int threads = argc > 6 ? atoi(argv[6]) : 512;
    int K = argc > 7 ? atoi(argv[7]) : 4;
    unsigned char* src;
    long long* out;
    unsigned long long* sink;
    cudaMalloc(&src, nbytes + 4096);
    cudaMemset(src, 1, nbytes + 4096);
    cudaMalloc(&out, ctas * 8);
    cudaMalloc(&sink, 8);
    auto fn = K == 2 ? k_fetch<2> : K == 4 ? k_fetch<4> : K == 8 ? k_fetch<8> : k_fetch<1>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, nbytes + 1024);
    fn<<<ctas, threads, nbytes + 1024>>>(src, nbytes, mode, piece, 10, out, sink);
    fn<<<ctas, threads, nbytes + 1024>>>(src, nbytes, mode, piece, iters, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<long long> h(ctas);
    cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("bytes=%d mode=%d piece=%d ctas=%d threads=%d K=%d cycles/fetch median=%lld p90=%lld max=%lld\n", nbytes, mode, piece,
           ctas, threads, K, h[ctas / 2], h[ctas * 9 / 10], h[ctas - 1]);
    return 0;
}
