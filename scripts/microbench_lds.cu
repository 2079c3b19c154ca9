// microbench_lds.cu -- shared-memory wavefronts per warp-wide LDS.64 / LDS.128 for the
// access patterns a broadcast-aware weight layout would produce (B200, sm_100a).
// pattern p: lane -> 8-byte (or 16-byte) word index
//   0 distinct consecutive   1 all lanes one word    2 word = lane & 15 (halves share)
//   3 word = lane >> 1 (pairs share)   4 word = lane >> 2   5 word = lane & 7
//   6 word = (lane >> 1) * 2 (pairs share, stride 2 words)   7 word = lane >> 3
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbl scripts/microbench_lds.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int W>
__global__ void k(int pat, int iters, unsigned long long* out, float* sink) {
    __shared__ __align__(16) unsigned char sm[32768];
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f + i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int word;
    switch (pat) {
        case 0: word = lane; break;
        case 1: word = 0; break;
        case 2: word = lane & 15; break;
        case 3: word = lane >> 1; break;
        case 4: word = lane >> 2; break;
        case 5: word = lane & 7; break;
        case 6: word = (lane >> 1) * 2; break;
        default: word = lane >> 3; break;
    }
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(sm)) + word * W + (warp & 7) * 512;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const unsigned a = base + ((it & 7) << 10);
        if (W == 8) {
            float x0, x1, y0, y1, z0, z1, w0, w1;
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x0), "=f"(x1) : "r"(a));
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2+4096];" : "=f"(y0), "=f"(y1) : "r"(a));
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2+8192];" : "=f"(z0), "=f"(z1) : "r"(a));
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2+12288];" : "=f"(w0), "=f"(w1) : "r"(a));
            acc += x0 + x1 + y0 + y1 + z0 + z1 + w0 + w1;
        } else {
            float4 x, y, z, w;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a));
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4+4096];" : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w) : "r"(a));
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4+8192];" : "=f"(z.x), "=f"(z.y), "=f"(z.z), "=f"(z.w) : "r"(a));
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4+12288];" : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w) : "r"(a));
            acc += x.x + y.y + z.z + w.w + x.w + y.x + z.y + w.z;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) *sink = acc;
}

int main() {
    unsigned long long* out;
    float* sink;
    cudaMalloc(&out, 8 * 148);
    cudaMalloc(&sink, 4);
    const int iters = 4096, threads = 512;
    for (int W : {8, 16}) {
        for (int pat = 0; pat < 8; ++pat) {
            auto fn = W == 8 ? k<8> : k<16>;
            fn<<<148, threads>>>(pat, iters, out, sink);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            const double instr = 4.0 * iters * (threads / 32);
            printf("LDS.%d pattern %d: %.3f cycles per warp-instruction (SM-wide)\n", W * 8, pat, h / instr);
        }
    }
    return 0;
}
