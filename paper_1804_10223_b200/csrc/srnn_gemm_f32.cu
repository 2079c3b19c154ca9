// srnn_gemm_f32.cu -- step a1 in fp32 mode: the non-recurrent input
// projection for all timesteps at once (Eq. 2: "W x_t ... has no
// dependency, so it can be processed in parallel and added to b, becoming
// b'"):
//
//     C[m][n] = bias[n] + sum_k A[m][k] * W[n][k]      (A = x [T*B][I], W [G*H][I])
//
// Exact fp32 FFMA on CUDA cores (the fp32 parity bound 1e-5 excludes TF32).
// 128x128 output tile per CTA, 256 threads, 8x8 outputs per thread, K staged
// through shared memory in slabs of 16 with a register double buffer.
#include <cuda_runtime.h>

#include "srnn_internal.h"

namespace srnn {

namespace {
constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8, NT = 256;

__global__ void __launch_bounds__(NT, 2) gemm_f32_nt_kernel(const GemmParams p) {
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Ws[2][BK][BN + 4];
    const int tid = threadIdx.x;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int n0 = blockIdx.x * BN;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);  // 16 x 16 thread grid

    // Each thread loads 8 elements of A and 8 of W per K slab: rows r = tid/2
    // (0..127), k = (tid%2)*8 .. +8.
    const int lr = tid >> 1, lk = (tid & 1) * 8;
    float ra[8], rw[8];
    auto load_slab = [&](int k0) {
        const int64_t am = m0 + lr;
        const int wn = n0 + lr;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + lk + i;
            ra[i] = (am < p.M && k < p.K) ? p.A[am * p.K + k] : 0.0f;
            rw[i] = (wn < p.N && k < p.K) ? p.W[static_cast<int64_t>(wn) * p.K + k] : 0.0f;
        }
    };
    auto store_slab = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            As[buf][lk + i][lr] = ra[i];
            Ws[buf][lk + i][lr] = rw[i];
        }
    };

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

    load_slab(0);
    store_slab(0);
    __syncthreads();
    const int nk = (p.K + BK - 1) / BK;
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load_slab((kt + 1) * BK);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float a[TM], w[TN];
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
            const float4 w0 = *reinterpret_cast<const float4*>(&Ws[buf][k][tx * 4]);
            const float4 w1 = *reinterpret_cast<const float4*>(&Ws[buf][k][64 + tx * 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
            w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
        }
        if (kt + 1 < nk) {
            store_slab(buf ^ 1);
            __syncthreads();
        }
    }
    // Epilogue: + bias, store.  Thread rows: ty*4+{0..3} and 64+ty*4+{0..3};
    // cols tx*4+{0..3} and 64+tx*4+{0..3}.
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (m >= p.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (n < p.N) p.C[m * p.N + n] = acc[i][j] + (p.bias ? p.bias[n] : 0.0f);
        }
    }
}
}  // namespace

int preload_gemm_f32() {
    cudaFuncAttributes a;
    return static_cast<int>(cudaFuncGetAttributes(&a, gemm_f32_nt_kernel));
}

int launch_gemm_f32(const GemmParams& p, void* stream) {
    if (p.M <= 0 || p.N <= 0) return 0;
    dim3 grid((p.N + BN - 1) / BN, static_cast<unsigned>((p.M + BM - 1) / BM));
    gemm_f32_nt_kernel<<<grid, NT, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace srnn
