// srnn_gemm_f32.cu -- step a1 in fp32 mode: the non-recurrent input
// projection for all timesteps at once (Eq. 2: "W x_t ... has no
// dependency, so it can be processed in parallel and added to b, becoming
// b'"):
//
//     C[m][n] = bias[n] + sum_k A[m][k] * W[n][k]      (A = x [T*B][I], W [G*H][I])
//
// Exact fp32 FFMA on CUDA cores (the fp32 parity bound 1e-5 excludes TF32).
// 128x128 (or 128x64) output tile per CTA, 256 threads, 8x8 (8x4) outputs per
// thread, K staged through shared memory in slabs of 16 with a register double
// buffer (float4 global loads when rows are 16-byte aligned).
#include <cuda_runtime.h>

#include <cstdlib>

#include "srnn_internal.h"

namespace srnn {

namespace {
constexpr int BM = 128, BK = 16, TM = 8, NT = 256;

// TBN = 128: 8x8 outputs per thread; TBN = 64: 8x4 (twice the CTAs, so a
// one-wave grid of 128-wide tiles fills two CTAs per SM instead of one).
template <int TBN>
__global__ void __launch_bounds__(NT, 2) gemm_f32_nt_kernel(const GemmParams p) {
    constexpr int TN = TBN / 16;               // outputs per thread along N (float4 groups of 4)
    constexpr int WPT = TBN * BK / NT;         // W slab elements per thread (8 or 4)
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Ws[2][BK][TBN + 4];
    const int tid = threadIdx.x;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int n0 = blockIdx.x * TBN;
    const int tx = tid % 16, ty = tid / 16;  // 16 x 16 thread grid

    // A slab: row lr = tid/2, k = (tid%2)*8 .. +8; W slab: row tid/(BK/WPT), WPT consecutive k.
    const int lr = tid >> 1, lk = (tid & 1) * 8;
    const int wr = tid / (BK / WPT), wk = (tid % (BK / WPT)) * WPT;
    const bool vec = (p.K & 3) == 0;  // 16-byte aligned rows: float4 loads
    float ra[8], rw[WPT];
    auto load_slab = [&](int k0) {
        const int64_t am = m0 + lr;
        const int wn = n0 + wr;
        if (vec && k0 + BK <= p.K) {
#pragma unroll
            for (int i = 0; i < 8; i += 4) {
                const float4 v = am < p.M ? *reinterpret_cast<const float4*>(p.A + am * p.K + k0 + lk + i)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                ra[i] = v.x; ra[i + 1] = v.y; ra[i + 2] = v.z; ra[i + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < WPT; i += 4) {
                const float4 v = wn < p.N ? *reinterpret_cast<const float4*>(p.W + static_cast<int64_t>(wn) * p.K + k0 + wk + i)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                rw[i] = v.x; rw[i + 1] = v.y; rw[i + 2] = v.z; rw[i + 3] = v.w;
            }
            return;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + lk + i;
            ra[i] = (am < p.M && k < p.K) ? p.A[am * p.K + k] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < WPT; ++i) {
            const int k = k0 + wk + i;
            rw[i] = (wn < p.N && k < p.K) ? p.W[static_cast<int64_t>(wn) * p.K + k] : 0.0f;
        }
    };
    auto store_slab = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) As[buf][lk + i][lr] = ra[i];
#pragma unroll
        for (int i = 0; i < WPT; ++i) Ws[buf][wk + i][wr] = rw[i];
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
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
#pragma unroll
            for (int g = 0; g < TN / 4; ++g) {
                const float4 wv = *reinterpret_cast<const float4*>(&Ws[buf][k][g * 64 + tx * 4]);
                w[4 * g] = wv.x; w[4 * g + 1] = wv.y; w[4 * g + 2] = wv.z; w[4 * g + 3] = wv.w;
            }
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
    // cols g*64 + tx*4+{0..3}.
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (m >= p.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + (j / 4) * 64 + tx * 4 + (j % 4);
            if (n < p.N) p.C[m * p.N + n] = acc[i][j] + (p.bias ? p.bias[n] : 0.0f);
        }
    }
}
}  // namespace

int preload_gemm_f32() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, gemm_f32_nt_kernel<128>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, gemm_f32_nt_kernel<64>);
    return static_cast<int>(e);
}

// 128-wide tiles unless the grid is small (measured on B200: C2 0.255 vs 0.278 ms,
// the C4 LSTM projection 0.121 vs 0.131 ms; C1's 2-tile grid 0.033 vs 0.021 ms).
int launch_gemm_f32(const GemmParams& p, void* stream) {
    if (p.M <= 0 || p.N <= 0) return 0;
    const int64_t mt = (p.M + BM - 1) / BM;
    const bool wide = mt * ((p.N + 127) / 128) >= 64 || std::getenv("SRNN_GEMM_F32_WIDE") != nullptr;
    if (wide) {
        dim3 grid((p.N + 127) / 128, static_cast<unsigned>(mt));
        gemm_f32_nt_kernel<128><<<grid, NT, 0, static_cast<cudaStream_t>(stream)>>>(p);
    } else {
        dim3 grid((p.N + 63) / 64, static_cast<unsigned>(mt));
        gemm_f32_nt_kernel<64><<<grid, NT, 0, static_cast<cudaStream_t>(stream)>>>(p);
    }
    return static_cast<int>(cudaGetLastError());
}

}  // namespace srnn
