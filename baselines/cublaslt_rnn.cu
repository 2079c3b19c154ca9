// cublaslt_rnn.cu -- the dense per-timestep cuBLAS baseline of SURVEY.md Sec. 8 d-v, as a
// library GEMM with a fused epilogue: ONE cublasLtMatmul per timestep,
//     h_{t+1} = relu(W_h h_t + b'_t)      (fp16 W_h / h / b', fp32 accumulate, RELU epilogue, beta = 1)
// over T steps, timed eager (T launches) and CUDA-graph captured (one replay).  Comparator
// only (bench.py loads it with ctypes); the product path never links cuBLAS.
// Layout: column-major H x B matrices = the [B][H] row-major buffers of the product.
#include <cublasLt.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace {
__global__ void fill_f16(__half* p, size_t n, unsigned seed, float scale) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned x = static_cast<unsigned>(i) * 2654435761u ^ seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = __float2half(scale * ((x & 0xffffu) / 32768.0f - 1.0f));
    }
}
}  // namespace

// Returns 0 on success; *eager_us / *graph_us = microseconds per timestep (median-free: mean of reps).
extern "C" int lt_rnn_bench(int H, int B, int T, int reps, double* eager_us, double* graph_us, int* launches_per_step) {
    cublasLtHandle_t lt;
    if (cublasLtCreate(&lt) != CUBLAS_STATUS_SUCCESS) return 1;
    __half *W, *bp, *h;
    const size_t nw = static_cast<size_t>(H) * H, nb = static_cast<size_t>(T) * B * H, nh = 2 * static_cast<size_t>(B) * H;
    if (cudaMalloc(&W, nw * 2) || cudaMalloc(&bp, nb * 2) || cudaMalloc(&h, nh * 2)) return 2;
    fill_f16<<<1024, 256>>>(W, nw, 1u, 0.8f * 1.7320508f / sqrtf(static_cast<float>(H)));
    fill_f16<<<1024, 256>>>(bp, nb, 2u, 0.5f);
    cudaMemset(h, 0, nh * 2);
    size_t ws_bytes = 32u << 20;
    void* ws;
    if (cudaMalloc(&ws, ws_bytes)) return 3;

    cublasLtMatmulDesc_t op;
    cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
    cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;  // W_h row-major = (col-major H x H)^T
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
    cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_RELU;
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
    cublasLtMatrixLayout_t la, lb, lc;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_16F, H, H, H);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_16F, H, B, H);
    cublasLtMatrixLayoutCreate(&lc, CUDA_R_16F, H, B, H);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes, sizeof(ws_bytes));
    cublasLtMatmulHeuristicResult_t heur;
    int found = 0;
    if (cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 1, &heur, &found) != CUBLAS_STATUS_SUCCESS || !found)
        return 4;
    const float alpha = 1.0f, beta = 1.0f;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    auto loop = [&]() -> int {
        for (int t = 0; t < T; ++t) {
            const __half* hin = h + static_cast<size_t>(t & 1) * B * H;
            __half* hout = h + static_cast<size_t>((t + 1) & 1) * B * H;
            const __half* c = bp + static_cast<size_t>(t) * B * H;
            if (cublasLtMatmul(lt, op, &alpha, W, la, hin, lb, &beta, c, lc, hout, lc, &heur.algo, ws, ws_bytes, st) !=
                CUBLAS_STATUS_SUCCESS)
                return 5;
        }
        return 0;
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (int r = loop()) return r;
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r)
        if (int rc = loop()) return rc;
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *eager_us = 1000.0 * ms / (static_cast<double>(reps) * T);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (int r = loop()) return r;
    if (cudaStreamEndCapture(st, &g) != cudaSuccess) return 6;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return 7;
    size_t nodes = 0;
    cudaGraphGetNodes(g, nullptr, &nodes);
    *launches_per_step = static_cast<int>(nodes / T);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    *graph_us = 1000.0 * ms / (static_cast<double>(reps) * T);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    cublasLtMatmulPreferenceDestroy(pref);
    cublasLtMatrixLayoutDestroy(la);
    cublasLtMatrixLayoutDestroy(lb);
    cublasLtMatrixLayoutDestroy(lc);
    cublasLtMatmulDescDestroy(op);
    cublasLtDestroy(lt);
    cudaFree(W);
    cudaFree(bp);
    cudaFree(h);
    cudaFree(ws);
    return cudaGetLastError() == cudaSuccess ? 0 : 8;
}
