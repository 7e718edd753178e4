// Diagnostic: one tcgen05.mma GEMM through the engine's operand-layout convention (umma.cuh),
// exposed as flw_selftest_umma so tests can pin descriptor/layout correctness against numpy.
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"
#include "umma.cuh"

namespace flw {

namespace {

__global__ void __launch_bounds__(128) k_umma_selftest(const float* A, int Ra, int Ca, const float* B, int Rb,
                                                       int Cb, int M, int N, int K, int a_mn, int b_mn,
                                                       int lane_off, float* D) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    uint8_t* As = smem;
    uint8_t* Bs = smem + ((Ra * Ca * 2 + 1023) / 1024) * 1024;
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    for (int i = t; i < Ra * Ca; i += 128)
        *reinterpret_cast<__nv_bfloat16*>(As + umma::tile_offset(i / Ca, i % Ca, Ca)) = __float2bfloat16(A[i]);
    for (int i = t; i < Rb * Cb; i += 128)
        *reinterpret_cast<__nv_bfloat16*>(Bs + umma::tile_offset(i / Cb, i % Cb, Cb)) = __float2bfloat16(B[i]);
    umma::fence_async_smem();
    if (w == 0) umma::tmem_alloc<256>(&tslot);
    if (t == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tslot;
    if (t == 0) {
        const uint32_t a0 = umma::smem_u32(As), b0 = umma::smem_u32(Bs);
        const uint32_t idesc = umma::idesc_bf16(M, N, a_mn != 0, b_mn != 0);
        for (int kb = 0; kb < K / 16; ++kb) {
            uint64_t ad = a_mn ? umma::desc_mnmajor(a0, Ca, kb) : umma::desc_kmajor(a0, Ca, kb);
            uint64_t bd = b_mn ? umma::desc_mnmajor(b0, Cb, kb) : umma::desc_kmajor(b0, Cb, kb);
            umma::mma_bf16(tmem + (static_cast<uint32_t>(lane_off) << 16), ad, bd, idesc, kb > 0);
        }
        umma::commit(&bar);
    }
    umma::mbar_wait(&bar, 0);
    umma::fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        umma::tmem_ld16(tmem + (static_cast<uint32_t>(32 * w) << 16) + c0, v);
        umma::tmem_ld_wait();
        int m = -1;
        if (M == 128) {
            m = 32 * w + lane;
        } else {
            int l = lane - lane_off;
            if (l >= 0 && l < 16) m = l + 16 * w;
        }
        if (m >= 0)
            for (int j = 0; j < 16 && c0 + j < N; ++j) D[m * N + c0 + j] = v[j];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_free<256>(tmem);
}

}  // namespace

int umma_selftest(int M, int N, int K, int a_mn, int b_mn, int lane_off, const float* A_h, const float* B_h,
                  float* D_h) {
    const int Ra = a_mn ? K : M, Ca = a_mn ? M : K;
    const int Rb = b_mn ? K : N, Cb = b_mn ? N : K;
    float *A, *B, *D;
    FLW_CUDA(cudaMalloc(&A, sizeof(float) * Ra * Ca));
    FLW_CUDA(cudaMalloc(&B, sizeof(float) * Rb * Cb));
    FLW_CUDA(cudaMalloc(&D, sizeof(float) * M * N));
    FLW_CUDA(cudaMemcpy(A, A_h, sizeof(float) * Ra * Ca, cudaMemcpyHostToDevice));
    FLW_CUDA(cudaMemcpy(B, B_h, sizeof(float) * Rb * Cb, cudaMemcpyHostToDevice));
    FLW_CUDA(cudaMemset(D, 0, sizeof(float) * M * N));
    size_t smem = ((Ra * Ca * 2 + 1023) / 1024) * 1024 + static_cast<size_t>(Rb) * Cb * 2 + 1024;
    FLW_CUDA(cudaFuncSetAttribute(k_umma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_umma_selftest<<<1, 128, smem>>>(A, Ra, Ca, B, Rb, Cb, M, N, K, a_mn, b_mn, lane_off, D);
    FLW_CUDA(cudaGetLastError());
    FLW_CUDA(cudaDeviceSynchronize());
    FLW_CUDA(cudaMemcpy(D_h, D, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    cudaFree(A);
    cudaFree(B);
    cudaFree(D);
    return 0;
}

}  // namespace flw
