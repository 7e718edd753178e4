// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion cycles per instruction for the
// shapes the learn kernel uses (one CTA, one issuing thread, operands in shared memory).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2210_00882_b200/csrc tools/umma_rate.cu -o /tmp/umma_rate
#include <cstdio>
#include "umma.cuh"
using namespace flw;

__global__ void k(int M, int N, int a_mn, int b_mn, int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    umma::fence_async_smem();
    if (threadIdx.x < 32) umma::tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); umma::fence_barrier_init(); }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (threadIdx.x == 0) {
        const uint32_t base = umma::smem_u32(smem);
        const uint32_t id = umma::idesc_bf16(M, N, a_mn, b_mn);
        const int K = 128;  // operand tiles: A [M x K], B [N x K]
        uint32_t ph = 0;
        long long best = 1LL << 60;
        for (int trial = 0; trial < 3; ++trial) {
            long long t0 = clock64();
            for (int r = 0; r < reps; ++r) {
                const int kb = r & 7;
                uint64_t ad = a_mn ? umma::desc_mnmajor(base, M, kb) : umma::desc_kmajor(base, K, kb);
                uint64_t bd = b_mn ? umma::desc_mnmajor(base + 32768, N, kb) : umma::desc_kmajor(base + 32768, K, kb);
                umma::mma_bf16(slot, ad, bd, id, r > 0);
            }
            umma::commit(&bar);
            umma::mbar_wait(&bar, ph);
            ph ^= 1;
            long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
        }
        out[0] = best;
    }
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free<512>(slot);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    int shapes[][4] = {{128, 64, 0, 0}, {128, 64, 0, 1}, {64, 64, 1, 1}, {128, 128, 0, 0}, {128, 256, 0, 0},
                       {64, 256, 0, 0}, {128, 32, 0, 0}, {128, 16, 0, 0}, {64, 64, 0, 0}};
    for (auto& s : shapes) {
        for (int reps : {1, 8, 64}) {
            k<<<1, 128, 96 * 1024>>>(s[0], s[1], s[2], s[3], reps, d);
            long long h = 0;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("M=%3d N=%3d a_mn=%d b_mn=%d reps=%2d cycles=%6lld per_mma=%7.1f  MAC/clk=%7.1f\n", s[0], s[1], s[2],
                   s[3], reps, h, double(h) / reps, double(s[0]) * s[1] * 16 * reps / h);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
