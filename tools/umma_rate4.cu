// Microbenchmark: warp-collective tcgen05.mma issue when the descriptors are NOT provably
// warp-uniform (read from shared memory per MMA -> R2UR.BROADCAST per operand) vs derived from
// uniform values (umma_rate3.cu). Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20
//   -I paper_2210_00882_b200/csrc tools/umma_rate4.cu -o tools/umma_rate4.bin
#include <cstdio>
#include "umma.cuh"
using namespace flw;

template <int M, int N, int AMN, int BMN, int MODE>
__global__ void k(int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ uint64_t dtab[16];
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    umma::fence_async_smem();
    if (threadIdx.x < 32) umma::tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_barrier_init();
        const uint32_t base = umma::smem_u32(smem);
        for (int kb = 0; kb < 8; ++kb) {
            dtab[kb] = AMN ? umma::desc_mnmajor(base, M, kb) : umma::desc_kmajor(base, 128, kb);
            dtab[8 + kb] = BMN ? umma::desc_mnmajor(base + 32768, N, kb) : umma::desc_kmajor(base + 32768, 128, kb);
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (threadIdx.x < 32) {
        const uint32_t base = umma::smem_u32(smem);
        constexpr uint32_t id = umma::idesc_bf16(M, N, AMN, BMN);
        const uint32_t tm = slot;
        uint32_t ph = 0;
        long long best = 1LL << 60;
        for (int trial = 0; trial < 4; ++trial) {
            __syncwarp();
            long long t0 = clock64();
            for (int r = 0; r < reps; r += 8) {
#pragma unroll
                for (int kb = 0; kb < 8; ++kb) {
                    uint64_t ad, bd;
                    if (MODE == 0) {
                        ad = AMN ? umma::desc_mnmajor(base, M, kb) : umma::desc_kmajor(base, 128, kb);
                        bd = BMN ? umma::desc_mnmajor(base + 32768, N, kb) : umma::desc_kmajor(base + 32768, 128, kb);
                    } else if (MODE == 1) {  // per-MMA shared-memory loads (not provably uniform)
                        ad = dtab[kb];
                        bd = dtab[8 + kb];
                    } else {  // lane-0 broadcast of the loaded values
                        ad = __shfl_sync(0xffffffffu, dtab[kb], 0);
                        bd = __shfl_sync(0xffffffffu, dtab[8 + kb], 0);
                    }
                    umma::mma_bf16_warp(tm, ad, bd, id, (r + kb) > 0);
                }
            }
            umma::commit_warp(&bar);
            umma::mbar_wait(&bar, ph);
            ph ^= 1;
            long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
        }
        if (threadIdx.x == 0) out[0] = best;
    }
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free<512>(slot);
}

template <int M, int N, int AMN, int BMN, int MODE>
void run(long long* d) {
    cudaFuncSetAttribute(k<M, N, AMN, BMN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    const int reps = 256;
    k<M, N, AMN, BMN, MODE><<<1, 128, 96 * 1024>>>(reps, d);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode=%d (0 uniform-computed, 1 smem-loaded, 2 smem+shfl) M=%3d N=%3d cycles/mma=%6.1f\n", MODE, M, N,
           double(h) / reps);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    run<128, 64, 0, 0, 0>(d);
    run<128, 64, 0, 0, 1>(d);
    run<128, 64, 0, 0, 2>(d);
    run<64, 64, 1, 1, 0>(d);
    run<64, 64, 1, 1, 1>(d);
    run<64, 64, 1, 1, 2>(d);
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
