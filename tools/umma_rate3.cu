// Microbenchmark: tcgen05.mma issue cost when the whole warp runs the issue loop with
// warp-uniform descriptors and an elect.sync inside the asm (no per-MMA R2UR / ELECT loop),
// vs. the single-thread issue of umma_rate2.cu.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2210_00882_b200/csrc tools/umma_rate3.cu -o tools/umma_rate3.bin
#include <cstdio>
#include "umma.cuh"
using namespace flw;

__device__ __forceinline__ void mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(umma::smem_u32(bar))
                 : "memory");
}

template <int M, int N, int AMN, int BMN, int NACC>
__global__ void k(int reps, long long* out) {
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
    if (threadIdx.x < 32) {
        const uint32_t base = umma::smem_u32(smem);
        constexpr uint32_t id = umma::idesc_bf16(M, N, AMN, BMN);
        constexpr int K = 128;
        const uint32_t tm = slot;
        constexpr uint32_t stride = N < 128 ? 128u : static_cast<uint32_t>(N);
        uint32_t ph = 0;
        long long best = 1LL << 60, best_issue = 0;
        for (int trial = 0; trial < 4; ++trial) {
            __syncwarp();
            long long t0 = clock64();
            for (int r = 0; r < reps; r += 8) {
#pragma unroll
                for (int kb = 0; kb < 8; ++kb) {
                    const uint64_t ad = AMN ? umma::desc_mnmajor(base, M, kb) : umma::desc_kmajor(base, K, kb);
                    const uint64_t bd = BMN ? umma::desc_mnmajor(base + 32768, N, kb) : umma::desc_kmajor(base + 32768, K, kb);
                    mma_elect(tm + stride * (kb % NACC), ad, bd, id, (r + kb) >= NACC);
                }
            }
            long long ti = clock64();
            commit_elect(&bar);
            umma::mbar_wait(&bar, ph);
            ph ^= 1;
            long long t1 = clock64();
            if (t1 - t0 < best) { best = t1 - t0; best_issue = ti - t0; }
        }
        if (threadIdx.x == 0) { out[0] = best; out[1] = best_issue; }
    }
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free<512>(slot);
}

template <int M, int N, int AMN, int BMN, int NACC>
void run(long long* d) {
    cudaFuncSetAttribute(k<M, N, AMN, BMN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int reps : {8, 64, 256}) {
        k<M, N, AMN, BMN, NACC><<<1, 128, 96 * 1024>>>(reps, d);
        long long h[2] = {0};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("warp-issue M=%3d N=%3d a_mn=%d b_mn=%d nacc=%d reps=%3d cycles=%6lld per_mma=%6.1f issue_per_mma=%6.1f MAC/clk=%7.1f\n",
               M, N, AMN, BMN, NACC, reps, h[0], double(h[0]) / reps, double(h[1]) / reps, double(M) * N * 16 * reps / h[0]);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    run<128, 64, 0, 0, 1>(d);
    run<128, 64, 0, 0, 2>(d);
    run<128, 64, 0, 1, 1>(d);
    run<64, 64, 1, 1, 1>(d);
    run<64, 64, 1, 1, 2>(d);
    run<128, 128, 0, 0, 1>(d);
    run<128, 256, 0, 0, 1>(d);
    run<128, 32, 0, 0, 1>(d);
    run<128, 16, 0, 0, 1>(d);
    run<128, 16, 0, 0, 2>(d);
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
