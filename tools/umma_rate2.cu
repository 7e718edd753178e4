// Microbenchmark (round 1, second pass): tcgen05.mma kind::f16 cost per instruction when the
// MMAs of a burst go to 1, 2 or 4 INDEPENDENT TMEM accumulators (round robin), with the
// descriptors precomputed; plus issue-only time (before the commit wait) and tcgen05.ld latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2210_00882_b200/csrc tools/umma_rate2.cu -o /tmp/umma_rate2
#include <cstdio>
#include "umma.cuh"
using namespace flw;

__global__ void k(int M, int N, int a_mn, int b_mn, int reps, int nacc, long long* out) {
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
        const int K = 128;
        uint64_t ad[8], bd[8];
        for (int kb = 0; kb < 8; ++kb) {
            ad[kb] = a_mn ? umma::desc_mnmajor(base, M, kb) : umma::desc_kmajor(base, K, kb);
            bd[kb] = b_mn ? umma::desc_mnmajor(base + 32768, N, kb) : umma::desc_kmajor(base + 32768, K, kb);
        }
        const uint32_t stride = N < 128 ? 128u : static_cast<uint32_t>(N);
        uint32_t ph = 0;
        long long best = 1LL << 60, best_issue = 0;
        for (int trial = 0; trial < 4; ++trial) {
            long long t0 = clock64();
#pragma unroll 8
            for (int r = 0; r < reps; ++r) {
                const int kb = r & 7;
                const uint32_t acc = slot + stride * static_cast<uint32_t>(r % nacc);
                umma::mma_bf16(acc, ad[kb], bd[kb], id, r >= nacc);
            }
            long long ti = clock64();
            umma::commit(&bar);
            umma::mbar_wait(&bar, ph);
            ph ^= 1;
            long long t1 = clock64();
            if (t1 - t0 < best) { best = t1 - t0; best_issue = ti - t0; }
        }
        out[0] = best;
        out[1] = best_issue;
    }
    __syncthreads();
    // TMEM load latency: one warp, x16 load + wait
    if (threadIdx.x < 32) {
        float v[16];
        long long t0 = clock64();
        umma::tmem_ld16(slot, v);
        umma::tmem_ld_wait();
        long long t1 = clock64();
        float s = 0; for (int i = 0; i < 16; ++i) s += v[i];
        if (threadIdx.x == 0) { out[2] = t1 - t0; out[3] = s == 12345.f; }
        t0 = clock64();
        umma::tmem_ld16(slot, v);
        umma::tmem_ld16(slot + 16, v);
        umma::tmem_ld16(slot + 32, v);
        umma::tmem_ld16(slot + 48, v);
        umma::tmem_ld_wait();
        t1 = clock64();
        if (threadIdx.x == 0) out[4] = t1 - t0;
        t0 = clock64();
        umma::fence_async_smem();
        t1 = clock64();
        if (threadIdx.x == 0) out[5] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free<512>(slot);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    int shapes[][4] = {{128, 64, 0, 0}, {128, 64, 0, 1}, {64, 64, 1, 1}, {128, 128, 0, 0}, {128, 256, 0, 0},
                       {128, 32, 0, 0}, {128, 16, 0, 0}};
    for (auto& s : shapes) {
        for (int nacc : {1, 2, 4}) {
            if (s[1] > 128 && nacc > 2) continue;
            int reps = 64;
            k<<<1, 128, 96 * 1024>>>(s[0], s[1], s[2], s[3], reps, nacc, d);
            long long h[6] = {0};
            cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
            printf("M=%3d N=%3d a_mn=%d b_mn=%d nacc=%d reps=%d cycles=%6lld per_mma=%6.1f issue_per_mma=%6.1f MAC/clk=%7.1f | ld16 %lld ld64 %lld fence %lld\n",
                   s[0], s[1], s[2], s[3], nacc, reps, h[0], double(h[0]) / reps, double(h[1]) / reps,
                   double(s[0]) * s[1] * 16 * reps / h[0], h[2], h[4], h[5]);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
