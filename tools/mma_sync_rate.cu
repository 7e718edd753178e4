// Microbenchmark: legacy warp-level mma.sync on sm_100a - dependent-chain latency and
// multi-warp throughput of m16n8k8 TF32 (the rollout MLP's instruction).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mma_sync_rate.cu -o tools/mma_sync_rate.bin
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_f16(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int CHAINS, bool F16 = false>
__global__ void k(int reps, long long* out, float* sink) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
    float acc[CHAINS][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (F16) mma_f16(acc[c], a, b);
            else mma_tf32(acc[c], a, b);
        }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
template <int CH, bool F16 = false>
void run(long long* d, float* sink, int warps) {
    const int reps = 256;
    k<CH, F16><<<1, 32 * warps>>>(reps, d, sink);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s chains/warp=%d warps=%2d cycles per mma per warp=%6.2f  SM mma/clk=%.3f\n", F16 ? "f16 m16n8k16" : "tf32 m16n8k8", CH, warps,
           double(h) / (reps * CH), double(reps) * CH * warps / h);
}
int main() {
    long long* d;
    float* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 1 << 20);
    for (int w : {1, 4, 8, 16}) { run<1>(d, sink, w); run<2>(d, sink, w); run<4>(d, sink, w); run<8>(d, sink, w); }
    for (int w : {1, 4, 8, 16}) { run<1, true>(d, sink, w); run<2, true>(d, sink, w); run<4, true>(d, sink, w); }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
