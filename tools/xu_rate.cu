// Pipe-rate probe (sm_100a): cycles per warp instruction per SM for MUFU.TANH, F2FP (f32 -> bf16x2
// pack), both interleaved, and the packed bf16x2 tanh, with 16 warps per SM and 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_rate tools/xu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    unsigned acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 2) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x[i]));
            if (MODE == 3) {
                unsigned v = __float_as_uint(x[i]);
                asm volatile("tanh.approx.bf16x2 %0, %0;" : "+r"(v));
                x[i] = __uint_as_float(v);
            }
            if (MODE == 4) {
                unsigned v = __float_as_uint(x[i]);
                asm volatile("tanh.approx.f16x2 %0, %0;" : "+r"(v));
                x[i] = __uint_as_float(v);
            }
            if (MODE == 1 || MODE == 2) {
                unsigned p;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(x[i]), "f"(x[(i + 1) & 7]));
                acc += p;
                x[i] = __uint_as_float(p & 0x3f800000u) ;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}
int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148, 512>>>(out, iters, cyc);
            if (mode == 1) k<1><<<148, 512>>>(out, iters, cyc);
            if (mode == 2) k<2><<<148, 512>>>(out, iters, cyc);
            if (mode == 3) k<3><<<148, 512>>>(out, iters, cyc);
            if (mode == 4) k<4><<<148, 512>>>(out, iters, cyc);
            cudaDeviceSynchronize();
        }
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double winstr = 16.0 * iters * 8;  // per SM per op type
        printf("mode %d (%s): %lld cycles, %.2f cycles per warp-op per SM\n", mode,
               mode == 0 ? "MUFU.TANH" : mode == 1 ? "F2FP+LOP" : mode == 2 ? "TANH+F2FP" : mode == 3 ? "TANH.BF16x2 (2 values/lane)" : "TANH.F16x2 (2 values/lane)", c, c / winstr);
    }
    return 0;
}
