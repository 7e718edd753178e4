// Scaled-size HBM microbenchmarks of the DP-D element-wise kernels (at C2 these
// move < 20 MB and are launch/L2 bound, so their roofline is reported on scaled sizes):
//   env_step : batched synth17x6 step over E envs, SoA double state in/out, f32 obs/reward,
//              u8 done, i32 action                      -> 8*17*2 + 4 + 4*17 + 4 + 1 = 349 B/env
//   gae      : GAE + returns over T*E rows (T = 32)     -> r, V, done (f32) in; adv, ret out = 20 B/row
//   adam     : Adam with f64 moments over P params      -> g,p (f32) + m,v (f64) in; p,m,v out = 44 B/param
// Inputs are device-resident and larger than L2 at the sizes bench.py uses; each launch is
// timed with CUDA events on the launching stream, after warm-up.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "engine.hpp"
#include "envs.cuh"
#include "fast.cuh"
#include "kernels.cuh"

namespace flw {

namespace {

__global__ void k_init_u64(double* x, int64_t n, uint64_t seed, double lo, double hi) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = rng_uniform_range(rng_key(seed, static_cast<uint64_t>(i)), lo, hi);
}

__global__ void k_init_f32(float* x, int64_t n, uint64_t seed, float lo, float hi) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = static_cast<float>(rng_uniform_range(rng_key(seed, static_cast<uint64_t>(i)), lo, hi));
}

__global__ void k_init_i32(int32_t* x, int64_t n, uint64_t seed, int mod) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = static_cast<int32_t>(rng_key(seed, static_cast<uint64_t>(i)) % static_cast<uint64_t>(mod));
}

// Standalone batched env step (synth17x6), thread per env, SoA state: the same dynamics as the
// fused rollout (envs.cuh env_step1), with the state streamed from/to HBM.
__global__ void __launch_bounds__(256) k_env_step_soa(double* __restrict__ est, const int32_t* __restrict__ act,
                                                      float* __restrict__ obs, float* __restrict__ rew,
                                                      uint8_t* __restrict__ done, const double* __restrict__ tab,
                                                      int64_t E) {
    int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= E) return;
    const int a = act[e];
    double old[kSynthObs];
#pragma unroll
    for (int i = 0; i < kSynthObs; ++i) old[i] = est[i * E + e];
    double sq = 0.0, mx = 0.0;
#pragma unroll
    for (int i = 0; i < kSynthObs; ++i) {
        double t4 = __dadd_rn(__dsub_rn(__dmul_rn(0.3, old[(i + 1) % kSynthObs]), __dmul_rn(0.5, old[i])),
                              tab[a * kSynthObs + i]);
        double nv = __dadd_rn(old[i], __dmul_rn(0.05, t4));
        est[i * E + e] = nv;
        obs[i * E + e] = static_cast<float>(nv);
        sq = __dadd_rn(sq, __dmul_rn(nv, nv));
        double av = nv < 0.0 ? -nv : nv;
        mx = av > mx ? av : mx;
    }
    rew[e] = static_cast<float>(__dsub_rn(1.0, __ddiv_rn(sq, static_cast<double>(kSynthObs))));
    done[e] = mx > 2.0 ? 1 : 0;
}

template <typename F>
double time_launches(F&& launch, int iters) {
    cudaEvent_t a, b;
    FLW_CUDA(cudaEventCreate(&a));
    FLW_CUDA(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) launch();  // warm-up
    FLW_CUDA(cudaDeviceSynchronize());
    FLW_CUDA(cudaEventRecord(a, 0));
    for (int i = 0; i < iters; ++i) launch();
    FLW_CUDA(cudaEventRecord(b, 0));
    FLW_CUDA(cudaEventSynchronize(b));
    float ms = 0.0f;
    FLW_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / iters;
}

struct DevBuf {
    std::vector<void*> ptrs;
    template <typename T>
    T* get(int64_t n) {
        void* p = nullptr;
        FLW_CUDA(cudaMalloc(&p, static_cast<size_t>(n) * sizeof(T)));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
};

}  // namespace

// Returns ms per launch and the algorithmic bytes one launch moves.
void microbench(const std::string& which, int64_t n, int iters, double* ms, double* bytes) {
    DevBuf d;
    const dim3 g(1184), blk(256);
    if (which == "env_step") {
        double* est = d.get<double>(kSynthObs * n);
        int32_t* act = d.get<int32_t>(n);
        float* obs = d.get<float>(kSynthObs * n);
        float* rew = d.get<float>(n);
        uint8_t* done = d.get<uint8_t>(n);
        double* tab = d.get<double>(kSynthAct * kSynthObs);
        k_init_u64<<<g, blk>>>(est, kSynthObs * n, 1, -0.1, 0.1);
        k_init_u64<<<g, blk>>>(tab, kSynthAct * kSynthObs, 2, -1.0, 1.0);
        k_init_i32<<<g, blk>>>(act, n, 3, kSynthAct);
        FLW_CUDA(cudaGetLastError());
        *ms = time_launches([&] { k_env_step_soa<<<static_cast<unsigned>((n + 255) / 256), 256>>>(est, act, obs, rew, done, tab, n); },
                            iters);
        *bytes = static_cast<double>(n) * (8.0 * kSynthObs * 2 + 4 + 4.0 * kSynthObs + 4 + 1);
    } else if (which == "gae") {
        const int64_t T = 32, R = n / T;
        float* r = d.get<float>(T * R);
        float* v = d.get<float>(T * R);
        float* dn = d.get<float>(T * R);
        float* lv = d.get<float>(R);
        float* adv = d.get<float>(T * R);
        float* ret = d.get<float>(T * R);
        double* bs = d.get<double>(2 * ((R + 31) / 32));
        double* st = d.get<double>(2);
        unsigned* cnt = d.get<unsigned>(1);
        FLW_CUDA(cudaMemset(cnt, 0, sizeof(unsigned)));
        k_init_f32<<<g, blk>>>(r, T * R, 1, -1.f, 1.f);
        k_init_f32<<<g, blk>>>(v, T * R, 2, -1.f, 1.f);
        k_init_f32<<<g, blk>>>(dn, T * R, 3, -18.f, 1.f);  // > 0.5 with probability ~0.03 (done)
        k_init_f32<<<g, blk>>>(lv, R, 4, -1.f, 1.f);
        FLW_CUDA(cudaGetLastError());
        *ms = time_launches([&] { fast_gae(0, r, v, dn, lv, T * R, R, 0.99, 0.95, adv, ret, true, bs, st, cnt); },
                            iters);
        *bytes = static_cast<double>(T * R) * 20.0 + static_cast<double>(R) * 4.0;
    } else if (which == "adam") {
        float* p = d.get<float>(n);
        float* gr = d.get<float>(n);
        double* m = d.get<double>(n);
        double* v = d.get<double>(n);
        DeviceCtx* ctx = d.get<DeviceCtx>(1);
        DeviceCtx c{};
        c.adam_t = 1;
        c.bc1 = 0.1;
        c.bc2 = 0.001;
        FLW_CUDA(cudaMemcpy(ctx, &c, sizeof(c), cudaMemcpyHostToDevice));
        k_init_f32<<<g, blk>>>(p, n, 1, -0.1f, 0.1f);
        k_init_f32<<<g, blk>>>(gr, n, 2, -1e-3f, 1e-3f);
        FLW_CUDA(cudaMemset(m, 0, n * sizeof(double)));
        FLW_CUDA(cudaMemset(v, 0, n * sizeof(double)));
        FLW_CUDA(cudaGetLastError());
        *ms = time_launches([&] { exact_adam(0, ctx, p, gr, nullptr, m, v, n, 3e-3, 0.9, 0.999, 1e-8); }, iters);
        *bytes = static_cast<double>(n) * 44.0;
    } else {
        fail(Errc::Config, "unknown microbenchmark '" + which + "'");
    }
    FLW_CUDA(cudaGetLastError());
}

}  // namespace flw
