// Scaled-size HBM microbenchmarks of the DP-D element-wise kernels the episodes launch (SURVEY
// §8(d): at C2 these move < 20 MB and are launch/L2 bound, so their roofline is reported on
// scaled sizes). Algorithmic bytes are the survey's per-unit figures:
//   rollout_env : k_rollout (PolicyApply + synth17x6 step, the per-step env kernel of the exact,
//                 layer-wise and split-GEMM rollouts) over E envs: (8S+9) B/env-step (state in/out,
//                 action, reward, done) + 4A logits in + 4 logp out = 173 B (the kernel keeps the
//                 env state in f64, so it moves more than this)
//   gae_scan32  : k_gae_scan32 (the episode's GAE + returns + advantage statistics, T = 32) at
//                 T*R rows (>= 2^22 rows: inputs > L2; smaller: four rotating sets): 17 B/row + 4 B/stream
//   gae         : k_fast_gae<8,4> (fast_gae's kernel for T != 32) at T*R rows
//   reduce_adam : k_reduce_adam (the fused per-iteration update: partial reduction + Adam with f64
//                 moments) over P params and 8 partial slots: 44 B/param (g in, p, m, v in/out) + 4 B
//                 per partial slot
//   exchange_adam: k_exchange_adam (the k-GPU peer-memory update) with k = 1: same bytes
//   env_step / adam: the standalone microbenchmark kernels of round 1 (kept for comparison)
// Each launch is timed with CUDA events on the launching stream, after warm-up.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "engine.hpp"
#include "envs.cuh"
#include "fast.cuh"
#include "kernels.cuh"
#include "p2p.cuh"

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
        // algorithmic 17 B/row (done as one byte); the kernel reads done as f32 (20 B)
        *bytes = static_cast<double>(T * R) * 17.0 + static_cast<double>(R) * 4.0;
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
    } else if (which == "rollout_env") {  // k_rollout: PolicyApply + env step, E = n envs
        const int S = kSynthObs, A = kSynthAct;
        float* logits = d.get<float>(A * n);
        double* est = d.get<double>(S * n);
        uint8_t* done = d.get<uint8_t>(n);
        int32_t* stepc = d.get<int32_t>(n);
        int32_t* act = d.get<int32_t>(n);
        float* lp = d.get<float>(n);
        float* rw = d.get<float>(n);
        double* rwd = d.get<double>(n);
        float* dnf = d.get<float>(n);
        float* obs = d.get<float>(S * n);
        double* tab = d.get<double>(A * S);
        DeviceCtx* ctx = d.get<DeviceCtx>(1);
        FLW_CUDA(cudaMemset(ctx, 0, sizeof(DeviceCtx)));
        FLW_CUDA(cudaMemset(done, 0, n));
        FLW_CUDA(cudaMemset(stepc, 0, n * sizeof(int32_t)));
        k_init_f32<<<g, blk>>>(logits, A * n, 1, -1.f, 1.f);
        k_init_u64<<<g, blk>>>(est, S * n, 2, -0.1, 0.1);
        k_init_u64<<<g, blk>>>(tab, A * S, 3, -1.0, 1.0);
        FLW_CUDA(cudaGetLastError());
        RolloutArgs a{};
        a.logits = logits;
        a.est = est;
        a.done = done;
        a.stepc = stepc;
        a.actions = act;
        a.logp = lp;
        a.reward = rw;
        a.reward_d = rwd;
        a.done_f = dnf;
        a.next_obs = obs;
        a.E = n;
        a.S = S;
        a.A = A;
        a.seed = 7;
        a.env.kind = static_cast<int>(EnvKind::Synth17x6);
        a.env.synth_b = tab;
        *ms = time_launches([&] { exact_rollout(0, ctx, a); }, iters);
        *bytes = static_cast<double>(n) * (8.0 * S + 9 + 4.0 * A + 4);
    } else if (which == "gae_scan32") {  // the episode's GAE kernel (T = 32) at R = n / 32 streams
        const int64_t T = 32, R = n / T;
        const int kSets = n <= (1 << 22) ? 4 : 1;  // small sizes: 4 rotating sets > L2
        float *r[4], *v[4], *dn[4], *lv[4], *adv[4], *ret[4];
        for (int k = 0; k < kSets; ++k) {
            r[k] = d.get<float>(T * R);
            v[k] = d.get<float>(T * R);
            dn[k] = d.get<float>(T * R);
            lv[k] = d.get<float>(R);
            adv[k] = d.get<float>(T * R);
            ret[k] = d.get<float>(T * R);
            k_init_f32<<<g, blk>>>(r[k], T * R, 1 + k, -1.f, 1.f);
            k_init_f32<<<g, blk>>>(v[k], T * R, 11 + k, -1.f, 1.f);
            k_init_f32<<<g, blk>>>(dn[k], T * R, 21 + k, -18.f, 1.f);
            k_init_f32<<<g, blk>>>(lv[k], R, 31 + k, -1.f, 1.f);
        }
        double* bs = d.get<double>(2 * ((R + 31) / 32));
        double* st = d.get<double>(2);
        unsigned* cnt = d.get<unsigned>(1);
        FLW_CUDA(cudaMemset(cnt, 0, sizeof(unsigned)));
        FLW_CUDA(cudaGetLastError());
        int it = 0;  // k_gae_scan32 directly (fast_gae routes R > 65536 to the thread-per-stream kernel)
        *ms = time_launches([&] {
            const int k = it++ % kSets;
            fast_gae_scan32(0, r[k], v[k], dn[k], lv[k], R, 0.99, 0.95, adv[k], ret[k], true, bs, st, cnt);
        }, iters);
        *bytes = static_cast<double>(T * R) * 17.0 + static_cast<double>(R) * 4.0;
    } else if (which == "reduce_adam" || which == "exchange_adam") {  // the fused update kernels, P = n
        // partial slots (the episode's learn kernels write 59-148; FLW_MB_PARTS overrides the 8)
        const int kParts = std::getenv("FLW_MB_PARTS") ? std::atoi(std::getenv("FLW_MB_PARTS")) : 8;
        const int64_t npad = (n + 3) / 4 * 4;
        float* part = d.get<float>(kParts * npad);
        float* p = d.get<float>(n);
        float* gr = d.get<float>(n);
        double* m = d.get<double>(n);
        double* v = d.get<double>(n);
        DeviceCtx* ctx = d.get<DeviceCtx>(1);
        constexpr int kBc = 256;  // the engine's host-computed bias-correction table (t <= kBc here)
        double2* bct = d.get<double2>(kBc);
        unsigned* cnt = d.get<unsigned>(1);
        {
            std::vector<double2> tab(kBc);
            for (int t = 1; t <= kBc; ++t) tab[t - 1] = double2{1.0 - std::pow(0.9, t), 1.0 - std::pow(0.999, t)};
            FLW_CUDA(cudaMemcpy(bct, tab.data(), kBc * sizeof(double2), cudaMemcpyHostToDevice));
        }
        DeviceCtx c{};
        c.bc1 = 0.1;
        c.bc2 = 0.001;
        FLW_CUDA(cudaMemcpy(ctx, &c, sizeof(c), cudaMemcpyHostToDevice));
        FLW_CUDA(cudaMemset(cnt, 0, sizeof(unsigned)));
        k_init_f32<<<g, blk>>>(p, n, 1, -0.1f, 0.1f);
        k_init_f32<<<g, blk>>>(part, kParts * npad, 2, -1e-3f, 1e-3f);
        FLW_CUDA(cudaMemset(m, 0, n * sizeof(double)));
        FLW_CUDA(cudaMemset(v, 0, n * sizeof(double)));
        FLW_CUDA(cudaGetLastError());
        if (which == "reduce_adam") {
            FastUpdateArgs u{};
            u.pp = part;
            u.pc = part;
            u.np = kParts;
            u.nc = 0;
            u.Pp = n;
            u.Pc = 0;
            u.ctx = ctx;
            u.bc_table = bct;
            u.bc_len = kBc;
            u.params = p;
            u.grads = gr;
            u.m = m;
            u.v = v;
            u.lr = 3e-3;
            u.b1 = 0.9;
            u.b2 = 0.999;
            u.eps = 1e-8;
            u.counter = cnt;  // pol / crit: L = 0 (no weight-image entries)
            *ms = time_launches([&] { fast_reduce_adam(0, u); }, iters);
        } else {
            const P2pLayout L = p2p_layout(1, n);
            uint8_t* region = d.get<uint8_t>(L.bytes);
            FLW_CUDA(cudaMemset(region, 0, L.bytes));
            uint8_t** peers = d.get<uint8_t*>(1);
            FLW_CUDA(cudaMemcpy(peers, &region, sizeof(region), cudaMemcpyHostToDevice));
            unsigned* abort_word = d.get<unsigned>(1);
            FLW_CUDA(cudaMemset(abort_word, 0, sizeof(unsigned)));
            P2pArgs a{};
            a.part_p = part;
            a.part_c = part;
            a.np = kParts;
            a.nc = 0;
            a.Pp = n;
            a.Pc = 0;
            a.rank = 0;
            a.k = 1;
            a.peers = peers;
            a.off_inbox = L.off_inbox;
            a.off_grads = L.off_grads;
            a.off_sflag = L.off_sflag;
            a.off_dflag = L.off_dflag;
            a.ctx = ctx;
            a.abort_flag = abort_word;
            a.params = p;
            a.m = m;
            a.v = v;
            a.lr = 3e-3;
            a.b1 = 0.9;
            a.b2 = 0.999;
            a.eps = 1e-8;
            a.gscale = 1.0;
            a.Ptot = n;
            *ms = time_launches([&] {
                coll_tick(0, ctx);
                reduce_allreduce_adam(0, a, true);  // k = 1: waits on its own push only
            }, iters);
        }
        // survey: 44 B/param of Adam with f64 moments + 4 B per partial slot of the reduction
        *bytes = static_cast<double>(n) * (44.0 + 4.0 * kParts);
    } else {
        fail(Errc::Config, "unknown microbenchmark '" + which + "'");
    }
    FLW_CUDA(cudaGetLastError());
}

}  // namespace flw
