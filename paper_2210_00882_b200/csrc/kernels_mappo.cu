// MAPPO on spread_lite (exact numerics): env reset/step for n agents per env and the per-step
// PolicyApply over the agent-major policy rows (programs.cpp:349-454; envs.cpp:86-150;
// interp.cpp:175-262). One thread per env; state SoA est[i * E + e], i < 4n.
//
// Layouts written per step t (R = n*E agent-major rows, W = n*(2+2n) joint obs width,
// C = W + n critic input width):
//   joint[t][e][W]            the env observation (state_in of the reference)
//   prows[t][a*E+e][S]        policy input rows (the per-agent Slice + Concat, programs.cpp:100-109)
//   cin[t][a*E+e][C]          critic input rows [joint(t,e) | onehot(a)] (programs.cpp:390-402);
//                             optional: the engine's compact critic reads joint + the agent id instead
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.hpp"
#include "kernels.cuh"

namespace flw {

namespace {

__device__ __forceinline__ double dmaxm(double a, double b) { return a < b ? b : a; }

// observe (envs.cpp:96-109) -> the three row layouts for step block `blk`
__device__ void spread_emit(const double* est, int64_t E, int64_t e, int n, float* joint, float* prows, float* cin,
                            int64_t blk) {
    const int S = 2 + 2 * n, W = n * S, C = W + n;
    const int64_t R = static_cast<int64_t>(n) * E;
    float* jrow = joint + (blk * E + e) * W;
    for (int a = 0; a < n; ++a) {
        const double xa = est[(2 * a) * E + e], ya = est[(2 * a + 1) * E + e];
        float* pr = prows + (blk * R + static_cast<int64_t>(a) * E + e) * S;
        float o[2] = {static_cast<float>(xa), static_cast<float>(ya)};
        jrow[a * S] = pr[0] = o[0];
        jrow[a * S + 1] = pr[1] = o[1];
        for (int l = 0; l < n; ++l) {
            const float dx = static_cast<float>(__dsub_rn(est[(2 * n + 2 * l) * E + e], xa));
            const float dy = static_cast<float>(__dsub_rn(est[(2 * n + 2 * l + 1) * E + e], ya));
            jrow[a * S + 2 + 2 * l] = pr[2 + 2 * l] = dx;
            jrow[a * S + 3 + 2 * l] = pr[3 + 2 * l] = dy;
        }
    }
    if (!cin) return;  // compact critic (the engine default): [joint | one-hot] is never materialised
    for (int a = 0; a < n; ++a) {
        float* crow = cin + (blk * R + static_cast<int64_t>(a) * E + e) * C;
        for (int j = 0; j < W; ++j) crow[j] = jrow[j];
        for (int j = 0; j < n; ++j) crow[W + j] = j == a ? 1.0f : 0.0f;
    }
}

__global__ void k_reset_mappo(const DeviceCtx* __restrict__ ctx, int n, double* est, uint8_t* done, int32_t* stepc,
                              float* joint, float* prows, float* cin, int64_t E, int64_t env_lo, uint64_t seed) {
    int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= E) return;
    uint64_t es = rng_key(seed, kEnvStream, static_cast<uint64_t>(env_lo + e), static_cast<uint64_t>(ctx->episode));
    for (int i = 0; i < 4 * n; ++i)  // envs.cpp:88-94
        est[i * E + e] = rng_uniform_range(rng_key(es, kResetTag, 0, static_cast<uint64_t>(i)), -1.0, 1.0);
    done[e] = 0;
    stepc[e] = 0;
    spread_emit(est, E, e, n, joint, prows, cin, 0);
}

// PolicyApply for every agent row of env e, then the joint env step, then the step's rows.
__global__ void k_rollout_mappo(const DeviceCtx* __restrict__ ctx, MappoStepArgs a) {
    int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= a.E) return;
    const int n = a.n, A = a.A;
    const int64_t R = static_cast<int64_t>(n) * a.E, st = a.step;
    int acts[64];
    for (int ag = 0; ag < n; ++ag) {
        const int64_t row = static_cast<int64_t>(ag) * a.E + e;
        const float* lg = a.logits + row * A;
        double l[16], p[16];
        double mx = lg[0];
        for (int c = 0; c < A; ++c) {
            l[c] = lg[c];
            mx = dmaxm(mx, l[c]);
        }
        double den = 0.0;
        for (int c = 0; c < A; ++c) {
            p[c] = exp(__dsub_rn(l[c], mx));
            den = __dadd_rn(den, p[c]);
        }
        for (int c = 0; c < A; ++c) p[c] = f32r(__ddiv_rn(p[c], den));
        const uint64_t global_row = static_cast<uint64_t>(ag * a.env_total + a.env_lo + e);
        const double u = rng_uniform(rng_key(a.seed, kActionStream, static_cast<uint64_t>(ctx->episode),
                                             static_cast<uint64_t>(st), global_row));
        double cum = 0.0;
        int chosen = A - 1;
        for (int c = 0; c < A; ++c) {
            cum = __dadd_rn(cum, p[c]);
            if (u < cum) {
                chosen = c;
                break;
            }
        }
        acts[ag] = chosen;
        a.actions[st * R + row] = chosen;
        a.logp[st * R + row] = static_cast<float>(log(dmaxm(p[chosen], 1e-30)));
    }
    double* s = a.est;
    const int64_t E = a.E;
    double total = 0.0;
    bool d;
    if (a.done[e]) {  // absorbing: repeat obs, zero rewards, done 1 (interp.cpp:239-245)
        for (int ag = 0; ag < n; ++ag) a.reward[st * R + static_cast<int64_t>(ag) * E + e] = 0.0f;
        d = true;
    } else {
        for (int ag = 0; ag < n; ++ag) {  // moves (envs.cpp:114-126)
            double dx = 0.0, dy = 0.0;
            switch (acts[ag]) {
                case 1: dx = 0.1; break;
                case 2: dx = -0.1; break;
                case 3: dy = 0.1; break;
                case 4: dy = -0.1; break;
                default: break;
            }
            s[(2 * ag) * E + e] = __dadd_rn(s[(2 * ag) * E + e], dx);
            s[(2 * ag + 1) * E + e] = __dadd_rn(s[(2 * ag + 1) * E + e], dy);
        }
        for (int ag = 0; ag < n; ++ag) {  // rewards (envs.cpp:128-144)
            const double xa = s[(2 * ag) * E + e], ya = s[(2 * ag + 1) * E + e];
            double best = 1e18;
            for (int l = 0; l < n; ++l) {
                double dx = __dsub_rn(s[(2 * n + 2 * l) * E + e], xa);
                double dy = __dsub_rn(s[(2 * n + 2 * l + 1) * E + e], ya);
                double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
                best = dist < best ? dist : best;
            }
            double r = -best;
            for (int b = 0; b < n; ++b) {
                if (b == ag) continue;
                double dx = __dsub_rn(s[(2 * b) * E + e], xa);
                double dy = __dsub_rn(s[(2 * b + 1) * E + e], ya);
                if (__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))) < 0.1) r = __dsub_rn(r, 0.5);
            }
            total = __dadd_rn(total, r);
            a.reward[st * R + static_cast<int64_t>(ag) * E + e] = static_cast<float>(r);
        }
        const int32_t sc = a.stepc[e];
        d = a.max_steps > 0 && sc + 1 >= a.max_steps;
        a.stepc[e] = sc + 1;
        a.done[e] = d ? 1 : 0;
    }
    a.reward_d[st * E + e] = total;
    for (int ag = 0; ag < n; ++ag) a.done_f[st * R + static_cast<int64_t>(ag) * E + e] = d ? 1.0f : 0.0f;
    spread_emit(s, E, e, n, a.joint, a.prows, a.cin, st + 1);
}

// The same step with one block per env and one thread per agent (n > 4, compact critic: no
// [joint | one-hot] rows): every per-row computation is the serial kernel's, in the same
// operation order (each agent's PolicyApply, move, and reward against the moved positions), and
// thread 0 adds the agents' rewards in agent order - bit-identical to k_rollout_mappo. The
// step's joint row and policy rows are written cooperatively (coalesced) from shared memory.
__global__ void k_rollout_mappo_par(const DeviceCtx* __restrict__ ctx, MappoStepArgs a) {
    extern __shared__ double sm[];  // positions [4n] (agents then landmarks), rewards [n]
    const int64_t e = blockIdx.x;
    const int n = a.n, A = a.A, ag = threadIdx.x;
    const int64_t E = a.E, R = static_cast<int64_t>(n) * E, st = a.step;
    double* pos = sm;
    double* rw = sm + 4 * n;
    __shared__ int dn;
    for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) pos[i] = a.est[i * E + e];
    if (threadIdx.x == 0) dn = a.done[e];
    __syncthreads();
    int chosen = 0;
    if (ag < n) {  // PolicyApply (interp.cpp:175-203): double softmax, the reference's draw and walk
        const int64_t row = static_cast<int64_t>(ag) * E + e;
        const float* lg = a.logits + row * A;
        double l[16], p[16];
        double mx = lg[0];
        for (int c = 0; c < A; ++c) {
            l[c] = lg[c];
            mx = dmaxm(mx, l[c]);
        }
        double den = 0.0;
        for (int c = 0; c < A; ++c) {
            p[c] = exp(__dsub_rn(l[c], mx));
            den = __dadd_rn(den, p[c]);
        }
        for (int c = 0; c < A; ++c) p[c] = f32r(__ddiv_rn(p[c], den));
        const uint64_t global_row = static_cast<uint64_t>(ag * a.env_total + a.env_lo + e);
        const double u = rng_uniform(rng_key(a.seed, kActionStream, static_cast<uint64_t>(ctx->episode),
                                             static_cast<uint64_t>(st), global_row));
        double cum = 0.0;
        chosen = A - 1;
        for (int c = 0; c < A; ++c) {
            cum = __dadd_rn(cum, p[c]);
            if (u < cum) {
                chosen = c;
                break;
            }
        }
        a.actions[st * R + row] = chosen;
        a.logp[st * R + row] = static_cast<float>(log(dmaxm(p[chosen], 1e-30)));
    }
    const bool live = !dn;
    if (live && ag < n) {  // moves (envs.cpp:114-126)
        double dx = 0.0, dy = 0.0;
        switch (chosen) {
            case 1: dx = 0.1; break;
            case 2: dx = -0.1; break;
            case 3: dy = 0.1; break;
            case 4: dy = -0.1; break;
            default: break;
        }
        pos[2 * ag] = __dadd_rn(pos[2 * ag], dx);
        pos[2 * ag + 1] = __dadd_rn(pos[2 * ag + 1], dy);
    }
    __syncthreads();
    if (ag < n) {  // rewards (envs.cpp:128-144); absorbing after done: 0 (interp.cpp:239-245)
        double r = 0.0;
        if (live) {
            const double xa = pos[2 * ag], ya = pos[2 * ag + 1];
            double best = 1e18;
            for (int lm = 0; lm < n; ++lm) {
                const double dx = __dsub_rn(pos[2 * n + 2 * lm], xa);
                const double dy = __dsub_rn(pos[2 * n + 2 * lm + 1], ya);
                const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
                best = dist < best ? dist : best;
            }
            r = -best;
            for (int b = 0; b < n; ++b) {
                if (b == ag) continue;
                const double dx = __dsub_rn(pos[2 * b], xa);
                const double dy = __dsub_rn(pos[2 * b + 1], ya);
                if (__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))) < 0.1) r = __dsub_rn(r, 0.5);
            }
        }
        rw[ag] = r;
        a.reward[st * R + static_cast<int64_t>(ag) * E + e] = static_cast<float>(r);
        a.done_f[st * R + static_cast<int64_t>(ag) * E + e] = 0.0f;  // set below when the env is done
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double total = 0.0;
        bool d = true;
        if (live) {
            for (int b = 0; b < n; ++b) total = __dadd_rn(total, rw[b]);
            const int32_t sc = a.stepc[e];
            d = a.max_steps > 0 && sc + 1 >= a.max_steps;
            a.stepc[e] = sc + 1;
            a.done[e] = d ? 1 : 0;
        }
        a.reward_d[st * E + e] = total;
        dn = d ? 1 : 0;
    }
    __syncthreads();
    if (dn && ag < n) a.done_f[st * R + static_cast<int64_t>(ag) * E + e] = 1.0f;
    for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) a.est[i * E + e] = pos[i];  // moved agents
    // observe (envs.cpp:96-109): joint row and the n policy rows of step block st + 1
    const int S = 2 + 2 * n, W = n * S;
    const int64_t blk = st + 1;
    float* jrow = a.joint + (blk * E + e) * W;
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
        const int b = j / S, c = j - b * S;
        float v;
        if (c < 2) {
            v = static_cast<float>(pos[2 * b + c]);
        } else {
            const int lm = (c - 2) >> 1, xy = (c - 2) & 1;
            v = static_cast<float>(__dsub_rn(pos[2 * n + 2 * lm + xy], pos[2 * b + xy]));
        }
        jrow[j] = v;
        a.prows[(blk * R + static_cast<int64_t>(b) * E + e) * S + c] = v;
    }
}

}  // namespace

void mappo_reset(cudaStream_t s, const DeviceCtx* ctx, int n, double* est, uint8_t* done, int32_t* stepc, float* joint,
                 float* prows, float* cin, int64_t E, int64_t env_lo, uint64_t seed) {
    k_reset_mappo<<<static_cast<unsigned>((E + 127) / 128), 128, 0, s>>>(ctx, n, est, done, stepc, joint, prows, cin,
                                                                          E, env_lo, seed);
}

void mappo_rollout(cudaStream_t s, const DeviceCtx* ctx, const MappoStepArgs& a) {
    if (!a.cin && a.n > 4) {  // one block per env, one thread per agent (bit-identical)
        const unsigned threads = static_cast<unsigned>((a.n + 31) / 32 * 32);
        const size_t smem = static_cast<size_t>(5 * a.n) * sizeof(double);
        k_rollout_mappo_par<<<static_cast<unsigned>(a.E), threads, smem, s>>>(ctx, a);
        return;
    }
    k_rollout_mappo<<<static_cast<unsigned>((a.E + 127) / 128), 128, 0, s>>>(ctx, a);
}

}  // namespace flw
