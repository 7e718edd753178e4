// Batched environments on the device: one thread per env, state in SoA layout
// (est[j * E + e]) so that a warp touches 32 consecutive doubles per state component.
//
// Arithmetic is IEEE double with every +,-,*,/ individually rounded (explicit _rn intrinsics,
// no FMA contraction), i.e. the same operation sequence the reference's x86-64 -O2 build runs
// (/root/reference/proj/src/envs/envs.cpp), so given identical actions the device dynamics are
// bit-identical to the reference (gridline, spread_lite) and to the builder env synth17x6.
#pragma once

#include "common.cuh"

namespace flw {

constexpr int kSynthObs = 17;
constexpr int kSynthAct = 6;
constexpr uint64_t kSynthTableSeed = 0x73796eULL;

struct EnvParams {
    int kind;          // EnvKind
    int n_agents;      // spread_lite agents
    int64_t max_steps; // 0: none
    int64_t length;    // gridline length
    // synth17x6 action table B[a][i] = U(key(0x73796e, a, i), -1, 1), device memory filled at
    // engine creation from the host RNG (identical arithmetic).
    const double* synth_b;
};

// ------------------------------------------------------------------ reset (envs.cpp:181-194)
__device__ __forceinline__ void env_reset_dev(const EnvParams& p, uint64_t env_seed, double* est, int64_t E,
                                              int64_t e) {
    if (p.kind == 0) {  // gridline, envs.cpp:26-31
        int64_t len = p.length;
        int64_t start = static_cast<int64_t>(__dmul_rn(rng_uniform(rng_key(env_seed, kResetTag, 0)),
                                                       static_cast<double>(len / 2)));
        est[e] = static_cast<double>(start);
        est[E + e] = static_cast<double>(len);
    } else if (p.kind == 1) {  // synth17x6: U(key(seed, reset, 0, i), -0.1, 0.1)
#pragma unroll
        for (int i = 0; i < kSynthObs; ++i)
            est[i * E + e] = rng_uniform_range(rng_key(env_seed, kResetTag, 0, static_cast<uint64_t>(i)), -0.1, 0.1);
    } else {  // spread_lite, envs.cpp:88-94
        for (int i = 0; i < 4 * p.n_agents; ++i)
            est[i * E + e] = rng_uniform_range(rng_key(env_seed, kResetTag, 0, static_cast<uint64_t>(i)), -1.0, 1.0);
    }
}

// Observation (single-agent envs): gridline x/(len-1) (envs.cpp:33-36); synth: the state.
__device__ __forceinline__ double env_obs1(const EnvParams& p, const double* est, int64_t E, int64_t e, int j) {
    if (p.kind == 0) return __ddiv_rn(est[e], __dsub_rn(est[E + e], 1.0));
    return est[j * E + e];
}

// One step of a single-agent env. Returns done; *reward is the double reward.
__device__ __forceinline__ bool env_step1(const EnvParams& p, double* est, int64_t E, int64_t e, int action,
                                          int64_t step_count, double* reward) {
    bool done = false;
    if (p.kind == 0) {  // gridline, envs.cpp:38-53
        int64_t len = static_cast<int64_t>(est[E + e]);
        int64_t x = static_cast<int64_t>(est[e]);
        x += action == 1 ? 1 : -1;
        if (x < 0) x = 0;
        if (x > len - 1) x = len - 1;
        est[e] = static_cast<double>(x);
        *reward = 0.0;
        if (x == len - 1) {
            *reward = 1.0;
            done = true;
        }
    } else {  // synth17x6 (oracle/refx/env_ext.cpp)
        double old[kSynthObs];
#pragma unroll
        for (int i = 0; i < kSynthObs; ++i) old[i] = est[i * E + e];
        double sq = 0.0, mx = 0.0;
#pragma unroll
        for (int i = 0; i < kSynthObs; ++i) {
            double t1 = __dmul_rn(0.3, old[(i + 1) % kSynthObs]);
            double t2 = __dmul_rn(0.5, old[i]);
            double t3 = __dsub_rn(t1, t2);
            double t4 = __dadd_rn(t3, p.synth_b[action * kSynthObs + i]);
            double t5 = __dmul_rn(0.05, t4);
            double n = __dadd_rn(old[i], t5);
            est[i * E + e] = n;
            sq = __dadd_rn(sq, __dmul_rn(n, n));
            double m = n < 0.0 ? -n : n;
            mx = m > mx ? m : mx;
        }
        *reward = __dsub_rn(1.0, __ddiv_rn(sq, static_cast<double>(kSynthObs)));
        done = mx > 2.0;
    }
    if (p.max_steps > 0 && step_count + 1 >= p.max_steps) done = true;
    return done;
}

}  // namespace flw
