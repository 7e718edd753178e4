// Launchers for the DP-D kernels. Every launcher enqueues on the given stream and returns
// immediately; shapes are in rows (M), reduction width (K) and output width (N).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "envs.cuh"

namespace flw {

struct DeviceCtx;

// Activation of a hidden layer (programs.cpp:67-68): 0 tanh, 1 relu; 2 = none (last layer).
enum Act : int { kTanh = 0, kRelu = 1, kNone = 2 };

struct RolloutArgs {      // one rollout step over E envs (single-agent PPO/A3C)
    const float* logits;  // [E, A]
    double* est;          // env state SoA [sw, E]
    uint8_t* done;        // [E]
    int32_t* stepc;       // [E]
    int32_t* actions;     // [E]   (this step's slice of the trajectory)
    float* logp;          // [E]
    float* reward;        // [E]
    double* reward_d;     // [E]   unrounded env reward (episode reward sum)
    float* done_f;        // [E]   0/1
    float* next_obs;      // [E, S] next step's policy input (or last_next)
    int64_t E, env_lo;
    int S, A;
    uint64_t seed;
    int64_t step;
    EnvParams env;
};

struct MappoStepArgs {    // one MAPPO rollout step over E envs x n agents (spread_lite)
    const float* logits;  // [n*E, A] agent-major
    double* est;          // [4n, E]
    uint8_t* done;
    int32_t* stepc;
    int32_t* actions;     // [T, n*E]
    float *logp, *reward, *done_f;  // [T, n*E]
    double* reward_d;     // [T, E] env total reward
    float *joint, *prows, *cin;     // step-block layouts (see kernels_mappo.cu)
    int64_t E, env_lo, env_total, step, max_steps;
    int n, A;
    uint64_t seed;
};

void mappo_reset(cudaStream_t s, const DeviceCtx* ctx, int n, double* est, uint8_t* done, int32_t* stepc, float* joint,
                 float* prows, float* cin, int64_t E, int64_t env_lo, uint64_t seed);
void mappo_rollout(cudaStream_t s, const DeviceCtx* ctx, const MappoStepArgs& a);

struct DwTile {           // one 32(t) x 32(j) block of dW_l = H_{l-1}^T dZ_l (+ bias row t == K)
    const float* H;       // [M, K]
    const float* DZ;      // [M, N]
    float* gW;            // [K, N] slice of the flat gradient
    float* gB;            // [N]
    int K, N, t0, j0;
    int64_t rows;         // M: rows of this chain (one replica's T*E_r rows)
    // MAPPO compact critic layer 0 (cn > 0): the input row (t, a*E+e) is [joint(t,e) | onehot(a)],
    // read from H = joint [(T+1)*E, cJ] by index - same values, same row order as the reference
    int cn = 0, cJ = 0;
    int64_t cE = 0;
};

// ---------------------------------------------------------------- exact (FP64-accumulate) path
// begin != null (the episode graph): the reset also does begin_episode's counter update
void exact_reset(cudaStream_t s, DeviceCtx* ctx, const EnvParams& env, double* est, uint8_t* done,
                 int32_t* stepc, float* obs0, int64_t E, int64_t env_lo, int S, uint64_t seed,
                 unsigned* begin = nullptr);
void exact_layer_fwd(cudaStream_t s, const float* in, const float* W, const float* b, float* out, int64_t M, int K,
                     int N, int act);
void exact_layer_dh(cudaStream_t s, const float* dz, const float* W, const float* hprev, float* dzprev, int64_t M,
                    int K, int N, int act);
void exact_rollout(cudaStream_t s, const DeviceCtx* ctx, const RolloutArgs& a);
void exact_seq_sum(cudaStream_t s, const double* x, int64_t n, double* out);
void exact_gae(cudaStream_t s, const float* rew, const float* values, const float* done_f, const float* last_value,
               int64_t TR, int64_t R, double gamma, double lam, double* adv_d, float* ret, bool with_adv);
void exact_normalize(cudaStream_t s, const double* adv_d, int64_t n, bool normalize, double* stats, float* adv);
void exact_loss_rows(cudaStream_t s, int algo, const float* logits, const float* values, const int32_t* actions,
                     const float* logp_old, const float* adv, const float* ret, int64_t n, int A, double clip_eps,
                     double value_coef, double entropy_coef, float* dlogits, float* dvalues, double* terms);
void exact_loss_reduce(cudaStream_t s, const double* terms, int64_t n, double entropy_coef, float* loss);
void exact_dw(cudaStream_t s, const DwTile* tiles, int ntiles);
// MAPPO critic layer 0 without materialising [joint | one-hot] (programs.cpp:390-402): the
// reference's left-to-right dot over the row is the joint prefix chain (identical for the n
// agents of an env) followed by +1*W[J+a] (the one-hot zeros add exact zeros). prefix[blk*E+e]
// is that chain in double; rows (blk, a, e) then get f32(f32(prefix + W[J+a]) + b) and act.
void exact_mappo_critic0(cudaStream_t s, const float* joint, const float* W0, const float* b0, int64_t blocks,
                         int64_t E, int n, int J, int N, double* prefix, float* out_rows, float* out_last, int act);
// R replicas per unit: t-major [T, E, w] trajectory rows -> replica-major [r][T][E_r][w] so that
// every replica's rows (its own unit's BufferSample, interp.cpp:297-301) are contiguous.
struct ReplicaMap {
    const int32_t* rep_of_env;  // [E]
    const int64_t* rep_off;     // [R] first env of replica r (relative to the unit)
    const int64_t* rep_n;       // [R] envs of replica r
};
void permute_rows_f32(cudaStream_t s, const float* src, float* dst, int64_t T, int64_t E, int w, const ReplicaMap& m);
void permute_rows_i32(cudaStream_t s, const int32_t* src, int32_t* dst, int64_t T, int64_t E, const ReplicaMap& m);
void permute_rows_f64(cudaStream_t s, const double* src, double* dst, int64_t T, int64_t E, const ReplicaMap& m);
void exact_grad_mean(cudaStream_t s, const float* gathered, int k, int64_t P, double* mean);
void begin_episode(cudaStream_t s, DeviceCtx* ctx);  // ctx->episode = ctx->next_episode++
// Engine::init_params: params[woff[l] + i] = f32(U(-a[l], a[l]) keyed (seed, kParamStream,
// node[l], i)) for i < n[l], every other parameter 0; m, v (if given) zeroed. One launch.
struct XavierTable {
    int count;
    int64_t woff[16], n[16];
    uint64_t node[16];
    double a[16];
};
void param_init(cudaStream_t s, const XavierTable& t, float* params, int64_t P, double* m, double* v,
                uint64_t seed);
// rsum[0, n) -> ring[(ctx->runs % slots) * n, +n) (host-mapped), then ++ctx->runs
void publish_rsum(cudaStream_t s, DeviceCtx* ctx, const double* rsum, int n, double* ring, int slots);
void adam_tick(cudaStream_t s, DeviceCtx* ctx, const double2* bc_table, int64_t table_len);
void exact_adam(cudaStream_t s, const DeviceCtx* ctx, float* params, const float* g32, const double* g64, double* m,
                double* v, int64_t P, double lr, double b1, double b2, double eps, double gscale = 1.0);

}  // namespace flw
