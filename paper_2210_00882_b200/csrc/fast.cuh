// Fast-numerics (tensor-core learn phase, f32 rollout) kernel interfaces.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "envs.cuh"

namespace flw {

constexpr int kMaxLayers = 8;

enum NetKind : int { kNetPolicyPpo = 0, kNetPolicyA3c = 1, kNetCritic = 2 };

struct FastNet {                       // one MLP, dims padded to multiples of 16 (<= 64)
    int L;
    int din[kMaxLayers], dout[kMaxLayers];   // padded
    int rin[kMaxLayers], rout[kMaxLayers];   // real
    int64_t woff[kMaxLayers], boff[kMaxLayers];  // offsets in the flat parameter vector
};

struct FastLearnArgs {
    FastNet net;
    int kind;            // NetKind
    int mode;            // 0: forward only (values_out), 1: learn (partials)
    int act;             // 0 tanh, 1 relu
    const float* params; // flat f32 parameters
    const float* X;      // input rows [rows, in_cols]
    int in_cols;
    int64_t rows;
    // per-row learn inputs
    const int32_t* actions;
    const float* logp_old;
    const float* adv;          // raw GAE advantages (normalised on the fly with adv_stats)
    const double* adv_stats;   // {mean, sd} or null (no normalisation)
    const float* ret;
    const float* values_in;    // critic values (A3C advantage)
    float* values_out;         // mode 0: rows [0, split_rows)
    float* values_out2;        // mode 0: rows [split_rows, rows) (when split_rows >= 0)
    int64_t split_rows;
    const __nv_bfloat16* wimg; // pre-built shared-memory image of the weight tiles (bf16)
    // Critic activation reuse: mode 0 stores each tile's hidden-activation tiles (the exact
    // shared-memory bytes, bf16) for tiles < save_tiles; mode 1 with hload set skips the
    // forward pass and bulk-copies them back (values come from values_in).
    uint8_t* hsave;
    int64_t save_tiles;
    int hload;
    uint8_t* hscratch;         // k_learn: per (CTA, group) activation scratch [grid * groups][hbytes]
    // R > 1 replicas folded into the unit: row -> replica via env (row % rep_E); per-replica row
    // weight (1 / (R * T * E_r)) replaces inv_n and adv_stats is indexed [replica][2]
    const int32_t* rep_of_env;
    const float* rep_w;
    int64_t rep_E;
    // learn mode: also write dZ wrt the input pre-activation, dH_0 * act'(X) (X = the input rows
    // are activations of an outer layer): f32 [rows, in_cols]. The MAPPO compact critic uses it.
    float* dx_out;
    double inv_n, value_coef, entropy_coef;
    float clip_eps;
    float* partials;           // [grid, part_stride]
    int64_t part_stride;       // = parameter count of this net
    float* loss_partials;      // [grid, 3]
    // launched as a programmatic dependent of the kernel before it on the stream (the update):
    // the setup runs, then griddepcontrol.wait before the weight image and the biases are read
    int pdl = 0;
};

size_t fast_wimg_bytes(const FastNet& n);  // bytes of the weight-tile image (smem prefix)
size_t fast_hsave_bytes(const FastNet& n); // bytes of one tile's saved tiles (X, hidden activations)
// Builds the bf16 W^T tile image of one net from the f32 params (once per train iteration,
// shared by every CTA of the critic-forward / learn kernels that follow).
void fast_build_wimg(cudaStream_t s, const float* params, const FastNet& n0, __nv_bfloat16* img0, const FastNet& n1,
                     __nv_bfloat16* img1);  // both nets in one launch
// Warp-specialised two-tiles-per-SM learn kernel (kernels_learn.cu): mode 0 values pass,
// mode 1 one train iteration of one net.
void fast_learn(cudaStream_t s, const FastLearnArgs& a, int grid);
size_t fast_learn_smem_bytes(const FastNet& n);
size_t fast_learn_scratch_bytes(const FastNet& n);  // hidden bytes of one 128-row tile
int fast_learn_groups();   // tiles in flight per k_learn CTA (learn modes)
int fast_values_groups();  // ... in the values pass (forward only)
// fixed-order sums of the per-CTA partial slots: np policy slots, nc critic slots
// Element index of flat parameter p (absolute, params layout) in its net's bf16 weight-tile image
// (W_l^T as [dout x din] K-major core-matrix tiles at 128-byte aligned per-layer offsets, the
// layout k_build_wimg writes), or -1 when p is not a weight of this net.
__host__ __device__ inline int64_t wimg_elem(const FastNet& n, int64_t p) {
    uint32_t off = 0;
    for (int l = 0; l < n.L; ++l) {
        const int64_t r = p - n.woff[l];
        if (r >= 0 && r < static_cast<int64_t>(n.rin[l]) * n.rout[l]) {
            const int c = static_cast<int>(r / n.rout[l]), o = static_cast<int>(r % n.rout[l]), C = n.din[l];
            const uint32_t t = static_cast<uint32_t>((o >> 3) * (C * 16) + (c >> 3) * 128 + (o & 7) * 16 + (c & 7) * 2);
            return static_cast<int64_t>((off + t) / 2);
        }
        off = (off + static_cast<uint32_t>(n.dout[l] * n.din[l] * 2) + 127u) / 128u * 128u;
    }
    return -1;
}

struct DeviceCtx;
struct FastUpdateArgs {      // k_reduce_adam: partial reduction + Adam + weight image, one launch
    const float *pp, *pc;    // per-CTA dW partials of the policy / critic learn kernels
    int np, nc;
    int64_t Pp, Pc;          // policy / critic parameter counts (critic follows the policy)
    DeviceCtx* ctx;          // Adam step counter and bias corrections
    const double2* bc_table;
    int64_t bc_len;
    float* params;
    float* grads;            // the reduced gradient (kept for read-back)
    double *m, *v;
    double lr, b1, b2, eps;
    FastNet pol, crit;
    __nv_bfloat16 *img_p, *img_c;
    unsigned* counter;       // zero between launches
    // split update (the critic's update runs as soon as the critic learn finishes, while the
    // policy learn still runs): a launch over one net only - off = its first flat parameter,
    // critic_only = the rows are critic parameters; advance = this launch advances the Adam
    // step counter (the iteration's last launch)
    int64_t off = 0;
    bool critic_only = false;
    bool advance = true;
};
// pdl: a programmatic dependent launch of the preceding learn kernel (same stream)
void fast_reduce_adam(cudaStream_t s, const FastUpdateArgs& a, bool pdl = false);
void fast_reduce_partials(cudaStream_t s, const float* part_p, const float* part_c, int np, int nc, int64_t Pp,
                          int64_t Pc, float* grads, int64_t c_off = 0);  // critic slots land at Pp + c_off
// MAPPO compact critic (fast numerics, n > 4): layer-0 rows from the joint GEMM P, and the
// layer-0 gradients (per-env agent sums S for the joint GEMM, one-hot rows, bias) from dz0.
void mappo_fast_h0(cudaStream_t s, const float* P, const float* W0, const float* b0, int64_t blocks, int64_t E, int n,
                   int J, int H, int act, float* h0);
void mappo_fast_layer0_grads(cudaStream_t s, const float* dz0, int64_t T, int64_t E, int n, int H, float* S,
                             float* part, float* gWoh, float* gb0);  // part: scratch [T, n, H]
void fast_reduce_loss(cudaStream_t s, const float* loss_parts, int np, int nc, double entropy_coef, float* loss);
void fast_gae(cudaStream_t s, const float* rew, const float* values, const float* done_f, const float* last_value,
              int64_t TR, int64_t R, double gamma, double lam, float* adv, float* ret, bool with_adv,
              double* block_sums, double* stats, unsigned* done_counter = nullptr,  // counter: fused stats
              bool pdl = false);  // k_gae_scan32 as a programmatic dependent of the values pass
// k_gae_scan32 for any stream count (T = 32), persistent over 32-stream tiles (microbenchmarks)
void fast_gae_scan32(cudaStream_t s, const float* rew, const float* values, const float* done_f,
                     const float* last_value, int64_t R, double gamma, double lam, float* adv, float* ret,
                     bool with_adv, double* block_sums, double* stats, unsigned* done_counter);
void fast_sum(cudaStream_t s, const double* x, int64_t n, double* scratch, double* out);
void fast_rep_adv_stats(cudaStream_t s, const float* adv, int64_t T, int64_t E, const int64_t* rep_off,
                        const int64_t* rep_n, int R, double* stats);

struct FastRolloutArgs {     // whole-episode rollout, all T steps in one launch
    const float* params;     // policy params (flat, reference layout)
    int L;
    int dims[kMaxLayers + 1];
    int64_t woff[kMaxLayers], boff[kMaxLayers];
    int act;
    double* est;
    uint8_t* done;
    int32_t* stepc;
    float* states;           // [(T+1), E, S]
    int32_t* actions;        // [T, E]
    float *logp, *reward, *done_f;
    double* reward_d;
    int64_t E, env_lo;
    int64_t step0, nsteps;   // steps [step0, step0 + nsteps) of the episode
    int S, A;
    uint64_t seed;
    EnvParams env;
    // MAPPO (spread_lite): agent-major rows a*E + e; the step-block layouts of kernels_mappo.cu
    int64_t env_total;
    float *joint, *cin;      // cin: null with the compact critic
};

struct DeviceCtx;
size_t fast_rollout_smem_bytes(const FastRolloutArgs& a);
void fast_rollout(cudaStream_t s, const DeviceCtx* ctx, const FastRolloutArgs& a);
// MAPPO fused fast rollout (n <= 16 agents, hidden <= 64); false: shape not supported
bool fast_rollout_mappo_ok(const FastRolloutArgs& a);
void fast_rollout_mappo(cudaStream_t s, const DeviceCtx* ctx, const FastRolloutArgs& a);

}  // namespace flw
