/* fraglow_b200: B200-native engine for the GPU-only distribution policy (DP-D) of fraglow
 * (the reference's MSRL re-implementation, /root/reference/proj).
 *
 * Two surfaces, both plain C (no torch or CUDA types), implemented in libfraglow_b200.so:
 *
 *  1. The reference's public API for the DP-D path, same names / argument meaning / error
 *     codes / string ownership as /root/reference/proj/include/fraglow.h. A program whose
 *     deploy config selects "dp-d" (alias "GPU_only") runs its fused training loop on B200s:
 *     one unit (replica) per accelerator slot = per GPU, gradients averaged over NVLink.
 *
 *  2. The engine seam the reference's run_unit (/root/reference/proj/src/run/local_run.cpp:367-501)
 *     would call per unit: flw_dpd_*. It also exposes phase-level entry points and named
 *     tensors so parity tests can drive it step by step against the reference oracle.
 *
 * Conventions (capi.cpp:14-60 in the reference): functions return 0 or an error code;
 * flw_last_error() describes the failure for the calling thread; out strings are malloc'd and
 * released with flw_string_free(); exceptions never cross the ABI. */
#ifndef FRAGLOW_B200_H
#define FRAGLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- reference API (DP-D) */

typedef struct flw_program flw_program;

enum {
    FLW_OK = 0,
    FLW_ERR_CONFIG = 2,  /* bad configuration or policy not applicable (fraglow.h:19) */
    FLW_ERR_RUNTIME = 3, /* execution failure (fraglow.h:20) */
    FLW_ERR_BIND = 4,    /* (fraglow.h:21; unused by the DP-D engine) */
    FLW_ERR_CHECK = 5    /* (fraglow.h:22; unused by the DP-D engine) */
};

enum {
    FLW_DUMP_DFG = 0, /* fraglow.h:26-29; only FLW_DUMP_PLAN is served by the engine */
    FLW_DUMP_FDG = 1,
    FLW_DUMP_PLAN = 2,
    FLW_DUMP_DOT = 3
};

/* Same layout and meaning as fraglow.h:32-39. latency_us is accepted and ignored (no TCP legs
 * on a single NVSwitch node); unpartitioned runs the whole env range as one unit (== DP-D k=1). */
typedef struct {
    uint64_t seed;
    int64_t episodes;        /* 0: take from the algorithm config */
    int64_t latency_us;
    int64_t timeout_ms;      /* 0: default (30 s) */
    double reward_threshold; /* <0: no threshold tracking */
    int unpartitioned;
} flw_run_options;

/* Replaces fraglow.h:43 / capi.cpp:207-219 for dp-d. Parses and validates both documents
 * (config.cpp:24-103) and builds the DP-D placement (plan.cpp:308-417). Non-dp-d policies and
 * envs without an accelerator implementation fail with FLW_ERR_CONFIG ("PolicyInapplicable: ..."). */
int flw_program_create(const char* algo_json, const char* deploy_json, flw_program** out);
void flw_program_destroy(flw_program* p);                              /* fraglow.h:44 */
int flw_program_dump(const flw_program* p, int what, char** out_text); /* fraglow.h:46 */
/* The seam's graph input: the dataflow graph JSON a reference worker receives
 * (dfg::dump_json, graph.cpp:468-507; coordinator.cpp:75-84) of a PPO / MAPPO standard program
 * -> the equivalent algo JSON (free with flw_string_free). flw_dpd_create and
 * flw_dpd_create_replicas accept either JSON directly. */
int flw_algo_from_graph(const char* graph_json, char** out_algo_json);
int flw_validate_plan(const flw_program* p, char** out_report, int* n_violations); /* fraglow.h:49 */
/* Replaces fraglow.h:55 / capi.cpp:249-265: runs every unit on its own GPU (one host thread per
 * unit, local_run.cpp:532-535), same CSV schema (episode,wall_ms,reward,bytes_total) and summary
 * JSON keys (capi.cpp:74-113). */
int flw_run_local(const flw_program* p, const flw_run_options* opts, char** metrics_csv, char** summary_json);
void flw_string_free(char* s);     /* fraglow.h:72 */
const char* flw_last_error(void);  /* fraglow.h:73 */

/* ---------------------------------------------------------------- engine seam (per unit) */

typedef struct flw_dpd flw_dpd;

enum { FLW_NUMERICS_EXACT = 0, FLW_NUMERICS_FAST = 1 };

/* One DP-D unit (the reference's Interp over the fused fragment, interp.hpp:34-115) owning envs
 * [env_lo, env_hi) of env_total on CUDA device `device`. */
int flw_dpd_create(const char* algo_json, int device, uint64_t seed, int64_t env_lo, int64_t env_hi,
                   int64_t env_total, int numerics, flw_dpd** out);
/* R consecutive units folded into one engine on one GPU (R > #GPUs replicas):
 * [env_lo, env_hi) is split like split_envs (plan.cpp:46-55); each replica keeps its own
 * advantage statistics, loss mean, gradient and reward sum, and the gradients are averaged in
 * unit order (local_run.cpp:408-411). A gradient group then has R units per rank. */
int flw_dpd_create_replicas(const char* algo_json, int device, uint64_t seed, int64_t env_lo, int64_t env_hi,
                            int64_t env_total, int numerics, int replicas, flw_dpd** out);
/* Per-replica reward sums of the last episode, unit order (exact numerics). */
int flw_dpd_replica_rewards(flw_dpd* e, double* out, int64_t cap);
int flw_dpd_destroy(flw_dpd* e);

/* Gradient group (GradSync, local_run.cpp:379-414): rank 0 creates an id (128 bytes), the
 * caller distributes it, every unit joins with its rank (= unit id). */
int flw_dpd_comm_unique_id(char* out_id, int64_t cap);
int flw_dpd_comm_init(flw_dpd* e, const char* id, int64_t id_len, int rank, int nranks);

/* Fast numerics, one unit per GPU: gradient exchange over NVLink peer memory instead of NCCL
 * (reduce of the per-CTA partials + all-reduce + Adam in one kernel). Every rank exports the
 * CUDA IPC handle (64 bytes) of its exchange region, the caller gathers the k handles in rank
 * order and every rank imports them. */
/* exchange handle: the region's CUDA IPC handle + the exporting GPU's UUID */
#define FLW_P2P_HANDLE_BYTES 80
int flw_dpd_p2p_export(flw_dpd* e, int nranks, char* out_handle, int64_t cap);
int flw_dpd_p2p_import(flw_dpd* e, const char* handles, int64_t len, int rank, int nranks);
/* Back to the NCCL exchange (every rank of the group must make the same choice). */
int flw_dpd_p2p_disable(flw_dpd* e);
/* Bounded group waits (the reference's receive timeouts, local_run.cpp:543-546 / fraglow.h:36):
 * a unit in a gradient group fails its episode / learn call with Timeout (code 3) once it has
 * waited timeout_ms (<= 0: 30 s) for its peers, and aborts the group (NCCL communicator abort +
 * the peer-memory exchange's abort word). flw_dpd_abort aborts the group from the caller
 * (a peer failed); the unit's next waits fail with PeerFailure. Either leaves the unit unusable
 * for further grouped episodes: destroy it. */
int flw_dpd_set_timeout(flw_dpd* e, int64_t timeout_ms);
int flw_dpd_abort(flw_dpd* e);

/* One whole episode (Reset, T x Step, I x Learn) as a replayed CUDA graph. reward_sum is the
 * episode's summed env reward over this unit's envs (interp.cpp:257); device_ms the graph time. */
int flw_dpd_run_episode(flw_dpd* e, int64_t episode, double* reward_sum, float* device_ms);
/* Pipelined episodes: launch_episode enqueues an episode (at most 2 in flight) and returns;
 * finish_episode waits (bounded like run_episode for a unit in a gradient group) for the oldest
 * enqueued one and returns its reward sum. Launching episode e+1 before finishing e overlaps the
 * host's per-episode gate with the GPU (flw_run_local does this on one GPU). */
int flw_dpd_launch_episode(flw_dpd* e, int64_t episode);
int flw_dpd_finish_episode(flw_dpd* e, double* reward_sum);
/* Back-to-back episodes without host synchronisation in between (throughput timing). */
int flw_dpd_run_episodes(flw_dpd* e, int64_t first_episode, int64_t count, float* device_ms);
int flw_dpd_reinit(flw_dpd* e, uint64_t seed);

int flw_dpd_param_count(const flw_dpd* e, int64_t* n);
int flw_dpd_get_params(flw_dpd* e, double* out, int64_t n);
int flw_dpd_set_params(flw_dpd* e, const double* in, int64_t n);
int flw_dpd_stats(const flw_dpd* e, int64_t* steps, int64_t* env_count, int64_t* learn_iters, int64_t* graph_kernels);

/* Phase-level entry points (the reference's Interp::eval_phase per phase, interp.cpp:137-144). */
int flw_dpd_reset(flw_dpd* e, int64_t episode);
int flw_dpd_step(flw_dpd* e, int64_t episode, int64_t step);
int flw_dpd_learn(flw_dpd* e, int64_t episode, int64_t iter);
int flw_dpd_learn_grads(flw_dpd* e, int64_t episode, int64_t iter);
int flw_dpd_apply_grads(flw_dpd* e, const double* grads, int64_t n); /* grads NULL: own f32 grads */

/* Named tensors (reset_obs, state_in, logits, pa, envstep, sample, values, last_value, adv, ret,
 * logits_new, dlogits, loss, grads, env_state), reference row-major layouts, as doubles. */
int flw_dpd_tensor_size(const flw_dpd* e, const char* name, int64_t* n);
int flw_dpd_read(flw_dpd* e, const char* name, double* out, int64_t n);
int flw_dpd_write(flw_dpd* e, const char* name, const double* in, int64_t n);

/* Scaled-size HBM microbenchmark of one element-wise DP-D kernel on the current device:
 * which = "env_step" (n envs), "gae" (n = T*E rows, T=32) or "adam" (n params). Returns the
 * mean ms per launch (CUDA events, after warm-up) and the algorithmic bytes per launch. */
int flw_microbench(const char* which, int64_t n, int iters, double* ms_per_launch, double* bytes_per_launch);

/* Per-kernel device times (ms) of the most recent episode replay, measured by CUDA events
 * captured inside the episode graph; probes are enabled by this call (the graph is rebuilt).
 * JSON object: {"rollout": x, "critic_fwd": [..], "learn_policy": [..], "learn_critic": [..],
 * "gae": [..], "reduce": [..], "adam": [..]}; malloc'd, release with flw_string_free. */
int flw_dpd_enable_probes(flw_dpd* e, int on);
int flw_dpd_probe_times(flw_dpd* e, char** json);

/* Diagnostic (tests only): one tcgen05.mma GEMM D[M,N] = op(A) op(B) through the engine's
 * shared-memory operand convention. a_mn=0: A is [M,K] row-major; a_mn=1: A is stored [K,M].
 * b_mn=0: B is stored [N,K]; b_mn=1: B is [K,N]. lane_off = TMEM lane offset of D (M=64 only). */
int flw_selftest_umma(int M, int N, int K, int a_mn, int b_mn, int lane_off, const float* A, const float* B, float* D);

/* Diagnostic (tests only): D[M,N] = op(A) op(B) through the generic TMA + tcgen05 GEMM of the
 * layer-wise learn path (kernels_tgemm.cu), K split `splits` ways (partials summed on the host).
 * a_mn: A given as [K,M] (else [M,K]); b_mn: B given as [K,N] (else [N,K]); tf32: kind::tf32 on
 * the f32 values, else kind::f16 on their bf16 roundings; bn: N tile (64, 128 or 256). */
int flw_selftest_tgemm(int64_t M, int64_t N, int64_t K, int a_mn, int b_mn, int tf32, int splits, int bn,
                       const float* A, const float* B, float* D);

/* Diagnostic: mean ms per launch of that GEMM for one shape and epilogue (synthetic operands).
 * dt: 0 bf16, 1 f16, 2 f32/tf32; mode: 0 f32 store, 1 bias + tanh -> bf16, 4 f16 hi|lo|hi. */
int flw_bench_tgemm(int64_t M, int64_t N, int64_t K, int dt, int mode, int bn, int iters, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* FRAGLOW_B200_H */
