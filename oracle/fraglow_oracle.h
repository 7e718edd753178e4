/* fraglow_oracle: CPU restatement of the reference DP-D unit (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library, and only as the checker. The product (paper_2210_00882_b200) never links it.
 *
 * Semantics follow /root/reference/proj (cited per function in fraglow_oracle.c): every
 * tensor value is an f32-representable double ("store" rounds through float,
 * core/tensor.hpp:74-79); reductions accumulate left-to-right in double from 0.0; the RNG is
 * splitmix64-keyed (core/rng.hpp:12-38). Pinned against the reference itself: see
 * tests/golden/make_golden.py and tests/test_oracle_golden.py. */
#ifndef FRAGLOW_ORACLE_H
#define FRAGLOW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_PPO = 0, ORC_A3C = 1, ORC_MAPPO = 2 };
enum { ORC_GRIDLINE = 0, ORC_SYNTH17X6 = 1, ORC_SPREAD = 2 };

typedef struct {
    int32_t algo;
    int32_t env;
    int32_t n_agents;     /* MAPPO agents (spread_lite n_agents); 1 otherwise */
    int32_t activation;   /* 0 tanh, 1 relu */
    int32_t n_hidden;
    int32_t hidden[8];
    int32_t normalize_adv;
    int64_t steps_per_episode;
    int64_t train_iters;
    int64_t max_steps;    /* env param max_steps (0: none) */
    double env_length;    /* gridline param length (default 8) */
    double gamma, lam, clip_eps, lr, value_coef, entropy_coef;
} orc_cfg;

typedef struct orc_unit orc_unit;

uint64_t orc_mix(uint64_t x);
uint64_t orc_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d);
double orc_uniform(uint64_t k);

orc_unit* orc_unit_new(const orc_cfg* cfg, uint64_t seed, int64_t env_lo, int64_t env_hi, int64_t env_total);
void orc_unit_free(orc_unit* u);
int64_t orc_param_count(const orc_unit* u);
int64_t orc_learn_iters(const orc_unit* u);
void orc_get_params(const orc_unit* u, double* out);
void orc_set_params(orc_unit* u, const double* in);

void orc_reset(orc_unit* u, int64_t ep);
void orc_step(orc_unit* u, int64_t ep, int64_t st);
double orc_reward_sum(const orc_unit* u);
int64_t orc_steps(const orc_unit* u);
/* One train iteration up to the flat f32 gradient (GradCompute); grads_out may be NULL. */
int orc_learn_grads(orc_unit* u, int64_t ep, int64_t k, double* grads_out);
/* OptimStep on an already-synchronised gradient (interp.cpp:368-387). */
void orc_apply_grads(orc_unit* u, const double* grads);
void orc_learn(orc_unit* u, int64_t ep, int64_t k);

/* Named tensors of the last evaluation: reset_obs, state_in, logits, pa, envstep, sample,
 * values, last_value, adv, ret, logits_new, loss, grads, dlogits. -1 if unknown/empty. */
int64_t orc_size(const orc_unit* u, const char* name);
int orc_get(const orc_unit* u, const char* name, double* out);
/* Teacher forcing: state_in (next step's policy input) and sample (the learn batch). */
int orc_set(orc_unit* u, const char* name, const double* in, int64_t n);

/* DP-D plan with k replicas over contiguous env ranges (plan.cpp:46-55,365-411) and the
 * GradSync ordered mean (local_run.cpp:379-414); returns 0 on success. */
int orc_run(const orc_cfg* cfg, uint64_t seed, int64_t env_total, int32_t k, int64_t episodes,
            double* episode_rewards, double* final_params, int64_t* steps_out);

/* Kernel-level restatements used directly by tests. */
void orc_gae_streams(const double* r, const double* v, const double* d, const double* lv, int64_t n,
                     int64_t streams, double gamma, double lam, double* out);
void orc_returns_streams(const double* r, const double* d, const double* lv, int64_t n, int64_t streams,
                         double gamma, double* out);
void orc_normalize(double* a, int64_t n);
void orc_adam(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr, double b1,
              double b2, double eps);
double orc_ppo_loss(const double* logits, const double* values, const double* actions, const double* logp_old,
                    const double* adv, const double* ret, int64_t n, int64_t a_dim, double clip_eps,
                    double value_coef, double entropy_coef, double* dlogits, double* dvalues);

#ifdef __cplusplus
}
#endif
#endif
