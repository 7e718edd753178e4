/* fraglow_oracle.c -- CPU restatement of the reference DP-D unit. TEST INFRASTRUCTURE ONLY:
 * the checker for the B200 engine, never part of the product path. Build flags
 * (oracle/Makefile): -O2 -ffp-contract=off, plain IEEE double, glibc libm, like the
 * reference's g++ -O2 build (proj/CMakeLists.txt:11).
 *
 * Citations are /root/reference/proj/<file>:<line>. Parity status: pinned bit-exactly to the
 * reference itself (tests/golden/*.npz produced by oracle/_ref/ref_tool; see
 * tests/test_oracle_golden.py). */
#include "fraglow_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng (core/rng.hpp:12-38) */
uint64_t orc_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t orc_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    uint64_t h = orc_mix(seed);
    h = orc_mix(h ^ a);
    h = orc_mix(h ^ b);
    h = orc_mix(h ^ c);
    h = orc_mix(h ^ d);
    return h;
}

double orc_uniform(uint64_t k) { return (double)(k >> 11) * (1.0 / 9007199254740992.0); }

static double uniform_range(uint64_t k, double lo, double hi) { return lo + (hi - lo) * orc_uniform(k); }

/* Tensor::store for F32/I64/Bool (core/tensor.hpp:74). */
static double f32(double v) { return (double)(float)v; }

/* stream tags: interp.cpp:15-17, envs.cpp:13 */
#define K_PARAM 0x706172ULL
#define K_ACTION 0x616374ULL
#define K_ENV 0x656e76ULL
#define K_RESET 0x7265736574ULL
/* builder env synth17x6 (oracle/refx/synth_env.hpp) */
#define SYN_OBS 17
#define SYN_ACT 6
#define SYN_DT 0.05
#define SYN_C 0.3
#define SYN_D 0.5
#define SYN_BOUND 2.0
#define SYN_TABLE 0x73796eULL

#define MAXL 10

struct orc_unit {
    orc_cfg c;
    uint64_t seed;
    int64_t lo, hi, etot, E;
    int n_ag, s_dim, A, state_w, joint, L, sw; /* sw: env state width */
    int64_t rows; /* policy rows per step */
    int pdims[MAXL + 1], cdims[MAXL + 1];
    int64_t woff[2][MAXL], boff[2][MAXL];
    int64_t P;
    double* params;
    double *m, *v;
    int64_t t;
    int adam_ready;
    /* env group (interp.cpp:204-262) */
    double* est;
    int64_t* step_count;
    unsigned char* done;
    double* last_obs;
    double reward_sum;
    int64_t steps;
    double *state_in, *reset_obs, *logits, *pa, *envstep;
    /* buffer (interp.cpp:263-307) */
    int width;
    double* blocks;
    int64_t nblocks;
    double* sample;
    int64_t cached_ep;
    /* learn byproducts */
    double *values, *last_value, *adv, *ret, *logits_new, *dlogits, *grads;
    double loss;
};

/* -------------------------------------------------------------------------------- envs */
static double synth_b(int a, int i) { return uniform_range(orc_key(SYN_TABLE, (uint64_t)a, (uint64_t)i, 0, 0), -1.0, 1.0); }

/* observation of env e into obs[0..state_w) */
static void env_observe(const orc_unit* u, int64_t e, double* obs) {
    const double* s = u->est + e * u->sw;
    if (u->c.env == ORC_GRIDLINE) { /* envs.cpp:33-36 */
        obs[0] = s[0] / (s[1] - 1.0);
    } else if (u->c.env == ORC_SYNTH17X6) {
        for (int i = 0; i < SYN_OBS; ++i) obs[i] = s[i];
    } else { /* spread_lite observe, envs.cpp:96-109 */
        int n = u->n_ag, k = 0;
        for (int a = 0; a < n; ++a) {
            obs[k++] = s[2 * a];
            obs[k++] = s[2 * a + 1];
            for (int l = 0; l < n; ++l) {
                obs[k++] = s[2 * n + 2 * l] - s[2 * a];
                obs[k++] = s[2 * n + 2 * l + 1] - s[2 * a + 1];
            }
        }
    }
}

/* env_reset (envs.cpp:181-194) with seed = key(seed, kEnvStream, env_lo+e, ep) (interp.cpp:214) */
static void env_reset(orc_unit* u, int64_t e, uint64_t env_seed) {
    double* s = u->est + e * u->sw;
    if (u->c.env == ORC_GRIDLINE) { /* envs.cpp:26-31 */
        int64_t len = (int64_t)u->c.env_length;
        int64_t start = (int64_t)(orc_uniform(orc_key(env_seed, K_RESET, 0, 0, 0)) * (double)(len / 2));
        s[0] = (double)start;
        s[1] = (double)len;
    } else if (u->c.env == ORC_SYNTH17X6) {
        for (int i = 0; i < SYN_OBS; ++i) s[i] = uniform_range(orc_key(env_seed, K_RESET, 0, (uint64_t)i, 0), -0.1, 0.1);
    } else { /* envs.cpp:88-94 */
        for (int i = 0; i < 4 * u->n_ag; ++i) s[i] = uniform_range(orc_key(env_seed, K_RESET, 0, (uint64_t)i, 0), -1.0, 1.0);
    }
    u->step_count[e] = 0;
    u->done[e] = 0;
}

/* env_step (envs.cpp:196-222 and the per-env step bodies); rewards[n_ag], returns done */
static int env_step(orc_unit* u, int64_t e, const int64_t* acts, double* rewards, double* reward_total) {
    double* s = u->est + e * u->sw;
    int done = 0;
    int64_t ms = u->c.max_steps;
    if (u->c.env == ORC_GRIDLINE) { /* envs.cpp:38-53 */
        int64_t len = (int64_t)s[1], x = (int64_t)s[0];
        double r = 0.0;
        x += acts[0] == 1 ? 1 : -1;
        if (x < 0) x = 0;
        if (x > len - 1) x = len - 1;
        s[0] = (double)x;
        if (x == len - 1) {
            r = 1.0;
            done = 1;
        }
        if (ms > 0 && u->step_count[e] + 1 >= ms) done = 1;
        rewards[0] = r;
        *reward_total = r;
    } else if (u->c.env == ORC_SYNTH17X6) { /* oracle/refx/env_ext.cpp */
        double old[SYN_OBS], sq = 0.0, mx = 0.0;
        for (int i = 0; i < SYN_OBS; ++i) old[i] = s[i];
        for (int i = 0; i < SYN_OBS; ++i) {
            double t1 = SYN_C * old[(i + 1) % SYN_OBS];
            double t2 = SYN_D * old[i];
            double t3 = t1 - t2;
            double t4 = t3 + synth_b((int)acts[0], i);
            double t5 = SYN_DT * t4;
            s[i] = old[i] + t5;
        }
        for (int i = 0; i < SYN_OBS; ++i) {
            double n = s[i];
            sq = sq + n * n;
            double m = n < 0.0 ? -n : n;
            if (m > mx) mx = m;
        }
        double r = 1.0 - sq / (double)SYN_OBS;
        done = mx > SYN_BOUND || (ms > 0 && u->step_count[e] + 1 >= ms);
        rewards[0] = r;
        *reward_total = r;
    } else { /* spread_lite, envs.cpp:111-148 */
        int n = u->n_ag;
        const double move = 0.1, collide_radius = 0.1, collide_penalty = 0.5;
        for (int a = 0; a < n; ++a) {
            double dx = 0, dy = 0;
            switch (acts[a]) {
                case 1: dx = move; break;
                case 2: dx = -move; break;
                case 3: dy = move; break;
                case 4: dy = -move; break;
                default: break;
            }
            s[2 * a] += dx;
            s[2 * a + 1] += dy;
        }
        double total = 0.0;
        for (int a = 0; a < n; ++a) {
            double best = 1e18;
            for (int l = 0; l < n; ++l) {
                double dx = s[2 * n + 2 * l] - s[2 * a];
                double dy = s[2 * n + 2 * l + 1] - s[2 * a + 1];
                double dist = sqrt(dx * dx + dy * dy);
                best = dist < best ? dist : best;
            }
            rewards[a] = -best;
            for (int b = 0; b < n; ++b) {
                if (b == a) continue;
                double dx = s[2 * b] - s[2 * a];
                double dy = s[2 * b + 1] - s[2 * a + 1];
                if (sqrt(dx * dx + dy * dy) < collide_radius) rewards[a] -= collide_penalty;
            }
            total += rewards[a];
        }
        done = ms > 0 && u->step_count[e] + 1 >= ms;
        *reward_total = total;
    }
    u->step_count[e] += 1;
    u->done[e] = (unsigned char)done;
    return done;
}

/* --------------------------------------------------------------------------- unit setup */
static void* zalloc(size_t n) { return calloc(n ? n : 1, 1); }

orc_unit* orc_unit_new(const orc_cfg* cfg, uint64_t seed, int64_t env_lo, int64_t env_hi, int64_t env_total) {
    orc_unit* u = (orc_unit*)zalloc(sizeof(orc_unit));
    u->c = *cfg;
    if (u->c.env_length <= 0) u->c.env_length = 8; /* envs.cpp:24 */
    u->seed = seed;
    u->lo = env_lo;
    u->hi = env_hi;
    u->etot = env_total;
    u->E = env_hi - env_lo;
    u->n_ag = cfg->algo == ORC_MAPPO ? cfg->n_agents : 1;
    if (cfg->env == ORC_GRIDLINE) {
        u->s_dim = 1, u->A = 2, u->sw = 2;
    } else if (cfg->env == ORC_SYNTH17X6) {
        u->s_dim = SYN_OBS, u->A = SYN_ACT, u->sw = SYN_OBS;
    } else {
        u->s_dim = 2 + 2 * cfg->n_agents, u->A = 5, u->sw = 4 * cfg->n_agents;
    }
    u->state_w = u->n_ag * u->s_dim;
    u->joint = u->state_w + u->n_ag;
    u->rows = (int64_t)u->n_ag * u->E;
    u->L = cfg->n_hidden + 1;
    /* programs.cpp:204-214 (PPO/A3C), 349-363 (MAPPO): policy [s, hidden..., A]; critic [s or
     * joint, hidden..., 1] */
    u->pdims[0] = u->s_dim;
    u->cdims[0] = cfg->algo == ORC_MAPPO ? u->joint : u->s_dim;
    for (int l = 0; l < cfg->n_hidden; ++l) u->pdims[l + 1] = u->cdims[l + 1] = cfg->hidden[l];
    u->pdims[u->L] = u->A;
    u->cdims[u->L] = 1;
    int64_t off = 0;
    for (int net = 0; net < 2; ++net) {
        const int* d = net == 0 ? u->pdims : u->cdims;
        for (int l = 0; l < u->L; ++l) {
            u->woff[net][l] = off;
            off += (int64_t)d[l] * d[l + 1];
            u->boff[net][l] = off;
            off += d[l + 1];
        }
    }
    u->P = off;
    u->params = (double*)zalloc(sizeof(double) * u->P);
    /* Param init, interp.cpp:71-85: node id of W_l is 2l (policy) / 2L+2l (critic), ids follow
     * make_mlp_params order (programs.cpp:42-54); biases zero. */
    for (int net = 0; net < 2; ++net) {
        const int* d = net == 0 ? u->pdims : u->cdims;
        for (int l = 0; l < u->L; ++l) {
            uint64_t node = (uint64_t)(net * 2 * u->L + 2 * l);
            double a = sqrt(6.0 / ((double)d[l] + (double)d[l + 1]));
            int64_t n = (int64_t)d[l] * d[l + 1];
            for (int64_t i = 0; i < n; ++i)
                u->params[u->woff[net][l] + i] = f32(uniform_range(orc_key(seed, K_PARAM, node, (uint64_t)i, 0), -a, a));
        }
    }
    u->m = (double*)zalloc(sizeof(double) * u->P);
    u->v = (double*)zalloc(sizeof(double) * u->P);
    u->est = (double*)zalloc(sizeof(double) * u->E * u->sw);
    u->step_count = (int64_t*)zalloc(sizeof(int64_t) * u->E);
    u->done = (unsigned char*)zalloc(u->E);
    u->last_obs = (double*)zalloc(sizeof(double) * u->E * u->state_w);
    u->state_in = (double*)zalloc(sizeof(double) * u->E * u->state_w);
    u->reset_obs = (double*)zalloc(sizeof(double) * u->E * u->state_w);
    u->logits = (double*)zalloc(sizeof(double) * u->rows * u->A);
    u->pa = (double*)zalloc(sizeof(double) * u->rows * 2);
    u->envstep = (double*)zalloc(sizeof(double) * u->E * (u->state_w + u->n_ag + 1));
    u->width = cfg->algo == ORC_MAPPO ? u->s_dim + 4 + 2 * u->joint : 2 * u->s_dim + 4;
    int64_t T = cfg->steps_per_episode, tr = T * u->rows;
    u->blocks = (double*)zalloc(sizeof(double) * tr * u->width);
    u->sample = (double*)zalloc(sizeof(double) * tr * u->width);
    u->cached_ep = -1;
    u->values = (double*)zalloc(sizeof(double) * tr);
    u->last_value = (double*)zalloc(sizeof(double) * u->rows);
    u->adv = (double*)zalloc(sizeof(double) * tr);
    u->ret = (double*)zalloc(sizeof(double) * tr);
    u->logits_new = (double*)zalloc(sizeof(double) * tr * u->A);
    u->dlogits = (double*)zalloc(sizeof(double) * tr * u->A);
    u->grads = (double*)zalloc(sizeof(double) * u->P);
    return u;
}

void orc_unit_free(orc_unit* u) {
    if (!u) return;
    double* bufs[] = {u->params, u->m,      u->v,          u->est,    u->last_obs, u->state_in, u->reset_obs,
                      u->logits, u->pa,     u->envstep,    u->blocks, u->sample,   u->values,   u->last_value,
                      u->adv,    u->ret,    u->logits_new, u->dlogits, u->grads};
    for (size_t i = 0; i < sizeof(bufs) / sizeof(bufs[0]); ++i) free(bufs[i]);
    free(u->step_count);
    free(u->done);
    free(u);
}

int64_t orc_param_count(const orc_unit* u) { return u->P; }
/* interp.cpp:127-135: PPO/MAPPO carry train_iters on GradCompute/OptimStep; A3C does not. */
int64_t orc_learn_iters(const orc_unit* u) { return u->c.algo == ORC_A3C ? 1 : u->c.train_iters; }
void orc_get_params(const orc_unit* u, double* out) { memcpy(out, u->params, sizeof(double) * u->P); }
void orc_set_params(orc_unit* u, const double* in) {
    for (int64_t i = 0; i < u->P; ++i) u->params[i] = f32(in[i]);
}
double orc_reward_sum(const orc_unit* u) { return u->reward_sum; }
int64_t orc_steps(const orc_unit* u) { return u->steps; }

/* ---------------------------------------------------------------------------------- MLP */
/* apply_mlp (programs.cpp:56-72) evaluated by ops::matmul (ops.cpp:75-106), ops::add
 * (ops.cpp:28-47) and ops::tanh/relu (ops.cpp:63-73); each op output rounded to f32.
 * H[l] receives layer l's output ([M, d[l+1]]): post-activation, or the Add output for the
 * last layer. */
static void mlp_forward(const orc_unit* u, int net, const double* X, int64_t M, double** H) {
    const int* d = net == 0 ? u->pdims : u->cdims;
    const double* in = X;
    for (int l = 0; l < u->L; ++l) {
        int K = d[l], N = d[l + 1];
        const double* W = u->params + u->woff[net][l];
        const double* b = u->params + u->boff[net][l];
        double* out = H[l];
        for (int64_t i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double acc = 0.0;
                for (int t = 0; t < K; ++t) acc += in[i * K + t] * W[(int64_t)t * N + j];
                double z = f32(acc);
                double za = f32(z + b[j]);
                double h = za;
                if (l + 1 < u->L) h = u->c.activation == 0 ? f32(tanh(za)) : (za > 0 ? za : 0.0);
                out[i * N + j] = h;
            }
        in = out;
    }
}

static double** alloc_acts(const orc_unit* u, int net, int64_t M) {
    const int* d = net == 0 ? u->pdims : u->cdims;
    double** H = (double**)zalloc(sizeof(double*) * u->L);
    for (int l = 0; l < u->L; ++l) H[l] = (double*)zalloc(sizeof(double) * M * d[l + 1]);
    return H;
}

static void free_acts(const orc_unit* u, double** H) {
    for (int l = 0; l < u->L; ++l) free(H[l]);
    free(H);
}

/* backward_flat (interp.cpp:392-499) restricted to one MLP: dZ is the adjoint of the last
 * layer's Add output. MatMul -> matmul_grad_rhs/lhs (ops.cpp:213-240), Add -> reduce_to_shape
 * for the bias (ops.cpp:267-277), Tanh -> tanh_grad (ops.cpp:242-246), Relu -> relu_grad
 * (ops.cpp:248-252). Writes f32-rounded dW/db into g at the flat offsets. */
static void mlp_backward(const orc_unit* u, int net, const double* X, int64_t M, double** H, const double* dZtop,
                         double* g) {
    const int* d = net == 0 ? u->pdims : u->cdims;
    int maxw = 0;
    for (int l = 0; l <= u->L; ++l) maxw = d[l] > maxw ? d[l] : maxw;
    double* dz = (double*)zalloc(sizeof(double) * M * maxw);
    double* dh = (double*)zalloc(sizeof(double) * M * maxw);
    memcpy(dz, dZtop, sizeof(double) * M * d[u->L]);
    for (int l = u->L - 1; l >= 0; --l) {
        int K = d[l], N = d[l + 1];
        const double* hin = l == 0 ? X : H[l - 1];
        const double* W = u->params + u->woff[net][l];
        double* dW = g + u->woff[net][l];
        double* db = g + u->boff[net][l];
        for (int t = 0; t < K; ++t)
            for (int j = 0; j < N; ++j) {
                double acc = 0.0;
                for (int64_t i = 0; i < M; ++i) acc += hin[i * K + t] * dz[i * N + j];
                dW[(int64_t)t * N + j] = f32(acc);
            }
        for (int j = 0; j < N; ++j) {
            double acc = 0.0;
            for (int64_t i = 0; i < M; ++i) acc += dz[i * N + j];
            db[j] = f32(acc);
        }
        if (l == 0) break;
        for (int64_t i = 0; i < M; ++i)
            for (int t = 0; t < K; ++t) {
                double acc = 0.0;
                for (int j = 0; j < N; ++j) acc += dz[i * N + j] * W[(int64_t)t * N + j];
                dh[i * K + t] = f32(acc);
            }
        for (int64_t i = 0; i < M * K; ++i) {
            double y = hin[i];
            dz[i] = u->c.activation == 0 ? f32(dh[i] * (1.0 - y * y)) : (y > 0 ? dh[i] : 0.0);
        }
    }
    free(dz);
    free(dh);
}

/* ---------------------------------------------------------------------------------- Reset */
void orc_reset(orc_unit* u, int64_t ep) {
    /* EnvReset, interp.cpp:204-226 */
    for (int64_t e = 0; e < u->E; ++e) {
        uint64_t env_seed = orc_key(u->seed, K_ENV, (uint64_t)(u->lo + e), (uint64_t)ep, 0);
        env_reset(u, e, env_seed);
        double* obs = u->reset_obs + e * u->state_w;
        env_observe(u, e, obs);
        for (int j = 0; j < u->state_w; ++j) obs[j] = f32(obs[j]);
        /* last_obs keeps the unrounded vector (interp.cpp:221) */
        env_observe(u, e, u->last_obs + e * u->state_w);
    }
    u->reward_sum = 0.0;
    /* feedback state_in <- env_reset (local_run.cpp:422-426) */
    memcpy(u->state_in, u->reset_obs, sizeof(double) * u->E * u->state_w);
    u->nblocks = 0;
}

/* ----------------------------------------------------------------------------------- Step */
void orc_step(orc_unit* u, int64_t ep, int64_t st) {
    int64_t E = u->E, R = u->rows;
    int n = u->n_ag, S = u->s_dim, A = u->A, W = u->state_w;
    /* rows_state: MAPPO per-agent Slice + Concat axis 0 (programs.cpp:100-109) */
    double* rs = (double*)zalloc(sizeof(double) * R * S);
    for (int a = 0; a < n; ++a)
        for (int64_t e = 0; e < E; ++e)
            for (int j = 0; j < S; ++j) rs[((int64_t)a * E + e) * S + j] = u->state_in[e * W + a * S + j];
    double** H = alloc_acts(u, 0, R);
    mlp_forward(u, 0, rs, R, H);
    memcpy(u->logits, H[u->L - 1], sizeof(double) * R * A);
    free_acts(u, H);
    /* PolicyApply, interp.cpp:175-203, with ops::softmax (ops.cpp:108-122) */
    for (int64_t r = 0; r < R; ++r) {
        const double* lg = u->logits + r * A;
        double mx = lg[0], p[64], denom = 0.0;
        for (int c = 1; c < A; ++c) mx = lg[c] > mx ? lg[c] : mx;
        for (int c = 0; c < A; ++c) denom += exp(lg[c] - mx);
        for (int c = 0; c < A; ++c) p[c] = f32(exp(lg[c] - mx) / denom);
        int64_t agent = r / E, env = r % E;
        uint64_t global_row = (uint64_t)(agent * u->etot + u->lo + env);
        double uu = orc_uniform(orc_key(u->seed, K_ACTION, (uint64_t)ep, (uint64_t)st, global_row));
        double cum = 0.0;
        int chosen = A - 1;
        for (int a = 0; a < A; ++a) {
            cum += p[a];
            if (uu < cum) {
                chosen = a;
                break;
            }
        }
        u->pa[r * 2] = (double)chosen;
        u->pa[r * 2 + 1] = f32(log(p[chosen] > 1e-30 ? p[chosen] : 1e-30));
    }
    /* EnvStep, interp.cpp:227-262 (absorbing after done, no auto-reset) */
    int ow = W + n + 1;
    for (int64_t e = 0; e < E; ++e) {
        double* out = u->envstep + e * ow;
        if (u->done[e]) {
            for (int j = 0; j < W; ++j) out[j] = f32(u->last_obs[e * W + j]);
            for (int a = 0; a < n; ++a) out[W + a] = 0.0;
            out[W + n] = 1.0;
            continue;
        }
        int64_t acts[64];
        double rew[64], total = 0.0;
        for (int a = 0; a < n; ++a) acts[a] = (int64_t)(u->pa[((int64_t)a * E + e) * 2] + 0.5);
        int d = env_step(u, e, acts, rew, &total);
        double obs[4096];
        env_observe(u, e, obs);
        for (int j = 0; j < W; ++j) out[j] = f32(obs[j]);
        for (int a = 0; a < n; ++a) out[W + a] = f32(rew[a]);
        out[W + n] = d ? 1.0 : 0.0;
        memcpy(u->last_obs + e * W, obs, sizeof(double) * W);
        u->reward_sum += total;
    }
    u->steps += 1;
    /* BufferInsert (interp.cpp:263-286) of the programs.cpp:229-230 / 410-411 field list */
    double* blk = u->blocks + u->nblocks * R * u->width;
    int wd = u->width;
    for (int64_t r = 0; r < R; ++r) {
        int64_t a = r / E, e = r % E;
        double* row = blk + r * wd;
        const double* es = u->envstep + e * ow;
        int c = 0;
        if (u->c.algo != ORC_MAPPO) {
            for (int j = 0; j < S; ++j) row[c++] = u->state_in[e * W + j];
            row[c++] = u->pa[r * 2];
            row[c++] = es[W];
            for (int j = 0; j < S; ++j) row[c++] = es[j];
            row[c++] = es[W + 1];
            row[c++] = u->pa[r * 2 + 1];
        } else {
            for (int j = 0; j < S; ++j) row[c++] = rs[r * S + j];
            row[c++] = u->pa[r * 2];
            row[c++] = es[W + a];
            for (int j = 0; j < W; ++j) row[c++] = u->state_in[e * W + j];
            for (int j = 0; j < n; ++j) row[c++] = j == a ? 1.0 : 0.0;
            for (int j = 0; j < W; ++j) row[c++] = es[j];
            for (int j = 0; j < n; ++j) row[c++] = j == a ? 1.0 : 0.0;
            row[c++] = es[W + n];
            row[c++] = u->pa[r * 2 + 1];
        }
    }
    u->nblocks += 1;
    free(rs);
    /* feedback state_in <- new_state (local_run.cpp:431-441) */
    for (int64_t e = 0; e < E; ++e) memcpy(u->state_in + e * W, u->envstep + e * ow, sizeof(double) * W);
}

/* ------------------------------------------------------------------------------- RL math */
/* gae (rl.cpp:28-47) over gae_streams' t-major interleave (rl.cpp:81-95) */
void orc_gae_streams(const double* r, const double* v, const double* d, const double* lv, int64_t n,
                     int64_t streams, double gamma, double lam, double* out) {
    int64_t T = n / streams;
    for (int64_t s = 0; s < streams; ++s) {
        double acc = 0.0;
        for (int64_t t = T - 1; t >= 0; --t) {
            int64_t i = t * streams + s;
            int done = d[i] > 0.5;
            double next_v = t + 1 < T ? v[i + streams] : lv[s];
            if (done) {
                next_v = 0.0;
                acc = 0.0;
            }
            double delta = r[i] + gamma * next_v - v[i];
            acc = delta + gamma * lam * acc;
            out[i] = acc;
        }
    }
}

/* discounted_return (rl.cpp:14-26) over discounted_return_streams (rl.cpp:66-79) */
void orc_returns_streams(const double* r, const double* d, const double* lv, int64_t n, int64_t streams,
                         double gamma, double* out) {
    int64_t T = n / streams;
    for (int64_t s = 0; s < streams; ++s) {
        double running = lv[s];
        for (int64_t t = T - 1; t >= 0; --t) {
            int64_t i = t * streams + s;
            if (d[i] > 0.5) running = 0.0;
            running = r[i] + gamma * running;
            out[i] = running;
        }
    }
}

/* normalize_advantages (rl.cpp:97-107) */
void orc_normalize(double* a, int64_t n) {
    if (n == 0) return;
    double mean = 0.0;
    for (int64_t i = 0; i < n; ++i) mean += a[i];
    mean /= (double)n;
    double var = 0.0;
    for (int64_t i = 0; i < n; ++i) var += (a[i] - mean) * (a[i] - mean);
    double sd = sqrt(var / (double)n);
    if (sd < 1e-8) return;
    for (int64_t i = 0; i < n; ++i) a[i] = (a[i] - mean) / (sd + 1e-8);
}

/* row_dist (rl.cpp:117-133) */
static double row_dist(const double* lg, int A, double* p, double* logp) {
    double mx = lg[0], denom = 0.0, ent = 0.0;
    for (int j = 1; j < A; ++j) mx = lg[j] > mx ? lg[j] : mx;
    for (int j = 0; j < A; ++j) denom += exp(lg[j] - mx);
    double log_denom = log(denom);
    for (int j = 0; j < A; ++j) {
        logp[j] = lg[j] - mx - log_denom;
        p[j] = exp(logp[j]);
        ent -= p[j] * logp[j];
    }
    return ent;
}

/* ppo_loss_core (rl.cpp:137-172); dlogits f32-rounded (Tensor::set), dvalues double */
double orc_ppo_loss(const double* logits, const double* values, const double* actions, const double* logp_old,
                    const double* adv, const double* ret, int64_t n, int64_t A, double clip_eps,
                    double value_coef, double entropy_coef, double* dlogits, double* dvalues) {
    double inv_n = 1.0 / (double)n;
    double policy_loss = 0.0, value_loss = 0.0, entropy = 0.0;
    double p[64], logp[64];
    for (int64_t i = 0; i < n; ++i) {
        double H = row_dist(logits + i * A, (int)A, p, logp);
        int64_t a = (int64_t)(actions[i] + 0.5); /* interp.cpp:337-339 */
        double ratio = exp(logp[a] - logp_old[i]);
        double lo = ratio > 1.0 - clip_eps ? ratio : 1.0 - clip_eps;
        double clipped = lo < 1.0 + clip_eps ? lo : 1.0 + clip_eps;
        double s1 = ratio * adv[i];
        double s2 = clipped * adv[i];
        policy_loss -= (s1 < s2 ? s1 : s2) * inv_n;
        double dlogp_coef = s1 <= s2 ? -inv_n * ratio * adv[i] : 0.0;
        double verr = values[i] - ret[i];
        value_loss += value_coef * verr * verr * inv_n;
        dvalues[i] = 2.0 * value_coef * verr * inv_n;
        entropy += H * inv_n;
        for (int64_t j = 0; j < A; ++j) {
            double g = dlogp_coef * ((j == a ? 1.0 : 0.0) - p[j]);
            g += (entropy_coef * inv_n) * p[j] * (logp[j] + H);
            dlogits[i * A + j] = f32(g);
        }
    }
    return policy_loss + value_loss - entropy_coef * entropy;
}

/* a3c_loss_core (rl.cpp:174-202) */
static double a3c_loss(const double* logits, const double* values, const double* actions, const double* ret,
                       int64_t n, int64_t A, double value_coef, double entropy_coef, double* dlogits,
                       double* dvalues) {
    double inv_n = 1.0 / (double)n;
    double policy_loss = 0.0, value_loss = 0.0, entropy = 0.0;
    double p[64], logp[64];
    for (int64_t i = 0; i < n; ++i) {
        double H = row_dist(logits + i * A, (int)A, p, logp);
        int64_t a = (int64_t)(actions[i] + 0.5);
        double adv = ret[i] - values[i];
        policy_loss -= logp[a] * adv * inv_n;
        double verr = values[i] - ret[i];
        value_loss += value_coef * verr * verr * inv_n;
        dvalues[i] = 2.0 * value_coef * verr * inv_n;
        entropy += H * inv_n;
        for (int64_t j = 0; j < A; ++j) {
            double g = -inv_n * adv * ((j == a ? 1.0 : 0.0) - p[j]);
            g += (entropy_coef * inv_n) * p[j] * (logp[j] + H);
            dlogits[i * A + j] = f32(g);
        }
    }
    return policy_loss + value_loss - entropy_coef * entropy;
}

/* adam_step (mlp.cpp:480-495), params rounded to f32 */
void orc_adam(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr, double b1,
              double b2, double eps) {
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        double mhat = m[i] / bc1;
        double vhat = v[i] / bc2;
        double next = p[i] - lr * mhat / (sqrt(vhat) + eps);
        p[i] = f32(next);
    }
}

/* ---------------------------------------------------------------------------------- Learn */
int orc_learn_grads(orc_unit* u, int64_t ep, int64_t k, double* grads_out) {
    (void)k;
    int64_t R = u->rows, T = u->c.steps_per_episode, TR = T * R;
    int S = u->s_dim, A = u->A, wd = u->width, n = u->n_ag, W = u->state_w;
    /* BufferSample: t-major concat, cached across the train iterations (interp.cpp:287-307) */
    if (u->cached_ep != ep) {
        if (u->nblocks == 0) return -1;
        memcpy(u->sample, u->blocks, sizeof(double) * u->nblocks * R * wd);
        u->nblocks = 0;
        u->cached_ep = ep;
    }
    /* column slices (programs.cpp:233-243 / 414-425) */
    int cin = u->c.algo == ORC_MAPPO ? u->joint : S;
    int o_act = S, o_rew = S + 1, o_cin = u->c.algo == ORC_MAPPO ? S + 2 : 0;
    int o_next = u->c.algo == ORC_MAPPO ? S + 2 + u->joint : S + 2;
    int o_done = u->c.algo == ORC_MAPPO ? S + 2 + 2 * u->joint : 2 * S + 2;
    int o_logp = o_done + 1;
    double* states = (double*)zalloc(sizeof(double) * TR * S);
    double* cinput = (double*)zalloc(sizeof(double) * TR * cin);
    double *act = (double*)zalloc(sizeof(double) * TR), *rew = (double*)zalloc(sizeof(double) * TR);
    double *don = (double*)zalloc(sizeof(double) * TR), *lpo = (double*)zalloc(sizeof(double) * TR);
    double* last_in = (double*)zalloc(sizeof(double) * R * cin);
    for (int64_t i = 0; i < TR; ++i) {
        const double* row = u->sample + i * wd;
        for (int j = 0; j < S; ++j) states[i * S + j] = row[j];
        for (int j = 0; j < cin; ++j) cinput[i * cin + j] = row[o_cin + j];
        act[i] = row[o_act];
        rew[i] = row[o_rew];
        don[i] = row[o_done];
        lpo[i] = row[o_logp];
    }
    /* last_step_of slice: rows [TR - TR/T, TR) of nexts (interp.cpp:34-45) */
    for (int64_t i = 0; i < R; ++i) {
        const double* row = u->sample + (TR - R + i) * wd;
        for (int j = 0; j < cin; ++j) last_in[i * cin + j] = row[o_next + j];
    }
    (void)n;
    (void)W;
    double** HC = alloc_acts(u, 1, TR);
    mlp_forward(u, 1, cinput, TR, HC);
    memcpy(u->values, HC[u->L - 1], sizeof(double) * TR);
    double** HL = alloc_acts(u, 1, R);
    mlp_forward(u, 1, last_in, R, HL);
    memcpy(u->last_value, HL[u->L - 1], sizeof(double) * R);
    free_acts(u, HL);
    /* GaeAdv (interp.cpp:308-319) and DiscountedReturn (interp.cpp:320-329), outputs f32 */
    if (u->c.algo != ORC_A3C) {
        orc_gae_streams(rew, u->values, don, u->last_value, TR, R, u->c.gamma, u->c.lam, u->adv);
        if (u->c.normalize_adv) orc_normalize(u->adv, TR);
        for (int64_t i = 0; i < TR; ++i) u->adv[i] = f32(u->adv[i]);
    }
    orc_returns_streams(rew, don, u->last_value, TR, R, u->c.gamma, u->ret);
    for (int64_t i = 0; i < TR; ++i) u->ret[i] = f32(u->ret[i]);
    double** HP = alloc_acts(u, 0, TR);
    mlp_forward(u, 0, states, TR, HP);
    memcpy(u->logits_new, HP[u->L - 1], sizeof(double) * TR * A);
    double* dvals = (double*)zalloc(sizeof(double) * TR);
    double loss;
    if (u->c.algo == ORC_A3C)
        loss = a3c_loss(u->logits_new, u->values, act, u->ret, TR, A, u->c.value_coef, u->c.entropy_coef, u->dlogits,
                        dvals);
    else
        loss = orc_ppo_loss(u->logits_new, u->values, act, lpo, u->adv, u->ret, TR, A, u->c.clip_eps, u->c.value_coef,
                            u->c.entropy_coef, u->dlogits, dvals);
    u->loss = f32(loss);
    /* backward_flat: loss adjoint 1.0 -> dlogits*1 and dv = f32(1*dvalues) (interp.cpp:472-483) */
    for (int64_t i = 0; i < TR; ++i) dvals[i] = f32(dvals[i]);
    memset(u->grads, 0, sizeof(double) * u->P);
    mlp_backward(u, 0, states, TR, HP, u->dlogits, u->grads);
    mlp_backward(u, 1, cinput, TR, HC, dvals, u->grads);
    free_acts(u, HP);
    free_acts(u, HC);
    if (grads_out) memcpy(grads_out, u->grads, sizeof(double) * u->P);
    free(states);
    free(cinput);
    free(act);
    free(rew);
    free(don);
    free(lpo);
    free(last_in);
    free(dvals);
    return 0;
}

/* OptimStep (interp.cpp:368-387): lazily initialised Adam with programs.cpp:197-200 attrs */
void orc_apply_grads(orc_unit* u, const double* grads) {
    u->t += 1;
    orc_adam(u->params, grads, u->m, u->v, u->P, u->t, u->c.lr, 0.9, 0.999, 1e-8);
}

void orc_learn(orc_unit* u, int64_t ep, int64_t k) {
    orc_learn_grads(u, ep, k, NULL);
    orc_apply_grads(u, u->grads);
}

/* ------------------------------------------------------------------------ named tensors */
static double* named(const orc_unit* u, const char* name, int64_t* n) {
    int64_t T = u->c.steps_per_episode, R = u->rows, TR = T * R;
#define NM(s, ptr, cnt)            \
    if (strcmp(name, s) == 0) {    \
        *n = (cnt);                \
        return (double*)(ptr);     \
    }
    NM("reset_obs", u->reset_obs, u->E * u->state_w)
    NM("state_in", u->state_in, u->E * u->state_w)
    NM("logits", u->logits, R * u->A)
    NM("pa", u->pa, R * 2)
    NM("envstep", u->envstep, u->E * (u->state_w + u->n_ag + 1))
    NM("sample", u->sample, TR * u->width)
    NM("values", u->values, TR)
    NM("last_value", u->last_value, R)
    NM("adv", u->adv, TR)
    NM("ret", u->ret, TR)
    NM("logits_new", u->logits_new, TR * u->A)
    NM("dlogits", u->dlogits, TR * u->A)
    NM("grads", u->grads, u->P)
    NM("loss", &u->loss, 1)
    NM("env_state", u->est, u->E * u->sw)
#undef NM
    *n = -1;
    return NULL;
}

int64_t orc_size(const orc_unit* u, const char* name) {
    int64_t n;
    named(u, name, &n);
    return n;
}

int orc_get(const orc_unit* u, const char* name, double* out) {
    int64_t n;
    double* p = named(u, name, &n);
    if (!p) return -1;
    memcpy(out, p, sizeof(double) * n);
    return 0;
}

int orc_set(orc_unit* u, const char* name, const double* in, int64_t cnt) {
    int64_t n;
    double* p = named(u, name, &n);
    if (!p || cnt != n) return -1;
    for (int64_t i = 0; i < n; ++i) p[i] = in[i];
    if (strcmp(name, "sample") == 0) u->cached_ep = -2; /* pinned: learn_grads reuses it */
    return 0;
}

/* --------------------------------------------------------------------------- plan + run */
int orc_run(const orc_cfg* cfg, uint64_t seed, int64_t env_total, int32_t k, int64_t episodes,
            double* episode_rewards, double* final_params, int64_t* steps_out) {
    if (k < 1) return -1;
    orc_unit** us = (orc_unit**)zalloc(sizeof(orc_unit*) * k);
    int64_t base = env_total / k, rem = env_total % k, lo = 0; /* split_envs, plan.cpp:46-55 */
    for (int r = 0; r < k; ++r) {
        int64_t cnt = base + (r < rem ? 1 : 0);
        us[r] = orc_unit_new(cfg, seed, lo, lo + cnt, env_total);
        lo += cnt;
    }
    int64_t P = us[0]->P, iters = orc_learn_iters(us[0]);
    double* mean = (double*)zalloc(sizeof(double) * P);
    for (int64_t ep = 0; ep < episodes; ++ep) {
        for (int r = 0; r < k; ++r) {
            orc_reset(us[r], ep);
            for (int64_t st = 0; st < cfg->steps_per_episode; ++st) orc_step(us[r], ep, st);
        }
        for (int64_t it = 0; it < iters; ++it) {
            for (int r = 0; r < k; ++r) orc_learn_grads(us[r], ep, it, NULL);
            if (k == 1) {
                orc_apply_grads(us[0], us[0]->grads);
            } else {
                /* GradSync: AllGather then the mean in unit-id order (local_run.cpp:397-412) */
                for (int64_t i = 0; i < P; ++i) {
                    double acc = 0.0;
                    for (int r = 0; r < k; ++r) acc += us[r]->grads[i];
                    mean[i] = acc / (double)k;
                }
                for (int r = 0; r < k; ++r) orc_apply_grads(us[r], mean);
            }
        }
        /* per-episode reward: sum over units / env count (local_run.cpp:560-570) */
        double sum = 0.0;
        for (int r = 0; r < k; ++r) sum += us[r]->reward_sum;
        if (episode_rewards) episode_rewards[ep] = sum / (double)env_total;
    }
    if (final_params) memcpy(final_params, us[0]->params, sizeof(double) * P);
    if (steps_out) {
        int64_t s = 0;
        for (int r = 0; r < k; ++r) s += us[r]->steps;
        *steps_out = s;
    }
    for (int r = 0; r < k; ++r) orc_unit_free(us[r]);
    free(us);
    free(mean);
    return 0;
}
