// DP-D unit engine: buffer layout, phase sequencing and per-episode CUDA graph.
//
// HBM layout for one unit with E envs, T steps, obs width S (PPO/A3C):
//   states  f32 [(T+1), E, S]   block t = policy input of step t (== trajectory state column);
//                               block T = the last step's next obs (last_next, programs.cpp:240)
//   actions i32 [T, E], logp/reward/done f32 [T, E], reward_d f64 [T, E]  (t-major == the
//                               reference's BufferSample row order t*E + e, interp.cpp:297-301)
//   est     f64 [sw, E]         env state, structure-of-arrays
//   H/DZ    f32 [T*E, width]    learn-phase activations / adjoints per layer and net
//   params  f32 [P], m/v f64 [P], grads f32 [P]   flat, reference parameter order
#include "engine.hpp"


#include <cmath>
#include <cstddef>
#include <cstring>
#include <vector>

#include <mutex>

#include "comm.hpp"
#include "common.cuh"
#include "fast.cuh"
#include "p2p.cuh"
#include "tgemm.cuh"
#include "wide.cuh"
#include <cuda_fp16.h>

#include <chrono>
#include <thread>
#include "kernels.cuh"

namespace flw {

struct Engine::Bufs {
    DeviceCtx* ctx = nullptr;
    double2* bc_table = nullptr;
    int64_t bc_len = 0;
    float* params = nullptr;
    double *m = nullptr, *v = nullptr;
    float* grads = nullptr;
    float* gather = nullptr;
    double* gmean = nullptr;
    double* est = nullptr;
    uint8_t* done = nullptr;
    int32_t* stepc = nullptr;
    float* states = nullptr;
    float *act0 = nullptr, *act1 = nullptr, *logits = nullptr;
    int32_t* actions = nullptr;
    float *logp = nullptr, *rew = nullptr, *done_f = nullptr;
    double* rew_d = nullptr;
    std::vector<float*> Hp, Hc, Hl, DZp, DZc;
    double* adv_d = nullptr;
    float *adv = nullptr, *ret = nullptr;
    double* terms = nullptr;
    double* stats = nullptr;
    float* loss = nullptr;
    double* rsum = nullptr;
    double* synth_b = nullptr;
    DwTile* tiles = nullptr;
    int ntiles = 0;
    // both modes: critic outputs consumed by GAE and the loss
    float *values = nullptr, *last_value = nullptr;
    // MAPPO: joint observation blocks [(T+1), E, W] and critic input rows [(T+1), n*E, W+n]
    float *joint = nullptr, *cin = nullptr;
    double* cprefix = nullptr;  // MAPPO compact critic: joint prefix chains [(T+1)*E, H0]
    // fast MAPPO compact critic (n > 4): joint GEMM, layer-0 rows, input gradients, per-env sums
    float *h0 = nullptr, *cP = nullptr, *dz0 = nullptr, *cS = nullptr, *cpart = nullptr;
    __nv_bfloat16 *jb = nullptr, *wjb = nullptr, *Sb = nullptr;  // bf16 joint rows, W_J, S
    float* jpart = nullptr;                                        // dW_J split-K partials
    int64_t jld = 0, hld0 = 0;
    int jsplits = 1;
    // fast MAPPO compact policy (n > 31): layer 0 on tcgen05 GEMMs around the fused kernel
    __nv_bfloat16 *w0b = nullptr, *pdz0b = nullptr;
    float *ph0 = nullptr, *pdz0 = nullptr, *ppart0 = nullptr;
    int64_t hld0p = 0;
    int psplits = 1;
    // fast numerics
    FastNet pol{}, crit{};
    int grid = 0;                       // persistent CTAs of the fused learn kernel
    float *part_p = nullptr, *part_c = nullptr, *loss_parts = nullptr;
    __nv_bfloat16 *wimg_p = nullptr, *wimg_c = nullptr;
    uint8_t* hsave = nullptr;           // critic hidden activations of the values pass (bf16 tiles)
    uint8_t* hscratch = nullptr;        // k_learn per-(CTA, group) activation scratch
    int grid2 = 0;                      // k_learn grid (fast_learn_groups() tiles per CTA in flight)
    int lgrid_p = 0, lgrid_c = 0;       // CTA partial slots written by the last policy / critic learn
    double *block_sums = nullptr, *rsum_scratch = nullptr;
    unsigned* gae_counter = nullptr;  // last-block-done counter of the fused GAE statistics
    unsigned* upd_counter = nullptr;  // last-block-done counter of k_reduce_adam
    unsigned* begin_counter = nullptr;  // last-block-done counter of the episode-begin reset
    // R > 1 replicas: env -> replica map, replica-major trajectory copies (exact), per-replica
    // gradient slots [R, P], advantage statistics [R, 2] and row weights (fast)
    int32_t* rep_of_env = nullptr;
    int64_t *rep_off = nullptr, *rep_n = nullptr;
    float *pstates = nullptr, *plogp = nullptr, *prew = nullptr, *pdone = nullptr;
    int32_t* pact = nullptr;
    double* prew_d = nullptr;
    float* gslots = nullptr;
    float* rep_w = nullptr;
    // layer-wise learn path (fast numerics, an MLP wider than the fused kernel's 64 columns):
    // bf16 weight copies, the input rows and every hidden activation as bf16 in HBM, dZ ping-pong
    WideNet wpol{}, wcrit{};
    __nv_bfloat16 *wb_p = nullptr, *wb_c = nullptr;
    __nv_bfloat16* xb = nullptr;
    int64_t xld = 0;
    std::vector<__nv_bfloat16*> hw_p, hw_c;
    std::vector<int64_t> hld_p, hld_c;
    float* wlogits = nullptr;
    __nv_bfloat16 *wdz0 = nullptr, *wdz1 = nullptr;
    int64_t dzld = 0;
    int wsplits = 0;
    // f32-accurate rollout of wide policies: split f16 operands (hi | lo | hi), f16 weight image
    __half *wr_x = nullptr, *wr_h0 = nullptr, *wr_h1 = nullptr, *wr_w = nullptr;
    int64_t wr_ldx = 0, wr_ldh = 0;
    std::vector<void*> owned;

    template <typename T>
    T* alloc(int64_t n) {
        void* p = nullptr;
        FLW_CUDA(cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T)));
        FLW_CUDA(cudaMemset(p, 0, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T)));
        owned.push_back(p);
        return static_cast<T*>(p);
    }
    ~Bufs() {
        for (void* p : owned) cudaFree(p);
    }
};

namespace {

EnvParams env_params(const AlgoConfig& c, const ProgramShape& s, const double* synth_b) {
    EnvParams p{};
    p.synth_b = synth_b;
    p.kind = static_cast<int>(s.env);
    p.n_agents = s.n_agents;
    p.max_steps = static_cast<int64_t>(c.env_param("max_steps", 0));
    p.length = static_cast<int64_t>(c.env_param("length", 8));  // envs.cpp:24,27
    return p;
}

int act_of(const AlgoConfig& c) { return c.activation == "relu" ? kRelu : kTanh; }

}  // namespace

Engine::Engine(const AlgoConfig& cfg, int device, uint64_t seed, int64_t env_lo, int64_t env_hi, int64_t env_total,
               Numerics numerics, int replicas)
    : cfg_(cfg), device_(device), seed_(seed), lo_(env_lo), hi_(env_hi), etot_(env_total), numerics_(numerics),
      nrep_(replicas) {
    cfg_.validate();
    shape_ = program_shape(cfg_);
    if (!shape_.accel_capable)
        fail(Errc::PolicyInapplicable, "dp-d requires an accelerator-capable environment implementation");
    mappo_ = shape_.algo == Algo::Mappo;
    if (mappo_ && shape_.env != EnvKind::SpreadLite)
        fail(Errc::PolicyInapplicable, "MAPPO runs on spread_lite (the reference's multi-agent env)");
    // fast MAPPO with a policy wider than the fused kernel (per-agent observation 2 + 2n > 64,
    // i.e. n > 31 agents, or hidden > 64): the policy learns on the layer-wise GEMM path
    if (mappo_ && numerics == Numerics::Fast) {
        bool hw = false;
        for (int l = 1; l < shape_.L; ++l) hw = hw || shape_.pdims[l] > 64;
        pwide_ = hw;  // hidden > 64: the whole policy on the layer-wise path
        // per-agent observation > 64 (n > 31) with hidden <= 64: layer 0 as tcgen05 GEMMs, the
        // rest in the fused learn kernel (the compact critic's split, for the policy)
        pcompact_ = !hw && shape_.obs_dim > 64 && shape_.L >= 2;
    }
    // fast MAPPO with a critic input wider than the fused kernel's 64 columns (n > 4): the
    // compact critic - layer 0 as a joint GEMM once per env + W[J+a], the rest fused
    cfast_ = mappo_ && numerics == Numerics::Fast && shape_.crit_in > 64;
    if (mappo_ && shape_.n_agents > 64) fail(Errc::Config, "at most 64 agents");
    if (!mappo_ && shape_.env == EnvKind::SpreadLite)
        fail(Errc::PolicyInapplicable, "PPO/A3C need a single-agent env (spread_lite is multi-agent)");
    {  // fast numerics with a layer wider than the fused kernel's 64 columns: layer-wise GEMMs
        int maxw = 0;
        for (int l = 1; l < shape_.L; ++l) maxw = std::max({maxw, shape_.pdims[l], shape_.cdims[l]});
        wide_ = numerics == Numerics::Fast && !mappo_ && (maxw > 64 || shape_.obs_dim > 64);
        if (wide_ && replicas > 1)
            fail(Errc::Config, "the layer-wise fast path (hidden > 64) runs one replica per engine");
    }
    if (env_hi <= env_lo || env_lo < 0 || env_hi > env_total) fail(Errc::Config, "bad env range");
    if (shape_.n_actions > 16) fail(Errc::Config, "at most 16 discrete actions are supported");
    E_ = env_hi - env_lo;
    if (nrep_ < 1 || nrep_ > E_) fail(Errc::Config, "replicas per engine must be in [1, envs]");
    if (nrep_ > 1 && mappo_) fail(Errc::Config, "MAPPO runs one replica per GPU in this build");
    {  // split_envs (plan.cpp:46-55): contiguous ranges, the remainder to the low replicas
        const int64_t base = E_ / nrep_, rem = E_ % nrep_;
        int64_t off = 0;
        for (int r = 0; r < nrep_; ++r) {
            const int64_t n = base + (r < rem ? 1 : 0);
            rep_off_.push_back(off);
            rep_n_.push_back(n);
            off += n;
        }
    }
    R_ = static_cast<int64_t>(shape_.n_agents) * E_;
    T_ = cfg_.steps_per_episode;
    TR_ = T_ * R_;
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    FLW_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    FLW_CUDA(cudaStreamCreateWithFlags(&side2_, cudaStreamNonBlocking));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_lfork_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_ljoin_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_plearn_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_gae_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreateWithFlags(&ev_wimg_, cudaEventDisableTiming));
    FLW_CUDA(cudaEventCreate(&ev_t0_));
    FLW_CUDA(cudaEventCreate(&ev_t1_));
    // group abort word in host-mapped memory: the host sets it (deadline passed, a peer failed)
    // and the peer-memory exchange's flag waits give up (kernels_p2p.cu)
    FLW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&abort_h_), sizeof(unsigned), cudaHostAllocMapped | cudaHostAllocPortable));
    *abort_h_ = 0;
    FLW_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&abort_d_), abort_h_, 0));
    alloc();
    FLW_CUDA(cudaDeviceSynchronize());  // alloc's zero-fills (legacy stream) before the stream's work
    init_params();
}

Engine::~Engine() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    destroy_graph();
    comm_.reset();
    for (void* q : p2p_ipc_opened_) cudaIpcCloseMemHandle(q);
    if (p2p_region_ptr_) cudaFree(p2p_region_ptr_);
    b_.reset();
    for (cudaEvent_t e : {ev_fork_, ev_join_, ev_wimg_, ev_t0_, ev_t1_, ev_lfork_, ev_ljoin_, ev_plearn_, ev_gae_})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_done_)
        if (e) cudaEventDestroy(e);
    if (rs_pinned_) cudaFreeHost(rs_pinned_);
    if (side_) cudaStreamDestroy(side_);
    if (side2_) cudaStreamDestroy(side2_);
    if (stream_) cudaStreamDestroy(stream_);
    if (abort_h_) cudaFreeHost(abort_h_);
}

void Engine::abort_group() {
    if (abort_h_) *reinterpret_cast<volatile unsigned*>(abort_h_) = 1u;
    if (comm_) comm_->abort();
}

bool Engine::grouped() const { return p2p_enabled() || (comm_ && comm_->nranks() > 1); }

// Waits for the engine stream. A unit in a gradient group can block on its peers (flag waits of
// the peer-memory exchange, NCCL collectives), so its wait is bounded like the reference's
// channel receives (local_run.cpp:543-546): past timeout_ms the group is aborted and the call
// fails with Timeout. A unit without a group cannot block on anything: plain synchronize.
void Engine::wait_stream(const char* what) { wait_event(nullptr, what); }

// (ev null: the whole stream)
void Engine::wait_event(cudaEvent_t ev, const char* what) {
    if (!grouped()) {
        if (ev)
            FLW_CUDA(cudaEventSynchronize(ev));
        else
            FLW_CUDA(cudaStreamSynchronize(stream_));
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t st = ev ? cudaEventQuery(ev) : cudaStreamQuery(stream_);
        if (st == cudaSuccess) break;
        if (st != cudaErrorNotReady) FLW_CUDA(st);
        if (*reinterpret_cast<volatile unsigned*>(abort_h_)) {
            FLW_CUDA(cudaStreamSynchronize(stream_));  // the exchange gives up on the abort word
            fail(Errc::PeerFailure, std::string(what) + ": the gradient group was aborted (a peer failed)");
        }
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > static_cast<double>(timeout_ms_)) {
            abort_group();
            FLW_CUDA(cudaStreamSynchronize(stream_));
            fail(Errc::Timeout, std::string(what) + ": no progress from the gradient group within " +
                                    std::to_string(timeout_ms_) + " ms (a peer did not reach the exchange)");
        }
        if (spin < 2000)
            std::this_thread::yield();
        else
            std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void Engine::destroy_graph() {
    for (cudaGraphExec_t g : segs_) cudaGraphExecDestroy(g);
    segs_.clear();
    between_.clear();
    graph_ = nullptr;
}

void Engine::set_eager_collectives(bool on) {
    if (on != eager_coll_) destroy_graph();
    eager_coll_ = on;
}

int64_t Engine::p2p_region_bytes() const { return p2p_layout(p2p_k_ > 0 ? p2p_k_ : 1, shape_.P).bytes; }

void* Engine::p2p_region() {
    if (numerics_ != Numerics::Fast || nrep_ > 1 || cfast_ || wide_)
        fail(Errc::Config, "the peer-memory exchange serves fast numerics with one unit per GPU");
    if (!p2p_region_ptr_) fail(Errc::Config, "call set_p2p_group first (region size depends on k)");
    return p2p_region_ptr_;
}

void Engine::set_p2p_peers(int rank, int k, const std::vector<void*>& regions, bool peers_elsewhere) {
    FLW_CUDA(cudaSetDevice(device_));
    if (static_cast<int>(regions.size()) != k || rank < 0 || rank >= k) fail(Errc::Config, "bad p2p group");
    destroy_graph();
    if (!p2p_peers_dev_) p2p_peers_dev_ = reinterpret_cast<uint8_t**>(b_->alloc<uint8_t*>(64));
    if (k > 64) fail(Errc::Config, "at most 64 ranks");
    FLW_CUDA(cudaMemcpy(p2p_peers_dev_, regions.data(), sizeof(void*) * regions.size(), cudaMemcpyHostToDevice));
    p2p_rank_ = rank;
    p2p_k_ = k;
    // the fused exchange kernel's blocks wait for the other ranks' blocks: only safe when no two
    // ranks share a GPU (FLW_P2P_FUSED=0 forces the two-kernel form, A/B)
    static const char* fz = std::getenv("FLW_P2P_FUSED");
    p2p_fused_ = peers_elsewhere && !(fz && fz[0] == '0');
}

void Engine::alloc_p2p_region(int k) {
    FLW_CUDA(cudaSetDevice(device_));
    if (numerics_ != Numerics::Fast || nrep_ > 1 || cfast_ || wide_)
        fail(Errc::Config, "the peer-memory exchange serves fast numerics with one unit per GPU");
    const P2pLayout L = p2p_layout(k, shape_.P);
    if (!p2p_region_ptr_) {
        FLW_CUDA(cudaMalloc(&p2p_region_ptr_, static_cast<size_t>(L.bytes)));  // plain cudaMalloc: IPC-exportable
        FLW_CUDA(cudaMemset(p2p_region_ptr_, 0, static_cast<size_t>(L.bytes)));
        p2p_alloc_k_ = k;
    } else if (p2p_alloc_k_ != k) {
        fail(Errc::Config, "p2p region already sized for another group");
    }
}

void Engine::set_comm(std::unique_ptr<Comm> comm) {
    if (graph_) destroy_graph();
    comm_ = std::move(comm);
    FLW_CUDA(cudaSetDevice(device_));  // the gather buffer must live on this engine's GPU
    if (comm_ && numerics_ == Numerics::Exact && !b_->gather) {
        b_->gather = b_->alloc<float>(static_cast<int64_t>(comm_->nranks()) * nrep_ * shape_.P);
    }
}

void Engine::alloc() {
    b_ = std::make_unique<Bufs>();
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int S = s.obs_dim, A = s.n_actions, L = s.L;
    b.ctx = b.alloc<DeviceCtx>(1);
    b.begin_counter = b.alloc<unsigned>(1);
    // Adam bias-correction table 1 - beta^t computed with the host libm pow, the reference's
    // arithmetic (mlp.cpp:151-152), for every step this run can take (+ slack).
    b.bc_len = std::max<int64_t>(4096, (cfg_.episodes + 16) * s.learn_iters);
    {
        std::vector<double2> tab(static_cast<size_t>(b.bc_len));
        for (int64_t t = 1; t <= b.bc_len; ++t) {
            tab[static_cast<size_t>(t - 1)].x = 1.0 - std::pow(0.9, static_cast<double>(t));
            tab[static_cast<size_t>(t - 1)].y = 1.0 - std::pow(0.999, static_cast<double>(t));
        }
        b.bc_table = b.alloc<double2>(b.bc_len);
        FLW_CUDA(cudaMemcpy(b.bc_table, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
    if (s.env == EnvKind::Synth17x6) {
        double tab[kSynthAct * kSynthObs];
        for (int a = 0; a < kSynthAct; ++a)
            for (int i = 0; i < kSynthObs; ++i)
                tab[a * kSynthObs + i] = rng_uniform_range(
                    rng_key(kSynthTableSeed, static_cast<uint64_t>(a), static_cast<uint64_t>(i)), -1.0, 1.0);
        b.synth_b = b.alloc<double>(kSynthAct * kSynthObs);
        FLW_CUDA(cudaMemcpy(b.synth_b, tab, sizeof(tab), cudaMemcpyHostToDevice));
    }
    b.params = b.alloc<float>(s.P);
    b.m = b.alloc<double>(s.P);
    b.v = b.alloc<double>(s.P);
    b.grads = b.alloc<float>(s.P);
    b.gmean = b.alloc<double>(s.P);
    b.est = b.alloc<double>(static_cast<int64_t>(s.env_state_w) * E_);
    b.done = b.alloc<uint8_t>(E_);
    b.stepc = b.alloc<int32_t>(E_);
    // policy rows per step: R = E (PPO/A3C) or n*E agent-major (MAPPO)
    b.states = b.alloc<float>((T_ + 1) * R_ * S);
    int maxw = 0;
    for (int d : s.pdims) maxw = std::max(maxw, d);
    for (int d : s.cdims) maxw = std::max(maxw, d);
    b.act0 = b.alloc<float>(R_ * maxw);
    b.act1 = b.alloc<float>(R_ * maxw);
    b.logits = b.alloc<float>(R_ * A);
    b.actions = b.alloc<int32_t>(T_ * R_);
    b.logp = b.alloc<float>(T_ * R_);
    b.rew = b.alloc<float>(T_ * R_);
    b.done_f = b.alloc<float>(T_ * R_);
    b.rew_d = b.alloc<double>(T_ * E_);
    if (mappo_) {  // joint obs per env and the critic rows [joint | one-hot] per (agent, env)
        b.joint = b.alloc<float>((T_ + 1) * E_ * s.state_w);
        // compact critic: [joint | one-hot] rows are never materialised (n x smaller; n=64,
        // E=2048 would need 145 GB), layer 0 reads the joint prefix chains + W[J+a]
        b.cprefix = b.alloc<double>((T_ + 1) * E_ * s.cdims[1]);
        // fast numerics (n <= 4): the tensor-core learn kernels read [joint | one-hot] rows
        if (numerics_ == Numerics::Fast && !cfast_) b.cin = b.alloc<float>((T_ + 1) * R_ * s.crit_in);
    }
    b.adv = b.alloc<float>(TR_);
    b.ret = b.alloc<float>(TR_);
    b.stats = b.alloc<double>(2 * nrep_);
    b.loss = b.alloc<float>(1);
    b.rsum = b.alloc<double>(nrep_);
    if (nrep_ > 1) {
        std::vector<int32_t> roe(static_cast<size_t>(E_));
        for (int r = 0; r < nrep_; ++r)
            for (int64_t e = rep_off_[r]; e < rep_off_[r] + rep_n_[r]; ++e) roe[static_cast<size_t>(e)] = r;
        b.rep_of_env = b.alloc<int32_t>(E_);
        b.rep_off = b.alloc<int64_t>(nrep_);
        b.rep_n = b.alloc<int64_t>(nrep_);
        FLW_CUDA(cudaMemcpy(b.rep_of_env, roe.data(), roe.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        FLW_CUDA(cudaMemcpy(b.rep_off, rep_off_.data(), rep_off_.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        FLW_CUDA(cudaMemcpy(b.rep_n, rep_n_.data(), rep_n_.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        if (numerics_ == Numerics::Exact) {
            b.pstates = b.alloc<float>(TR_ * S);
            b.pact = b.alloc<int32_t>(TR_);
            b.plogp = b.alloc<float>(TR_);
            b.prew = b.alloc<float>(TR_);
            b.pdone = b.alloc<float>(TR_);
            b.prew_d = b.alloc<double>(TR_);
            b.gslots = b.alloc<float>(static_cast<int64_t>(nrep_) * s.P);
        } else {
            // fast: row weight 1 / (R * T * E_r) folds the replica means and their average
            std::vector<float> w(static_cast<size_t>(nrep_));
            for (int r = 0; r < nrep_; ++r)
                w[static_cast<size_t>(r)] = static_cast<float>(1.0 / (static_cast<double>(nrep_) * T_ * rep_n_[r]));
            b.rep_w = b.alloc<float>(nrep_);
            FLW_CUDA(cudaMemcpy(b.rep_w, w.data(), w.size() * sizeof(float), cudaMemcpyHostToDevice));
        }
    }
    if (numerics_ == Numerics::Fast && wide_) {
        gemm_roll_ = true;
        alloc_wide();
        return;
    }
    if (numerics_ == Numerics::Fast) {
        // Fused tensor-core learn kernels: per-CTA dW partials replace the per-layer activations.
        auto make_net = [&](int net, int first = 0) {  // layers [first, L) of the net
            const auto& d = net == 0 ? s.pdims : s.cdims;
            FastNet n{};
            n.L = L - first;
            for (int l = 0; l < n.L; ++l) {
                const int ll = l + first;
                n.rin[l] = d[ll];
                n.rout[l] = d[ll + 1];
                n.din[l] = (d[ll] + 15) / 16 * 16;
                n.dout[l] = (d[ll + 1] + 15) / 16 * 16;
                n.woff[l] = s.woff[net][ll];
                n.boff[l] = s.boff[net][ll];
                if (n.din[l] > 64 || n.dout[l] > 64)
                    fail(Errc::Config, "fast numerics supports MLP widths up to 64 (use numerics=exact)");
            }
            return n;
        };
        if (L > kMaxLayers) fail(Errc::Config, "fast numerics supports at most 8 layers");
        {  // MAPPO policies the fused rollout kernel cannot hold roll out on split GEMMs
            FastRolloutArgs ra{};
            ra.L = L;
            for (int l = 0; l <= L; ++l) ra.dims[l] = s.pdims[l];
            ra.S = S;
            ra.A = A;
            ra.env = env_params(cfg_, shape_, nullptr);
            gemm_roll_ = mappo_ && !fast_rollout_mappo_ok(ra);
            // A/B: FLW_ROLLOUT=tcgen05 runs the PPO / A3C rollout's policy MLP as the split-f16
            // tcgen05 GEMMs (per layer, TMA + TMEM) instead of the fused mma.sync kernel
            static const char* rv = std::getenv("FLW_ROLLOUT");
            if (rv && std::string(rv) == "tcgen05") gemm_roll_ = true;
        }
        if (gemm_roll_ || pwide_) setup_wide_net(0, b.wpol);
        if (gemm_roll_) alloc_split_rollout();
        if (pwide_) alloc_wide_policy(TR_, 1);
        b.pol = pwide_ ? FastNet{} : make_net(0, pcompact_ ? 1 : 0);
        if (pcompact_) {  // compact policy: layer-0 GEMM operands and products
            const int H0 = s.pdims[1];
            auto pad8 = [](int64_t x) { return (x + 7) / 8 * 8; };
            b.xld = pad8(S + 1);  // + a column of ones: the bias-gradient row of dW0
            b.xb = b.alloc<__nv_bfloat16>(TR_ * b.xld);
            b.w0b = b.alloc<__nv_bfloat16>(static_cast<int64_t>(S) * pad8(H0));
            b.ph0 = b.alloc<float>(TR_ * H0);
            b.pdz0 = b.alloc<float>(TR_ * H0);
            b.hld0p = pad8(H0);
            b.pdz0b = b.alloc<__nv_bfloat16>(TR_ * b.hld0p);
            const int64_t mt = (S + 1 + 127) / 128, kb = (TR_ + 63) / 64;
            b.psplits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kb, 148 / mt)));
            b.ppart0 = b.alloc<float>(static_cast<int64_t>(b.psplits) * (S + 1) * H0);
            FLW_CUDA(cudaDeviceSynchronize());
            wide_fill_col(stream_, b.xb, TR_, b.xld, S, 1.0f);
        }
        if (cfast_) {
            if (L < 2 || s.cdims[1] > 64 || s.cdims[1] % 4 != 0)
                fail(Errc::Config, "compact fast critic needs >= 2 layers, hidden <= 64 and a multiple of 4");
            b.crit = make_net(1, 1);  // the critic without its layer 0
            const int H0 = s.cdims[1];
            b.h0 = b.alloc<float>((T_ + 1) * R_ * H0);
            b.cP = b.alloc<float>((T_ + 1) * E_ * H0);
            b.dz0 = b.alloc<float>(TR_ * H0);
            b.cS = b.alloc<float>(T_ * E_ * H0);
            b.cpart = b.alloc<float>(T_ * s.n_agents * H0);
            // the joint GEMMs (P = joint . W_J, dW_J = joint^T . S) on tcgen05 (kernels_tgemm.cu):
            // bf16 copies of the joint rows, W_J and S, split-K partials of dW_J
            const int J = s.state_w;
            b.jld = (J + 7) / 8 * 8;
            b.hld0 = (H0 + 7) / 8 * 8;
            b.jb = b.alloc<__nv_bfloat16>((T_ + 1) * E_ * b.jld);
            b.wjb = b.alloc<__nv_bfloat16>(static_cast<int64_t>(J) * b.hld0);
            b.Sb = b.alloc<__nv_bfloat16>(T_ * E_ * b.hld0);
            const int64_t mt = (J + 127) / 128, kb = (T_ * E_ + 63) / 64;
            b.jsplits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kb, 148 / mt)));
            b.jpart = b.alloc<float>(static_cast<int64_t>(b.jsplits) * J * H0);
        } else {
            b.crit = make_net(1);
        }
        int sms = 0;
        FLW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
        b.grid = static_cast<int>(std::min<int64_t>(sms, (TR_ + 127) / 128));
        // rows padded to 4 floats: the fused update reads them as float4
        b.part_p = b.alloc<float>(static_cast<int64_t>(std::max(b.grid, b.wsplits)) * ((s.P_policy + 3) / 4 * 4));
        b.part_c = b.alloc<float>(static_cast<int64_t>(b.grid) * ((s.P - s.P_policy + 3) / 4 * 4));
        b.loss_parts = b.alloc<float>(3 * (2 * b.grid + wide_loss_blocks(TR_)));
        b.wimg_p = b.alloc<__nv_bfloat16>(static_cast<int64_t>(fast_wimg_bytes(b.pol) / 2));
        b.wimg_c = b.alloc<__nv_bfloat16>(static_cast<int64_t>(fast_wimg_bytes(b.crit) / 2));
        b.hsave = b.alloc<uint8_t>(static_cast<int64_t>(fast_hsave_bytes(b.crit)) * ((TR_ + 127) / 128));
        const int64_t grp = fast_learn_groups();
        b.grid2 = static_cast<int>(std::min<int64_t>(sms, ((TR_ + 127) / 128 + grp - 1) / grp));
        b.hscratch = b.alloc<uint8_t>(static_cast<int64_t>(
            std::max(fast_learn_scratch_bytes(b.pol), fast_learn_scratch_bytes(b.crit)) * grp * b.grid2));
        b.block_sums = b.alloc<double>(2 * ((R_ + 31) / 32));  // per GAE block (32 or 256 streams)
        b.gae_counter = b.alloc<unsigned>(1);
        b.upd_counter = b.alloc<unsigned>(1);
        b.rsum_scratch = b.alloc<double>(256);
        b.values = b.alloc<float>(TR_);
        b.last_value = b.alloc<float>(R_);
        return;
    }
    for (int l = 0; l < L; ++l) {
        b.Hp.push_back(b.alloc<float>(TR_ * s.pdims[l + 1]));
        b.DZp.push_back(b.alloc<float>(TR_ * s.pdims[l + 1]));
        b.Hc.push_back(b.alloc<float>(TR_ * s.cdims[l + 1]));
        b.DZc.push_back(b.alloc<float>(TR_ * s.cdims[l + 1]));
        b.Hl.push_back(b.alloc<float>(R_ * s.cdims[l + 1]));
    }
    b.values = b.Hc[L - 1];
    b.last_value = b.Hl[L - 1];
    b.adv_d = b.alloc<double>(TR_);
    b.terms = b.alloc<double>(3 * TR_);
    // dW tile table: every (replica, net, layer) as 32(t, incl. the bias row t == K) x 32(j)
    // tiles; replica r's chains run over its own T*E_r rows (replica-major copies) into its
    // gradient slot.
    std::vector<DwTile> tiles;
    for (int r = 0; r < nrep_; ++r) {
        const int64_t row0 = T_ * rep_off_[r];
        float* g = nrep_ > 1 ? b.gslots + static_cast<int64_t>(r) * s.P : b.grads;
        const float* X0 = nrep_ > 1 ? b.pstates : b.states;
        for (int net = 0; net < 2; ++net) {
            const auto& d = net == 0 ? s.pdims : s.cdims;
            const auto& H = net == 0 ? b.Hp : b.Hc;
            const auto& DZ = net == 0 ? b.DZp : b.DZc;
            for (int l = 0; l < L; ++l) {
                int K = d[l], N = d[l + 1];
                for (int t0 = 0; t0 <= K; t0 += 32)
                    for (int j0 = 0; j0 < N; j0 += 32) {
                        DwTile t{};
                        t.H = (l == 0 ? X0 : H[l - 1]) + row0 * K;
                        if (l == 0 && net == 1 && mappo_) {  // compact [joint | one-hot] by index
                            t.H = b.joint;
                            t.cn = s.n_agents;
                            t.cE = E_;
                            t.cJ = s.state_w;
                        }
                        t.DZ = DZ[l] + row0 * N;
                        t.gW = g + s.woff[net][l];
                        t.gB = g + s.boff[net][l];
                        t.K = K, t.N = N, t.t0 = t0, t.j0 = j0;
                        t.rows = T_ * rep_n_[r] * (mappo_ ? s.n_agents : 1);
                        tiles.push_back(t);
                    }
            }
        }
    }
    b.ntiles = static_cast<int>(tiles.size());
    b.tiles = b.alloc<DwTile>(b.ntiles);
    FLW_CUDA(cudaMemcpy(b.tiles, tiles.data(), tiles.size() * sizeof(DwTile), cudaMemcpyHostToDevice));
}

// Xavier-uniform weights keyed by (seed, param stream, node id, i), zero biases, rounded to
// f32 (interp.cpp:71-85); node ids follow make_mlp_params order (programs.cpp:42-54).
void Engine::init_params(bool moments) {
    // Xavier-uniform weights, zero biases (interp.cpp init) in one kernel computing the same keyed
    // draws as the host would (rng_uniform_range rounds every operation on both sides; the bounds
    // are computed here), on the engine's stream - no host loop, no blocking copy
    const ProgramShape& s = shape_;
    FLW_CUDA(cudaSetDevice(device_));
    XavierTable t{};
    for (int net = 0; net < 2; ++net) {
        const auto& d = net == 0 ? s.pdims : s.cdims;
        for (int l = 0; l < s.L; ++l) {
            if (t.count == 16) fail(Errc::Config, "more than 8 layers per net");
            t.node[t.count] = static_cast<uint64_t>(net * 2 * s.L + 2 * l);
            t.a[t.count] = std::sqrt(6.0 / (static_cast<double>(d[l]) + static_cast<double>(d[l + 1])));
            t.n[t.count] = static_cast<int64_t>(d[l]) * d[l + 1];
            t.woff[t.count] = s.woff[net][l];
            ++t.count;
        }
    }
    param_init(stream_, t, b_->params, s.P, moments ? b_->m : nullptr, moments ? b_->v : nullptr, seed_);
}

void Engine::reinit(uint64_t seed) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    if (seed != seed_ && graph_) destroy_graph();  // the seed is baked into the captured kernel arguments
    seed_ = seed;
    init_params(true);  // (and the Adam moments)
    FLW_CUDA(cudaMemsetAsync(b_->ctx, 0, offsetof(DeviceCtx, coll_seq), stream_));  // keep the exchange epoch
    next_ep_dev_ = -1;
    steps_ = 0;
    cur_step_ = 0;
}

// ------------------------------------------------------------------------------ probes
void Engine::probe_begin(const char* tag) {
    if (!probes_on_ || !capturing_) return;
    Probe p{tag, nullptr, nullptr};
    FLW_CUDA(cudaEventCreate(&p.a));
    FLW_CUDA(cudaEventCreate(&p.b));
    // External: a real event-record node in the captured graph (a plain record during capture
    // only expresses an intra-graph dependency and cannot be timed).
    FLW_CUDA(cudaEventRecordWithFlags(p.a, stream_, cudaEventRecordExternal));
    probes_.push_back(p);
    open_probe_ = static_cast<int>(probes_.size()) - 1;
}

void Engine::probe_end() {
    if (open_probe_ < 0) return;
    FLW_CUDA(cudaEventRecordWithFlags(probes_[static_cast<size_t>(open_probe_)].b, stream_, cudaEventRecordExternal));
    open_probe_ = -1;
}

void Engine::clear_probes() {
    for (auto& p : probes_) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    probes_.clear();
    open_probe_ = -1;
}

void Engine::enable_probes(bool on) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    probes_on_ = on;
    if (graph_) destroy_graph();
    clear_probes();
}

std::string Engine::probe_times_json() {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    std::map<std::string, std::vector<float>> by;
    std::vector<std::string> order;
    for (auto& p : probes_) {
        float ms = 0.0f;
        FLW_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        if (!by.count(p.tag)) order.push_back(p.tag);
        by[p.tag].push_back(ms);
    }
    std::string s = "{";
    for (size_t i = 0; i < order.size(); ++i) {
        s += (i ? ", \"" : "\"") + order[i] + "\": [";
        const auto& v = by[order[i]];
        for (size_t j = 0; j < v.size(); ++j) s += (j ? ", " : "") + std::to_string(v[j]);
        s += "]";
    }
    return s + "}";
}

// Pageable H2D copies are staged before cudaMemcpyAsync returns, so `ep` may live on the stack.
void Engine::set_episode(int64_t ep) {
    FLW_CUDA(cudaMemcpyAsync(&b_->ctx->episode, &ep, sizeof(int64_t), cudaMemcpyHostToDevice, stream_));
}

// ----------------------------------------------------------------------------- phases
void Engine::enq_reset(bool begin) {
    Bufs& b = *b_;
    if (mappo_) {
        if (begin) begin_episode(stream_, b.ctx);
        mappo_reset(stream_, b.ctx, shape_.n_agents, b.est, b.done, b.stepc, b.joint, b.states, b.cin, E_, lo_, seed_);
    } else {
        exact_reset(stream_, b.ctx, env_params(cfg_, shape_, b_->synth_b), b.est, b.done, b.stepc, b.states, E_, lo_,
                    shape_.obs_dim, seed_, begin ? b.begin_counter : nullptr);
    }
}

void Engine::enq_mlp_forward(int net, const float* X, int64_t M, float* const* H, int first_layer) {
    const ProgramShape& s = shape_;
    const auto& d = net == 0 ? s.pdims : s.cdims;
    const float* in = first_layer > 0 ? H[first_layer - 1] : X;
    for (int l = first_layer; l < s.L; ++l) {
        exact_layer_fwd(stream_, in, b_->params + s.woff[net][l], b_->params + s.boff[net][l], H[l], M, d[l], d[l + 1],
                        l + 1 < s.L ? act_of(cfg_) : kNone);
        in = H[l];
    }
}

void Engine::enq_rollout_fast(int64_t step0, int64_t nsteps) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    FastRolloutArgs a{};
    a.params = b.params;
    a.L = s.L;
    for (int l = 0; l <= s.L; ++l) a.dims[l] = s.pdims[l];
    for (int l = 0; l < s.L; ++l) {
        a.woff[l] = s.woff[0][l];
        a.boff[l] = s.boff[0][l];
    }
    a.act = act_of(cfg_);
    a.est = b.est;
    a.done = b.done;
    a.stepc = b.stepc;
    a.states = b.states;
    a.actions = b.actions;
    a.logp = b.logp;
    a.reward = b.rew;
    a.done_f = b.done_f;
    a.reward_d = b.rew_d;
    a.E = E_;
    a.env_lo = lo_;
    a.step0 = step0;
    a.nsteps = nsteps;
    a.S = s.obs_dim;
    a.A = s.n_actions;
    a.seed = seed_;
    a.env = env_params(cfg_, shape_, b.synth_b);
    fast_rollout(stream_, b.ctx, a);
}

// MAPPO, fast numerics: the fused episode rollout (tensor-core MLP, one launch) when the shape
// fits (n <= 16 agents, widths <= 64); false: the exact per-step rollout is used.
bool Engine::enq_rollout_fast_mappo(int64_t step0, int64_t nsteps) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    FastRolloutArgs a{};
    a.params = b.params;
    a.L = s.L;
    for (int l = 0; l <= s.L; ++l) a.dims[l] = s.pdims[l];
    for (int l = 0; l < s.L; ++l) {
        a.woff[l] = s.woff[0][l];
        a.boff[l] = s.boff[0][l];
    }
    a.act = act_of(cfg_);
    a.est = b.est;
    a.done = b.done;
    a.stepc = b.stepc;
    a.states = b.states;  // the policy rows prows[T+1][n*E][S]
    a.actions = b.actions;
    a.logp = b.logp;
    a.reward = b.rew;
    a.done_f = b.done_f;
    a.reward_d = b.rew_d;
    a.E = E_;
    a.env_lo = lo_;
    a.env_total = etot_;
    a.step0 = step0;
    a.nsteps = nsteps;
    a.S = s.obs_dim;
    a.A = s.n_actions;
    a.seed = seed_;
    a.env = env_params(cfg_, shape_, b.synth_b);
    a.joint = b.joint;
    a.cin = b.cin;
    static const bool off = std::getenv("FLW_MAPPO_EXACT_ROLLOUT") != nullptr;  // A/B only
    if (off || !fast_rollout_mappo_ok(a)) return false;
    fast_rollout_mappo(stream_, b.ctx, a);
    return true;
}

void Engine::enq_step(int64_t st) {
    if (numerics_ == Numerics::Fast && !mappo_ && !wide_ && !gemm_roll_) return enq_rollout_fast(st, 1);
    if (numerics_ == Numerics::Fast && mappo_ && !gemm_roll_ && enq_rollout_fast_mappo(st, 1)) return;
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int S = s.obs_dim, A = s.n_actions;
    if (gemm_roll_) {
        enq_policy_fwd_split(st);  // f32-accurate tensor-core policy forward -> b.logits
    } else {
        const float* in = b.states + st * R_ * S;
        float* bufs[2] = {b.act0, b.act1};
        for (int l = 0; l < s.L; ++l) {
            float* out = l + 1 == s.L ? b.logits : bufs[l & 1];
            exact_layer_fwd(stream_, in, b.params + s.woff[0][l], b.params + s.boff[0][l], out, R_, s.pdims[l],
                            s.pdims[l + 1], l + 1 < s.L ? act_of(cfg_) : kNone);
            in = out;
        }
    }
    if (mappo_) {
        MappoStepArgs m{};
        m.logits = b.logits;
        m.est = b.est;
        m.done = b.done;
        m.stepc = b.stepc;
        m.actions = b.actions;
        m.logp = b.logp;
        m.reward = b.rew;
        m.done_f = b.done_f;
        m.reward_d = b.rew_d;
        m.joint = b.joint;
        m.prows = b.states;
        m.cin = b.cin;
        m.E = E_;
        m.env_lo = lo_;
        m.env_total = etot_;
        m.step = st;
        m.max_steps = static_cast<int64_t>(cfg_.env_param("max_steps", 0));
        m.n = s.n_agents;
        m.A = A;
        m.seed = seed_;
        mappo_rollout(stream_, b.ctx, m);
        return;
    }
    enq_step_env(st);
}

// PolicyApply + env step of one rollout step on the f32 logits in b.logits (PPO / A3C).
void Engine::enq_step_env(int64_t st) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int S = s.obs_dim, A = s.n_actions;
    RolloutArgs a{};
    a.logits = b.logits;
    a.est = b.est;
    a.done = b.done;
    a.stepc = b.stepc;
    a.actions = b.actions + st * E_;
    a.logp = b.logp + st * E_;
    a.reward = b.rew + st * E_;
    a.reward_d = b.rew_d + st * E_;
    a.done_f = b.done_f + st * E_;
    a.next_obs = b.states + (st + 1) * E_ * S;
    a.E = E_;
    a.env_lo = lo_;
    a.S = S;
    a.A = A;
    a.seed = seed_;
    a.step = st;
    a.env = env_params(cfg_, shape_, b_->synth_b);
    exact_rollout(stream_, b.ctx, a);
}

// Fast numerics: critic forward (tensor cores) -> GAE + advantage stats -> fused policy and
// critic learn kernels (forward, loss, backward, TMEM-resident dW) -> deterministic reduction.
void Engine::enq_learn_fast() {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int S = s.obs_dim;
    const bool ppo = s.algo != Algo::A3c;
    FastLearnArgs f{};
    f.act = act_of(cfg_);
    f.params = b.params;
    f.in_cols = S;
    f.inv_n = 1.0 / static_cast<double>(TR_);
    f.value_coef = cfg_.value_coef;
    f.entropy_coef = cfg_.entropy_coef;
    f.clip_eps = static_cast<float>(cfg_.clip_eps);
    f.split_rows = -1;
    f.rep_of_env = nrep_ > 1 ? b.rep_of_env : nullptr;
    f.rep_w = b.rep_w;
    f.rep_E = E_;
    // the weight images: built at the first train iteration of an episode (in the episode graph:
    // on the side stream during the rollout, build_graph); later iterations use the images the
    // previous iteration's fused update (k_reduce_adam) wrote
    if (learn_iter_ == 0 ? !wimg_early_ : !prev_fused_)
        fast_build_wimg(stream_, b.params, b.crit, b.wimg_c, b.pol, b.wimg_p);
    // values = critic(states), last_value = critic(last_next)
    f.net = b.crit;
    f.wimg = b.wimg_c;
    f.kind = kNetCritic;
    f.mode = 0;
    // critic rows: the states (PPO/A3C), [joint | one-hot] per agent row (MAPPO, n <= 4), or
    // the compact critic's layer-0 activations (MAPPO, n > 4)
    const int H0 = s.cdims[1], J = s.state_w;
    if (cfast_) {
        // P[(T+1)*E, H0] = joint . W_J on the tensor cores (bf16 operands, f32 accumulation)
        if (learn_iter_ == 0)  // the joint rows change once per episode (the rollout)
            wide_to_bf16(stream_, b.joint, (T_ + 1) * E_, J, b.jb, b.jld);
        wide_to_bf16(stream_, b.params + s.woff[1][0], J, H0, b.wjb, b.hld0);
        TgEpilogue pe;
        pe.mode = kTgStoreF32;
        pe.c32 = b.cP;
        pe.ldc32 = H0;
        tgemm(stream_, TgOperand{b.jb, (T_ + 1) * E_, J, b.jld, kTgBF16}, false, TgOperand{b.wjb, J, H0, b.hld0, kTgBF16},
              true, (T_ + 1) * E_, H0, J, 1, pe, 64);
        mappo_fast_h0(stream_, b.cP, b.params + s.woff[1][0], b.params + s.boff[1][0], T_ + 1, E_, s.n_agents, J, H0,
                      act_of(cfg_), b.h0);
    }
    const float* Xc = cfast_ ? b.h0 : (mappo_ ? b.cin : b.states);
    const int Cin = cfast_ ? H0 : (mappo_ ? s.crit_in : S);
    f.X = Xc;
    f.in_cols = Cin;
    f.rows = TR_;
    // states block T (= last_next) directly follows the T*E trajectory rows, so ONE launch over
    // T*E + E rows yields values and last_value (values_out rows >= T*E go to last_value).
    f.rows = TR_ + R_;
    f.split_rows = TR_;
    f.values_out = b.values;
    f.values_out2 = b.last_value;
    // Keep the trajectory tiles' hidden activations for the critic learn pass (FLW_NO_HREUSE
    // disables the reuse, for A/B measurement only).
    static const bool hreuse = std::getenv("FLW_NO_HREUSE") == nullptr;
    f.hsave = hreuse ? b.hsave : nullptr;
    f.save_tiles = hreuse ? (TR_ + 127) / 128 : 0;
    // k_learn: warp-specialised, two tiles per SM in flight
    const int lgrid = b.grid2;
    auto launch = [&](int grid) { fast_learn(stream_, f, grid); };
    f.hscratch = b.hscratch;
    const int64_t grp = fast_values_groups();
    const int vgrid = static_cast<int>(std::min<int64_t>(lgrid, ((f.rows + 127) / 128 + grp - 1) / grp));
    // the values pass and the policy learn start as programmatic dependents of the kernel before
    // them on their stream (setup overlapped; griddepcontrol.wait before any input is read)
    f.pdl = pdl_ok() && !probes_on_ ? 1 : 0;
    const FastLearnArgs fv = f;  // the values pass (kept for the next iteration's, see below)
    if (vg_ready_) {
        // the previous iteration enqueued this one's values pass + GAE on side2_ (pipelined)
        vg_ready_ = false;
        FLW_CUDA(cudaStreamWaitEvent(stream_, ev_gae_, 0));
    } else {
        probe_begin("critic_fwd");
        launch(vgrid);
        probe_end();
        probe_begin("gae");
        fast_gae(stream_, b.rew, b.values, b.done_f, b.last_value, TR_, R_, cfg_.gamma, cfg_.lam, b.adv, b.ret, ppo,
                 b.block_sums, b.stats, b.gae_counter, f.pdl != 0);
        if (nrep_ > 1 && ppo && cfg_.normalize_adv)  // each folded unit normalises over its own rows
            fast_rep_adv_stats(stream_, b.adv, T_, E_, b.rep_off, b.rep_n, nrep_, b.stats);
        probe_end();
    }
    f.split_rows = -1;
    // learn: policy then critic, each a persistent fused kernel
    f.mode = 1;
    f.X = b.states;
    f.in_cols = S;
    f.rows = TR_;
    f.actions = b.actions;
    f.logp_old = b.logp;
    f.adv = b.adv;
    f.adv_stats = (ppo && cfg_.normalize_adv) ? b.stats : nullptr;
    f.ret = b.ret;
    f.values_in = b.values;
    f.net = b.pol;
    f.wimg = b.wimg_p;
    f.hsave = nullptr;
    f.hload = 0;
    f.kind = ppo ? kNetPolicyPpo : kNetPolicyA3c;
    f.partials = b.part_p;
    // one GPU, one unit, no exchange: the reduction is fused with Adam (enq_grad_sync_and_adam)
    // and reads 16-byte aligned partial rows
    fused_pending_ = fuse_ok_ && !p2p_enabled() && !(comm_ && comm_->nranks() > 1) && !cfast_ && nrep_ == 1;
    const bool padded = fused_pending_ || (p2p_enabled() && !cfast_);  // float4 partial rows
    f.part_stride = padded ? (s.P_policy + 3) / 4 * 4 : s.P_policy;
    f.loss_partials = b.loss_parts;
    // The policy and critic learn kernels run CONCURRENTLY on disjoint SMs (two streams), the
    // SMs split in proportion to their per-tile cost (the critic skips its forward), so both
    // finish together instead of each paying its own tail.
    int gp = lgrid, gc = lgrid;
    // (a layer-wise policy runs after the critic on the whole GPU)
    const bool concurrent = hreuse && lgrid >= 8 && !pwide_;  // the critic reads hsave, not hscratch
    if (concurrent) {
        // measured (C2 sweep 0.58-0.70, profiles/r02_learn_split.txt): 60/40
        static const char* env_split = std::getenv("FLW_LEARN_SPLIT");
        const double split = env_split ? std::atof(env_split) : 0.6;
        gp = std::max(1, std::min(lgrid - 1, static_cast<int>(lgrid * split + 0.5)));
        gc = std::max(1, lgrid - gp);
        FLW_CUDA(cudaEventRecord(ev_lfork_, stream_));
        FLW_CUDA(cudaStreamWaitEvent(side2_, ev_lfork_, 0));
    }
    int64_t p_off = 0;  // compact policy: the fused kernel owns layers 1.., its partials start there
    if (pcompact_) {
        // layer 0: h0 = act(X W0 + b0) as one tcgen05 GEMM over the policy rows (bf16 operands)
        const int H0 = s.pdims[1];
        p_off = static_cast<int64_t>(S) * H0 + H0;
        if (learn_iter_ == 0) wide_to_bf16(stream_, b.states, TR_, S, b.xb, b.xld);  // once per episode
        wide_to_bf16(stream_, b.params + s.woff[0][0], S, H0, b.w0b, b.hld0p);
        TgEpilogue he;
        he.mode = kTgBiasAct;
        he.act = act_of(cfg_);
        he.bias = b.params + s.boff[0][0];
        he.c32 = b.ph0;
        he.ldc32 = H0;
        tgemm(stream_, TgOperand{b.xb, TR_, S, b.xld, kTgBF16}, false, TgOperand{b.w0b, S, H0, b.hld0p, kTgBF16}, true,
              TR_, H0, S, 1, he, 64);
        f.X = b.ph0;
        f.in_cols = H0;
        f.dx_out = b.pdz0;  // dZ0 = dH0 * act'(h0) from the kernel's input-gradient stage
        f.part_stride = s.P_policy - p_off;
    }
    f.loss_partials = b.loss_parts;
    const int np_loss = pwide_ ? wide_loss_blocks(TR_) : gp;  // policy loss-partial slots
    if (!pwide_) {
        probe_begin("learn_policy");
        launch(gp);
        probe_end();
    }
    if (concurrent) FLW_CUDA(cudaEventRecord(ev_plearn_, stream_));  // the policy learn read adv
    FastLearnArgs fc = f;
    fc.pdl = 0;
    fc.X = Xc;
    fc.in_cols = Cin;
    fc.net = b.crit;
    fc.wimg = b.wimg_c;
    fc.hsave = hreuse ? b.hsave : nullptr;  // same params as the values pass: same activations
    fc.hload = hreuse ? 1 : 0;
    fc.kind = kNetCritic;
    fc.partials = b.part_c;
    // compact critic: the fused kernel owns layers 1.. (and reports dZ wrt its input rows)
    const int64_t c_off = cfast_ ? static_cast<int64_t>(J + s.n_agents) * H0 + H0 : 0;
    fc.part_stride = padded ? (s.P - s.P_policy + 3) / 4 * 4 : s.P - s.P_policy - c_off;
    fc.dx_out = cfast_ ? b.dz0 : nullptr;
    fc.loss_partials = b.loss_parts + 3 * np_loss;
    if (concurrent) {
        fast_learn(side2_, fc, gc);
        if (split_update_ok()) enq_critic_update(side2_, gc);
        FLW_CUDA(cudaEventRecord(ev_ljoin_, side2_));
        FLW_CUDA(cudaStreamWaitEvent(stream_, ev_ljoin_, 0));
        // Train-iteration pipelining: the next iteration's values pass needs only the updated
        // critic, so it starts here on the critic's stream - on the SMs the critic learn freed -
        // while the policy learn and the policy update still run; its GAE waits for the policy
        // learn (which reads adv). PPO only (an A3C policy reads the values).
        if (pipe_next_ok_ && split_done_ && ppo && nrep_ == 1 && !eager_coll_ && hreuse) {
            fast_learn(side2_, fv, vgrid);
            FLW_CUDA(cudaStreamWaitEvent(side2_, ev_plearn_, 0));
            fast_gae(side2_, b.rew, b.values, b.done_f, b.last_value, TR_, R_, cfg_.gamma, cfg_.lam, b.adv, b.ret, ppo,
                     b.block_sums, b.stats, b.gae_counter, fv.pdl != 0);
            FLW_CUDA(cudaEventRecord(ev_gae_, side2_));
            vg_ready_ = true;
        }
    } else {
        probe_begin("learn_critic");
        fast_learn(stream_, fc, gc);
        probe_end();
    }
    if (pwide_) {
        probe_begin("learn_policy");
        enq_learn_policy_wide(b.loss_parts);
        probe_end();
    }
    if (pcompact_) {  // [dW0 ; db0] = [X | 1]^T dZ0: split-K tcgen05 GEMM + fixed-order sum
        const int H0 = s.pdims[1];
        wide_to_bf16(stream_, b.pdz0, TR_, H0, b.pdz0b, b.hld0p);
        TgEpilogue we;
        we.mode = kTgStoreF32;
        we.c32 = b.ppart0;
        we.ldc32 = H0;
        we.split_stride = static_cast<int64_t>(S + 1) * H0;
        tgemm(stream_, TgOperand{b.xb, TR_, S + 1, b.xld, kTgBF16}, true, TgOperand{b.pdz0b, TR_, H0, b.hld0p, kTgBF16},
              true, S + 1, H0, TR_, b.psplits, we, 64);
        wide_sum_partials(stream_, b.ppart0, b.psplits, static_cast<int64_t>(S + 1) * H0, b.grads + s.woff[0][0]);
    }
    b.lgrid_p = pwide_ ? np_loss : gp;
    b.lgrid_c = gc;
    if (!p2p_enabled() && !fused_pending_) {  // with peer-memory exchange the reduction is fused into the exchange
        probe_begin("reduce");
        // (compact policy: partial index i is parameter p_off + i; the critic's offset is unchanged)
        fast_reduce_partials(stream_, b.part_p, b.part_c, pwide_ ? b.wsplits : gp, gc, s.P_policy - p_off,
                             s.P - s.P_policy - c_off, b.grads + p_off, c_off);
        probe_end();
    }
    if (cfast_) {  // critic layer-0 gradients: one-hot rows, bias, and dW_J = joint^T . S
        float* g0 = b.grads + s.woff[1][0];
        mappo_fast_layer0_grads(stream_, b.dz0, T_, E_, s.n_agents, H0, b.cS, b.cpart,
                                g0 + static_cast<int64_t>(J) * H0, b.grads + s.boff[1][0]);
        // dW_J = joint^T . S over the T*E trajectory envs: split-K tcgen05 GEMM + fixed-order sum
        wide_to_bf16(stream_, b.cS, T_ * E_, H0, b.Sb, b.hld0);
        TgEpilogue we;
        we.mode = kTgStoreF32;
        we.c32 = b.jpart;
        we.ldc32 = H0;
        we.split_stride = static_cast<int64_t>(J) * H0;
        tgemm(stream_, TgOperand{b.jb, T_ * E_, J, b.jld, kTgBF16}, true, TgOperand{b.Sb, T_ * E_, H0, b.hld0, kTgBF16},
              true, J, H0, T_ * E_, b.jsplits, we, 64);
        wide_sum_partials(stream_, b.jpart, b.jsplits, static_cast<int64_t>(J) * H0, g0);
    }
    // the scalar loss is not an input of anything downstream: reduced on demand (read_tensor)
}

// Fast numerics, policy forward of one rollout step as f32-accurate split GEMMs on the tensor
// cores (x = hi + lo, W = hi + lo in f16; x.W ~ hi.hi + lo.hi + hi.lo with f32 accumulation, one
// GEMM with K = 3 segments per layer; tanh in f32) into the f32 logits b.logits; the reference's
// PolicyApply + env step follow (enq_step). Used when the fused rollout kernel does not fit the
// policy (hidden > 64, or MAPPO with n > 16 agents).
void Engine::enq_policy_fwd_split(int64_t st) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int L = s.L, S = s.obs_dim;
    const WideNet& n = b.wpol;
    if (st == 0 || !capturing_) wide_build_split_weights(stream_, b.params, n, b.wr_w);
    wide_split_input(stream_, b.states + st * R_ * S, R_, S, b.wr_x, n.dp[0]);
    auto bn_for = [](int64_t x) { return x > 128 ? 256 : (x > 64 ? 128 : 64); };
    const __half* in = b.wr_x;
    int64_t inld = b.wr_ldx;
    __half* outs[2] = {b.wr_h0, b.wr_h1};
    for (int l = 0; l < L; ++l) {
        const TgOperand A{in, R_, 3 * n.dp[l], inld, kTgF16};
        const TgOperand B{b.wr_w + n.sofs[l], 3 * n.dp[l], n.dout[l], n.wld[l], kTgF16};
        TgEpilogue e;
        e.bias = b.params + n.boff[l];
        if (l + 1 < L) {
            e.mode = kTgSplit3;
            e.act = act_of(cfg_);
            e.c16h = outs[l & 1];
            e.ldc16 = 3 * n.dp[l + 1];
            e.seg = n.dp[l + 1];
        } else {
            e.mode = kTgBias;
            e.c32 = b.logits;
            e.ldc32 = n.dout[l];
        }
        // few rows per step: narrow N tiles spread the layer over more SMs
        tgemm(stream_, A, false, B, true, R_, n.dout[l], 3 * n.dp[l], 1, e, R_ <= 16384 ? 64 : bn_for(n.dout[l]));
        if (l + 1 < L) {
            in = outs[l & 1];
            inld = 3 * n.dp[l + 1];
        }
    }
}

void Engine::setup_wide_net(int net, WideNet& n) const {
    const ProgramShape& s = shape_;
    const auto& d = net == 0 ? s.pdims : s.cdims;
    const int L = s.L;
    if (L > kMaxLayers) fail(Errc::Config, "fast numerics supports at most 8 layers");
    auto pad8 = [](int64_t x) { return (x + 7) / 8 * 8; };
    n = WideNet{};
    n.L = L;
    int64_t off = 0, so = 0;
    for (int l = 0; l < L; ++l) {
        n.din[l] = d[l];
        n.dout[l] = d[l + 1];
        n.woff[l] = s.woff[net][l];
        n.boff[l] = s.boff[net][l];
        n.wofs[l] = off;
        n.wld[l] = pad8(d[l + 1]);
        off += (static_cast<int64_t>(d[l]) * n.wld[l] + 7) / 8 * 8;  // 16-byte aligned layers
        n.dp[l] = (d[l] + 63) / 64 * 64;
        n.sofs[l] = so;
        so += 3 * n.dp[l] * n.wld[l];
    }
    n.wbytes = off;
    n.sbytes = so;
}

// split-GEMM rollout buffers of the policy (R_ rows per step; pad columns stay zero)
void Engine::alloc_split_rollout() {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    int64_t maxh = 64;
    for (int l = 1; l < s.L; ++l) maxh = std::max<int64_t>(maxh, (s.pdims[l] + 63) / 64 * 64);
    b.wr_ldx = 3 * b.wpol.dp[0];
    b.wr_ldh = 3 * maxh;
    b.wr_x = b.alloc<__half>(R_ * b.wr_ldx);
    b.wr_h0 = b.alloc<__half>(R_ * b.wr_ldh);
    b.wr_h1 = b.alloc<__half>(R_ * b.wr_ldh);
    b.wr_w = b.alloc<__half>(b.wpol.sbytes);
}

// layer-wise learn buffers of the policy: bf16 weights, input rows, hidden activations, dZ
// ping-pong (sized for `maxw` columns), outputs, split-K partial slots
void Engine::alloc_wide_policy(int64_t xrows, int maxw) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    auto pad8 = [](int64_t x) { return (x + 7) / 8 * 8; };
    b.wb_p = b.alloc<__nv_bfloat16>(b.wpol.wbytes);
    // activation buffers carry a column of ones after the data (the bias-gradient row of the
    // weight-gradient GEMM)
    b.xld = pad8(s.obs_dim + 1);
    b.xb = b.alloc<__nv_bfloat16>(xrows * b.xld);
    for (int l = 0; l + 1 < s.L; ++l) {
        b.hld_p.push_back(pad8(s.pdims[l + 1] + 1));
        b.hw_p.push_back(b.alloc<__nv_bfloat16>(TR_ * b.hld_p.back()));
    }
    FLW_CUDA(cudaDeviceSynchronize());  // the allocations' memsets before the fills on stream_
    wide_fill_col(stream_, b.xb, xrows, b.xld, s.obs_dim, 1.0f);
    for (int l = 0; l + 1 < s.L; ++l) wide_fill_col(stream_, b.hw_p[l], TR_, b.hld_p[l], s.pdims[l + 1], 1.0f);
    for (int l = 0; l <= s.L; ++l) maxw = std::max(maxw, s.pdims[l]);
    b.dzld = pad8(maxw);
    b.wdz0 = b.alloc<__nv_bfloat16>(TR_ * b.dzld);
    b.wdz1 = b.alloc<__nv_bfloat16>(TR_ * b.dzld);
    b.wlogits = b.alloc<float>(TR_ * s.n_actions);
    // partial slots of the weight-gradient GEMMs (<= tgemm's clamp of one k-block per split):
    // 128 for nets of <= 200 k parameters (one 148-CTA wave for 64-wide layers), 64 above (the
    // reduction reads every slot)
    const int64_t pmax = std::max<int64_t>(s.P_policy, s.P - s.P_policy);
    b.wsplits = static_cast<int>(std::min<int64_t>(pmax <= 200000 ? 128 : 64, (TR_ + 63) / 64));
}

void Engine::alloc_wide() {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int L = s.L;
    auto pad8 = [](int64_t x) { return (x + 7) / 8 * 8; };
    setup_wide_net(0, b.wpol);
    setup_wide_net(1, b.wcrit);
    const int64_t Rc = TR_ + R_;
    int maxw = 1;
    for (int l = 0; l <= L; ++l) maxw = std::max(maxw, s.cdims[l]);
    alloc_wide_policy(Rc, maxw);  // the critic reads the same input rows (+ last_next)
    b.wb_c = b.alloc<__nv_bfloat16>(b.wcrit.wbytes);
    for (int l = 0; l + 1 < L; ++l) {
        b.hld_c.push_back(pad8(s.cdims[l + 1] + 1));
        b.hw_c.push_back(b.alloc<__nv_bfloat16>(Rc * b.hld_c.back()));
    }
    FLW_CUDA(cudaDeviceSynchronize());
    for (int l = 0; l + 1 < L; ++l) wide_fill_col(stream_, b.hw_c[l], Rc, b.hld_c[l], s.cdims[l + 1], 1.0f);
    alloc_split_rollout();
    b.values = b.alloc<float>(Rc);  // values | last_value: one critic forward over all rows
    b.last_value = b.values + TR_;
    b.grid = b.wsplits;
    b.part_p = b.alloc<float>(static_cast<int64_t>(b.wsplits) * s.P_policy);
    b.part_c = b.alloc<float>(static_cast<int64_t>(b.wsplits) * (s.P - s.P_policy));
    b.loss_parts = b.alloc<float>(2 * 3 * wide_loss_blocks(TR_));
    b.block_sums = b.alloc<double>(2 * ((R_ + 31) / 32));
    b.gae_counter = b.alloc<unsigned>(1);
    b.upd_counter = b.alloc<unsigned>(1);
    b.rsum_scratch = b.alloc<double>(256);
}

// Layer-wise forward of one net over `rows` rows of b.xb: hidden activations to H (bf16), the
// output layer to `out` (f32).
void Engine::wide_forward(const WideNet& n, const __nv_bfloat16* wb, const std::vector<__nv_bfloat16*>& H,
                          const std::vector<int64_t>& ld, int64_t rows, float* out) {
    Bufs& b = *b_;
    auto bn_for = [](int64_t x) { return x > 128 ? 256 : (x > 64 ? 128 : 64); };
    for (int l = 0; l < n.L; ++l) {
        const TgOperand A{l == 0 ? b.xb : H[l - 1], rows, n.din[l], l == 0 ? b.xld : ld[l - 1], kTgBF16};
        const TgOperand B{wb + n.wofs[l], n.din[l], n.dout[l], n.wld[l], kTgBF16};
        TgEpilogue e;
        e.bias = b.params + n.boff[l];
        if (l + 1 < n.L) {
            e.mode = kTgBiasAct;
            e.act = act_of(cfg_);
            e.c16 = H[l];
            e.ldc16 = ld[l];
        } else {
            e.mode = kTgBias;
            e.c32 = out;
            e.ldc32 = n.dout[l];
        }
        tgemm(stream_, A, false, B, true, rows, n.dout[l], n.din[l], 1, e, bn_for(n.dout[l]));
    }
}

// Layer-wise backward over the TR_ trajectory rows from dZ_{L-1} in b.wdz0: per layer dW_m
// (split-K partial slots, stride pstride) and db_m, then dZ_{m-1} = (dZ_m W_m^T) * act'(H_{m-1}).
void Engine::wide_backward(const WideNet& n, const __nv_bfloat16* wb, const std::vector<__nv_bfloat16*>& H,
                           const std::vector<int64_t>& ld, float* part, int64_t pstride) {
    Bufs& b = *b_;
    auto bn_for = [](int64_t x) { return x > 128 ? 256 : (x > 64 ? 128 : 64); };
    const int splits = b.wsplits;
    __nv_bfloat16 *dz = b.wdz0, *other = b.wdz1;
    for (int m = n.L - 1; m >= 0; --m) {
        const int din = n.din[m], dout = n.dout[m];
        // dW_m = H_{m-1}^T dZ_m (K = rows split `splits` ways) -> partial slots
        // [dW_m ; db_m] = [H_{m-1} | 1]^T dZ_m (K = rows split `splits` ways) -> partial slots:
        // column din of every activation buffer holds ones, so output row din is the bias
        // gradient (the column sums of dZ_m), landing at boff = woff + din*dout
        const TgOperand Hin{m == 0 ? b.xb : H[m - 1], TR_, din + 1, m == 0 ? b.xld : ld[m - 1], kTgBF16};
        const TgOperand Dz{dz, TR_, dout, b.dzld, kTgBF16};
        TgEpilogue e;
        e.mode = kTgStoreF32;
        e.c32 = part + (n.woff[m] - n.woff[0]);
        e.ldc32 = dout;
        e.split_stride = pstride;
        // one wave: this layer's K split so that (M tiles x N tiles x splits) <= 148; rows of
        // the partial buffer beyond its split count are never written (stay zero)
        const int64_t tiles = ((din + 1 + 127) / 128) * ((dout + bn_for(dout) - 1) / bn_for(dout));
        const int lsplits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(splits, 148 / tiles)));
        tgemm(stream_, Hin, true, Dz, true, din + 1, dout, TR_, lsplits, e, bn_for(dout));
        if (m == 0) break;
        const TgOperand Wk{wb + n.wofs[m], din, dout, n.wld[m], kTgBF16};
        TgEpilogue g;
        g.mode = kTgActGrad;
        g.act = act_of(cfg_);
        g.h = H[m - 1];
        g.ldh = ld[m - 1];
        g.c16 = other;
        g.ldc16 = b.dzld;
        tgemm(stream_, Dz, false, Wk, false, TR_, din, dout, 1, g, bn_for(din));
        std::swap(dz, other);
    }
}

// PPO / A3C loss rows over the output layer (rl.cpp:137-202) -> dZ_{L-1} in b.wdz0
void Engine::wide_loss_rows(int kind, const float* out, int A, float* loss_partials) {
    Bufs& b = *b_;
    WideLossArgs la{};
    la.rows = TR_;
    la.actions = b.actions;
    la.logp_old = b.logp;
    la.adv = b.adv;
    la.ret = b.ret;
    la.values_in = b.values;
    la.adv_stats = (shape_.algo != Algo::A3c && cfg_.normalize_adv) ? b.stats : nullptr;
    la.inv_n = 1.0 / static_cast<double>(TR_);
    la.value_coef = cfg_.value_coef;
    la.entropy_coef = cfg_.entropy_coef;
    la.clip_eps = static_cast<float>(cfg_.clip_eps);
    la.ld = b.dzld;
    la.kind = kind;
    la.out = out;
    la.A = A;
    la.width = A;
    la.dz = b.wdz0;
    la.loss_partials = loss_partials;
    wide_loss(stream_, la);
}

// MAPPO with a policy wider than the fused kernel (n > 31 agents: per-agent observation
// 2 + 2n > 64): the policy's train iteration on the layer-wise path, into part_p
void Engine::enq_learn_policy_wide(float* loss_partials) {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    WideNet none{};
    wide_build_weights(stream_, b.params, b.wpol, b.wb_p, none, nullptr);
    if (learn_iter_ == 0) wide_to_bf16(stream_, b.states, TR_, s.obs_dim, b.xb, b.xld);  // once per episode
    wide_forward(b.wpol, b.wb_p, b.hw_p, b.hld_p, TR_, b.wlogits);
    wide_loss_rows(s.algo != Algo::A3c ? kNetPolicyPpo : kNetPolicyA3c, b.wlogits, s.n_actions, loss_partials);
    wide_backward(b.wpol, b.wb_p, b.hw_p, b.hld_p, b.part_p, s.P_policy);
}

// Fast numerics, widths > 64: one train iteration as layer-wise tcgen05 GEMMs (kernels_tgemm.cu)
// with bf16 activations in HBM: critic forward (values | last_value) -> GAE -> policy forward ->
// losses (dZ of the output layers) -> per layer dW (split-K partials) + db + dZ of the layer
// below -> fixed-order reduction of the partials. Same operand precision as the fused kernel
// (bf16 operands, f32 accumulation, bf16 activations and adjoints).
void Engine::enq_learn_wide() {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const bool ppo = s.algo != Algo::A3c;
    const int64_t Rc = TR_ + R_;
    wide_build_weights(stream_, b.params, b.wpol, b.wb_p, b.wcrit, b.wb_c);
    if (learn_iter_ == 0)  // states blocks 0..T (last_next): once per episode
        wide_to_bf16(stream_, b.states, Rc, s.obs_dim, b.xb, b.xld);
    probe_begin("critic_fwd");
    wide_forward(b.wcrit, b.wb_c, b.hw_c, b.hld_c, Rc, b.values);
    probe_end();
    probe_begin("gae");
    fast_gae(stream_, b.rew, b.values, b.done_f, b.last_value, TR_, R_, cfg_.gamma, cfg_.lam, b.adv, b.ret, ppo,
             b.block_sums, b.stats, b.gae_counter);
    probe_end();
    probe_begin("learn_policy");
    wide_forward(b.wpol, b.wb_p, b.hw_p, b.hld_p, TR_, b.wlogits);
    const int nlb = wide_loss_blocks(TR_);
    wide_loss_rows(ppo ? kNetPolicyPpo : kNetPolicyA3c, b.wlogits, s.n_actions, b.loss_parts);
    wide_backward(b.wpol, b.wb_p, b.hw_p, b.hld_p, b.part_p, s.P_policy);
    wide_loss_rows(kNetCritic, b.values, 1, b.loss_parts + 3 * nlb);
    wide_backward(b.wcrit, b.wb_c, b.hw_c, b.hld_c, b.part_c, s.P - s.P_policy);
    b.lgrid_p = b.lgrid_c = nlb;
    fast_reduce_partials(stream_, b.part_p, b.part_c, b.wsplits, b.wsplits, s.P_policy, s.P - s.P_policy, b.grads, 0);
    probe_end();
}

void Engine::enq_learn_grads() {
    if (numerics_ == Numerics::Fast) return wide_ ? enq_learn_wide() : enq_learn_fast();
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const int S = s.obs_dim, A = s.n_actions, L = s.L;
    // R > 1: the replica-major copies made after the rollout (enq_permute_replicas), so every
    // replica's rows are one contiguous t-major block [T, E_r]
    const bool rep = nrep_ > 1;
    const float* X = rep ? b.pstates : b.states;  // [T*R, S] t-major policy rows
    // critic rows: the states themselves (PPO/A3C) or [joint | one-hot] (MAPPO); block T holds
    // the last step's next rows (last_next / last nci, programs.cpp:240-245, 422-427)
    const float* Xc = X;
    const float* last_next = b.states + T_ * R_ * s.crit_in;
    const float* rew = rep ? b.prew : b.rew;
    const float* done_f = rep ? b.pdone : b.done_f;
    const int32_t* actions = rep ? b.pact : b.actions;
    const float* logp = rep ? b.plogp : b.logp;
    (void)S;
    if (mappo_) {  // compact critic layer 0 over all T+1 blocks, then layers 1.. per row
        exact_mappo_critic0(stream_, b.joint, b.params + s.woff[1][0], b.params + s.boff[1][0], T_ + 1, E_,
                            s.n_agents, s.state_w, s.cdims[1], b.cprefix, b.Hc[0], b.Hl[0],
                            L > 1 ? act_of(cfg_) : kNone);
        enq_mlp_forward(1, nullptr, TR_, b.Hc.data(), 1);
        enq_mlp_forward(1, nullptr, R_, b.Hl.data(), 1);
    } else {
        enq_mlp_forward(1, Xc, TR_, b.Hc.data());         // values = critic(states | ci)
        enq_mlp_forward(1, last_next, R_, b.Hl.data());   // last_value = critic(last_next | last nci)
    }
    const bool ppo = s.algo != Algo::A3c;
    enq_mlp_forward(0, X, TR_, b.Hp.data());          // logits_new = policy(states)
    // Per replica (= per reference unit): GAE over its E_r streams, advantage normalisation
    // with its own statistics, loss mean over its T*E_r rows.
    for (int r = 0; r < nrep_; ++r) {
        const int64_t ro = T_ * rep_off_[r] * (mappo_ ? s.n_agents : 1);
        const int64_t nr = rep_n_[r] * (mappo_ ? s.n_agents : 1), tr = T_ * nr;
        const int64_t lo = rep_off_[r] * (mappo_ ? s.n_agents : 1);
        exact_gae(stream_, rew + ro, b.Hc[L - 1] + ro, done_f + ro, b.Hl[L - 1] + lo, tr, nr, cfg_.gamma, cfg_.lam,
                  b.adv_d + ro, b.ret + ro, ppo);
        if (ppo) exact_normalize(stream_, b.adv_d + ro, tr, cfg_.normalize_adv, b.stats + 2 * r, b.adv + ro);
        exact_loss_rows(stream_, ppo ? 0 : 1, b.Hp[L - 1] + ro * A, b.Hc[L - 1] + ro, actions + ro, logp + ro,
                        b.adv + ro, b.ret + ro, tr, A, cfg_.clip_eps, cfg_.value_coef, cfg_.entropy_coef,
                        b.DZp[L - 1] + ro * A, b.DZc[L - 1] + ro, b.terms + 3 * ro);
    }
    // Adjoint chains (row-parallel), then every dW/db chain of both nets (and replicas) in one launch.
    for (int net = 0; net < 2; ++net) {
        const auto& d = net == 0 ? s.pdims : s.cdims;
        const auto& H = net == 0 ? b.Hp : b.Hc;
        const auto& DZ = net == 0 ? b.DZp : b.DZc;
        for (int l = L - 1; l >= 1; --l)
            exact_layer_dh(stream_, DZ[l], b.params + s.woff[net][l], H[l - 1], DZ[l - 1], TR_, d[l], d[l + 1],
                           act_of(cfg_));
    }
    exact_dw(stream_, b.tiles, b.ntiles);
}

void Engine::enq_permute_replicas() {
    Bufs& b = *b_;
    ReplicaMap m{b.rep_of_env, b.rep_off, b.rep_n};
    permute_rows_f32(stream_, b.states, b.pstates, T_, E_, shape_.obs_dim, m);
    permute_rows_i32(stream_, b.actions, b.pact, T_, E_, m);
    permute_rows_f32(stream_, b.logp, b.plogp, T_, E_, 1, m);
    permute_rows_f32(stream_, b.rew, b.prew, T_, E_, 1, m);
    permute_rows_f32(stream_, b.done_f, b.pdone, T_, E_, 1, m);
    permute_rows_f64(stream_, b.rew_d, b.prew_d, T_, E_, m);
}

FastUpdateArgs Engine::update_args() const {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    FastUpdateArgs u{};
    u.pp = b.part_p;
    u.pc = b.part_c;
    u.np = b.lgrid_p;
    u.nc = b.lgrid_c;
    u.Pp = s.P_policy;
    u.Pc = s.P - s.P_policy;
    u.ctx = b.ctx;
    u.bc_table = b.bc_table;
    u.bc_len = b.bc_len;
    u.params = b.params;
    u.grads = b.grads;
    u.m = b.m;
    u.v = b.v;
    u.lr = cfg_.lr;
    u.b1 = 0.9;
    u.b2 = 0.999;
    u.eps = 1e-8;
    u.pol = b.pol;
    u.crit = b.crit;
    u.img_p = b.wimg_p;
    u.img_c = b.wimg_c;
    u.counter = b.upd_counter;
    return u;
}

P2pArgs Engine::p2p_args() const {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    const P2pLayout Lo = p2p_layout(p2p_k_, s.P);
    P2pArgs a{};
    a.part_p = b.part_p;
    a.part_c = b.part_c;
    a.np = b.lgrid_p;
    a.nc = b.lgrid_c;
    a.Pp = s.P_policy;
    a.Pc = s.P - s.P_policy;
    a.rank = p2p_rank_;
    a.k = p2p_k_;
    a.peers = p2p_peers_dev_;
    a.off_inbox = Lo.off_inbox;
    a.off_grads = Lo.off_grads;
    a.off_sflag = Lo.off_sflag;
    a.off_dflag = Lo.off_dflag;
    a.ctx = b.ctx;
    a.abort_flag = abort_d_;
    a.params = b.params;
    a.m = b.m;
    a.v = b.v;
    a.lr = cfg_.lr;
    a.b1 = 0.9;
    a.b2 = 0.999;
    a.eps = 1e-8;
    a.gscale = 1.0 / static_cast<double>(p2p_k_);
    a.Ptot = s.P;
    if (!cfast_) {  // the exchange's Adam also refreshes the weight images
        a.pol = b.pol;
        a.crit = b.crit;
        a.img_p = b.wimg_p;
        a.img_c = b.wimg_c;
    }
    return a;
}

// The critic's half of the update, enqueued on the critic learn's stream right after it (the
// policy learn is still running on the other SMs): its partials reduced (and exchanged over
// peer memory with k GPUs) and Adam applied to the critic parameters. The policy half follows
// the join in enq_grad_sync_and_adam. Same arithmetic per parameter as the one-launch update.
// The fused update as a programmatic dependent launch of the learn kernel before it (k_learn
// triggers its dependents once its tiles are done). FLW_NO_PDL: plain launches (A/B only).
bool Engine::pdl_ok() const {
    static const bool off = std::getenv("FLW_NO_PDL") != nullptr;
    return !off && !cfast_ && !pcompact_ && !pwide_;
}

bool Engine::split_update_ok() const {
    // (fuse_ok_: the update follows this learn; peer exchange only between distinct GPUs - a
    // co-located rank's waiting exchange could hold the SMs its peer's critic learn needs)
    return fuse_ok_ && !cfast_ && !pcompact_ && !pwide_ && nrep_ == 1 && numerics_ == Numerics::Fast &&
           (fused_pending_ || (p2p_enabled() && p2p_fused_));
}

void Engine::enq_critic_update(cudaStream_t st, int ncrit) {
    const ProgramShape& s = shape_;
    split_done_ = true;
    if (fused_pending_) {
        FastUpdateArgs u = update_args();
        u.pp = b_->part_c;
        u.np = ncrit;
        u.Pp = s.P - s.P_policy;
        u.Pc = 0;
        u.nc = 0;
        u.off = s.P_policy;
        u.critic_only = true;
        u.advance = false;  // the policy launch (the iteration's last) advances the step counter
        fast_reduce_adam(st, u, pdl_ok());
        return;
    }
    adam_tick(st, b_->ctx, b_->bc_table, b_->bc_len);  // once per iteration: before both halves
    P2pArgs a = p2p_args();
    a.part_p = b_->part_c;
    a.np = ncrit;
    a.Pp = s.P - s.P_policy;
    a.Pc = 0;
    a.nc = 0;
    a.off = s.P_policy;
    a.critic_only = true;
    a.flag0 = static_cast<int>(((s.P_policy + 3) / 4 * 4 + 127) / 128);  // after the policy launch's hint rows
    coll_tick(st, b_->ctx);
    reduce_allreduce_adam(st, a, p2p_fused_);
}

void Engine::enq_grad_sync_and_adam() {
    Bufs& b = *b_;
    const ProgramShape& s = shape_;
    prev_fused_ = fused_pending_;
    const bool split = split_done_;
    split_done_ = false;
    if (fused_pending_) {  // partial reduction + Adam + weight images, one launch
        fused_pending_ = false;
        FastUpdateArgs u = update_args();
        if (split) {  // the critic's half already ran after the critic learn
            u.Pc = 0;
            u.nc = 0;
        }
        probe_begin("reduce");
        fast_reduce_adam(stream_, u, pdl_ok() && !probes_on_);
        probe_end();
        return;
    }
    if (!split) adam_tick(stream_, b.ctx, b.bc_table, b.bc_len);
    if (p2p_enabled() && numerics_ == Numerics::Fast) {
        // reduce the CTA partials + all-reduce over NVLink peer memory + Adam: one kernel
        P2pArgs a = p2p_args();
        if (split) {
            a.Pc = 0;
            a.nc = 0;
        }
        if (!cfast_) prev_fused_ = true;
        coll_tick(stream_, b.ctx);
        probe_begin("exchange_adam");
        reduce_allreduce_adam(stream_, a, p2p_fused_);
        probe_end();
        return;
    }
    const double* g64 = nullptr;
    double gscale = 1.0;
    const bool rep = nrep_ > 1 && numerics_ == Numerics::Exact;
    if (comm_ && comm_->nranks() > 1) {
        if (numerics_ == Numerics::Exact) {
            // GradSync (local_run.cpp:379-414): AllGather then the mean in unit-id order; with
            // R replicas per GPU each rank contributes its R consecutive units' gradients.
            const float* send = rep ? b.gslots : b.grads;
            const int64_t cnt = static_cast<int64_t>(nrep_) * s.P;
            const int k = comm_->nranks() * nrep_;
            auto op = [this, &b, send, cnt] { comm_->all_gather(send, b.gather, cnt, stream_); };
            if (eager_coll_ && capturing_)
                segment_break(op);
            else
                op();
            exact_grad_mean(stream_, b.gather, k, s.P, b.gmean);
            g64 = b.gmean;
        } else {
            // Fast: in-place NCCL sum over NVLink, the 1/k of the mean folded into Adam.
            auto op = [this, &b, P = s.P] { comm_->all_reduce_sum(b.grads, b.grads, P, stream_); };
            if (eager_coll_ && capturing_)
                segment_break(op);
            else
                op();
            gscale = 1.0 / static_cast<double>(comm_->nranks());
        }
    } else if (rep) {  // one GPU, R units: the ordered mean of the local slots
        exact_grad_mean(stream_, b.gslots, nrep_, s.P, b.gmean);
        g64 = b.gmean;
    }
    probe_begin("adam");
    exact_adam(stream_, b.ctx, b.params, b.grads, g64, b.m, b.v, s.P, cfg_.lr, 0.9, 0.999, 1e-8, gscale);
    probe_end();
}

void Engine::enq_reward_sum() {
    // Episode reward sum in the reference's order: steps outer, envs inner (interp.cpp:257),
    // one chain per replica (= unit) over its own envs.
    if (numerics_ == Numerics::Fast) {
        fast_sum(side_, b_->rew_d, T_ * E_, b_->rsum_scratch, b_->rsum);
    } else if (nrep_ == 1) {
        exact_seq_sum(side_, b_->rew_d, T_ * E_, b_->rsum);
    } else {
        for (int r = 0; r < nrep_; ++r)
            exact_seq_sum(side_, b_->prew_d + T_ * rep_off_[r], T_ * rep_n_[r], b_->rsum + r);
    }
}

// ------------------------------------------------------------------- phase-level API
void Engine::reset(int64_t ep) {
    if (nrep_ > 1) fail(Errc::Config, "the phase-level API drives one replica per engine (use run_episode)");
    FLW_CUDA(cudaSetDevice(device_));
    set_episode(ep);
    enq_reset();
    FLW_CUDA(cudaMemsetAsync(b_->rew_d, 0, static_cast<size_t>(T_ * E_) * sizeof(double), stream_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    cur_step_ = 0;
}

void Engine::step(int64_t ep, int64_t st) {
    FLW_CUDA(cudaSetDevice(device_));
    if (st < 0 || st >= T_) fail(Errc::Config, "step index outside the episode");
    set_episode(ep);
    enq_step(st);
    FLW_CUDA(cudaStreamSynchronize(stream_));
    cur_step_ = st + 1;
    steps_ += 1;
}

void Engine::learn_grads(int64_t ep, int64_t k) {
    (void)k;
    FLW_CUDA(cudaSetDevice(device_));
    set_episode(ep);
    learn_iter_ = 0;
    enq_learn_grads();
    if (numerics_ == Numerics::Exact) exact_loss_reduce(stream_, b_->terms, TR_, cfg_.entropy_coef, b_->loss);
    FLW_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::apply_grads(const double* host_grads) {
    FLW_CUDA(cudaSetDevice(device_));
    Bufs& b = *b_;
    adam_tick(stream_, b.ctx, b.bc_table, b.bc_len);
    const double* g64 = nullptr;
    if (host_grads) {
        FLW_CUDA(cudaMemcpyAsync(b.gmean, host_grads, static_cast<size_t>(shape_.P) * sizeof(double),
                                 cudaMemcpyHostToDevice, stream_));
        g64 = b.gmean;
    }
    exact_adam(stream_, b.ctx, b.params, b.grads, g64, b.m, b.v, shape_.P, cfg_.lr, 0.9, 0.999, 1e-8);
    FLW_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::learn(int64_t ep, int64_t k) {
    (void)k;
    FLW_CUDA(cudaSetDevice(device_));
    set_episode(ep);
    learn_iter_ = 0;
    fuse_ok_ = true;  // the update follows right away
    enq_learn_grads();
    fuse_ok_ = false;
    if (numerics_ == Numerics::Exact) exact_loss_reduce(stream_, b_->terms, TR_, cfg_.entropy_coef, b_->loss);
    enq_grad_sync_and_adam();
    wait_stream("learn");
}

// ------------------------------------------------------------------------ episode graph
void Engine::build_graph() {
    FLW_CUDA(cudaSetDevice(device_));
    if (!rs_pinned_) {  // [kInFlight][nrep_] reward sums (mapped), then [kInFlight] episode indices
        FLW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&rs_pinned_),
                               sizeof(double) * static_cast<size_t>(kInFlight * (nrep_ + 1)), cudaHostAllocMapped));
        FLW_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&rs_ring_d_), rs_pinned_, 0));
        for (cudaEvent_t& e : ev_done_) FLW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    flw_trace("build_graph: capture");
    destroy_graph();
    graph_kernels_ = 0;
    clear_probes();
    FLW_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    capturing_ = true;
    // (the episode begin - ctx->episode = ctx->next_episode++ - runs inside the reset launch)
    trace_capture("begin");
    // The first train iteration's weight images depend only on the params the previous episode
    // left: built on the side stream while the episode resets and rolls out (fast k_learn path)
    wimg_early_ = numerics_ == Numerics::Fast && !mappo_ && !wide_ && !gemm_roll_ && !eager_coll_;
    if (wimg_early_) {
        FLW_CUDA(cudaEventRecord(ev_wimg_, stream_));
        FLW_CUDA(cudaStreamWaitEvent(side_, ev_wimg_, 0));
        fast_build_wimg(side_, b_->params, b_->crit, b_->wimg_c, b_->pol, b_->wimg_p);
        FLW_CUDA(cudaEventRecord(ev_wimg_, side_));
    }
    enq_reset(true);
    trace_capture("reset");
    probe_begin("rollout");
    if (numerics_ == Numerics::Fast && !mappo_ && !wide_ && !gemm_roll_)
        enq_rollout_fast(0, T_);
    else if (!(numerics_ == Numerics::Fast && mappo_ && !gemm_roll_ && enq_rollout_fast_mappo(0, T_)))
        for (int64_t st = 0; st < T_; ++st) enq_step(st);  // per-step rollout (exact or split GEMMs)
    probe_end();
    if (nrep_ > 1 && numerics_ == Numerics::Exact) enq_permute_replicas();
    FLW_CUDA(cudaEventRecord(ev_fork_, stream_));
    FLW_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    enq_reward_sum();
    publish_rsum(side_, b_->ctx, b_->rsum, numerics_ == Numerics::Exact ? nrep_ : 1, rs_ring_d_, kInFlight);
    FLW_CUDA(cudaEventRecord(ev_join_, side_));
    if (wimg_early_) FLW_CUDA(cudaStreamWaitEvent(stream_, ev_wimg_, 0));
    // a capture segment cannot end with the side stream still forked
    if (eager_coll_) FLW_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
    trace_capture("rollout+reward");
    for (int64_t k = 0; k < shape_.learn_iters; ++k) {
        if (numerics_ == Numerics::Exact) probe_begin("learn_grads");
        learn_iter_ = k;
        fuse_ok_ = true;  // the update follows right away
        pipe_next_ok_ = k + 1 < shape_.learn_iters;
        enq_learn_grads();
        pipe_next_ok_ = false;
        fuse_ok_ = false;
        trace_capture("learn_grads");
        if (numerics_ == Numerics::Exact) probe_end();
        enq_grad_sync_and_adam();
        trace_capture("sync+adam");
    }
    learn_iter_ = 0;
    wimg_early_ = false;
    if (!eager_coll_) FLW_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
    end_segment();
    graph_ = segs_.front();
    flw_trace("build_graph: done");
}

void Engine::trace_capture(const char* where) {
    static const bool on = std::getenv("FLW_TRACE") != nullptr;
    if (!on) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(stream_, &st);
    std::fprintf(stderr, "[flw] dev %d %s: capture status %d (%s)\n", device_, where, static_cast<int>(st),
                 cudaGetErrorString(e));
}

void Engine::end_segment() {
    trace_capture("end_segment");
    cudaGraph_t g;
    capturing_ = false;
    FLW_CUDA(cudaStreamEndCapture(stream_, &g));
    size_t n = 0;
    FLW_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    FLW_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    for (auto nd : nodes) {
        cudaGraphNodeType ty;
        FLW_CUDA(cudaGraphNodeGetType(nd, &ty));
        if (ty == cudaGraphNodeTypeKernel) ++graph_kernels_;
    }
    cudaGraphExec_t exec = nullptr;
    FLW_CUDA(cudaGraphInstantiate(&exec, g, 0));
    FLW_CUDA(cudaGraphDestroy(g));
    segs_.push_back(exec);
}

void Engine::segment_break(std::function<void()> op) {
    end_segment();
    between_.push_back(std::move(op));
    FLW_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    capturing_ = true;
}

void Engine::launch_graph() {
    for (size_t i = 0; i < segs_.size(); ++i) {
        FLW_CUDA(cudaGraphLaunch(segs_[i], stream_));
        if (i < between_.size()) between_[i]();
    }
    ++graph_runs_;
}

void Engine::prepare() {
    FLW_CUDA(cudaSetDevice(device_));
    if (!graph_) build_graph();
    FLW_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::enqueue_episodes(int64_t first, int64_t count) {
    FLW_CUDA(cudaSetDevice(device_));
    if (fl_head_ != fl_tail_) fail(Errc::Config, "enqueue_episodes: pipelined episodes still in flight");
    if (!graph_) build_graph();
    FLW_CUDA(cudaMemcpyAsync(&b_->ctx->next_episode, &first, sizeof(int64_t), cudaMemcpyHostToDevice, stream_));
    for (int64_t i = 0; i < count; ++i) launch_graph();
    next_ep_dev_ = first + count;
    steps_ += T_ * count * nrep_;
    cur_step_ = T_;
}

double Engine::last_reward_sum() {
    double total = 0.0;
    for (double v : replica_reward_sums()) total += v;
    return total;
}

std::vector<double> Engine::replica_reward_sums() {
    FLW_CUDA(cudaSetDevice(device_));
    std::vector<double> r(static_cast<size_t>(nrep_), 0.0);
    const int n = numerics_ == Numerics::Exact ? nrep_ : 1;
    FLW_CUDA(cudaMemcpy(r.data(), b_->rsum, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost));
    return r;
}

void Engine::sync() {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
}

double Engine::run_episode(int64_t ep, float* device_ms) {
    FLW_CUDA(cudaSetDevice(device_));
    if (fl_head_ != fl_tail_) fail(Errc::Config, "run_episode: pipelined episodes still in flight");
    if (!graph_) build_graph();
    FLW_CUDA(cudaMemcpyAsync(&b_->ctx->next_episode, &ep, sizeof(int64_t), cudaMemcpyHostToDevice, stream_));
    FLW_CUDA(cudaEventRecord(ev_t0_, stream_));
    launch_graph();
    next_ep_dev_ = ep + 1;
    FLW_CUDA(cudaEventRecord(ev_t1_, stream_));
    flw_trace("run_episode: launched");
    wait_stream("run_episode");
    flw_trace("run_episode: synced");
    steps_ += T_ * nrep_;
    cur_step_ = T_;
    if (device_ms) FLW_CUDA(cudaEventElapsedTime(device_ms, ev_t0_, ev_t1_));
    const double r = last_reward_sum();
    if (std::isnan(r) && numerics_ == Numerics::Fast)
        fail(Errc::Runtime, "fast numerics: an observation left the f16 range (|x| >= 65504) of the rollout's "
                            "split tensor-core MLP; use numerics=exact");
    return r;
}

void Engine::launch_episode(int64_t ep) {
    FLW_CUDA(cudaSetDevice(device_));
    if (fl_head_ - fl_tail_ >= kInFlight) fail(Errc::Config, "launch_episode: too many episodes in flight");
    if (!graph_) build_graph();
    const int slot = static_cast<int>(fl_head_ % kInFlight);
    // the episode index from a pinned slot: a truly asynchronous copy (the slot is reused only
    // after finish_episode has waited for this episode)
    int64_t* ep_pinned = reinterpret_cast<int64_t*>(rs_pinned_ + static_cast<size_t>(kInFlight) * nrep_) + slot;
    *ep_pinned = ep;
    // consecutive episodes: the previous graph's k_begin_episode already advanced the device
    // counter to ep, so no copy sits between the two graphs
    if (ep != next_ep_dev_)
        FLW_CUDA(cudaMemcpyAsync(&b_->ctx->next_episode, ep_pinned, sizeof(int64_t), cudaMemcpyHostToDevice, stream_));
    // the graph publishes its reward sums into ring slot graph_runs_ % kInFlight (k_publish_rsum):
    // nothing but the completion event follows it on the stream
    fl_slot_[slot] = graph_runs_ % kInFlight;
    launch_graph();
    next_ep_dev_ = ep + 1;
    FLW_CUDA(cudaEventRecord(ev_done_[slot], stream_));
    ++fl_head_;
}

std::vector<double> Engine::finish_episode() {
    FLW_CUDA(cudaSetDevice(device_));
    if (fl_tail_ == fl_head_) fail(Errc::Config, "finish_episode: no episode in flight");
    const int slot = static_cast<int>(fl_tail_ % kInFlight);
    wait_event(ev_done_[slot], "finish_episode");
    ++fl_tail_;
    steps_ += T_ * nrep_;
    cur_step_ = T_;
    const int n = numerics_ == Numerics::Exact ? nrep_ : 1;  // (fast: the total in entry 0)
    std::vector<double> r(static_cast<size_t>(nrep_), 0.0);
    const double* ring = rs_pinned_ + static_cast<size_t>(fl_slot_[slot]) * n;
    for (int i = 0; i < n; ++i) r[static_cast<size_t>(i)] = ring[i];
    double total = 0.0;
    for (double v : r) total += v;
    if (std::isnan(total) && numerics_ == Numerics::Fast)
        fail(Errc::Runtime, "fast numerics: an observation left the f16 range (|x| >= 65504) of the rollout's "
                            "split tensor-core MLP; use numerics=exact");
    return r;
}

void Engine::drain_episodes() {
    cudaSetDevice(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    fl_tail_ = fl_head_;
}

// --------------------------------------------------------------------------- params
void Engine::get_params(double* out) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));  // (params are written on the engine's stream)
    std::vector<float> p(static_cast<size_t>(shape_.P));
    FLW_CUDA(cudaMemcpy(p.data(), b_->params, p.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < p.size(); ++i) out[i] = static_cast<double>(p[i]);
}

void Engine::set_params(const double* in) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    std::vector<float> p(static_cast<size_t>(shape_.P));
    for (size_t i = 0; i < p.size(); ++i) p[i] = static_cast<float>(in[i]);
    FLW_CUDA(cudaMemcpy(b_->params, p.data(), p.size() * sizeof(float), cudaMemcpyHostToDevice));
}

// ----------------------------------------------------------------- named tensors (tests)
namespace {
template <typename T>
std::vector<T> d2h(const T* p, int64_t n) {
    std::vector<T> v(static_cast<size_t>(n));
    if (n) FLW_CUDA(cudaMemcpy(v.data(), p, static_cast<size_t>(n) * sizeof(T), cudaMemcpyDeviceToHost));
    return v;
}
template <typename T>
void h2d(T* p, const std::vector<T>& v) {
    if (!v.empty()) FLW_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}
}  // namespace

int64_t Engine::tensor_size(const std::string& n) const {
    const int64_t S = shape_.obs_dim, A = shape_.n_actions;
    if (mappo_) {  // MAPPO layouts (programs.cpp:349-454)
        const int64_t W = shape_.state_w, C = shape_.crit_in, na = shape_.n_agents;
        if (n == "reset_obs" || n == "state_in") return E_ * W;
        if (n == "logits") return R_ * A;
        if (n == "pa") return R_ * 2;
        if (n == "envstep") return E_ * (W + na + 1);
        if (n == "sample") return TR_ * (S + 4 + 2 * C);
    }
    if (n == "reset_obs" || n == "state_in") return E_ * S;
    if (n == "logits") return E_ * A;
    if (n == "pa") return E_ * 2;
    if (n == "envstep") return E_ * (S + 2);
    if (n == "sample") return TR_ * (2 * S + 4);
    if (n == "values" || n == "adv" || n == "ret") return TR_;
    if (n == "last_value") return R_;
    if (n == "logits_new" || n == "dlogits") return TR_ * A;
    if (n == "loss") return 1;
    if (n == "grads") return shape_.P;
    if (n == "env_state") return E_ * shape_.env_state_w;
    if (n == "env_full") return E_ * (shape_.env_state_w + 2);  // [env state | done | step count]
    return -1;
}

void Engine::read_tensor(const std::string& n, double* out) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    Bufs& b = *b_;
    const int64_t S = shape_.obs_dim, A = shape_.n_actions, L = shape_.L;
    auto put = [&](const auto& v) {
        for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<double>(v[i]);
    };
    const int64_t last = std::max<int64_t>(cur_step_ - 1, 0);
    if (mappo_) {
        const int64_t W = shape_.state_w, C = shape_.crit_in, na = shape_.n_agents;
        if (n == "reset_obs") return put(d2h(b.joint, E_ * W));
        if (n == "state_in") return put(d2h(b.joint + cur_step_ * E_ * W, E_ * W));
        if (n == "logits") return put(d2h(b.logits, R_ * A));
        if (n == "pa") {
            auto act = d2h(b.actions + last * R_, R_);
            auto lp = d2h(b.logp + last * R_, R_);
            for (int64_t r = 0; r < R_; ++r) {
                out[2 * r] = act[static_cast<size_t>(r)];
                out[2 * r + 1] = lp[static_cast<size_t>(r)];
            }
            return;
        }
        if (n == "envstep") {  // [joint | per-agent rewards | done] (programs.cpp:366-367)
            auto obs = d2h(b.joint + (last + 1) * E_ * W, E_ * W);
            auto rw = d2h(b.rew + last * R_, R_);
            auto dn = d2h(b.done_f + last * R_, R_);
            const int64_t ow = W + na + 1;
            for (int64_t e = 0; e < E_; ++e) {
                for (int64_t j = 0; j < W; ++j) out[e * ow + j] = obs[static_cast<size_t>(e * W + j)];
                for (int64_t a = 0; a < na; ++a) out[e * ow + W + a] = rw[static_cast<size_t>(a * E_ + e)];
                out[e * ow + W + na] = dn[static_cast<size_t>(e)];
            }
            return;
        }
        if (n == "sample") {  // rows_state | action | reward | ci | nci | done | logp (programs.cpp:410-411)
            auto st = d2h(b.states, TR_ * S);
            // critic input rows [joint(t,e) | onehot(a)] rebuilt from the compact joint blocks
            const int64_t Wj = C - shape_.n_agents;
            auto jt = d2h(b.joint, (T_ + 1) * E_ * Wj);
            std::vector<double> ci(static_cast<size_t>((T_ + 1) * R_ * C), 0.0);
            for (int64_t blk = 0; blk <= T_; ++blk)
                for (int64_t a = 0; a < shape_.n_agents; ++a)
                    for (int64_t e = 0; e < E_; ++e) {
                        double* crow = ci.data() + ((blk * R_) + a * E_ + e) * C;
                        for (int64_t j = 0; j < Wj; ++j) crow[j] = jt[static_cast<size_t>((blk * E_ + e) * Wj + j)];
                        crow[Wj + a] = 1.0;
                    }
            auto act = d2h(b.actions, TR_);
            auto rw = d2h(b.rew, TR_);
            auto dn = d2h(b.done_f, TR_);
            auto lp = d2h(b.logp, TR_);
            const int64_t wd = S + 4 + 2 * C;
            for (int64_t i = 0; i < TR_; ++i) {
                double* row = out + i * wd;
                int64_t c = 0;
                for (int64_t j = 0; j < S; ++j) row[c++] = st[static_cast<size_t>(i * S + j)];
                row[c++] = act[static_cast<size_t>(i)];
                row[c++] = rw[static_cast<size_t>(i)];
                for (int64_t j = 0; j < C; ++j) row[c++] = ci[static_cast<size_t>(i * C + j)];
                for (int64_t j = 0; j < C; ++j) row[c++] = ci[static_cast<size_t>((i + R_) * C + j)];
                row[c++] = dn[static_cast<size_t>(i)];
                row[c++] = lp[static_cast<size_t>(i)];
            }
            return;
        }
    }
    if (n == "reset_obs") return put(d2h(b.states, E_ * S));
    if (n == "state_in") return put(d2h(b.states + cur_step_ * E_ * S, E_ * S));
    const bool fast = numerics_ == Numerics::Fast;
    if (fast && (n == "logits" || n == "logits_new" || n == "dlogits"))
        fail(Errc::Config, "tensor '" + n + "' is only materialised by numerics=exact (fused away in fast)");
    if (n == "logits") return put(d2h(b.logits, E_ * A));
    if (n == "values") return put(d2h(b.values, TR_));
    if (n == "last_value") return put(d2h(b.last_value, R_));
    if (n == "adv" && fast) {  // fast keeps raw GAE advantages; normalised on the fly by the loss
        auto raw = d2h(b.adv, TR_);
        auto st = d2h(b.stats, 2);
        const bool norm = cfg_.normalize_adv && !(st[1] < 1e-8);
        for (int64_t i = 0; i < TR_; ++i)
            out[i] = norm ? static_cast<float>((raw[static_cast<size_t>(i)] - st[0]) / (st[1] + 1e-8))
                          : raw[static_cast<size_t>(i)];
        return;
    }
    if (n == "adv") return put(d2h(b.adv, TR_));
    if (n == "ret") return put(d2h(b.ret, TR_));
    if (n == "logits_new") return put(d2h(b.Hp[L - 1], TR_ * A));
    if (n == "dlogits") return put(d2h(b.DZp[L - 1], TR_ * A));
    if (n == "loss") {
        if (fast) {  // reduce the last learn launch's per-CTA loss partials now
            fast_reduce_loss(stream_, b.loss_parts, b.lgrid_p, b.lgrid_c, cfg_.entropy_coef, b.loss);
            FLW_CUDA(cudaStreamSynchronize(stream_));
        }
        return put(d2h(b.loss, 1));
    }
    if (n == "grads") return put(d2h(b.grads, shape_.P));
    if (n == "pa" || n == "envstep") {
        auto act = d2h(b.actions + last * E_, E_);
        auto lp = d2h(b.logp + last * E_, E_);
        if (n == "pa") {
            for (int64_t e = 0; e < E_; ++e) {
                out[2 * e] = act[static_cast<size_t>(e)];
                out[2 * e + 1] = lp[static_cast<size_t>(e)];
            }
            return;
        }
        auto obs = d2h(b.states + (last + 1) * E_ * S, E_ * S);
        auto rw = d2h(b.rew + last * E_, E_);
        auto dn = d2h(b.done_f + last * E_, E_);
        for (int64_t e = 0; e < E_; ++e) {
            for (int64_t j = 0; j < S; ++j) out[e * (S + 2) + j] = obs[static_cast<size_t>(e * S + j)];
            out[e * (S + 2) + S] = rw[static_cast<size_t>(e)];
            out[e * (S + 2) + S + 1] = dn[static_cast<size_t>(e)];
        }
        return;
    }
    if (n == "sample") {  // [T*E, 2S+4] = state | action | reward | next | done | logp (programs.cpp:229-230)
        auto st = d2h(b.states, (T_ + 1) * E_ * S);
        auto act = d2h(b.actions, TR_);
        auto rw = d2h(b.rew, TR_);
        auto dn = d2h(b.done_f, TR_);
        auto lp = d2h(b.logp, TR_);
        const int64_t W = 2 * S + 4;
        for (int64_t i = 0; i < TR_; ++i) {
            double* row = out + i * W;
            for (int64_t j = 0; j < S; ++j) row[j] = st[static_cast<size_t>(i * S + j)];
            row[S] = act[static_cast<size_t>(i)];
            row[S + 1] = rw[static_cast<size_t>(i)];
            for (int64_t j = 0; j < S; ++j) row[S + 2 + j] = st[static_cast<size_t>((i + E_) * S + j)];
            row[2 * S + 2] = dn[static_cast<size_t>(i)];
            row[2 * S + 3] = lp[static_cast<size_t>(i)];
        }
        return;
    }
    if (n == "env_state" || n == "env_full") {
        const int64_t sw = shape_.env_state_w, w = n == "env_full" ? sw + 2 : sw;
        auto est = d2h(b.est, E_ * sw);
        auto dn = d2h(b.done, E_);
        auto sc = d2h(b.stepc, E_);
        for (int64_t e = 0; e < E_; ++e) {
            for (int64_t j = 0; j < sw; ++j) out[e * w + j] = est[static_cast<size_t>(j * E_ + e)];
            if (w > sw) {
                out[e * w + sw] = dn[static_cast<size_t>(e)];
                out[e * w + sw + 1] = sc[static_cast<size_t>(e)];
            }
        }
        return;
    }
    fail(Errc::Config, "unknown tensor '" + n + "'");
}

void Engine::write_tensor(const std::string& n, const double* in, int64_t cnt) {
    FLW_CUDA(cudaSetDevice(device_));
    FLW_CUDA(cudaStreamSynchronize(stream_));
    if (cnt != tensor_size(n)) fail(Errc::Shape, "tensor '" + n + "' expects " + std::to_string(tensor_size(n)));
    if (mappo_) fail(Errc::Config, "teacher forcing is not implemented for MAPPO layouts");
    Bufs& b = *b_;
    const int64_t S = shape_.obs_dim;
    auto f = [&](int64_t off, int64_t len, int64_t stride = 1) {
        std::vector<float> v(static_cast<size_t>(len));
        for (int64_t i = 0; i < len; ++i) v[static_cast<size_t>(i)] = static_cast<float>(in[off + i * stride]);
        return v;
    };
    if (n == "state_in") return h2d(b.states + cur_step_ * E_ * S, f(0, E_ * S));
    if (n == "env_full") {  // teacher forcing of the env state (SoA on the device)
        const int64_t sw = shape_.env_state_w, w = sw + 2;
        std::vector<double> est(static_cast<size_t>(E_ * sw));
        std::vector<uint8_t> dn(static_cast<size_t>(E_));
        std::vector<int32_t> sc(static_cast<size_t>(E_));
        for (int64_t e = 0; e < E_; ++e) {
            for (int64_t j = 0; j < sw; ++j) est[static_cast<size_t>(j * E_ + e)] = in[e * w + j];
            dn[static_cast<size_t>(e)] = static_cast<uint8_t>(in[e * w + sw] != 0.0);
            sc[static_cast<size_t>(e)] = static_cast<int32_t>(in[e * w + sw + 1]);
        }
        h2d(b.est, est);
        h2d(b.done, dn);
        h2d(b.stepc, sc);
        return;
    }
    if (n == "sample") {  // teacher forcing of the learn batch
        const int64_t W = 2 * S + 4;
        std::vector<float> st(static_cast<size_t>((T_ + 1) * E_ * S)), rw(TR_), dn(TR_), lp(TR_);
        std::vector<int32_t> act(static_cast<size_t>(TR_));
        for (int64_t i = 0; i < TR_; ++i) {
            const double* row = in + i * W;
            for (int64_t j = 0; j < S; ++j) st[static_cast<size_t>(i * S + j)] = static_cast<float>(row[j]);
            act[static_cast<size_t>(i)] = static_cast<int32_t>(row[S] + 0.5);
            rw[static_cast<size_t>(i)] = static_cast<float>(row[S + 1]);
            dn[static_cast<size_t>(i)] = static_cast<float>(row[2 * S + 2]);
            lp[static_cast<size_t>(i)] = static_cast<float>(row[2 * S + 3]);
        }
        for (int64_t e = 0; e < E_; ++e)  // last_next = next-state column of the last E rows
            for (int64_t j = 0; j < S; ++j)
                st[static_cast<size_t>((TR_ + e) * S + j)] = static_cast<float>(in[(TR_ - E_ + e) * W + S + 2 + j]);
        h2d(b.states, st);
        h2d(b.actions, act);
        h2d(b.rew, rw);
        h2d(b.done_f, dn);
        h2d(b.logp, lp);
        return;
    }
    fail(Errc::Config, "tensor '" + n + "' is not writable");
}

}  // namespace flw
