// The B200 DP-D unit engine: one instance owns one fused-loop replica (the reference's
// run_unit + Interp over the fused fragment, local_run.cpp:367-501 / interp.hpp:34-115) with
// ALL of its state resident in HBM: parameters, Adam moments, env state (SoA), trajectory,
// activations. The host only drives phases (or replays a captured CUDA graph per episode) and
// reads back per-episode scalars.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "config.hpp"

namespace flw {

struct FastUpdateArgs;  // fast.cuh
struct P2pArgs;         // p2p.cuh

enum class Numerics : int {
    Exact = 0,  // FP64-accumulate CUDA-core path, bit-exact with the reference's per-op f32 rounding
    Fast = 1,   // tensor-core (tcgen05) path, fp32 accumulate, tolerance-checked
};

struct DeviceCtx {      // device-resident episode context (read by kernels inside captured graphs)
    int64_t episode;
    int64_t next_episode;  // consumed by the graph's first node, so replays can be queued back to back
    int64_t adam_t;
    double bc1, bc2;    // Adam bias corrections 1 - beta^t, from a host-computed table
    uint64_t coll_seq;  // peer-memory exchange epoch: monotonically increasing, never reset
    uint64_t runs;      // episode graphs completed (k_publish_rsum's ring slot), never reset
};

class Comm;  // NCCL gradient group (comm.hpp)
struct WideNet;  // layer-wise learn path net description (wide.cuh)

class Engine {
  public:
    // `replicas` > 1 folds that many consecutive units (reference replicas with contiguous env
    // ranges split like split_envs, plan.cpp:46-55) into this engine: each keeps its own
    // advantage statistics, loss mean, gradient and reward sum; gradients are averaged in unit
    // order (local_run.cpp:408-411) before Adam.
    Engine(const AlgoConfig& cfg, int device, uint64_t seed, int64_t env_lo, int64_t env_hi, int64_t env_total,
           Numerics numerics, int replicas = 1);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Gradient group (GradSync): rank = unit id, nranks = k. Takes ownership.
    void set_comm(std::unique_ptr<Comm> comm);
    Comm* comm() { return comm_.get(); }
    // Peer-memory gradient exchange (fast numerics, k GPUs): this rank's exchange region, and
    // the regions of all k ranks as mapped into this process (own entry included). When set,
    // reduce + all-reduce + Adam run as one kernel (kernels_p2p.cu) instead of NCCL.
    void* p2p_region();
    int64_t p2p_region_bytes() const;
    void alloc_p2p_region(int k);  // before p2p_region(): the layout depends on k
    void adopt_ipc_mapping(void* p) { p2p_ipc_opened_.push_back(p); }  // closed by the destructor
    // peers_elsewhere: every other rank's region lives on another GPU (the one-kernel exchange
    // and the split update are then allowed; co-located ranks use the two-kernel form)
    void set_p2p_peers(int rank, int k, const std::vector<void*>& regions, bool peers_elsewhere);
    bool p2p_enabled() const { return p2p_k_ > 1; }
    bool p2p_capable() const { return numerics_ == Numerics::Fast && nrep_ == 1 && !cfast_ && !wide_; }
    void disable_p2p() {  // back to the NCCL exchange (the group must agree; see bench.py)
        destroy_graph();
        p2p_k_ = 0;
    }
    void set_eager_collectives(bool on);
    // Bounded waits (reference: channel receive timeouts, local_run.cpp:543-546): a grouped
    // unit's episode / learn call fails with Timeout after timeout_ms and aborts its group.
    void set_timeout_ms(int64_t ms) { timeout_ms_ = ms > 0 ? ms : 30000; }
    int64_t timeout_ms() const { return timeout_ms_; }
    // Sets the group abort word (peer-memory flag waits give up) and aborts the NCCL group.
    void abort_group();
    bool grouped() const;
    void prepare();  // captures the episode graph now (before any peer launches its own)

    // Phase-level API (each enqueues on the engine stream and synchronises before returning).
    void reset(int64_t ep);
    void step(int64_t ep, int64_t st);
    void learn_grads(int64_t ep, int64_t k);       // up to GradCompute (flat f32 gradient)
    void apply_grads(const double* host_grads);     // OptimStep on given (already synced) grads
    void learn(int64_t ep, int64_t k);              // grads + GradSync + Adam

    // Whole episode: Reset, T x Step, I x Learn as one captured CUDA graph. Returns the
    // episode reward sum (sum over this unit's envs, interp.cpp:257) and the device time.
    double run_episode(int64_t ep, float* device_ms = nullptr);
    // Pipelined episodes (flw_run_local on one GPU, flw_dpd_launch/finish_episode): launch_episode
    // enqueues episode ep (its index, the episode graph, an async copy of its reward sums into a
    // pinned slot); finish_episode waits for the oldest enqueued episode and returns its
    // per-replica reward sums. At most kInFlight are enqueued, so the host's per-episode gate
    // (wait, read the reward, record the episode) overlaps the next episode on the GPU.
    static constexpr int kInFlight = 2;
    void launch_episode(int64_t ep);
    std::vector<double> finish_episode();
    void drain_episodes();  // after a failure: wait for and discard the in-flight episodes
    // Enqueue `count` episodes starting at `first` back to back (no host sync in between).
    void enqueue_episodes(int64_t first, int64_t count);
    double last_reward_sum();
    // Per-replica reward sums of the last episode, in unit order (exact numerics; fast numerics
    // report the unit total in slot 0).
    std::vector<double> replica_reward_sums();
    int replicas() const { return nrep_; }
    void sync();
    cudaStream_t stream() const { return stream_; }

    int64_t param_count() const { return shape_.P; }
    // Fresh run on the same buffers: re-initialised params (new seed), Adam state and counters.
    void reinit(uint64_t seed);
    void get_params(double* out);
    void set_params(const double* in);
    int64_t steps_executed() const { return steps_; }
    int64_t env_count() const { return E_; }
    int64_t learn_iters() const { return shape_.learn_iters; }
    const ProgramShape& shape() const { return shape_; }
    Numerics numerics() const { return numerics_; }
    int device() const { return device_; }

    // Named tensors for parity tests (same names as the oracle): reset_obs, state_in, logits,
    // pa, envstep, sample, values, last_value, adv, ret, logits_new, loss, grads, dlogits,
    // env_state. Values are returned as doubles in the reference's row-major layouts.
    int64_t tensor_size(const std::string& name) const;
    void read_tensor(const std::string& name, double* out);
    void write_tensor(const std::string& name, const double* in, int64_t n);

    // Launch statistics of the last captured episode graph (kernel nodes).
    int64_t graph_kernel_nodes() const { return graph_kernels_; }

    // CUDA-event probes around the main kernels, recorded inside the episode graph.
    void enable_probes(bool on);
    std::string probe_times_json();

  private:
    struct Bufs;
    void alloc();
    void init_params(bool moments = false);
    void set_episode(int64_t ep);
    void enq_reset(bool begin = false);
    void enq_step(int64_t st);
    void enq_rollout_fast(int64_t step0, int64_t nsteps);
    bool enq_rollout_fast_mappo(int64_t step0, int64_t nsteps);
    void enq_learn_fast();
    void alloc_wide();
    void setup_wide_net(int net, WideNet& n) const;
    void alloc_split_rollout();
    void alloc_wide_policy(int64_t xrows, int maxw);
    void enq_policy_fwd_split(int64_t st);
    void enq_step_env(int64_t st);
    void wide_forward(const WideNet& n, const __nv_bfloat16* wb, const std::vector<__nv_bfloat16*>& H,
                      const std::vector<int64_t>& ld, int64_t rows, float* out);
    void wide_backward(const WideNet& n, const __nv_bfloat16* wb, const std::vector<__nv_bfloat16*>& H,
                       const std::vector<int64_t>& ld, float* part, int64_t pstride);
    void wide_loss_rows(int kind, const float* out, int A, float* loss_partials);
    void enq_learn_policy_wide(float* loss_partials);
    void enq_learn_wide();
    void enq_learn_grads();
    void enq_grad_sync_and_adam();
    void enq_reward_sum();
    void enq_mlp_forward(int net, const float* X, int64_t M, float* const* H, int first_layer = 0);
    void build_graph();
    void wait_stream(const char* what);
    void wait_event(cudaEvent_t ev, const char* what);  // bounded like wait_stream (grouped units)
    unsigned* abort_h_ = nullptr;  // host-mapped group abort word (host view)
    unsigned* abort_d_ = nullptr;  // ... device view
    int64_t timeout_ms_ = 30000;

    AlgoConfig cfg_;
    ProgramShape shape_;
    int device_;
    uint64_t seed_;
    int64_t lo_, hi_, etot_, E_, R_, T_, TR_;
    bool mappo_ = false;   // agent-major rows R = n*E, critic on [joint obs | agent one-hot]
    bool cfast_ = false;   // fast MAPPO with the compact critic (critic input > 64 wide)
    bool wide_ = false;    // fast numerics, a layer > 64 wide: layer-wise tcgen05 GEMM learn path
    bool pwide_ = false;   // fast MAPPO, policy hidden > 64: layer-wise policy learn
    bool pcompact_ = false;  // fast MAPPO, observation > 64, hidden <= 64: layer 0 on GEMMs
    bool gemm_roll_ = false;  // fast numerics: rollout policy forward as split-f16 GEMMs
    int p2p_rank_ = 0, p2p_k_ = 0;
    bool p2p_fused_ = false;  // every peer region on another GPU: the one-kernel exchange
    void* p2p_region_ptr_ = nullptr;
    int p2p_alloc_k_ = 0;
    std::vector<void*> p2p_ipc_opened_;
    uint8_t** p2p_peers_dev_ = nullptr;
    int nrep_ = 1;                          // replicas folded into this engine
    std::vector<int64_t> rep_off_, rep_n_;  // replica env offset (relative to lo_) and size
    void enq_permute_replicas();
    Numerics numerics_;
    cudaStream_t stream_ = nullptr, side_ = nullptr, side2_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_t0_ = nullptr, ev_t1_ = nullptr;
    cudaEvent_t ev_wimg_ = nullptr;  // the episode's first weight images, built on side_ (build_graph)
    bool wimg_early_ = false;        // ... so the first train iteration does not build them
    double* rs_pinned_ = nullptr;                  // [kInFlight][nrep_] reward sums of in-flight episodes
    cudaEvent_t ev_done_[kInFlight] = {};          // per slot: the episode and its reward copy finished
    int64_t fl_head_ = 0, fl_tail_ = 0;            // pipelined episodes launched / finished
    int64_t next_ep_dev_ = -1;  // ctx->next_episode once the enqueued work has run (-1: unknown)
    int64_t graph_runs_ = 0;    // episode graphs launched (= ctx->runs once they have run)
    int64_t fl_slot_[kInFlight] = {};  // ring slot (graph_runs_ % kInFlight) of each in-flight episode
    double* rs_ring_d_ = nullptr;      // device address of the mapped reward ring (rs_pinned_)
    cudaEvent_t ev_lfork_ = nullptr, ev_ljoin_ = nullptr;  // policy || critic learn fork/join
    std::unique_ptr<Bufs> b_;
    std::unique_ptr<Comm> comm_;
    cudaGraphExec_t graph_ = nullptr;  // == segs_[0]
    // Single-process multi-GPU: the collectives are issued eagerly between graph segments
    // (NCCL >= 2.28 cannot capture collectives of several communicators of one process).
    bool eager_coll_ = false;
    std::vector<cudaGraphExec_t> segs_;
    std::vector<std::function<void()>> between_;
    int64_t graph_kernels_ = 0;
    void destroy_graph();
    void segment_break(std::function<void()> op);
    void end_segment();
    void trace_capture(const char* where);
    void launch_graph();
    int64_t steps_ = 0;
    int64_t cur_step_ = 0;      // index of the trajectory block holding the current policy input

    struct Probe {
        std::string tag;
        cudaEvent_t a, b;
    };
    bool probes_on_ = false;
    bool capturing_ = false;
    // fast numerics, 1 GPU: the train iteration's update as one fused launch (k_reduce_adam)
    int64_t learn_iter_ = 0;      // train iteration being enqueued (0: weight images rebuilt)
    bool fuse_ok_ = false;        // enq_grad_sync_and_adam follows the learn being enqueued
    bool fused_pending_ = false;  // the learn left its partials for k_reduce_adam
    bool prev_fused_ = false;     // the last update also refreshed the weight images
    bool split_done_ = false;     // this iteration's critic update already ran (enq_critic_update)
    // Train-iteration pipelining (graph build only): another iteration follows this one, and
    // the next iteration's values pass + GAE are already enqueued on side2_ (ev_gae_)
    bool pipe_next_ok_ = false, vg_ready_ = false;
    cudaEvent_t ev_plearn_ = nullptr, ev_gae_ = nullptr;
    FastUpdateArgs update_args() const;
    P2pArgs p2p_args() const;
    bool split_update_ok() const;
    bool pdl_ok() const;
    void enq_critic_update(cudaStream_t st, int ncrit);
    std::vector<Probe> probes_;
    int open_probe_ = -1;
    void probe_begin(const char* tag);
    void probe_end();
    void clear_probes();
};

}  // namespace flw
