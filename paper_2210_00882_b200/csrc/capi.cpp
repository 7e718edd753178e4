// C-ABI of libfraglow_b200.so (include/fraglow_b200.h): the reference's public API for the
// DP-D path plus the per-unit engine seam. Conventions follow /root/reference/proj/src/capi.cpp:
// guarded() maps exceptions to codes, thread-local last error, malloc'd out strings.
#include <cuda_runtime.h>

#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

#include "../../include/fraglow_b200.h"
#include "comm.hpp"
#include "common.cuh"
#include "config.hpp"
#include "engine.hpp"
#include "nlohmann/json.hpp"

using namespace flw;

namespace flw {
int umma_selftest(int M, int N, int K, int a_mn, int b_mn, int lane_off, const float* A, const float* B, float* D);
}

struct flw_program {
    AlgoConfig algo;
    DeployConfig deploy;
    Plan plan;
    Numerics numerics = Numerics::Exact;
    int reps_per_gpu = 0;  // deploy "replicas_per_gpu": units folded per engine (0: only when k > #GPUs)
    std::string exchange = "p2p";  // deploy "exchange": gradient exchange of fast numerics, "p2p" | "nccl"
    // Engines persist across flw_run_local calls on the same program (re-initialised per run):
    // device buffers and the captured episode graph are set up once.
    std::vector<std::unique_ptr<Engine>> engines;
    bool unpartitioned_engines = false;
    std::mutex mu;
};

struct flw_dpd {
    std::unique_ptr<Engine> engine;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        g_last_error = std::string(errc_name(e.code())) + ": " + e.what();
        return c_code(e.code());
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FLW_ERR_RUNTIME;
    }
}

char* dup_string(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

Numerics numerics_from(const std::string& s) {
    if (s == "exact") return Numerics::Exact;
    if (s == "fast") return Numerics::Fast;
    fail(Errc::Config, "numerics must be 'exact' or 'fast'");
}

struct EpisodeMetrics {
    double wall_ms = 0.0, reward = 0.0;
    int64_t bytes_total = 0;
};

// capi.cpp:74-113 summary schema.
// The bytes the GPU gradient exchange really moves (all ranks, NVLink), next to the reference's
// message accounting in bytes_total: kind "p2p" (each rank stores its f32 gradient
// into every peer's inbox), "nccl_allreduce" (ring: 2(k-1)/k of the vector per rank) or
// "nccl_allgather" (exact numerics: every rank receives the other ranks' R unit gradients).
struct DeviceExchange {
    std::string kind = "none";
    int64_t bytes_per_episode = 0;
};

std::string summarize(const std::vector<EpisodeMetrics>& eps, int64_t steps, const std::vector<double>& params,
                      int64_t grad_bytes_total, const flw_run_options* opts, const DeviceExchange& dx) {
    nlohmann::ordered_json j;
    j["episodes"] = eps.size();
    j["steps"] = steps;
    j["grad_messages"] = 0;  // DP-D has no async gradient pushes (local_run.cpp:447-456)
    j["final_reward"] = eps.empty() ? 0.0 : eps.back().reward;
    double total_ms = 0.0;
    for (const auto& e : eps) total_ms += e.wall_ms;
    j["total_wall_ms"] = total_ms;
    j["bytes_total"] = grad_bytes_total;
    nlohmann::ordered_json per = nlohmann::ordered_json::object();
    if (grad_bytes_total > 0) per["0"] = grad_bytes_total;
    j["bytes_per_channel"] = per;
    nlohmann::ordered_json dev;
    dev["kind"] = dx.kind;
    dev["bytes_per_episode"] = dx.bytes_per_episode;
    dev["bytes_total"] = dx.bytes_per_episode * static_cast<int64_t>(eps.size());
    j["device_exchange"] = dev;
    double sum = 0.0, sumsq = 0.0;
    for (double v : params) {
        sum += v;
        sumsq += v * v;
    }
    j["param_count"] = params.size();
    j["param_checksum"] = sum;
    j["param_l2"] = std::sqrt(sumsq);
    if (opts && opts->reward_threshold >= 0.0) {
        double t = -1.0, acc = 0.0;
        for (const auto& e : eps) {
            acc += e.wall_ms;
            if (e.reward >= opts->reward_threshold) {
                t = acc;
                break;
            }
        }
        j["reward_threshold"] = opts->reward_threshold;
        j["time_to_threshold_ms"] = t;
    }
    return j.dump(2);
}

std::string to_csv(const std::vector<EpisodeMetrics>& eps) {  // local_run.cpp:503-510
    std::ostringstream os;
    os << "episode,wall_ms,reward,bytes_total\n";
    for (size_t i = 0; i < eps.size(); ++i)
        os << i << "," << eps[i].wall_ms << "," << eps[i].reward << "," << eps[i].bytes_total << "\n";
    return os.str();
}

// run_plan_local (local_run.cpp:512-581) for a DP-D plan: one host thread per unit, each unit
// on its own GPU, an episode lockstep gate driven by this thread, wall_ms per episode.
void run_local(flw_program& p, const flw_run_options* opts, std::vector<EpisodeMetrics>& eps, int64_t& steps,
               std::vector<double>& final_params, int64_t& grad_bytes, DeviceExchange& dx) {
    std::lock_guard<std::mutex> lk(p.mu);
    const uint64_t seed = opts ? opts->seed : 0;
    const int64_t episodes = opts && opts->episodes > 0 ? opts->episodes : p.algo.episodes;
    const bool unpart = opts && opts->unpartitioned;
    std::vector<Unit> units = p.plan.units;
    if (unpart) units = {Unit{0, 0, 0, 0, p.algo.envs}};
    const int k = static_cast<int>(units.size());
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        fail(Errc::Runtime, "no CUDA device visible: the DP-D engine has no CPU fallback");
    // One engine per GPU. More units than GPUs fold R = k / #GPUs consecutive units into each
    // engine (each keeps its own statistics, loss mean, gradient and reward sum).
    int R = 1;
    if (p.reps_per_gpu > 0) {
        R = p.reps_per_gpu;
        if (k % R != 0 || k / R > ndev)
            fail(Errc::InsufficientSlots, "replicas_per_gpu=" + std::to_string(R) + " does not fold " +
                                              std::to_string(k) + " units onto " + std::to_string(ndev) + " GPUs");
    } else if (k > ndev) {
        if (k % ndev != 0)
            fail(Errc::InsufficientSlots, "dp-d plan has " + std::to_string(k) + " units but " + std::to_string(ndev) +
                                              " GPUs are visible: folding needs k to be a multiple of the GPU count");
        R = k / ndev;
    }
    const int ng = k / R;
    bool reuse = static_cast<int>(p.engines.size()) == ng && p.unpartitioned_engines == unpart &&
                 (ng == 0 || p.engines[0]->replicas() == R);
    if (!reuse) {
        p.engines.clear();
        for (int g = 0; g < ng; ++g) {
            const Unit& first = units[static_cast<size_t>(g * R)];
            const Unit& last = units[static_cast<size_t>(g * R + R - 1)];
            p.engines.push_back(std::make_unique<Engine>(p.algo, g, seed, first.env_lo, last.env_hi, p.algo.envs,
                                                         p.numerics, R));
        }
        p.unpartitioned_engines = unpart;
        if (ng > 1) {
            std::vector<int> devs;
            for (int g = 0; g < ng; ++g) devs.push_back(g);
            auto comms = Comm::init_all(devs);
            std::vector<Comm*> cs;
            for (int g = 0; g < ng; ++g) {
                auto c = std::make_unique<Comm>(comms[g], g, ng);
                cs.push_back(c.get());
                p.engines[g]->set_eager_collectives(true);
                p.engines[g]->set_comm(std::move(c));
            }
            Comm::connect_all(cs, devs, static_cast<int64_t>(R) * p.engines[0]->shape().P);
            // fast numerics, one unit per GPU: gradient exchange over NVLink peer memory when
            // every pair of GPUs can address each other (deploy "exchange": "nccl" opts out)
            bool p2p = p.exchange != "nccl";
            for (auto& e : p.engines) p2p = p2p && e->p2p_capable();
            for (int a = 0; p2p && a < ng; ++a)
                for (int b2 = 0; p2p && b2 < ng; ++b2) {
                    int ok = 0;
                    if (a != b2 && (cudaDeviceCanAccessPeer(&ok, a, b2) != cudaSuccess || !ok)) p2p = false;
                }
            if (p2p) {
                std::vector<void*> regions;
                for (int g = 0; g < ng; ++g) {
                    p.engines[g]->alloc_p2p_region(ng);
                    regions.push_back(p.engines[g]->p2p_region());
                }
                for (int g = 0; g < ng; ++g) {
                    FLW_CUDA(cudaSetDevice(g));
                    for (int h = 0; h < ng; ++h)
                        if (h != g) {
                            cudaError_t err = cudaDeviceEnablePeerAccess(h, 0);
                            if (err == cudaErrorPeerAccessAlreadyEnabled)
                                cudaGetLastError();
                            else
                                FLW_CUDA(err);
                        }
                    p.engines[g]->set_p2p_peers(g, ng, regions, true);  // one engine per GPU
                }
            }
        }
    } else {
        for (auto& e : p.engines) e->reinit(seed);
    }
    for (auto& e : p.engines) e->set_timeout_ms(opts ? opts->timeout_ms : 0);  // 0: 30 s (fraglow.h:36)
    eps.assign(static_cast<size_t>(episodes), {});
    // reward sum of every unit and episode, folded in unit order below (local_run.cpp:560-570)
    std::vector<std::vector<double>> rsum(static_cast<size_t>(k), std::vector<double>(episodes, 0.0));
    const ProgramShape& s = p.engines[0]->shape();
    // Reference byte accounting of the GradSync channel: k(k-1) legs x learn iters x (14 + 8P).
    const int64_t per_ep_bytes = k > 1 ? static_cast<int64_t>(k) * (k - 1) * s.learn_iters * (14 + 8 * s.P) : 0;
    std::mutex err_mu;
    std::string first_error;          // guarded by err_mu
    std::atomic<bool> failed{false};  // lock-free "a unit failed" for the worker fast path
    auto run_one = [&](int g, int64_t ep) {
        p.engines[g]->run_episode(ep);
        const std::vector<double> v = p.engines[g]->replica_reward_sums();
        for (int r = 0; r < R; ++r) rsum[static_cast<size_t>(g * R + r)][static_cast<size_t>(ep)] = v[static_cast<size_t>(r)];
    };
    if (ng == 1) {
        // One GPU, no gradient group: the episode gate is pipelined - episode ep + 1 is already
        // enqueued while the host waits for episode ep and records its reward (same episode
        // order and results; wall_ms = time between consecutive episode completions).
        Engine& e0 = *p.engines[0];
        try {
            auto t_prev = std::chrono::steady_clock::now();
            if (episodes > 0) e0.launch_episode(0);
            for (int64_t ep = 0; ep < episodes; ++ep) {
                if (ep + 1 < episodes) e0.launch_episode(ep + 1);
                const std::vector<double> v = e0.finish_episode();
                for (int r = 0; r < R; ++r) rsum[static_cast<size_t>(r)][static_cast<size_t>(ep)] = v[static_cast<size_t>(r)];
                const auto t1 = std::chrono::steady_clock::now();
                eps[static_cast<size_t>(ep)].wall_ms = std::chrono::duration<double, std::milli>(t1 - t_prev).count();
                t_prev = t1;
            }
        } catch (...) {
            e0.drain_episodes();
            throw;
        }
    } else {
        // Every engine's episode graph segments are captured before any engine launches.
        for (auto& e : p.engines) e->prepare();
        std::barrier gate(ng + 1);
        std::vector<std::thread> threads;
        for (int g = 0; g < ng; ++g)
            threads.emplace_back([&, g] {
                for (int64_t ep = 0; ep < episodes; ++ep) {
                    gate.arrive_and_wait();  // raise_gate(ep)
                    try {
                        flw_trace(("engine " + std::to_string(g) + " episode " + std::to_string(ep)).c_str());
                        if (!failed.load(std::memory_order_acquire)) run_one(g, ep);
                    } catch (const std::exception& e) {
                        std::lock_guard<std::mutex> lk2(err_mu);
                        if (first_error.empty()) first_error = "unit " + std::to_string(g * R) + ": " + e.what();
                        failed.store(true, std::memory_order_release);
                        // peers may be blocked inside a collective or a peer-memory flag wait
                        // for this unit: abort the whole group (local_run.cpp:79-86)
                        for (auto& en : p.engines) en->abort_group();
                    }
                    gate.arrive_and_wait();  // on_episode_done
                }
            });
        for (int64_t ep = 0; ep < episodes; ++ep) {
            auto t0 = std::chrono::steady_clock::now();
            gate.arrive_and_wait();
            gate.arrive_and_wait();
            auto t1 = std::chrono::steady_clock::now();
            eps[static_cast<size_t>(ep)].wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
        for (auto& t : threads) t.join();
        if (failed.load()) {
            p.engines.clear();  // aborted communicators: rebuild on the next run
            fail(Errc::PeerFailure, first_error);
        }
    }
    for (int64_t ep = 0; ep < episodes; ++ep) {  // local_run.cpp:560-570
        double sum = 0.0;
        for (int r = 0; r < k; ++r) sum += rsum[r][static_cast<size_t>(ep)];
        eps[static_cast<size_t>(ep)].reward = sum / static_cast<double>(p.algo.envs);
        eps[static_cast<size_t>(ep)].bytes_total = per_ep_bytes;
    }
    steps = 0;
    for (auto& e : p.engines) steps += e->steps_executed();
    final_params.assign(static_cast<size_t>(s.P), 0.0);
    p.engines[0]->get_params(final_params.data());
    grad_bytes = per_ep_bytes * episodes;
    dx = DeviceExchange{};
    if (ng > 1) {
        const int64_t P4 = 4 * s.P, I = s.learn_iters;
        const Engine& e0 = *p.engines[0];
        if (e0.numerics() == Numerics::Exact) {
            dx.kind = "nccl_allgather";
            dx.bytes_per_episode = I * static_cast<int64_t>(ng) * (ng - 1) * R * P4;
        } else if (e0.p2p_enabled()) {
            dx.kind = "p2p";  // one 8-byte {value, epoch} word per parameter and peer
            dx.bytes_per_episode = I * static_cast<int64_t>(ng) * (ng - 1) * 2 * P4;
        } else {
            dx.kind = "nccl_allreduce";
            dx.bytes_per_episode = I * 2 * static_cast<int64_t>(ng - 1) * P4;
        }
    }
}

Engine& eng(flw_dpd* e) {
    if (!e || !e->engine) fail(Errc::Config, "null engine handle");
    return *e->engine;
}

}  // namespace

extern "C" {

int flw_program_create(const char* algo_json, const char* deploy_json, flw_program** out) {
    return guarded([&] {
        auto p = std::make_unique<flw_program>();
        p->algo = parse_algo_config(algo_json ? algo_json : "{}");
        if (deploy_json && *deploy_json) {
            p->deploy = parse_deploy_config(deploy_json);
            auto j = nlohmann::json::parse(deploy_json);
            if (j.contains("numerics")) p->numerics = numerics_from(j["numerics"].get<std::string>());
            if (j.contains("replicas_per_gpu")) p->reps_per_gpu = j["replicas_per_gpu"].get<int>();
            if (j.contains("exchange")) p->exchange = j["exchange"].get<std::string>();
        } else {
            p->deploy = DeployConfig{{"local"}, 8, 8, Policy::DpA};  // capi.cpp:211-212 default
        }
        if (const char* env = std::getenv("FLW_NUMERICS")) p->numerics = numerics_from(env);
        p->plan = make_dpd_plan(p->algo, p->deploy);
        *out = p.release();
        return FLW_OK;
    });
}

void flw_program_destroy(flw_program* p) { delete p; }

int flw_algo_from_graph(const char* graph_json, char** out_algo_json) {
    return guarded([&] {
        if (!out_algo_json) fail(Errc::Config, "null output pointer");
        *out_algo_json = dup_string(algo_to_json(algo_from_graph(graph_json ? graph_json : "{}")));
        return FLW_OK;
    });
}

int flw_program_dump(const flw_program* p, int what, char** out_text) {
    return guarded([&] {
        if (what != FLW_DUMP_PLAN)
            fail(Errc::Config, "the DP-D engine serves FLW_DUMP_PLAN only (the DFG/FDG are the reference's)");
        *out_text = dup_string(p->plan.to_json());
        return FLW_OK;
    });
}

int flw_validate_plan(const flw_program* p, char** out_report, int* n_violations) {
    return guarded([&] {
        auto v = p->plan.violations();
        nlohmann::ordered_json j = nlohmann::ordered_json::array();
        for (const auto& [code, msg] : v) j.push_back({{"code", code}, {"message", msg}});
        if (out_report) *out_report = dup_string(j.dump(2));
        if (n_violations) *n_violations = static_cast<int>(v.size());
        return FLW_OK;
    });
}

int flw_run_local(const flw_program* p, const flw_run_options* opts, char** metrics_csv, char** summary_json) {
    return guarded([&] {
        std::vector<EpisodeMetrics> eps;
        int64_t steps = 0, bytes = 0;
        std::vector<double> params;
        DeviceExchange dx;
        run_local(*const_cast<flw_program*>(p), opts, eps, steps, params, bytes, dx);
        if (metrics_csv) *metrics_csv = dup_string(to_csv(eps));
        if (summary_json) *summary_json = dup_string(summarize(eps, steps, params, bytes, opts, dx));
        return FLW_OK;
    });
}

void flw_string_free(char* s) { std::free(s); }

const char* flw_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------------ engine seam
int flw_dpd_create(const char* algo_json, int device, uint64_t seed, int64_t env_lo, int64_t env_hi,
                   int64_t env_total, int numerics, flw_dpd** out) {
    return guarded([&] {
        AlgoConfig a = parse_algo_or_graph(algo_json ? algo_json : "{}");
        if (numerics != FLW_NUMERICS_EXACT && numerics != FLW_NUMERICS_FAST) fail(Errc::Config, "bad numerics");
        auto h = std::make_unique<flw_dpd>();
        h->engine = std::make_unique<Engine>(a, device, seed, env_lo, env_hi, env_total, static_cast<Numerics>(numerics));
        *out = h.release();
        return FLW_OK;
    });
}

int flw_dpd_create_replicas(const char* algo_json, int device, uint64_t seed, int64_t env_lo, int64_t env_hi,
                            int64_t env_total, int numerics, int replicas, flw_dpd** out) {
    return guarded([&] {
        AlgoConfig a = parse_algo_or_graph(algo_json ? algo_json : "{}");
        if (numerics != FLW_NUMERICS_EXACT && numerics != FLW_NUMERICS_FAST) fail(Errc::Config, "bad numerics");
        auto h = std::make_unique<flw_dpd>();
        h->engine = std::make_unique<Engine>(a, device, seed, env_lo, env_hi, env_total, static_cast<Numerics>(numerics),
                                             replicas);
        *out = h.release();
        return FLW_OK;
    });
}

int flw_dpd_replica_rewards(flw_dpd* e, double* out, int64_t cap) {
    return guarded([&] {
        const std::vector<double> v = eng(e).replica_reward_sums();
        if (cap < static_cast<int64_t>(v.size())) fail(Errc::Config, "output buffer too small");
        std::copy(v.begin(), v.end(), out);
        return FLW_OK;
    });
}

int flw_dpd_destroy(flw_dpd* e) {
    return guarded([&] {
        delete e;
        return FLW_OK;
    });
}

int flw_dpd_comm_unique_id(char* out_id, int64_t cap) {
    return guarded([&] {
        std::string id = Comm::new_unique_id();
        if (cap < static_cast<int64_t>(id.size())) fail(Errc::Config, "unique id buffer too small");
        std::memcpy(out_id, id.data(), id.size());
        return FLW_OK;
    });
}

// The exported handle: the region's CUDA IPC handle followed by the exporting GPU's UUID (so an
// importer can tell co-located ranks from ranks on other GPUs).
constexpr int64_t kP2pHandleBytes = static_cast<int64_t>(sizeof(cudaIpcMemHandle_t)) + 16;
static_assert(kP2pHandleBytes == FLW_P2P_HANDLE_BYTES, "fraglow_b200.h FLW_P2P_HANDLE_BYTES");

static void device_uuid(int dev, char* out16) {
    cudaDeviceProp pr{};
    FLW_CUDA(cudaGetDeviceProperties(&pr, dev));
    std::memcpy(out16, &pr.uuid, 16);
}

int flw_dpd_p2p_export(flw_dpd* e, int nranks, char* out_handle, int64_t cap) {
    return guarded([&] {
        Engine& en = eng(e);
        if (cap < kP2pHandleBytes) fail(Errc::Config, "handle buffer too small (FLW_P2P_HANDLE_BYTES)");
        en.alloc_p2p_region(nranks);
        FLW_CUDA(cudaSetDevice(en.device()));
        cudaIpcMemHandle_t h;
        FLW_CUDA(cudaIpcGetMemHandle(&h, en.p2p_region()));
        std::memcpy(out_handle, &h, sizeof(h));
        device_uuid(en.device(), out_handle + sizeof(h));
        return FLW_OK;
    });
}

int flw_dpd_p2p_import(flw_dpd* e, const char* handles, int64_t len, int rank, int nranks) {
    return guarded([&] {
        Engine& en = eng(e);
        const int64_t hb = kP2pHandleBytes;
        if (len != hb * nranks) fail(Errc::Config, "expected nranks exchange handles (FLW_P2P_HANDLE_BYTES each)");
        en.alloc_p2p_region(nranks);
        FLW_CUDA(cudaSetDevice(en.device()));
        char mine[16];
        device_uuid(en.device(), mine);
        bool elsewhere = true;
        std::vector<void*> regions(static_cast<size_t>(nranks), nullptr);
        for (int r = 0; r < nranks; ++r) {
            if (r == rank) {
                regions[static_cast<size_t>(r)] = en.p2p_region();
                continue;
            }
            if (std::memcmp(handles + hb * r + sizeof(cudaIpcMemHandle_t), mine, 16) == 0) elsewhere = false;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + hb * r, sizeof(h));
            void* ptr = nullptr;
            FLW_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            en.adopt_ipc_mapping(ptr);
            regions[static_cast<size_t>(r)] = ptr;
        }
        en.set_p2p_peers(rank, nranks, regions, elsewhere);
        return FLW_OK;
    });
}

int flw_dpd_set_timeout(flw_dpd* e, int64_t timeout_ms) {
    return guarded([&] {
        eng(e).set_timeout_ms(timeout_ms);
        return FLW_OK;
    });
}

int flw_dpd_abort(flw_dpd* e) {
    return guarded([&] {
        eng(e).abort_group();
        return FLW_OK;
    });
}

int flw_dpd_p2p_disable(flw_dpd* e) {
    return guarded([&] {
        eng(e).disable_p2p();
        return FLW_OK;
    });
}

int flw_dpd_comm_init(flw_dpd* e, const char* id, int64_t id_len, int rank, int nranks) {
    return guarded([&] {
        Engine& en = eng(e);
        en.set_comm(std::make_unique<Comm>(std::string(id, static_cast<size_t>(id_len)), rank, nranks, en.device()));
        return FLW_OK;
    });
}

int flw_dpd_run_episode(flw_dpd* e, int64_t episode, double* reward_sum, float* device_ms) {
    return guarded([&] {
        double r = eng(e).run_episode(episode, device_ms);
        if (reward_sum) *reward_sum = r;
        return FLW_OK;
    });
}

int flw_dpd_launch_episode(flw_dpd* e, int64_t episode) {
    return guarded([&] {
        eng(e).launch_episode(episode);
        return FLW_OK;
    });
}

int flw_dpd_finish_episode(flw_dpd* e, double* reward_sum) {
    return guarded([&] {
        double total = 0.0;
        for (double v : eng(e).finish_episode()) total += v;
        if (reward_sum) *reward_sum = total;
        return FLW_OK;
    });
}

int flw_dpd_run_episodes(flw_dpd* e, int64_t first_episode, int64_t count, float* device_ms) {
    return guarded([&] {
        Engine& en = eng(e);
        cudaEvent_t a, b;
        FLW_CUDA(cudaSetDevice(en.device()));
        FLW_CUDA(cudaEventCreate(&a));
        FLW_CUDA(cudaEventCreate(&b));
        FLW_CUDA(cudaEventRecord(a, en.stream()));
        en.enqueue_episodes(first_episode, count);
        FLW_CUDA(cudaEventRecord(b, en.stream()));
        FLW_CUDA(cudaEventSynchronize(b));
        float ms = 0.0f;
        FLW_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (device_ms) *device_ms = ms;
        return FLW_OK;
    });
}

int flw_dpd_reinit(flw_dpd* e, uint64_t seed) {
    return guarded([&] {
        eng(e).reinit(seed);
        return FLW_OK;
    });
}

int flw_dpd_param_count(const flw_dpd* e, int64_t* n) {
    return guarded([&] {
        *n = eng(const_cast<flw_dpd*>(e)).param_count();
        return FLW_OK;
    });
}

int flw_dpd_get_params(flw_dpd* e, double* out, int64_t n) {
    return guarded([&] {
        if (n != eng(e).param_count()) fail(Errc::Shape, "param count mismatch");
        eng(e).get_params(out);
        return FLW_OK;
    });
}

int flw_dpd_set_params(flw_dpd* e, const double* in, int64_t n) {
    return guarded([&] {
        if (n != eng(e).param_count()) fail(Errc::Shape, "param count mismatch");
        eng(e).set_params(in);
        return FLW_OK;
    });
}

int flw_dpd_stats(const flw_dpd* e, int64_t* steps, int64_t* env_count, int64_t* learn_iters, int64_t* graph_kernels) {
    return guarded([&] {
        Engine& en = eng(const_cast<flw_dpd*>(e));
        if (steps) *steps = en.steps_executed();
        if (env_count) *env_count = en.env_count();
        if (learn_iters) *learn_iters = en.learn_iters();
        if (graph_kernels) *graph_kernels = en.graph_kernel_nodes();
        return FLW_OK;
    });
}

int flw_dpd_reset(flw_dpd* e, int64_t episode) {
    return guarded([&] {
        eng(e).reset(episode);
        return FLW_OK;
    });
}

int flw_dpd_step(flw_dpd* e, int64_t episode, int64_t step) {
    return guarded([&] {
        eng(e).step(episode, step);
        return FLW_OK;
    });
}

int flw_dpd_learn(flw_dpd* e, int64_t episode, int64_t iter) {
    return guarded([&] {
        eng(e).learn(episode, iter);
        return FLW_OK;
    });
}

int flw_dpd_learn_grads(flw_dpd* e, int64_t episode, int64_t iter) {
    return guarded([&] {
        eng(e).learn_grads(episode, iter);
        return FLW_OK;
    });
}

int flw_dpd_apply_grads(flw_dpd* e, const double* grads, int64_t n) {
    return guarded([&] {
        if (grads && n != eng(e).param_count()) fail(Errc::Shape, "gradient length mismatch");
        eng(e).apply_grads(grads);
        return FLW_OK;
    });
}

int flw_dpd_tensor_size(const flw_dpd* e, const char* name, int64_t* n) {
    return guarded([&] {
        *n = eng(const_cast<flw_dpd*>(e)).tensor_size(name);
        if (*n < 0) fail(Errc::Config, std::string("unknown tensor '") + name + "'");
        return FLW_OK;
    });
}

int flw_dpd_read(flw_dpd* e, const char* name, double* out, int64_t n) {
    return guarded([&] {
        if (n != eng(e).tensor_size(name)) fail(Errc::Shape, std::string("size mismatch for '") + name + "'");
        eng(e).read_tensor(name, out);
        return FLW_OK;
    });
}

int flw_dpd_write(flw_dpd* e, const char* name, const double* in, int64_t n) {
    return guarded([&] {
        eng(e).write_tensor(name, in, n);
        return FLW_OK;
    });
}

int flw_selftest_umma(int M, int N, int K, int a_mn, int b_mn, int lane_off, const float* A, const float* B,
                      float* D) {
    return guarded([&] {
        if (!((M == 64 || M == 128) && N % 16 == 0 && N >= 16 && N <= 256 && K % 16 == 0 && K > 0))
            fail(Errc::Config, "unsupported selftest shape");
        return umma_selftest(M, N, K, a_mn, b_mn, lane_off, A, B, D);
    });
}

}  // extern "C"

// ------------------------------------------------------------------ profiling helpers
namespace flw {
void microbench(const std::string& which, int64_t n, int iters, double* ms, double* bytes);
}

extern "C" {

int flw_microbench(const char* which, int64_t n, int iters, double* ms_per_launch, double* bytes_per_launch) {
    return guarded([&] {
        if (n < 1 || iters < 1) fail(Errc::Config, "microbench needs n >= 1 and iters >= 1");
        microbench(which ? which : "", n, iters, ms_per_launch, bytes_per_launch);
        return FLW_OK;
    });
}

int flw_dpd_enable_probes(flw_dpd* e, int on) {
    return guarded([&] {
        eng(e).enable_probes(on != 0);
        return FLW_OK;
    });
}

int flw_dpd_probe_times(flw_dpd* e, char** json) {
    return guarded([&] {
        *json = dup_string(eng(e).probe_times_json());
        return FLW_OK;
    });
}

}  // extern "C"
