// Host control plane for the DP-D drop-in: the reference's two JSON documents, their
// validation, and the DP-D placement (one fused-loop unit per accelerator slot).
//
// Mirrors, for the DP-D path only:
//   parse_algo_config / parse_deploy_config   /root/reference/proj/src/config.cpp:24-63,88-103
//   AlgoConfig::validate, Hyperparams::validate  dfg/programs.cpp:7-20, rl/rl.cpp:7-12
//   parse_policy (aliases)                   plan/plan.cpp:16-26
//   make_plan DP-D branch + split_envs        plan/plan.cpp:46-55,308-417
//   validate_plan DP-D rules                  plan/plan.cpp:567-576
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "errors.hpp"

namespace flw {

enum class Policy { DpA, DpB, DpC, DpD, DpE, DpF };
Policy parse_policy(const std::string& name);
const char* policy_name(Policy p);

enum class Algo { Ppo = 0, A3c = 1, Mappo = 2 };
enum class EnvKind { Gridline = 0, Synth17x6 = 1, SpreadLite = 2, CartpoleLite = 3 };

struct AlgoConfig {
    std::string algorithm = "ppo";
    int64_t agents = 1, actors = 1, envs = 1;
    std::string env_name = "gridline";
    std::map<std::string, double> env_params;
    std::vector<int64_t> hidden = {16, 16};
    std::string activation = "tanh";
    double gamma = 0.97, lam = 0.95, clip_eps = 0.2, lr = 3e-3;
    int64_t train_iters = 4;
    double value_coef = 0.5, entropy_coef = 0.01;
    bool normalize_adv = true;
    int64_t episodes = 1, steps_per_episode = 32;

    void validate() const;
    Algo algo() const;
    EnvKind env() const;
    double env_param(const std::string& k, double dflt) const {
        auto it = env_params.find(k);
        return it == env_params.end() ? dflt : it->second;
    }
};

AlgoConfig parse_algo_config(const std::string& json_text);
// the dataflow graph JSON of a PPO / MAPPO standard program (dfg::dump_json) -> its algo config
AlgoConfig algo_from_graph(const std::string& graph_json);
std::string algo_to_json(const AlgoConfig& c);
// algo JSON, or graph JSON when the object has a "nodes" array (the seam accepts either)
AlgoConfig parse_algo_or_graph(const std::string& text);

struct DeployConfig {
    std::vector<std::string> workers = {"local"};
    int cpu_slots = 4, accel_slots = 2;
    Policy policy = Policy::DpA;
    void validate() const;
    int worker_count() const { return static_cast<int>(workers.size()); }
};

DeployConfig parse_deploy_config(const std::string& json_text);

// Static shape of the standard program for an algo config (programs.cpp:204-454): obs widths,
// action count, MLP dims, flat parameter layout (policy W0,b0,..., critic W0,b0,...; W
// row-major [in,out]) and the Param node ids used as init keys (interp.cpp:71-85).
struct ProgramShape {
    Algo algo;
    EnvKind env;
    int n_agents = 1;   // MAPPO agents, 1 otherwise
    int obs_dim = 1;    // per-agent observation width
    int n_actions = 2;
    int state_w = 1;    // joint observation width (n_agents * obs_dim)
    int crit_in = 1;    // critic input width (obs_dim, or joint obs + agent one-hot for MAPPO)
    int env_state_w = 1;
    bool accel_capable = false;
    int L = 0;          // Linear layers per net
    std::vector<int> pdims, cdims;
    std::vector<int64_t> woff[2], boff[2];
    int64_t P = 0, P_policy = 0;
    int64_t learn_iters = 1;
};

ProgramShape program_shape(const AlgoConfig& a);

struct Unit {
    int id = 0;
    int worker = 0;
    int slot = 0;        // accel slot index on that worker
    int64_t env_lo = 0, env_hi = 0;
};

struct Plan {
    Policy policy = Policy::DpD;
    int64_t env_total = 0;
    std::vector<Unit> units;
    bool grad_sync = false;      // GradSync channel present (>= 2 units)
    std::string to_json() const;
    std::vector<std::pair<std::string, std::string>> violations() const;
};

std::vector<std::pair<int64_t, int64_t>> split_envs(int64_t total, int k);
Plan make_dpd_plan(const AlgoConfig& a, const DeployConfig& d);

}  // namespace flw
