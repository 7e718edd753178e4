// ref_tool: drives the UNMODIFIED reference (compiled from /root/reference/proj/src by
// oracle/Makefile) for two purposes, both test infrastructure:
//
//   ref_tool trace <algo.json> <seed> <out_prefix>
//       Interp::whole phase by phase (the single-process oracle, fdg_local.cpp:57-83, which is
//       bit-identical to a DP-D unit with k=1) and dumps every tensor the B200
//       engine produces: reset obs, per-step state/logits/PolicyApply/EnvStep, the buffer
//       sample, per-train-iteration values/last_value/adv/ret/logits/loss/grads/params.
//       Output: <out_prefix>.bin (float64 LE) + <out_prefix>.json (name, shape, offset).
//
//   ref_tool run <algo.json> <deploy.json> <seed> [--params] [--unpartitioned]
//       flw_run_local semantics (capi.cpp:170-186 -> local_run.cpp:512-581) on the deploy
//       config's policy; prints one JSON object: per-episode wall_ms/reward, steps,
//       grad_messages, bytes_total, env_total, and (with --params) the final flat params.
//       This is the CPU baseline arm of bench.py (cpu_baseline.kind = "reference").
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../include/fraglow.h"
#include "config.hpp"
#include "fdgc/fdg.hpp"
#include "plan/plan.hpp"
#include "run/interp.hpp"
#include "run/runner.hpp"

using namespace fraglow;
using dfg::NodeId;
using dfg::OpKind;

namespace {

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        std::cerr << "cannot read " << path << "\n";
        std::exit(2);
    }
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

struct Dump {
    std::ofstream bin;
    std::ostringstream man;
    int64_t offset = 0;
    bool first = true;

    explicit Dump(const std::string& prefix) : bin(prefix + ".bin", std::ios::binary) { man << "[\n"; }

    void put(const std::string& name, const Shape& shape, const std::vector<double>& data) {
        bin.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size() * 8));
        if (!first) man << ",\n";
        first = false;
        man << "  {\"name\": \"" << name << "\", \"shape\": [";
        for (size_t i = 0; i < shape.size(); ++i) man << (i ? ", " : "") << shape[i];
        man << "], \"offset\": " << offset << ", \"count\": " << data.size() << "}";
        offset += static_cast<int64_t>(data.size());
    }
    void put(const std::string& name, const Tensor& t) { put(name, t.shape(), t.data()); }
    void scalar(const std::string& name, double v) { put(name, {1}, {v}); }

    void finish(const std::string& prefix) {
        man << "\n]\n";
        std::ofstream(prefix + ".json") << man.str();
    }
};

NodeId find_kind(const dfg::DataflowGraph& g, OpKind k) {
    for (const auto& n : g.nodes)
        if (n.kind == k) return n.id;
    return -1;
}

int trace(const std::string& algo_path, uint64_t seed, const std::string& prefix) {
    dfg::AlgoConfig algo = parse_algo_config(slurp(algo_path));
    dfg::DataflowGraph g = dfg::standard_program(algo.algorithm, algo);
    run::Interp it = run::Interp::whole(&g, seed);
    auto fbs = g.feedbacks();

    NodeId n_reset = find_kind(g, OpKind::EnvReset), n_step = find_kind(g, OpKind::EnvStep);
    NodeId n_pa = find_kind(g, OpKind::PolicyApply), n_sample = find_kind(g, OpKind::BufferSample);
    NodeId n_gae = find_kind(g, OpKind::GaeAdv), n_ret = find_kind(g, OpKind::DiscountedReturn);
    NodeId n_ppo = find_kind(g, OpKind::PpoLoss), n_a3c = find_kind(g, OpKind::A3cLoss);
    NodeId n_grad = find_kind(g, OpKind::GradCompute), n_opt = find_kind(g, OpKind::OptimStep);
    NodeId n_loss = n_ppo >= 0 ? n_ppo : n_a3c;
    NodeId n_logits = g.node(n_pa).inputs[0];
    NodeId n_values = g.node(n_loss).inputs[1];
    NodeId n_logits_new = g.node(n_loss).inputs[0];
    NodeId n_last_value = g.node(n_ret).inputs[2];
    NodeId n_state_in = -1;
    for (const auto& fb : fbs) n_state_in = fb.input;
    auto params = dfg::param_list(g, g.node(n_opt));

    Dump d(prefix);
    d.put("params0", {static_cast<int64_t>(it.flat_params(params).size())}, it.flat_params(params));
    int64_t iters = it.learn_iters();
    for (int64_t ep = 0; ep < g.loop.episodes; ++ep) {
        std::string e = "ep" + std::to_string(ep) + "/";
        it.eval_phase(dfg::Phase::Reset, {ep, 0, 0});
        d.put(e + "reset_obs", it.value(n_reset));
        for (const auto& fb : fbs)
            if (fb.reset_from >= 0) it.bind(fb.input, it.value(fb.reset_from));
        for (int64_t st = 0; st < g.loop.steps_per_episode; ++st) {
            std::string s = e + "st" + std::to_string(st) + "/";
            d.put(s + "state_in", it.value(n_state_in));
            it.eval_phase(dfg::Phase::Step, {ep, st, 0});
            d.put(s + "logits", it.value(n_logits));
            d.put(s + "pa", it.value(n_pa));
            d.put(s + "envstep", it.value(n_step));
            for (const auto& fb : fbs)
                if (fb.step_from >= 0) it.bind(fb.input, it.value(fb.step_from));
        }
        d.scalar(e + "reward_sum", it.episode_reward_sum());
        d.scalar(e + "steps", static_cast<double>(it.steps_executed()));
        for (int64_t k = 0; k < iters; ++k) {
            std::string s = e + "it" + std::to_string(k) + "/";
            it.eval_phase(dfg::Phase::Learn, {ep, g.loop.steps_per_episode, k});
            if (k == 0) d.put(e + "sample", it.value(n_sample));
            d.put(s + "values", it.value(n_values));
            d.put(s + "last_value", it.value(n_last_value));
            if (n_gae >= 0) d.put(s + "adv", it.value(n_gae));
            d.put(s + "ret", it.value(n_ret));
            d.put(s + "logits_new", it.value(n_logits_new));
            d.put(s + "loss", it.value(n_loss));
            d.put(s + "grads", it.value(n_grad));
            auto p = it.flat_params(params);
            d.put(s + "params", {static_cast<int64_t>(p.size())}, p);
        }
    }
    d.finish(prefix);
    return 0;
}

int run_cmd(const std::string& algo_path, const std::string& deploy_path, uint64_t seed, bool with_params,
        bool unpartitioned, int64_t episodes_override) {
    dfg::AlgoConfig algo = parse_algo_config(slurp(algo_path));
    plan::DeploymentConfig deploy = parse_deploy_config(slurp(deploy_path));
    if (episodes_override > 0) algo.loop.episodes = episodes_override;
    dfg::DataflowGraph g = dfg::standard_program(algo.algorithm, algo);
    fdgc::FDG fdg = fdgc::generate_fdg(g);
    plan::PlacementPlan p = plan::make_plan(fdg, deploy, algo);
    run::RunOptions o;
    o.seed = seed;
    o.loop = g.loop;
    o.timeout_ms = 3600 * 1000;
    run::RunMetrics m;
    if (unpartitioned) {
        g.loop = o.loop;
        auto t0 = std::chrono::steady_clock::now();
        auto r = fdgc::run_unpartitioned(g, seed);
        auto t1 = std::chrono::steady_clock::now();
        double per = std::chrono::duration<double, std::milli>(t1 - t0).count() /
                     static_cast<double>(std::max<size_t>(1, r.episode_rewards.size()));
        for (double rew : r.episode_rewards) m.episodes.push_back({per, rew, 0});
        m.steps = r.steps;
        m.final_params = r.final_params;
    } else {
        m = run::run_plan_local(g, p, o);
    }
    std::ostringstream os;
    os.precision(17);
    os << "{\"policy\": \"" << plan::policy_name(p.policy) << "\", \"units\": " << p.units.size()
       << ", \"env_total\": " << p.env_total << ", \"steps_per_episode\": " << g.loop.steps_per_episode
       << ", \"steps\": " << m.steps << ", \"grad_messages\": " << m.grad_messages
       << ", \"hw_threads\": " << std::thread::hardware_concurrency() << ", \"episodes\": [";
    for (size_t i = 0; i < m.episodes.size(); ++i)
        os << (i ? ", " : "") << "{\"wall_ms\": " << m.episodes[i].wall_ms << ", \"reward\": " << m.episodes[i].reward
           << ", \"bytes_total\": " << m.episodes[i].bytes_total << "}";
    os << "]";
    if (with_params) {
        os << ", \"final_params\": [";
        for (size_t i = 0; i < m.final_params.size(); ++i) os << (i ? ", " : "") << m.final_params[i];
        os << "]";
    }
    os << "}\n";
    std::cout << os.str();
    return 0;
}

// ref_tool plan <algo.json> <deploy.json>: the reference C API's view of a program
// (flw_program_create / flw_program_dump(PLAN) / flw_validate_plan, capi.cpp:207-247).
int plan_cmd(const std::string& algo_path, const std::string& deploy_path) {
    std::string a = slurp(algo_path), d = slurp(deploy_path);
    flw_program* p = nullptr;
    int rc = flw_program_create(a.c_str(), d.c_str(), &p);
    std::cout << "{\"rc\": " << rc;
    if (rc != 0) {
        std::string err = flw_last_error();
        std::string esc;
        for (char c : err) {
            if (c == '"' || c == '\\') esc += '\\';
            esc += c;
        }
        std::cout << ", \"error\": \"" << esc << "\"}\n";
        return 0;
    }
    char* plan = nullptr;
    char* report = nullptr;
    int nv = 0;
    flw_program_dump(p, FLW_DUMP_PLAN, &plan);
    flw_validate_plan(p, &report, &nv);
    std::cout << ", \"plan\": " << plan << ", \"violations\": " << report << "}\n";
    flw_string_free(plan);
    flw_string_free(report);
    flw_program_destroy(p);
    return 0;
}

// ref_tool dfg <algo.json>: the dataflow graph JSON the reference ships to its workers
// (flw_program_dump(FLW_DUMP_DFG) = dfg::dump_json, graph.cpp:468-507).
int dfg_cmd(const std::string& algo_path) {
    std::string a = slurp(algo_path);
    flw_program* p = nullptr;
    if (flw_program_create(a.c_str(), nullptr, &p) != 0) {
        std::cerr << flw_last_error() << "\n";
        return 1;
    }
    char* g = nullptr;
    flw_program_dump(p, FLW_DUMP_DFG, &g);
    std::cout << g << "\n";
    flw_string_free(g);
    flw_program_destroy(p);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc >= 4 && std::string(argv[1]) == "plan") return plan_cmd(argv[2], argv[3]);
        if (argc >= 3 && std::string(argv[1]) == "dfg") return dfg_cmd(argv[2]);
        if (argc >= 5 && std::string(argv[1]) == "trace")
            return trace(argv[2], std::stoull(argv[3]), argv[4]);
        if (argc >= 5 && std::string(argv[1]) == "run") {
            bool params = false, unpart = false;
            int64_t eps = 0;
            for (int i = 5; i < argc; ++i) {
                std::string a = argv[i];
                if (a == "--params") params = true;
                else if (a == "--unpartitioned") unpart = true;
                else if (a.rfind("--episodes=", 0) == 0) eps = std::stoll(a.substr(11));
            }
            return run_cmd(argv[2], argv[3], std::stoull(argv[4]), params, unpart, eps);
        }
    } catch (const Error& e) {
        std::cerr << errc_name(e.code()) << ": " << e.what() << "\n";
        return static_cast<int>(e.code()) < 10 ? static_cast<int>(e.code()) : 3;
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\n";
        return 3;
    }
    std::cerr << "usage: ref_tool trace <algo.json> <seed> <out_prefix>\n"
                 "       ref_tool run <algo.json> <deploy.json> <seed> [--params] [--unpartitioned] [--episodes=N]\n";
    return 2;
}
