#include "config.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <sstream>

#include "nlohmann/json.hpp"

namespace flw {

using nlohmann::json;

Policy parse_policy(const std::string& name) {  // plan.cpp:16-26
    std::string n = name;
    std::transform(n.begin(), n.end(), n.begin(), [](unsigned char c) { return std::tolower(c); });
    if (n == "dp-a" || n == "single_learner_coarse") return Policy::DpA;
    if (n == "dp-b" || n == "single_learner_fine") return Policy::DpB;
    if (n == "dp-c" || n == "multiple_learners") return Policy::DpC;
    if (n == "dp-d" || n == "gpu_only") return Policy::DpD;
    if (n == "dp-e" || n == "environments") return Policy::DpE;
    if (n == "dp-f" || n == "central") return Policy::DpF;
    fail(Errc::Config, "unknown distribution policy '" + name + "'");
}

const char* policy_name(Policy p) {
    switch (p) {
        case Policy::DpA: return "dp-a";
        case Policy::DpB: return "dp-b";
        case Policy::DpC: return "dp-c";
        case Policy::DpD: return "dp-d";
        case Policy::DpE: return "dp-e";
        case Policy::DpF: return "dp-f";
    }
    return "?";
}

static bool env_known(const std::string& n) {
    return n == "gridline" || n == "cartpole_lite" || n == "spread_lite" || n == "synth17x6";
}

Algo AlgoConfig::algo() const {
    return algorithm == "ppo" ? Algo::Ppo : algorithm == "a3c" ? Algo::A3c : Algo::Mappo;
}

EnvKind AlgoConfig::env() const {
    if (env_name == "gridline") return EnvKind::Gridline;
    if (env_name == "synth17x6") return EnvKind::Synth17x6;
    if (env_name == "spread_lite") return EnvKind::SpreadLite;
    return EnvKind::CartpoleLite;
}

void AlgoConfig::validate() const {  // programs.cpp:7-20 + rl.cpp:7-12
    if (algorithm != "ppo" && algorithm != "a3c" && algorithm != "mappo")
        fail(Errc::Config, "unknown algorithm '" + algorithm + "'");
    if (agents < 1 || actors < 1 || envs < 1) fail(Errc::Config, "agent/actor/env counts must be >= 1");
    if (!env_known(env_name)) fail(Errc::UnknownEnv, "unknown environment '" + env_name + "'");
    if (activation != "tanh" && activation != "relu") fail(Errc::Config, "activation must be tanh or relu");
    if (hidden.empty()) fail(Errc::Config, "policy needs at least one hidden layer");
    for (int64_t h : hidden)
        if (h < 1) fail(Errc::Shape, "shape dims must be >= 1");
    if (episodes < 0 || steps_per_episode < 1) fail(Errc::Config, "bad loop spec");
    if (algorithm == "a3c" && envs != actors)
        fail(Errc::Config, "a3c pairs one environment per actor (envs must equal actors)");
    if (actors > envs) fail(Errc::Config, "more actors than environments");
    if (!(gamma > 0.0 && gamma <= 1.0)) fail(Errc::Config, "gamma must be in (0,1]");
    if (!(lam >= 0.0 && lam <= 1.0)) fail(Errc::Config, "lam must be in [0,1]");
    if (!(clip_eps > 0.0 && clip_eps < 1.0)) fail(Errc::Config, "clip_eps must be in (0,1)");
    if (train_iters < 1) fail(Errc::Config, "train_iters must be >= 1");
    if (env_name == "spread_lite") {
        double n = algorithm == "mappo" ? static_cast<double>(agents) : env_param("n_agents", 2);
        if (static_cast<int64_t>(n) < 1) fail(Errc::Config, "spread_lite needs n_agents >= 1");
    }
}

static json parse_or_fail(const std::string& text) {
    try {
        return json::parse(text);
    } catch (const json::parse_error& e) {
        fail(Errc::Config, std::string("config parse error: ") + e.what());
    }
}

// The seam's other input: the dataflow graph JSON a reference worker receives
// (dfg::dump_json, graph.cpp:468-507) of a PPO or MAPPO standard program (programs.cpp:204-272,
// 349-454) - its node attributes carry every hyper-parameter: EnvReset {env, num, ep_*},
// xavier Param {pgroup, fan_in, fan_out} (the MLP widths), Tanh / Relu, GaeAdv {gamma, lam,
// normalize}, PpoLoss {clip_eps, value_coef, entropy_coef}, OptimStep {lr, train_iters},
// PolicyApply {rows_n} (MAPPO agents) and loop {episodes, steps_per_episode}.
AlgoConfig algo_from_graph(const std::string& text) {
    json g = parse_or_fail(text);
    if (!g.contains("nodes") || !g["nodes"].is_array()) fail(Errc::Config, "graph JSON has no nodes array");
    AlgoConfig c;
    c.hidden.clear();
    bool env = false, loss = false, optim = false, gae = false;
    std::vector<int64_t> pol;  // policy layer widths: fan_in of layer 0, then every fan_out
    try {
        for (const auto& n : g["nodes"]) {
            const std::string kind = n.at("kind").get<std::string>();
            const json& a = n.contains("attrs") ? n["attrs"] : json::object();
            if (kind == "EnvReset") {
                env = true;
                c.env_name = a.at("env").get<std::string>();
                c.envs = a.at("num").get<int64_t>();
                for (auto it = a.begin(); it != a.end(); ++it)
                    if (it.key().rfind("ep_", 0) == 0 && it.key() != "ep_n_agents")
                        c.env_params[it.key().substr(3)] = it.value().get<double>();
            } else if (kind == "Param" && a.value("init", "") == "xavier" && a.value("pgroup", "") == "policy") {
                if (pol.empty()) pol.push_back(a.at("fan_in").get<int64_t>());
                pol.push_back(a.at("fan_out").get<int64_t>());
            } else if (kind == "Relu") {
                c.activation = "relu";
            } else if (kind == "GaeAdv") {
                gae = true;
                c.gamma = a.at("gamma").get<double>();
                c.lam = a.at("lam").get<double>();
                c.normalize_adv = a.value("normalize", int64_t{1}) != 0;
            } else if (kind == "PpoLoss") {
                loss = true;
                c.clip_eps = a.at("clip_eps").get<double>();
                c.value_coef = a.at("value_coef").get<double>();
                c.entropy_coef = a.at("entropy_coef").get<double>();
            } else if (kind == "A3cLoss") {
                fail(Errc::Config, "graph JSON input covers the PPO and MAPPO standard programs; pass an A3C "
                                   "program as its algo JSON");
            } else if (kind == "OptimStep") {
                optim = true;
                c.lr = a.at("lr").get<double>();
                c.train_iters = a.at("train_iters").get<int64_t>();
            } else if (kind == "PolicyApply") {
                c.agents = a.value("rows_n", int64_t{1});
            }
        }
        if (g.contains("loop")) {
            c.episodes = g["loop"].value("episodes", c.episodes);
            c.steps_per_episode = g["loop"].value("steps_per_episode", c.steps_per_episode);
        }
    } catch (const json::exception& e) {
        fail(Errc::Config, std::string("graph JSON: ") + e.what());
    }
    if (!env || !loss || !optim || !gae || pol.size() < 2)
        fail(Errc::Config, "graph JSON is not a PPO / MAPPO standard program (EnvReset, xavier policy Params, "
                           "GaeAdv, PpoLoss, OptimStep expected)");
    c.algorithm = c.agents > 1 ? "mappo" : "ppo";
    c.hidden.assign(pol.begin() + 1, pol.end() - 1);  // [obs, h1 .. hL-1, actions]
    c.validate();
    return c;
}

std::string algo_to_json(const AlgoConfig& c) {
    nlohmann::ordered_json j;
    j["algorithm"] = c.algorithm;
    j["agent"] = {{"num", c.agents}};
    j["actor"] = {{"num", c.actors}};
    nlohmann::ordered_json e = {{"type", c.env_name}, {"num", c.envs}};
    if (!c.env_params.empty()) e["params"] = c.env_params;
    j["env"] = e;
    j["learner"] = {{"params", {{"gamma", c.gamma}, {"lam", c.lam}, {"clip_eps", c.clip_eps}, {"lr", c.lr},
                                {"train_iters", c.train_iters}, {"value_coef", c.value_coef},
                                {"entropy_coef", c.entropy_coef}, {"normalize_adv", c.normalize_adv}}}};
    j["policy_net"] = {{"hidden", c.hidden}, {"activation", c.activation}};
    j["loop"] = {{"episodes", c.episodes}, {"steps_per_episode", c.steps_per_episode}};
    return j.dump();
}

AlgoConfig parse_algo_or_graph(const std::string& text) {
    const auto p = text.find_first_not_of(" \t\r\n");
    if (p != std::string::npos && text[p] == '{' && text.find("\"nodes\"") != std::string::npos) {
        json j = json::parse(text, nullptr, false);
        if (!j.is_discarded() && j.is_object() && j.contains("nodes")) return algo_from_graph(text);
    }
    return parse_algo_config(text);
}

AlgoConfig parse_algo_config(const std::string& text) {  // config.cpp:24-63
    json j = parse_or_fail(text);
    AlgoConfig c;
    try {
        c.algorithm = j.value("algorithm", "ppo");
        if (j.contains("agent")) c.agents = j["agent"].value("num", 1);
        if (j.contains("actor")) c.actors = j["actor"].value("num", 1);
        if (j.contains("env")) {
            c.env_name = j["env"].value("type", "gridline");
            c.envs = j["env"].value("num", 1);
            if (j["env"].contains("params"))
                for (auto it = j["env"]["params"].begin(); it != j["env"]["params"].end(); ++it)
                    c.env_params[it.key()] = it->get<double>();
        }
        if (j.contains("learner") && j["learner"].contains("params")) {
            const json& p = j["learner"]["params"];
            c.gamma = p.value("gamma", c.gamma);
            c.lam = p.value("lam", c.lam);
            c.clip_eps = p.value("clip_eps", c.clip_eps);
            c.lr = p.value("lr", c.lr);
            c.train_iters = p.value("train_iters", c.train_iters);
            c.value_coef = p.value("value_coef", c.value_coef);
            c.entropy_coef = p.value("entropy_coef", c.entropy_coef);
            c.normalize_adv = p.value("normalize_adv", c.normalize_adv);
        }
        if (j.contains("policy_net")) {
            if (j["policy_net"].contains("hidden")) c.hidden = j["policy_net"]["hidden"].get<std::vector<int64_t>>();
            c.activation = j["policy_net"].value("activation", c.activation);
        }
        if (j.contains("loop")) {
            c.episodes = j["loop"].value("episodes", c.episodes);
            c.steps_per_episode = j["loop"].value("steps_per_episode", c.steps_per_episode);
        }
    } catch (const json::exception& e) {
        fail(Errc::Config, std::string("algorithm config: ") + e.what());
    }
    c.validate();
    return c;
}

void DeployConfig::validate() const {  // plan.cpp:40-44
    if (workers.empty()) fail(Errc::Config, "deployment needs at least one worker");
    if (cpu_slots < 1) fail(Errc::Config, "each worker needs at least one cpu slot");
    if (accel_slots < 0) fail(Errc::Config, "negative accel slot count");
}

DeployConfig parse_deploy_config(const std::string& text) {  // config.cpp:88-103
    json j = parse_or_fail(text);
    DeployConfig c;
    try {
        c.workers = j.value("workers", std::vector<std::string>{"local"});
        if (j.contains("slots_per_worker")) {
            c.cpu_slots = j["slots_per_worker"].value("cpu", c.cpu_slots);
            c.accel_slots = j["slots_per_worker"].value("accel", c.accel_slots);
        }
        c.policy = parse_policy(j.value("distribution_policy", "dp-a"));
    } catch (const json::exception& e) {
        fail(Errc::Config, std::string("deployment config: ") + e.what());
    }
    c.validate();
    return c;
}

ProgramShape program_shape(const AlgoConfig& a) {
    ProgramShape s;
    s.algo = a.algo();
    s.env = a.env();
    s.n_agents = s.algo == Algo::Mappo ? static_cast<int>(a.agents) : 1;
    switch (s.env) {  // envs.cpp:157-179 (+ builder env synth17x6)
        case EnvKind::Gridline:
            s.obs_dim = 1, s.n_actions = 2, s.env_state_w = 2, s.accel_capable = true;
            break;
        case EnvKind::Synth17x6:
            s.obs_dim = 17, s.n_actions = 6, s.env_state_w = 17, s.accel_capable = true;
            break;
        case EnvKind::SpreadLite: {
            int n = s.algo == Algo::Mappo ? s.n_agents : static_cast<int>(a.env_param("n_agents", 2));
            s.obs_dim = 2 + 2 * n, s.n_actions = 5, s.env_state_w = 4 * n;
            // Builder extension: spread_lite is accel-capable when asked to be.
            s.accel_capable = a.env_param("accel", 0.0) != 0.0;
            break;
        }
        case EnvKind::CartpoleLite:
            s.obs_dim = 4, s.n_actions = 2, s.env_state_w = 4, s.accel_capable = false;
            break;
    }
    s.state_w = s.n_agents * s.obs_dim;
    s.crit_in = s.algo == Algo::Mappo ? s.state_w + s.n_agents : s.obs_dim;
    s.L = static_cast<int>(a.hidden.size()) + 1;
    s.pdims.push_back(s.obs_dim);
    s.cdims.push_back(s.crit_in);
    for (int64_t h : a.hidden) {
        s.pdims.push_back(static_cast<int>(h));
        s.cdims.push_back(static_cast<int>(h));
    }
    s.pdims.push_back(s.n_actions);
    s.cdims.push_back(1);
    int64_t off = 0;
    for (int net = 0; net < 2; ++net) {
        const auto& d = net == 0 ? s.pdims : s.cdims;
        for (int l = 0; l < s.L; ++l) {
            s.woff[net].push_back(off);
            off += static_cast<int64_t>(d[l]) * d[l + 1];
            s.boff[net].push_back(off);
            off += d[l + 1];
        }
        if (net == 0) s.P_policy = off;
    }
    s.P = off;
    s.learn_iters = s.algo == Algo::A3c ? 1 : a.train_iters;  // interp.cpp:127-135
    return s;
}

std::vector<std::pair<int64_t, int64_t>> split_envs(int64_t total, int k) {  // plan.cpp:46-55
    std::vector<std::pair<int64_t, int64_t>> out;
    int64_t base = total / k, rem = total % k, lo = 0;
    for (int r = 0; r < k; ++r) {
        int64_t n = base + (r < rem ? 1 : 0);
        out.emplace_back(lo, lo + n);
        lo += n;
    }
    return out;
}

Plan make_dpd_plan(const AlgoConfig& a, const DeployConfig& d) {  // plan.cpp:308-417 (DP-D)
    d.validate();
    a.validate();
    if (d.policy != Policy::DpD)
        fail(Errc::PolicyInapplicable, std::string("the B200 engine serves distribution_policy dp-d (GPU_only); '") +
                                           policy_name(d.policy) + "' runs on the reference CPU runtime");
    ProgramShape s = program_shape(a);
    if (!s.accel_capable)
        fail(Errc::PolicyInapplicable, "dp-d requires an accelerator-capable environment implementation");
    Plan p;
    p.policy = d.policy;
    p.env_total = a.envs;
    int k = static_cast<int>(a.actors);
    if (k < 1) fail(Errc::Config, "replica count must be >= 1");
    auto ranges = split_envs(a.envs, k);
    int nw = d.worker_count();
    std::vector<int> used(static_cast<size_t>(nw), 0);
    for (int r = 0; r < k; ++r) {
        Unit u;
        u.id = r;
        u.worker = static_cast<int>((static_cast<int64_t>(r) * nw) / k);
        if (used[static_cast<size_t>(u.worker)] >= d.accel_slots)
            fail(Errc::InsufficientSlots, "accel slots exhausted on worker " + std::to_string(u.worker));
        u.slot = used[static_cast<size_t>(u.worker)]++;
        u.env_lo = k > 1 ? ranges[static_cast<size_t>(r)].first : 0;
        u.env_hi = k > 1 ? ranges[static_cast<size_t>(r)].second : a.envs;
        p.units.push_back(u);
    }
    p.grad_sync = k >= 2;  // plan.cpp:164-181
    return p;
}

std::vector<std::pair<std::string, std::string>> Plan::violations() const {  // plan.cpp:567-576
    std::vector<std::pair<std::string, std::string>> out;
    std::set<std::pair<int, int>> slots;
    for (const Unit& u : units)
        if (!slots.insert({u.worker, u.slot}).second)
            out.emplace_back("SlotSharingViolated", "dp-d places one fragment per slot");
    return out;
}

std::string Plan::to_json() const {  // plan.cpp:605-637 schema
    nlohmann::ordered_json out;
    out["policy"] = policy_name(policy);
    out["env_total"] = env_total;
    out["instances"] = nlohmann::ordered_json::array();
    for (const Unit& u : units)
        out["instances"].push_back({{"fragment", 0},
                                    {"replica", u.id},
                                    {"worker", u.worker},
                                    {"slot", u.slot},
                                    {"kind", "accel"},
                                    {"env_lo", u.env_lo},
                                    {"env_hi", u.env_hi}});
    out["fusion_groups"] = nlohmann::ordered_json::array();
    out["channels"] = nlohmann::ordered_json::array();
    if (grad_sync) {
        nlohmann::ordered_json ch;
        ch["fdg_channel"] = -1;
        ch["kind"] = "grad_sync";
        ch["sync"] = "per_episode";
        ch["legs"] = nlohmann::ordered_json::array();
        for (const Unit& a : units)
            for (const Unit& b : units)
                if (a.id != b.id)
                    ch["legs"].push_back({{"from", a.id},
                                          {"to", b.id},
                                          {"transport", a.worker != b.worker ? "tcp" : "inproc"}});
        out["channels"].push_back(ch);
    }
    return out.dump(2);
}

}  // namespace flw
