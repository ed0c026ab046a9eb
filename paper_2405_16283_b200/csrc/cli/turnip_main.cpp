// `turnip` — command-line front end, flag-compatible with the reference
// `memplan` CLI (proj/tools/memplan_main.cpp:134-208; exit codes 0 ok /
// 1 check failed / 2 usage, parse, I/O or planning error, :23-25) plus an
// `execute` subcommand that runs a memgraph on the GPU (exit 3 on CUDA
// errors). The reference CLI needs CLI11, which is not vendored here; this
// one parses its own flags.
//
//   turnip validate   --graph G
//   turnip compile    --graph G [--capacities slots:N|bytes,..] [--order-policy P]
//                     [--order-file F] [--victim-policy V] [--alloc-horizon H]
//                     [--drop-superfluous] [--seed N] [--out F]
//   turnip verify     --graph G --memgraph M [--schedules N]
//   turnip simulate   --memgraph M [--profile P] [--policy ..] [--tie-break ..] [--seed N]
//                     [--out F] [--format json|csv]
//   turnip bench      --memgraph M [--profile P] [--trials N] [--seed N] [--out F]
//   turnip export-dot (--graph G | --memgraph M) [--out F]
//   turnip execute    --memgraph M --graph G [--config JSON] [--policy ..] [--tie-break ..]
//                     [--seed N] [--input ID=FILE]... [--output ID=FILE]... [--out TRACE]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../core/dispatch.hpp"
#include "../core/planner.hpp"
#include "../core/verify.hpp"
#include "../exec/executor.hpp"

using namespace tn;

namespace {

constexpr int kOk = 0, kCheckFailed = 1, kUsage = 2;

std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("cannot open " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return buf.str();
}

void write_file(const std::string& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write " + path);
    out << content;
}

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --key value / --flag parser with a per-subcommand whitelist.
struct Args {
    std::map<std::string, std::vector<std::string>> opts;
    std::map<std::string, bool> flags;
    bool has(const std::string& k) const { return opts.count(k) > 0; }
    std::string get(const std::string& k, const std::string& d = "") const {
        auto it = opts.find(k);
        return it == opts.end() ? d : it->second.back();
    }
    std::string need(const std::string& k) const {
        if (!has(k)) throw UsageError("--" + k + " is required");
        return get(k);
    }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& valued,
                const std::vector<std::string>& flag_names) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) != 0) throw UsageError("unexpected argument " + s);
        std::string key = s.substr(2), val;
        auto eq = key.find('=');
        bool inline_val = eq != std::string::npos;
        if (inline_val) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        }
        bool is_flag = std::find(flag_names.begin(), flag_names.end(), key) != flag_names.end();
        bool is_valued = std::find(valued.begin(), valued.end(), key) != valued.end();
        if (is_flag && !inline_val) {
            a.flags[key] = true;
            continue;
        }
        if (!is_valued) throw UsageError("unknown option --" + key);
        if (!inline_val) {
            if (i + 1 >= argc) throw UsageError("--" + key + " needs a value");
            val = argv[++i];
        }
        a.opts[key].push_back(val);
    }
    return a;
}

std::uint64_t default_seed() {
    if (const char* env = std::getenv("MEMPLAN_SEED")) return std::strtoull(env, nullptr, 10);
    return 0;
}

std::uint64_t seed_of(const Args& a) {
    return a.has("seed") ? std::strtoull(a.get("seed").c_str(), nullptr, 10) : default_seed();
}

// "slots:N", "slots:a,b,c", "a,b,c", or one byte count (memplan_main.cpp:41-63).
std::pair<std::vector<std::int64_t>, MemoryMode> parse_capacities(const std::string& text, int devices) {
    std::string spec = text;
    MemoryMode mode = MemoryMode::Byte;
    if (spec.rfind("slots:", 0) == 0) {
        mode = MemoryMode::Slot;
        spec = spec.substr(6);
    }
    std::vector<std::int64_t> values;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ',')) {
        if (item.empty()) continue;
        try {
            values.push_back(std::stoll(item));
        } catch (const std::exception&) {
            throw Error("bad capacity value: " + item);
        }
    }
    if (values.empty()) throw Error("empty capacity spec: " + text);
    if (values.size() == 1) values.assign(devices, values[0]);
    if (static_cast<int>(values.size()) != devices)
        throw Error("capacity spec names " + std::to_string(values.size()) + " devices, graph has " +
                    std::to_string(devices));
    return {values, mode};
}

int cmd_validate(const Args& a) {
    auto g = parse_taskgraph(read_file(a.need("graph")));
    auto v = validate_taskgraph(g);
    if (v.empty()) {
        std::cout << "ok\n";
        return kOk;
    }
    for (const auto& m : v) std::cout << "violation: " << m << "\n";
    return kCheckFailed;
}

int cmd_compile(const Args& a) {
    auto g = parse_taskgraph(read_file(a.need("graph")));
    auto v = validate_taskgraph(g);
    if (!v.empty()) {
        for (const auto& m : v) std::cerr << "invalid graph: " << m << "\n";
        return kCheckFailed;
    }
    auto [caps, mode] = parse_capacities(a.get("capacities", "slots:5"), g.device_count);
    const std::uint64_t seed = seed_of(a);
    VertexOrder order;
    if (a.has("order-file")) {
        auto j = nlohmann::json::parse(read_file(a.get("order-file")));
        if (!j.is_array()) throw ParseError("order file must be a JSON array of ids");
        for (const auto& x : j) order.push_back(x.get<VertexId>());
    } else {
        order = topological_order(g, order_policy_from_string(a.get("order-policy", "as-listed")), seed);
    }
    BuildOptions o;
    o.victim_policy = victim_policy_from_string(a.get("victim-policy", "farthest-next-use"));
    o.victim_seed = seed;
    o.alloc_horizon = alloc_horizon_from_string(a.get("alloc-horizon", "greedy"));
    o.keep_superfluous = !a.flags.count("drop-superfluous");
    auto r = build_memgraph(g, order, caps, mode, o);
    nlohmann::ordered_json s;
    s["offloads"] = r.stats.offload_count;
    s["reloads"] = r.stats.reload_count;
    s["memory_edges"] = r.stats.memory_edge_count;
    s["required_memory_edges"] = r.stats.required_memory_edge_count;
    s["peak_usage"] = r.stats.peak_usage;
    std::cout << s.dump(2) << "\n";
    if (a.has("out")) write_file(a.get("out"), serialize_memgraph(r.memgraph, r.memory_map));
    return kOk;
}

int cmd_verify(const Args& a) {
    auto g = parse_taskgraph(read_file(a.need("graph")));
    auto [m, map] = parse_memgraph(read_file(a.need("memgraph")));
    auto rep = verify_all(g, m, map, a.has("schedules") ? std::stoll(a.get("schedules")) : 0);
    std::cout << rep.to_json();
    return rep.all_passed() ? kOk : kCheckFailed;
}

SchedulerPolicy policy_of(const Args& a) {
    SchedulerPolicy p;
    p.kind = scheduler_kind_from_string(a.get("policy", "event-driven"));
    p.tie_break = tie_break_from_string(a.get("tie-break", "fifo"));
    return p;
}

int cmd_simulate(const Args& a) {
    auto [m, map] = parse_memgraph(read_file(a.need("memgraph")));
    DeviceProfile prof;
    if (a.has("profile")) prof = parse_profile(read_file(a.get("profile")));
    auto t = simulate(m, map, prof, policy_of(a), seed_of(a));
    std::string out = a.get("format", "json") == "csv" ? t.to_csv() : t.to_json();
    if (!a.has("out")) {
        std::cout << out;
    } else {
        write_file(a.get("out"), out);
        nlohmann::ordered_json s;
        s["makespan"] = t.makespan;
        s["host_bytes_transferred"] = t.host_bytes_transferred;
        std::cout << s.dump(2) << "\n";
    }
    return kOk;
}

int cmd_bench(const Args& a) {
    auto [m, map] = parse_memgraph(read_file(a.need("memgraph")));
    DeviceProfile prof;
    if (a.has("profile")) prof = parse_profile(read_file(a.get("profile")));
    auto s = compare_policies(m, map, prof, a.has("trials") ? std::stoll(a.get("trials")) : 20, seed_of(a));
    std::string out = s.to_json();
    if (a.has("out")) write_file(a.get("out"), out);
    else std::cout << out;
    std::printf("%-14s %12s %24s\n", "policy", "mean", "95% CI");
    std::printf("%-14s %12.4f [%10.4f, %10.4f]\n", "event-driven", s.event_driven.mean, s.event_driven.ci_low,
                s.event_driven.ci_high);
    std::printf("%-14s %12.4f [%10.4f, %10.4f]\n", "fixed-order", s.fixed_order.mean, s.fixed_order.ci_low,
                s.fixed_order.ci_high);
    std::printf("%-14s %11.2f%% [%9.2f%%, %9.2f%%]\n", "speedup", 100 * s.speedup_mean, 100 * s.speedup_ci_low,
                100 * s.speedup_ci_high);
    return kOk;
}

int cmd_export_dot(const Args& a) {
    std::string dot;
    if (a.has("memgraph")) dot = memgraph_to_dot(parse_memgraph(read_file(a.get("memgraph"))).first);
    else if (a.has("graph")) dot = taskgraph_to_dot(parse_taskgraph(read_file(a.get("graph"))));
    else {
        std::cerr << "export-dot needs --graph or --memgraph\n";
        return kUsage;
    }
    if (a.has("out")) write_file(a.get("out"), dot);
    else std::cout << dot;
    return kOk;
}

int cmd_execute(const Args& a) {
    const std::string mg = read_file(a.need("memgraph"));
    const std::string tg = read_file(a.need("graph"));
    Executor ex(mg, tg, parse_exec_config(a.get("config", "")));
    auto kv = [](const std::string& s) {
        auto eq = s.find('=');
        if (eq == std::string::npos) throw UsageError("expected ID=FILE, got " + s);
        return std::make_pair(static_cast<VertexId>(std::stoll(s.substr(0, eq))), s.substr(eq + 1));
    };
    if (a.opts.count("input"))
        for (const auto& s : a.opts.at("input")) {
            auto [id, path] = kv(s);
            std::string bytes = read_file(path);
            ex.set_input(id, bytes.data(), bytes.size(), false);
        }
    auto t = ex.run(policy_of(a), seed_of(a));
    if (a.opts.count("output"))
        for (const auto& s : a.opts.at("output")) {
            auto [id, path] = kv(s);
            auto [m, map] = parse_memgraph(mg);
            const std::int64_t n = map.placements.at(id).size;
            std::string buf(static_cast<size_t>(n), '\0');
            ex.get_output(id, buf.data(), buf.size());
            write_file(path, buf);
        }
    if (a.has("out")) write_file(a.get("out"), t.to_json());
    std::cout << ex.stats().to_json() << "\n";
    return kOk;
}

void usage() {
    std::cerr << "usage: turnip <validate|compile|verify|simulate|bench|export-dot|execute> [options]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kUsage;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        usage();
        return kOk;
    }
    try {
        if (cmd == "validate") return cmd_validate(parse_args(argc, argv, 2, {"graph"}, {}));
        if (cmd == "compile")
            return cmd_compile(parse_args(argc, argv, 2,
                                          {"graph", "capacities", "order-policy", "order-file", "victim-policy",
                                           "alloc-horizon", "seed", "out"},
                                          {"drop-superfluous"}));
        if (cmd == "verify") return cmd_verify(parse_args(argc, argv, 2, {"graph", "memgraph", "schedules"}, {}));
        if (cmd == "simulate")
            return cmd_simulate(parse_args(argc, argv, 2,
                                           {"memgraph", "profile", "policy", "tie-break", "seed", "out", "format"}, {}));
        if (cmd == "bench")
            return cmd_bench(parse_args(argc, argv, 2, {"memgraph", "profile", "trials", "seed", "out"}, {}));
        if (cmd == "export-dot") return cmd_export_dot(parse_args(argc, argv, 2, {"graph", "memgraph", "out"}, {}));
        if (cmd == "execute")
            return cmd_execute(parse_args(argc, argv, 2,
                                          {"memgraph", "graph", "config", "policy", "tie-break", "seed", "input",
                                           "output", "out"},
                                          {}));
        usage();
        return kUsage;
    } catch (const UsageError& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return kUsage;
    } catch (const ParseError& e) {
        std::cerr << "parse error: " << e.what() << "\n";
        return kUsage;
    } catch (const CudaError& e) {
        std::cerr << "cuda error: " << e.what() << "\n";
        return 3;
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kUsage;
    }
}
