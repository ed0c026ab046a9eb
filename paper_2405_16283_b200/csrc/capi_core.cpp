// C ABI for the planner and the virtual-time dispatcher (include/turnip.h).
// Each entry point mirrors one function of the reference pybind module
// (proj/python/bindings.cpp) with JSON strings across the boundary.
#include <cstdlib>
#include <cstring>
#include <exception>

#include <nlohmann/json.hpp>

#include "../../include/turnip.h"
#include "core/dispatch.hpp"
#include "core/planner.hpp"
#include "core/verify.hpp"

using namespace tn;

namespace {

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = 0;
    return p;
}

template <class F>
int guarded(char** err, F&& f) {
    try {
        f();
        return 0;
    } catch (const tn::Error& e) {
        if (err) *err = dup(e.what());
        return e.code;
    } catch (const std::exception& e) {
        if (err) *err = dup(e.what());
        return 2;
    } catch (...) {
        if (err) *err = dup("unknown error");
        return 2;
    }
}

std::string str(const char* s, const char* dflt = "") { return s ? std::string(s) : std::string(dflt); }

}  // namespace

extern "C" {

const char* tn_version(void) { return "turnip-b200 0.1"; }
void tn_free(void* p) { std::free(p); }

int tn_validate_taskgraph(const char* graph_json, char** out, char** err) {
    return guarded(err, [&] {
        auto v = validate_taskgraph(parse_taskgraph(str(graph_json)));
        *out = dup(nlohmann::json(v).dump());
    });
}

int tn_topological_order(const char* graph_json, const char* policy, uint64_t seed, char** out, char** err) {
    return guarded(err, [&] {
        auto g = parse_taskgraph(str(graph_json));
        auto o = topological_order(g, order_policy_from_string(str(policy, "as-listed")), seed);
        *out = dup(nlohmann::json(o).dump());
    });
}

int tn_taskgraph_to_dot(const char* graph_json, char** out, char** err) {
    return guarded(err, [&] { *out = dup(taskgraph_to_dot(parse_taskgraph(str(graph_json)))); });
}
int tn_memgraph_to_dot(const char* memgraph_json, char** out, char** err) {
    return guarded(err, [&] { *out = dup(memgraph_to_dot(parse_memgraph(str(memgraph_json)).first)); });
}

int tn_build_memgraph(const char* graph_json, const int64_t* caps, size_t ncaps, const char* mode,
                      const int64_t* order, size_t norder, const char* order_policy, const char* victim_policy,
                      uint64_t seed, const char* alloc_horizon, int keep_superfluous, int64_t host_capacity,
                      char** memgraph_json, char** stats_json, char** err) {
    return guarded(err, [&] {
        auto g = parse_taskgraph(str(graph_json));
        VertexOrder o(order, order + norder);
        if (o.empty()) o = topological_order(g, order_policy_from_string(str(order_policy, "as-listed")), seed);
        MemoryMode mm = str(mode, "slot") == "byte" ? MemoryMode::Byte : MemoryMode::Slot;
        BuildOptions opts;
        opts.victim_policy = victim_policy_from_string(str(victim_policy, "farthest-next-use"));
        opts.victim_seed = seed;
        opts.alloc_horizon = alloc_horizon_from_string(str(alloc_horizon, "greedy"));
        opts.keep_superfluous = keep_superfluous != 0;
        if (host_capacity >= 0) opts.host_capacity = host_capacity;
        std::vector<std::int64_t> c(caps, caps + ncaps);
        auto r = build_memgraph(g, o, c, mm, opts);
        *memgraph_json = dup(serialize_memgraph(r.memgraph, r.memory_map));
        if (stats_json) *stats_json = dup(stats_to_json(r.stats));
    });
}

int tn_simulate(const char* memgraph_json, const char* profile_json, const char* policy, const char* tie_break,
                uint64_t seed, const char* format, char** out, char** err) {
    return guarded(err, [&] {
        auto [m, map] = parse_memgraph(str(memgraph_json));
        DeviceProfile p;
        if (profile_json && *profile_json) p = parse_profile(profile_json);
        SchedulerPolicy pol;
        pol.kind = scheduler_kind_from_string(str(policy, "event-driven"));
        pol.tie_break = tie_break_from_string(str(tie_break, "fifo"));
        auto t = simulate(m, map, p, pol, seed);
        *out = dup(str(format, "json") == "csv" ? t.to_csv() : t.to_json());
    });
}

int tn_compare_policies(const char* memgraph_json, const char* profile_json, int64_t trials, uint64_t seed,
                        char** out, char** err) {
    return guarded(err, [&] {
        auto [m, map] = parse_memgraph(str(memgraph_json));
        DeviceProfile p;
        if (profile_json && *profile_json) p = parse_profile(profile_json);
        *out = dup(compare_policies(m, map, p, trials, seed).to_json());
    });
}

int tn_verify(const char* graph_json, const char* memgraph_json, int64_t schedule_limit, char** out, char** err) {
    return guarded(err, [&] {
        auto g = parse_taskgraph(str(graph_json));
        auto [m, map] = parse_memgraph(str(memgraph_json));
        *out = dup(verify_all(g, m, map, schedule_limit).to_json());
    });
}

int tn_check_capacity(const char* memgraph_json, const int64_t* order, size_t norder, char** out, char** err) {
    return guarded(err, [&] {
        auto [m, map] = parse_memgraph(str(memgraph_json));
        std::vector<VertexId> o(order, order + norder);
        auto r = check_capacity(m, map, o);
        nlohmann::ordered_json j;
        j["passed"] = r.passed;
        if (!r.passed) j["witness"] = r.witness;
        *out = dup(j.dump());
    });
}

int tn_make_fixed_order(const char* memgraph_json, char** out, char** err) {
    return guarded(err, [&] {
        auto [m, map] = parse_memgraph(str(memgraph_json));
        *out = dup(serialize_memgraph(make_fixed_order(m), map));
    });
}

}  // extern "C"
