// Memgraph construction (bit-exact vs the reference), taskgraph utilities and
// wire formats. Reference interfaces restated here:
//   build_memgraph / BuildOptions / BuildStats   proj/include/memplan/compiler.hpp:16-65
//   prune_superfluous_edges                      proj/include/memplan/compiler.hpp:70
//   validate/topological_order/generators        proj/include/memplan/taskgraph.hpp:55-95
//   serialize_/parse_ memgraph + taskgraph       memgraph.hpp:94-96, taskgraph.hpp:79-81
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "types.hpp"

namespace tn {

enum class VictimPolicy : std::uint8_t { FarthestNextUse, LastAllocated, SeededRandom };
enum class AllocHorizonMode : std::uint8_t { Greedy, Lazy };

VictimPolicy victim_policy_from_string(const std::string& s);
AllocHorizonMode alloc_horizon_from_string(const std::string& s);

struct BuildOptions {
    VictimPolicy victim_policy = VictimPolicy::FarthestNextUse;
    std::uint64_t victim_seed = 0;
    AllocHorizonMode alloc_horizon = AllocHorizonMode::Greedy;
    bool keep_superfluous = true;
    std::optional<std::int64_t> host_capacity;
    bool check_invariants = false;
};

struct BuildStats {
    std::int64_t offload_count = 0;
    std::int64_t reload_count = 0;
    std::int64_t memory_edge_count = 0;
    std::int64_t required_memory_edge_count = 0;
    std::vector<std::int64_t> peak_usage;
};

struct BuildResult {
    MemGraph memgraph;
    MemoryMap memory_map;
    BuildStats stats;
};

BuildResult build_memgraph(const TaskGraph& g, const VertexOrder& order,
                           const std::vector<std::int64_t>& capacities, MemoryMode mode,
                           const BuildOptions& options = {});

// Flags (or drops) every Memory edge (u,w) with another u->w path.
// Reachability is searched only inside the total-order window [u, w]:
// every edge points forward in total_order, so no u->w path can leave it.
void prune_superfluous_edges(MemGraph& m, bool drop);

// --- taskgraph utilities -----------------------------------------------------
std::vector<std::string> validate_taskgraph(const TaskGraph& g);
VertexOrder topological_order(const TaskGraph& g, OrderPolicy policy, std::uint64_t seed = 0);
bool is_linear_extension(const TaskGraph& g, const VertexOrder& order);


// --- wire formats -------------------------------------------------------------
std::string serialize_taskgraph(const TaskGraph& g);
TaskGraph parse_taskgraph(const std::string& text);
std::string taskgraph_to_dot(const TaskGraph& g);

std::string serialize_memgraph(const MemGraph& m, const MemoryMap& map);
std::pair<MemGraph, MemoryMap> parse_memgraph(const std::string& text);
std::string memgraph_to_dot(const MemGraph& m);
std::string stats_to_json(const BuildStats& s);

}  // namespace tn
