// Graph indices, taskgraph validation/ordering/generators, pruning and the
// JSON/DOT wire formats.
//
// The wire formats are the reference's (memgraph.cpp:72-182,
// taskgraph.cpp:344-414) and are produced with the same nlohmann
// ordered_json `dump(2)` so bytes match. The generators restate
// taskgraph.cpp:418-616 (same libstdc++ <random> draws, so the same graphs)
// because the differential corpus on the GPU box must not need the reference.
#include <algorithm>
#include <functional>
#include <map>
#include <queue>
#include <random>
#include <set>
#include <sstream>

#include <nlohmann/json.hpp>

// Byte-identical serialisation with the reference depends on the exact
// nlohmann/json release it links (number formatting, dump(2) layout).
#if NLOHMANN_JSON_VERSION_MAJOR != 3 || NLOHMANN_JSON_VERSION_MINOR != 11 || NLOHMANN_JSON_VERSION_PATCH != 3
#error "memgraph JSON must be serialised with nlohmann/json 3.11.3 (set JSONINC)"
#endif

#include "planner.hpp"

namespace tn {

using json = nlohmann::ordered_json;  // serialisation: the reference's key order and layout
// Parsing only reads keys, so it uses the std::map object type: an
// ordered_json object is a vector with linear key lookup, which made parsing
// a 38k-vertex memgraph (38k placement keys) quadratic (3.7 s vs 0.7 s).
using pjson = nlohmann::json;

// ------------------------------------------------------------------ basics --
void TaskGraph::reindex() {
    index.clear();
    index.reserve(vertices.size() * 2 + 1);
    for (size_t i = 0; i < vertices.size(); ++i) index.try_emplace(vertices[i].id, static_cast<std::int32_t>(i));
}
const TaskVertex* TaskGraph::find(VertexId id) const {
    auto it = index.find(id);
    return it == index.end() ? nullptr : &vertices[it->second];
}
const TaskVertex& TaskGraph::at(VertexId id) const {
    const TaskVertex* v = find(id);
    if (!v) throw Error("no vertex with id " + std::to_string(id));
    return *v;
}
void MemGraph::reindex() {
    index.clear();
    index.reserve(vertices.size() * 2 + 1);
    for (size_t i = 0; i < vertices.size(); ++i) index.try_emplace(vertices[i].id, static_cast<std::int32_t>(i));
}
std::int32_t MemGraph::idx(VertexId id) const {
    auto it = index.find(id);
    return it == index.end() ? -1 : it->second;
}
const MemVertex& MemGraph::at(VertexId id) const {
    auto i = idx(id);
    if (i < 0) throw Error("no memgraph vertex with id " + std::to_string(id));
    return vertices[i];
}

const char* to_string(VertexKind k) {
    switch (k) {
        case VertexKind::Input: return "input";
        case VertexKind::Kernel: return "kernel";
        case VertexKind::Transfer: return "transfer";
    }
    return "?";
}
const char* to_string(MemOriginKind k) {
    switch (k) {
        case MemOriginKind::Original: return "original";
        case MemOriginKind::Offload: return "offload";
        case MemOriginKind::Reload: return "reload";
    }
    return "?";
}
const char* to_string(MemOpKind k) {
    switch (k) {
        case MemOpKind::Input: return "input";
        case MemOpKind::Kernel: return "kernel";
        case MemOpKind::Transfer: return "transfer";
        case MemOpKind::Offload: return "offload";
        case MemOpKind::Reload: return "reload";
    }
    return "?";
}
const char* to_string(EdgeKind k) { return k == EdgeKind::Data ? "data" : "memory"; }
const char* to_string(OrderPolicy p) {
    switch (p) {
        case OrderPolicy::AsListed: return "as-listed";
        case OrderPolicy::DepthFirst: return "depth-first";
        case OrderPolicy::MinMemoryGreedy: return "min-memory-greedy";
    }
    return "?";
}
OrderPolicy order_policy_from_string(const std::string& s) {
    if (s == "as-listed") return OrderPolicy::AsListed;
    if (s == "depth-first") return OrderPolicy::DepthFirst;
    if (s == "min-memory-greedy") return OrderPolicy::MinMemoryGreedy;
    throw Error("unknown order policy: " + s);
}

// -------------------------------------------------------------- validation --
// Same checks and messages as taskgraph.cpp:100-201.
std::vector<std::string> validate_taskgraph(const TaskGraph& g) {
    std::vector<std::string> out;
    auto violate = [&](std::string m) { out.push_back(std::move(m)); };
    if (g.device_count < 1) violate("device_count must be >= 1");

    std::unordered_map<VertexId, const TaskVertex*> by_id;
    for (const auto& v : g.vertices) {
        if (!by_id.emplace(v.id, &v).second) violate("duplicate vertex id " + std::to_string(v.id));
        if (v.output_size <= 0) violate("vertex " + std::to_string(v.id) + ": output_size must be > 0");
        if (v.device < 0 || v.device >= g.device_count)
            violate("vertex " + std::to_string(v.id) + ": device out of range");
        if (v.kind == VertexKind::Transfer) {
            if (v.src_device < 0 || v.src_device >= g.device_count)
                violate("transfer " + std::to_string(v.id) + ": src_device out of range");
            else if (v.src_device == v.device)
                violate("transfer " + std::to_string(v.id) + ": source device equals destination device");
        }
        if (v.cost_hint < 0) violate("vertex " + std::to_string(v.id) + ": cost_hint must be >= 0");
    }
    std::set<std::pair<VertexId, VertexId>> seen;
    std::unordered_map<VertexId, int> indegree;
    for (const auto& [p, c] : g.edges) {
        if (p == c) {
            violate("self-loop at " + std::to_string(p));
            continue;
        }
        if (!by_id.count(p)) violate("edge references missing producer " + std::to_string(p));
        if (!by_id.count(c)) violate("edge references missing consumer " + std::to_string(c));
        if (!seen.insert({p, c}).second)
            violate("duplicate edge " + std::to_string(p) + "->" + std::to_string(c));
        indegree[c]++;
    }
    for (const auto& v : g.vertices) {
        int in = indegree.count(v.id) ? indegree[v.id] : 0;
        switch (v.kind) {
            case VertexKind::Input:
                if (in != 0) violate("input " + std::to_string(v.id) + " has inbound edges");
                break;
            case VertexKind::Transfer:
                if (in != 1) violate("transfer " + std::to_string(v.id) + " must have exactly one inbound edge");
                break;
            case VertexKind::Kernel:
                if (in < 1) violate("kernel " + std::to_string(v.id) + " has no inbound edges");
                break;
        }
    }
    for (const auto& [p, c] : g.edges) {
        auto pi = by_id.find(p), ci = by_id.find(c);
        if (pi == by_id.end() || ci == by_id.end()) continue;
        const TaskVertex& prod = *pi->second;
        const TaskVertex& cons = *ci->second;
        if (cons.kind == VertexKind::Kernel && prod.device != cons.device)
            violate("kernel " + std::to_string(c) + " on device " + std::to_string(cons.device) + " reads tensor " +
                    std::to_string(p) + " on device " + std::to_string(prod.device) + " without a transfer");
        if (cons.kind == VertexKind::Transfer && prod.device != cons.src_device)
            violate("transfer " + std::to_string(c) + " declares src_device " + std::to_string(cons.src_device) +
                    " but reads tensor on device " + std::to_string(prod.device));
    }
    if (!by_id.empty()) {
        // Kahn over the distinct-id vertex set (self-loops excluded).
        std::unordered_map<VertexId, int> deg;
        std::unordered_map<VertexId, std::vector<VertexId>> adj;
        for (const auto& v : g.vertices) deg[v.id] = 0;
        for (const auto& [p, c] : g.edges)
            if (by_id.count(p) && by_id.count(c) && p != c) {
                deg[c]++;
                adj[p].push_back(c);
            }
        std::vector<VertexId> ready;
        for (const auto& [id, d] : deg)
            if (d == 0) ready.push_back(id);
        size_t visited = 0;
        while (!ready.empty()) {
            VertexId u = ready.back();
            ready.pop_back();
            ++visited;
            auto it = adj.find(u);
            if (it == adj.end()) continue;
            for (VertexId w : it->second)
                if (--deg[w] == 0) ready.push_back(w);
        }
        if (visited != by_id.size()) violate("graph contains a cycle");
    }
    return out;
}

// --------------------------------------------------------------- ordering --
namespace {

std::vector<VertexId> find_cycle(const TaskGraph& g) {
    std::map<VertexId, int> color;
    std::map<VertexId, VertexId> parent;
    std::map<VertexId, std::vector<VertexId>> adj;
    for (const auto& [p, c] : g.edges) adj[p].push_back(c);
    for (const auto& v : g.vertices) color[v.id] = 0;
    std::vector<VertexId> cycle;
    std::function<bool(VertexId)> dfs = [&](VertexId u) {
        color[u] = 1;
        for (VertexId w : adj[u]) {
            if (color[w] == 1) {
                cycle.push_back(w);
                for (VertexId x = u; x != w; x = parent[x]) cycle.push_back(x);
                cycle.push_back(w);
                std::reverse(cycle.begin(), cycle.end());
                return true;
            }
            if (color[w] == 0) {
                parent[w] = u;
                if (dfs(w)) return true;
            }
        }
        color[u] = 2;
        return false;
    };
    for (const auto& v : g.vertices)
        if (color[v.id] == 0 && dfs(v.id)) return cycle;
    return {};
}

}  // namespace

// Same three policies as taskgraph.cpp:242-328 (the seed is ignored there too).
VertexOrder topological_order(const TaskGraph& g, OrderPolicy policy, std::uint64_t) {
    std::unordered_map<VertexId, size_t> listed;
    for (size_t i = 0; i < g.vertices.size(); ++i) listed[g.vertices[i].id] = i;
    std::unordered_map<VertexId, std::vector<VertexId>> adj, radj;
    std::unordered_map<VertexId, int> indeg;
    for (const auto& v : g.vertices) indeg[v.id] = 0;
    for (const auto& [p, c] : g.edges) {
        adj[p].push_back(c);
        radj[c].push_back(p);
        indeg[c]++;
    }
    for (auto& [id, list] : adj)
        std::stable_sort(list.begin(), list.end(), [&](VertexId a, VertexId b) { return listed[a] < listed[b]; });

    VertexOrder order;
    order.reserve(g.vertices.size());
    if (policy == OrderPolicy::DepthFirst) {
        // Reverse DFS finish order from roots in listed order (iterative).
        std::unordered_map<VertexId, int> state;
        std::vector<VertexId> finish;
        for (const auto& root : g.vertices) {
            if (state[root.id] != 0) continue;
            std::vector<std::pair<VertexId, size_t>> stack{{root.id, 0}};
            state[root.id] = 1;
            while (!stack.empty()) {
                auto& [u, i] = stack.back();
                auto it = adj.find(u);
                const size_t deg = it == adj.end() ? 0 : it->second.size();
                if (i < deg) {
                    VertexId w = it->second[i++];
                    int s = state[w];
                    if (s == 0) {
                        state[w] = 1;
                        stack.push_back({w, 0});
                    } else if (s == 1) {
                        throw CycleError("cycle detected", find_cycle(g));
                    }
                } else {
                    state[u] = 2;
                    finish.push_back(u);
                    stack.pop_back();
                }
            }
        }
        order.assign(finish.rbegin(), finish.rend());
        if (order.size() != g.vertices.size()) throw CycleError("cycle detected", find_cycle(g));
        return order;
    }

    // Kahn; ready kept ordered by listed position (AsListed picks the minimum).
    std::set<std::pair<size_t, VertexId>> ready;
    for (const auto& v : g.vertices)
        if (indeg[v.id] == 0) ready.insert({listed[v.id], v.id});
    std::unordered_map<VertexId, int> remaining;
    for (const auto& [p, c] : g.edges) remaining[p]++;

    while (!ready.empty()) {
        VertexId u;
        if (policy == OrderPolicy::AsListed) {
            u = ready.begin()->second;
            ready.erase(ready.begin());
        } else {
            // Min immediate live delta, ties by listed position: iterating in
            // listed order with strict < keeps the first minimum.
            VertexId best = 0;
            std::int64_t best_delta = 0;
            bool first = true;
            for (const auto& [lp, cand] : ready) {
                std::int64_t delta = g.at(cand).output_size;
                auto rit = radj.find(cand);
                if (rit != radj.end())
                    for (VertexId in : rit->second)
                        if (remaining[in] == 1) delta -= g.at(in).output_size;
                if (first || delta < best_delta) {
                    best = cand;
                    best_delta = delta;
                    first = false;
                }
            }
            u = best;
            ready.erase({listed[u], u});
        }
        order.push_back(u);
        auto rit = radj.find(u);
        if (rit != radj.end())
            for (VertexId in : rit->second) remaining[in]--;
        auto ait = adj.find(u);
        if (ait != adj.end())
            for (VertexId w : ait->second)
                if (--indeg[w] == 0) ready.insert({listed[w], w});
    }
    if (order.size() != g.vertices.size()) throw CycleError("cycle detected", find_cycle(g));
    return order;
}

bool is_linear_extension(const TaskGraph& g, const VertexOrder& order) {
    if (order.size() != g.vertices.size()) return false;
    std::unordered_map<VertexId, size_t> pos;
    pos.reserve(order.size() * 2 + 1);
    for (size_t i = 0; i < order.size(); ++i) {
        if (!g.find(order[i])) return false;
        if (!pos.emplace(order[i], i).second) return false;
    }
    for (const auto& [p, c] : g.edges) {
        auto pi = pos.find(p), ci = pos.find(c);
        size_t pp = pi == pos.end() ? 0 : pi->second;
        size_t cp = ci == pos.end() ? 0 : ci->second;
        if (pp >= cp) return false;
    }
    return true;
}

// ----------------------------------------------------------------- pruning --
// compiler.cpp:546-585 does one unbounded BFS per memory edge. Here each BFS
// is confined to total_order positions <= pos(w) (all edges point forward,
// so a u->w path never leaves [pos(u), pos(w)]), and the searches run in
// parallel: in flag mode they are independent, and in drop mode dropping a
// superfluous edge never changes reachability of a DAG, so the flag set is
// order-independent as well.
void prune_superfluous_edges(MemGraph& m, bool drop) {
    const size_t V = m.vertices.size();
    if (m.index.size() != V) m.reindex();
    std::vector<std::int32_t> pos(V, -1);
    for (size_t i = 0; i < m.total_order.size(); ++i) {
        auto ix = m.idx(m.total_order[i]);
        if (ix >= 0) pos[ix] = static_cast<std::int32_t>(i);
    }
    bool have_order = m.total_order.size() == V;
    for (size_t i = 0; have_order && i < V; ++i) have_order = pos[i] >= 0;
    // CSR over out-edges by edge index.
    const size_t E = m.edges.size();
    std::vector<std::int32_t> from(E), to(E), start(V + 1, 0), adj(E);
    for (size_t e = 0; e < E; ++e) {
        from[e] = m.idx(m.edges[e].from);
        to[e] = m.idx(m.edges[e].to);
        start[from[e] + 1]++;
    }
    for (size_t i = 0; i < V; ++i) start[i + 1] += start[i];
    {
        std::vector<std::int32_t> fill(start.begin(), start.end() - 1);
        for (size_t e = 0; e < E; ++e) adj[fill[from[e]]++] = static_cast<std::int32_t>(e);
    }
    std::vector<std::int32_t> mem_edges;
    for (size_t e = 0; e < E; ++e)
        if (m.edges[e].kind == EdgeKind::Memory) mem_edges.push_back(static_cast<std::int32_t>(e));
    std::vector<char> flag(E, 0);

#pragma omp parallel if (mem_edges.size() > 512)
    {
        std::vector<std::uint32_t> seen(V, 0);
        std::uint32_t epoch = 0;
        std::vector<std::int32_t> queue;
        queue.reserve(1024);
#pragma omp for schedule(dynamic, 16)
        for (std::int64_t k = 0; k < static_cast<std::int64_t>(mem_edges.size()); ++k) {
            const std::int32_t e = mem_edges[k];
            const std::int32_t u = from[e], w = to[e];
            const std::int32_t limit = have_order ? pos[w] : INT32_MAX;
            if (++epoch == 0) {
                std::fill(seen.begin(), seen.end(), 0);
                epoch = 1;
            }
            queue.clear();
            queue.push_back(u);
            seen[u] = epoch;
            bool found = false;
            for (size_t qi = 0; qi < queue.size() && !found; ++qi) {
                const std::int32_t x = queue[qi];
                for (std::int32_t a = start[x]; a < start[x + 1]; ++a) {
                    const std::int32_t ei = adj[a];
                    if (ei == e) continue;
                    const std::int32_t y = to[ei];
                    if (y == w) {
                        found = true;
                        break;
                    }
                    if (seen[y] == epoch) continue;
                    if (have_order && pos[y] > limit) continue;
                    seen[y] = epoch;
                    queue.push_back(y);
                }
            }
            flag[e] = found ? 1 : 0;
        }
    }
    for (size_t e = 0; e < E; ++e)
        if (flag[e]) m.edges[e].superfluous = true;
    if (drop) {
        std::vector<MemEdge> kept;
        kept.reserve(E);
        for (size_t e = 0; e < E; ++e)
            if (!flag[e]) kept.push_back(m.edges[e]);
        m.edges = std::move(kept);
    }
}

// -------------------------------------------------------------- taskgraph IO --
std::string serialize_taskgraph(const TaskGraph& g) {
    json j;
    j["device_count"] = g.device_count;
    j["vertices"] = json::array();
    for (const auto& v : g.vertices) {
        json jv;
        jv["id"] = v.id;
        jv["kind"] = to_string(v.kind);
        jv["device"] = v.device;
        if (v.kind == VertexKind::Transfer) jv["src_device"] = v.src_device;
        jv["output_size"] = v.output_size;
        jv["cost_hint"] = v.cost_hint;
        j["vertices"].push_back(std::move(jv));
    }
    j["edges"] = json::array();
    for (const auto& [p, c] : g.edges) j["edges"].push_back(json::array({p, c}));
    return j.dump(2) + "\n";
}

TaskGraph parse_taskgraph(const std::string& text) {
    pjson j;
    try {
        j = pjson::parse(text);
    } catch (const pjson::parse_error& e) {
        throw ParseError(std::string("invalid JSON: ") + e.what());
    }
    if (!j.is_object()) throw ParseError("top level must be an object");
    if (!j.contains("vertices")) throw ParseError("missing vertices");
    TaskGraph g;
    try {
        g.device_count = j.value("device_count", 1);
        for (const auto& jv : j["vertices"]) {
            TaskVertex v;
            if (!jv.contains("id")) throw ParseError("vertex missing id");
            v.id = jv["id"].get<VertexId>();
            std::string kind = jv.value("kind", "");
            if (kind == "input") v.kind = VertexKind::Input;
            else if (kind == "kernel") v.kind = VertexKind::Kernel;
            else if (kind == "transfer") v.kind = VertexKind::Transfer;
            else throw ParseError("vertex " + std::to_string(v.id) + ": unknown kind '" + kind + "'");
            v.device = jv.value("device", 0);
            v.src_device = jv.value("src_device", -1);
            v.output_size = jv.value("output_size", std::int64_t{1});
            v.cost_hint = jv.value("cost_hint", 1.0);
            g.vertices.push_back(v);
        }
        g.reindex();
        for (const auto& je : j.value("edges", json::array())) {
            if (!je.is_array() || je.size() != 2) throw ParseError("edge must be a [producer, consumer] pair");
            VertexId p = je[0].get<VertexId>(), c = je[1].get<VertexId>();
            if (!g.find(p)) throw ParseError("edge references unknown vertex " + std::to_string(p));
            if (!g.find(c)) throw ParseError("edge references unknown vertex " + std::to_string(c));
            g.edges.emplace_back(p, c);
        }
    } catch (const pjson::exception& e) {
        throw ParseError(std::string("invalid taskgraph: ") + e.what());
    }
    return g;
}

std::string taskgraph_to_dot(const TaskGraph& g) {
    std::ostringstream out;
    out << "digraph taskgraph {\n";
    for (const auto& v : g.vertices)
        out << "  v" << v.id << " [label=\"" << v.id << " " << to_string(v.kind) << "@" << v.device << "\"];\n";
    for (const auto& [p, c] : g.edges) out << "  v" << p << " -> v" << c << ";\n";
    out << "}\n";
    return out.str();
}

// --------------------------------------------------------------- memgraph IO --
std::string serialize_memgraph(const MemGraph& m, const MemoryMap& map) {
    json j;
    j["device_count"] = m.device_count;
    j["mode"] = map.mode == MemoryMode::Slot ? "slot" : "byte";
    j["capacities"] = map.capacities;
    j["vertices"] = json::array();
    for (const auto& v : m.vertices) {
        json jv;
        jv["id"] = v.id;
        jv["origin"] = {{"kind", to_string(v.origin.kind)}, {"ref", v.origin.ref}};
        if (v.origin.kind != MemOriginKind::Original) jv["origin"]["gen"] = v.origin.gen;
        jv["op"] = to_string(v.op);
        jv["device"] = v.device;
        if (v.op == MemOpKind::Transfer) jv["src_device"] = v.src_device;
        jv["size"] = v.size;
        jv["cost_hint"] = v.cost_hint;
        j["vertices"].push_back(std::move(jv));
    }
    j["edges"] = json::array();
    for (const auto& e : m.edges)
        j["edges"].push_back(
            {{"from", e.from}, {"to", e.to}, {"kind", to_string(e.kind)}, {"superfluous", e.superfluous}});
    j["total_order"] = m.total_order;
    j["placement"] = json::object();
    for (const auto& [id, p] : map.placements)
        j["placement"][std::to_string(id)] = {{"device", p.device}, {"offset", p.offset}, {"size", p.size}};
    j["history"] = json::array();
    for (const auto& h : map.history)
        j["history"].push_back({{"owner", h.owner}, {"device", h.device}, {"offset", h.offset}, {"size", h.size}});
    return j.dump(2) + "\n";
}

std::pair<MemGraph, MemoryMap> parse_memgraph(const std::string& text) {
    pjson j;
    try {
        j = pjson::parse(text);
    } catch (const pjson::parse_error& e) {
        throw ParseError(std::string("invalid JSON: ") + e.what());
    }
    if (!j.is_object() || !j.contains("vertices") || !j.contains("edges"))
        throw ParseError("memgraph file needs vertices and edges");
    MemGraph m;
    MemoryMap map;
    try {
        m.device_count = j.value("device_count", 1);
        map.mode = j.value("mode", "slot") == std::string("byte") ? MemoryMode::Byte : MemoryMode::Slot;
        map.capacities = j.value("capacities", std::vector<std::int64_t>{});
        for (const auto& jv : j["vertices"]) {
            MemVertex v;
            v.id = jv.at("id").get<VertexId>();
            std::string ok = jv.at("origin").value("kind", "original");
            if (ok == "original") v.origin.kind = MemOriginKind::Original;
            else if (ok == "offload") v.origin.kind = MemOriginKind::Offload;
            else if (ok == "reload") v.origin.kind = MemOriginKind::Reload;
            else throw ParseError("unknown origin kind '" + ok + "'");
            v.origin.ref = jv.at("origin").value("ref", VertexId{0});
            v.origin.gen = jv.at("origin").value("gen", 0);
            std::string op = jv.value("op", "kernel");
            if (op == "input") v.op = MemOpKind::Input;
            else if (op == "kernel") v.op = MemOpKind::Kernel;
            else if (op == "transfer") v.op = MemOpKind::Transfer;
            else if (op == "offload") v.op = MemOpKind::Offload;
            else if (op == "reload") v.op = MemOpKind::Reload;
            else throw ParseError("unknown op kind '" + op + "'");
            v.device = jv.value("device", 0);
            v.src_device = jv.value("src_device", -1);
            v.size = jv.value("size", std::int64_t{1});
            v.cost_hint = jv.value("cost_hint", 1.0);
            m.vertices.push_back(v);
        }
        m.reindex();
        for (const auto& je : j["edges"]) {
            MemEdge e;
            e.from = je.at("from").get<VertexId>();
            e.to = je.at("to").get<VertexId>();
            e.kind = je.value("kind", "data") == std::string("memory") ? EdgeKind::Memory : EdgeKind::Data;
            e.superfluous = je.value("superfluous", false);
            if (m.idx(e.from) < 0 || m.idx(e.to) < 0) throw ParseError("edge references unknown memgraph vertex");
            m.edges.push_back(e);
        }
        m.total_order = j.value("total_order", std::vector<VertexId>{});
        if (j.contains("placement")) {
            for (const auto& [key, jp] : j["placement"].items()) {
                Placement p;
                p.device = jp.value("device", 0);
                p.offset = jp.value("offset", std::int64_t{0});
                p.size = jp.value("size", std::int64_t{1});
                map.placements[std::stoll(key)] = p;
            }
        }
        if (j.contains("history")) {
            for (const auto& jh : j["history"]) {
                RegionClaim h;
                h.owner = jh.value("owner", VertexId{0});
                h.device = jh.value("device", 0);
                h.offset = jh.value("offset", std::int64_t{0});
                h.size = jh.value("size", std::int64_t{0});
                map.history.push_back(h);
            }
        }
    } catch (const pjson::exception& e) {
        throw ParseError(std::string("invalid memgraph: ") + e.what());
    }
    return {std::move(m), std::move(map)};
}

std::string memgraph_to_dot(const MemGraph& m) {
    std::ostringstream out;
    out << "digraph memgraph {\n";
    for (const auto& v : m.vertices) {
        std::string label;
        switch (v.origin.kind) {
            case MemOriginKind::Original:
                label = std::to_string(v.id) + " " + to_string(v.op) + "@" + std::to_string(v.device);
                break;
            case MemOriginKind::Offload:
                label = "offload_" + std::to_string(v.origin.ref) + "@" + std::to_string(v.device);
                break;
            case MemOriginKind::Reload:
                label = "reload_" + std::to_string(v.origin.ref) + "@" + std::to_string(v.device);
                break;
        }
        out << "  v" << v.id << " [label=\"" << label << "\"";
        if (v.origin.kind != MemOriginKind::Original) out << " shape=box";
        out << "];\n";
    }
    for (const auto& e : m.edges) {
        out << "  v" << e.from << " -> v" << e.to;
        if (e.superfluous) out << " [color=gray style=dashed]";
        else if (e.kind == EdgeKind::Memory) out << " [color=red]";
        out << ";\n";
    }
    out << "}\n";
    return out.str();
}

std::string stats_to_json(const BuildStats& s) {
    json j;
    j["offloads"] = s.offload_count;
    j["reloads"] = s.reload_count;
    j["memory_edges"] = s.memory_edge_count;
    j["required_memory_edges"] = s.required_memory_edge_count;
    j["peak_usage"] = s.peak_usage;
    return j.dump();
}

}  // namespace tn
