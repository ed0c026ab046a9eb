// Graph model shared by the memgraph builder, the virtual-time dispatcher and
// the CUDA executor.
//
// Mirrors the reference data model field-for-field so the wire formats stay
// drop-in compatible:
//   TaskVertex/TaskGraph  <- proj/include/memplan/taskgraph.hpp:24-47
//   MemVertex/MemEdge/MemGraph/MemoryMap <- proj/include/memplan/memgraph.hpp:25-89
// Unlike the reference (linear-scan find, memgraph.cpp:40-50) every graph
// carries a hash index so lookups are O(1) at 10^5 vertices.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace tn {

using VertexId = std::int64_t;
using DeviceId = std::int32_t;

// ---------------------------------------------------------------- errors ---
// Error taxonomy of the reference (taskgraph.hpp:100-112, compiler.hpp:72-84).
// `code` is the C-ABI return code: 1 check/deadlock, 2 usage/parse/IO,
// 3 CUDA failure (executor only).
struct Error : std::runtime_error {
    int code;
    explicit Error(const std::string& m, int c = 2) : std::runtime_error(m), code(c) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m) : Error(m, 2) {}
};
struct CycleError : Error {
    std::vector<VertexId> cycle;
    CycleError(const std::string& m, std::vector<VertexId> w) : Error(m, 2), cycle(std::move(w)) {}
};
struct SingleTensorTooLargeError : Error {
    VertexId vertex;
    SingleTensorTooLargeError(const std::string& m, VertexId v) : Error(m, 2), vertex(v) {}
};
struct OffloadOverflowError : Error {
    explicit OffloadOverflowError(const std::string& m) : Error(m, 2) {}
};
struct InternalError : Error {
    explicit InternalError(const std::string& m) : Error(m, 2) {}
};
struct DeadlockError : Error {
    explicit DeadlockError(const std::string& m) : Error(m, 1) {}
};
struct CudaError : Error {
    explicit CudaError(const std::string& m) : Error(m, 3) {}
};

// ------------------------------------------------------------- taskgraph ---
enum class VertexKind : std::uint8_t { Input, Kernel, Transfer };

struct TaskVertex {
    VertexId id = 0;
    VertexKind kind = VertexKind::Input;
    DeviceId device = 0;
    DeviceId src_device = -1;
    std::int64_t output_size = 1;
    double cost_hint = 1.0;
};

struct TaskGraph {
    std::int32_t device_count = 1;
    std::vector<TaskVertex> vertices;
    std::vector<std::pair<VertexId, VertexId>> edges;

    // id -> index into `vertices` (first occurrence wins, like the
    // reference's linear find).
    std::unordered_map<VertexId, std::int32_t> index;
    void reindex();
    const TaskVertex* find(VertexId id) const;
    const TaskVertex& at(VertexId id) const;
};

using VertexOrder = std::vector<VertexId>;

enum class OrderPolicy : std::uint8_t { AsListed, DepthFirst, MinMemoryGreedy };

// -------------------------------------------------------------- memgraph ---
enum class MemOriginKind : std::uint8_t { Original, Offload, Reload };
enum class MemOpKind : std::uint8_t { Input, Kernel, Transfer, Offload, Reload };
enum class EdgeKind : std::uint8_t { Data, Memory };
enum class MemoryMode : std::uint8_t { Slot, Byte };

struct MemOrigin {
    MemOriginKind kind = MemOriginKind::Original;
    VertexId ref = 0;
    std::int32_t gen = 0;
};

struct MemVertex {
    VertexId id = 0;
    MemOrigin origin;
    MemOpKind op = MemOpKind::Kernel;
    DeviceId device = 0;
    DeviceId src_device = -1;
    std::int64_t size = 1;
    double cost_hint = 1.0;
};

struct MemEdge {
    VertexId from = 0;
    VertexId to = 0;
    EdgeKind kind = EdgeKind::Data;
    bool superfluous = false;
};

struct MemGraph {
    std::vector<MemVertex> vertices;
    std::vector<MemEdge> edges;
    std::vector<VertexId> total_order;
    std::int32_t device_count = 1;

    std::unordered_map<VertexId, std::int32_t> index;
    void reindex();
    std::int32_t idx(VertexId id) const;  // -1 when absent
    const MemVertex& at(VertexId id) const;
};

struct Placement {
    DeviceId device = 0;
    std::int64_t offset = 0;
    std::int64_t size = 1;
};

struct RegionClaim {
    VertexId owner = 0;
    DeviceId device = 0;
    std::int64_t offset = 0;
    std::int64_t size = 0;
};

struct MemoryMap {
    MemoryMode mode = MemoryMode::Slot;
    std::vector<std::int64_t> capacities;
    std::map<VertexId, Placement> placements;  // ordered: JSON key order
    std::vector<RegionClaim> history;
};

inline bool overlaps(const Placement& a, const Placement& b) {
    if (a.device != b.device) return false;
    return a.offset < b.offset + b.size && b.offset < a.offset + a.size;
}

const char* to_string(VertexKind k);
const char* to_string(MemOriginKind k);
const char* to_string(MemOpKind k);
const char* to_string(EdgeKind k);
const char* to_string(OrderPolicy p);
OrderPolicy order_policy_from_string(const std::string& s);

}  // namespace tn
