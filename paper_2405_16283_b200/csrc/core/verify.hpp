// Memgraph verifier: drop-in for proj/include/memplan/verifier.hpp:17-72.
#pragma once

#include <string>
#include <vector>

#include "planner.hpp"

namespace tn {

struct CheckResult {
    bool passed = true;
    std::string witness;
    static CheckResult pass() { return {}; }
    static CheckResult fail(std::string w) { return {false, std::move(w)}; }
};

struct ScheduleCheckResult {
    bool passed = true;
    bool sampled = false;
    std::int64_t schedules_run = 0;
    std::string witness;
};

CheckResult check_acyclic(const MemGraph& m);
CheckResult check_data_preservation(const TaskGraph& g, const MemGraph& m);
CheckResult check_race_freedom(const MemGraph& m, const MemoryMap& map);
CheckResult check_capacity(const MemGraph& m, const MemoryMap& map, const std::vector<VertexId>& order);
ScheduleCheckResult enumerate_schedules_check(const MemGraph& m, const MemoryMap& map, std::int64_t limit,
                                              std::uint64_t seed = 0);

struct VerificationReport {
    CheckResult acyclic, data_preservation, race_freedom, capacity;
    bool has_schedules = false;
    ScheduleCheckResult schedules;
    bool all_passed() const;
    std::string to_json() const;
};

VerificationReport verify_all(const TaskGraph& g, const MemGraph& m, const MemoryMap& map,
                              std::int64_t schedule_limit = 0);

}  // namespace tn
