// Host-side cost of the dispatch contract on a large memgraph: parse, the
// virtual-time dispatch loop (SimBackend), finalize and trace serialisation,
// timed separately. Build: see tools/native/Makefile.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "core/dispatch.hpp"
#include "core/planner.hpp"

using namespace tn;
using clk = std::chrono::steady_clock;

static double since(clk::time_point t) { return std::chrono::duration<double>(clk::now() - t).count(); }

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    auto t0 = clk::now();
    auto [m, map] = parse_memgraph(ss.str());
    const double parse = since(t0);
    for (const char* tb : {"fifo", "lowest-id", "seeded-random"}) {
        SchedulerPolicy pol{SchedulerKind::EventDriven, tie_break_from_string(tb)};
        t0 = clk::now();
        auto t = simulate(m, map, DeviceProfile{}, pol, 0);
        const double sim = since(t0);
        t0 = clk::now();
        auto js = t.to_json();
        const double ser = since(t0);
        std::printf("%s: V=%zu parse %.3f s, simulate %.3f s (%.2f us/vertex), to_json %.3f s\n", tb, m.vertices.size(),
                    parse, sim, sim * 1e6 / m.vertices.size(), ser);
    }
    return 0;
}
