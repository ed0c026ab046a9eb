/*
 * turnip.h — C ABI of the B200-native memgraph planner + executor
 * (library: paper_2405_16283_b200/lib/libturnip_b200.so).
 *
 * Drop-in boundary for the reference memplan pybind module
 * (proj/python/bindings.cpp) and its C++ API (proj/include/memplan/{compiler,simulator}.hpp).
 * Graphs cross the boundary as the reference's own JSON formats
 * ("format-stable", bindings.cpp:36-37). Every entry point:
 *   - returns 0 on success, 1 check failed / deadlock, 2 usage / parse / IO /
 *     planning error (the reference's MemplanError family), 3 CUDA error;
 *   - on failure stores a malloc'd message in *err (if err != NULL);
 *   - never aborts the process.
 * Every char** output is malloc'd; release it with tn_free().
 */
#ifndef TURNIP_H
#define TURNIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tn_exec tn_exec;

/* Library version string (static storage). */
const char* tn_version(void);
void tn_free(void* p);

/* --- taskgraph utilities -------------------------------------------------- */
/* replaces bindings.cpp:39-45 validate_taskgraph(graph_json) -> list[str];
 * out: JSON array of violation messages. */
int tn_validate_taskgraph(const char* graph_json, char** violations_json, char** err);

/* replaces bindings.cpp:47-51 topological_order(graph_json, policy, seed);
 * policy: "as-listed" | "depth-first" | "min-memory-greedy"; out: JSON array. */
int tn_topological_order(const char* graph_json, const char* policy, uint64_t seed, char** order_json,
                         char** err);

/* bindings.cpp:53-59 gen_matmul / gen_layered / gen_random_dag (toy
 * generators, SURVEY §2 out of scope) are not part of this library; the tests
 * read the reference generators' outputs from tests/golden/taskgraphs.json. */

/* replaces bindings.cpp:118-124 taskgraph_to_dot / memgraph_to_dot. */
int tn_taskgraph_to_dot(const char* graph_json, char** dot, char** err);
int tn_memgraph_to_dot(const char* memgraph_json, char** dot, char** err);

/* --- memgraph construction (bit-exact with the reference) ----------------- */
/* replaces bindings.cpp:61-85 build_memgraph(graph_json, capacities, mode,
 * order, order_policy, victim_policy, seed, alloc_horizon, keep_superfluous)
 * and compiler.hpp:63-65 build_memgraph(g, order, capacities, mode, opts).
 * order == NULL / norder == 0 derives the order with `order_policy`.
 * host_capacity < 0 means unbounded (BuildOptions::host_capacity unset).
 * Outputs: memgraph JSON (serialize_memgraph format) and stats JSON
 * {offloads, reloads, memory_edges, required_memory_edges, peak_usage}. */
int tn_build_memgraph(const char* graph_json, const int64_t* capacities, size_t ncapacities,
                      const char* mode, const int64_t* order, size_t norder, const char* order_policy,
                      const char* victim_policy, uint64_t seed, const char* alloc_horizon,
                      int keep_superfluous, int64_t host_capacity, char** memgraph_json,
                      char** stats_json, char** err);

/* --- virtual-time dispatch (drop-in for the reference simulator) ---------- */
/* replaces bindings.cpp:95-107 simulate(memgraph_json, profile_json, policy,
 * tie_break, seed) -> trace JSON; format: "json" | "csv" (CLI --format,
 * memplan_main.cpp:240-259). */
int tn_simulate(const char* memgraph_json, const char* profile_json, const char* policy,
                const char* tie_break, uint64_t seed, const char* format, char** trace, char** err);

/* replaces bindings.cpp:109-116 compare_policies(memgraph_json, profile_json,
 * trials, seed) -> summary JSON. */
int tn_compare_policies(const char* memgraph_json, const char* profile_json, int64_t trials,
                        uint64_t seed, char** summary_json, char** err);

/* replaces bindings.cpp:87-93 verify(graph_json, memgraph_json,
 * schedule_limit) -> report JSON (verifier.cpp:474-492 format, same witnesses;
 * scalable pair/reachability algorithms so large plans can be certified). */
int tn_verify(const char* graph_json, const char* memgraph_json, int64_t schedule_limit, char** report_json,
              char** err);

/* replaces verifier.hpp:47-48 check_capacity(m, map, order): replays an
 * arbitrary order (e.g. an executor trace's completion order) against the
 * placement lifetimes. out: {"passed": bool[, "witness": str]}. */
int tn_check_capacity(const char* memgraph_json, const int64_t* order, size_t norder, char** result_json,
                      char** err);

/* replaces simulator.hpp:72-73 make_fixed_order(m): memgraph JSON in/out. */
int tn_make_fixed_order(const char* memgraph_json, char** memgraph_out, char** err);

/* --- CUDA executor: real execution of a memgraph on B200s ----------------- */
/* The slot of simulator.hpp:67-68 simulate(m, map, profile, policy, seed).
 * taskgraph_json: the taskgraph the memgraph was built from, whose vertices
 *   carry an extra "op" payload (ignored by the reference parser,
 *   taskgraph.cpp:375-389) naming the kernel and its argument producers.
 * config_json (all keys optional, defaults shown):
 *   "devices": [0, 1, ...]          memgraph device d -> CUDA ordinal (default d % #GPUs)
 *   "streams_per_device": 5         simulator.hpp:23
 *   "compute_tokens": 1             kernels running at once per device (reference: 1)
 *   "lookahead": 1                  kernels queued behind the running kernel (0 = exact contract)
 *   "kernel_slots": true            kernels hold a generic stream slot (reference model); false with
 *                                   lookahead: slots are for copies only (kernels use the compute stream)
 *   "dependencies": "host"          "host": a vertex dispatches once the host saw its predecessors
 *                                   complete; "device": once they are dispatched, the GPU waiting
 *                                   (CUDA events) for the unfinished ones, same resource tokens
 *   "completion": "poll"            "poll" (cudaEventQuery) | "callback" (cudaLaunchHostFunc)
 *   "input_residency": "host"       "host" (pinned pool, H2D at dispatch) | "device" (HBM staging)
 *   "device_inputs": "alias"        with device residency: "alias" (read in place) | "copy" (D2D)
 *   "zero_copy_gathers": true       host inputs read only by embedding gathers stay in mapped memory
 *   "timestamps": "traced"          "traced": runs without a trace record timing-free completion
 *                                   events only (a timing event between kernels costs ~3 us);
 *                                   "all": every run is timestamped (last_trace() after any run)
 *   "pdl": true                     programmatic dependent launch between kernels of untimed runs
 *   "execution": "events"           "events": the host event loop; "graph": untimed runs replay the
 *                                   memgraph as one CUDA graph (a node per vertex, dependencies =
 *                                   memgraph edges: the GPU dispatches each vertex when its
 *                                   predecessors finished); traced runs use the host loop
 *   "tie_break": "plan-order"       ready-list order when tn_exec_run names none: "plan-order" (the
 *                                   memgraph's total order: each copy engine takes the tensor the plan
 *                                   needs soonest) | "fifo" (reference default) | "lowest-id" |
 *                                   "seeded-random"
 *   "elide_input_offloads": true    an evicted input is reloaded from its own copy, never offloaded
 *   "materialize_inputs": true, "timeout_s": 600 */
int tn_exec_create(const char* memgraph_json, const char* taskgraph_json, const char* config_json,
                   tn_exec** out, char** err);

/* Host bytes of Input vertex `vertex_id` (its taskgraph output tensor). The
 * executor copies them into its pinned host pool; the H2D materialisation
 * happens when the Input vertex dispatches. */
int tn_exec_set_input(tn_exec* h, int64_t vertex_id, const void* host, size_t bytes, char** err);

/* Same as set_input but the bytes already live on device `cuda_ordinal` at
 * `device_ptr` (staged once with a D2H into the pinned pool). */
int tn_exec_set_input_device(tn_exec* h, int64_t vertex_id, const void* device_ptr, size_t bytes,
                             char** err);

/* One full execution. policy: "event-driven" | "fixed-order"; tie_break:
 * "fifo" | "seeded-random" | "lowest-id" | "plan-order" (memgraph total order;
 * an extension), NULL or "" = the executor config's "tie_break" (default
 * "plan-order"). Blocks until every vertex finished.
 * trace_json uses the reference ExecutionTrace schema (simulator.cpp:421-436)
 * with times in seconds measured by CUDA events; may be NULL. */
int tn_exec_run(tn_exec* h, const char* policy, const char* tie_break, uint64_t seed, char** trace_json,
                char** err);

/* Trace of the most recent tn_exec_run (built from that run's CUDA events),
 * for runs made with trace_json == NULL (no host work inside the timed loop). */
int tn_exec_last_trace(tn_exec* h, char** trace_json, char** err);

/* Copies graph output `vertex_id` (never freed or evicted) to host. */
int tn_exec_get_output(tn_exec* h, int64_t vertex_id, void* host, size_t bytes, char** err);

/* Device pointer of the region currently holding `vertex_id`'s placement. */
int tn_exec_placement_ptr(tn_exec* h, int64_t vertex_id, void** device_ptr, char** err);

/* JSON: per-run counters (kernel launches, H2D/D2H/P2P bytes, exposed
 * transfer time, per-op-type device time). */
int tn_exec_stats(tn_exec* h, char** stats_json, char** err);

/* replaces bindings.cpp:109-116 compare_policies(memgraph_json, profile_json,
 * trials, seed) with measured makespans: `trials` paired runs of this
 * executor's memgraph, event-driven vs make_fixed_order (simulator.cpp:86-104),
 * alternating which goes first, each makespan device-timed (CUDA events around
 * the whole run); summary JSON in the schema of tn_compare_policies with the
 * same 2000-resample bootstrap (simulator.cpp:365-417). */
int tn_exec_compare_policies(tn_exec* h, int64_t trials, uint64_t seed, char** summary_json, char** err);

void tn_exec_destroy(tn_exec* h);

#ifdef __cplusplus
}
#endif

#endif /* TURNIP_H */
