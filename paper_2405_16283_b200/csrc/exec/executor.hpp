// CUDA executor for memgraphs: the real-hardware slot of the reference
// simulate() (proj/include/memplan/simulator.hpp:67-68). See executor.cpp.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../core/dispatch.hpp"

namespace tn {

struct ExecConfig {
    std::vector<int> devices;        // memgraph device -> CUDA ordinal (default d % gpus)
    int streams_per_device = 5;      // simulator.hpp:23
    int compute_tokens = 1;          // concurrent kernels per device (reference: 1)
    bool device_deps = false;        // "dependencies": "host" (a vertex is dispatched once the host saw
                                     // its predecessors complete; kernels may chain, see lookahead) |
                                     // "device" (dispatched once its predecessors are dispatched,
                                     // waiting on the GPU for them: dispatch_loop_device_deps)
    bool kernel_slots = true;        // "kernel_slots": true (default) -> kernels also hold one of the
                                     // generic stream slots (the reference resource model); false (with
                                     // lookahead: kernels run on the compute stream) -> slots are for
                                     // copies only, so a FIFO backlog of ready input copies cannot hold
                                     // off a ready kernel. 7B value step, paired A/B: 53.59 vs 53.82 ms
                                     // (noise level) while the extra concurrent D2D copies stretch every
                                     // GEMM vertex by ~8 %, so the reference model stays the default
    int lookahead = 1;               // kernels queued behind the running one on the GPU
                                     // (0 = reference dispatch: only after host-observed completion)
    bool materialize_inputs = true;  // Input = a copy into its placement at dispatch
    bool inputs_on_device = false;   // "input_residency": "device" -> D2D from an HBM
                                     // staging copy (stream only); "host" -> H2D from the
                                     // pinned pool (stream + host_in channel)
    int timeout_s = 600;             // completion watchdog
    TieBreak tie_break = TieBreak::PlanOrder;  // "tie_break": the event-driven ready-list order when a
                                          // run names none: "plan-order" (default; ready copies / kernels
                                          // in the memgraph's total order, so the H2D engine loads the
                                          // tensor the plan needs next instead of the one that became
                                          // ready first: config-4 step 0.586 -> 0.537 s, config 5
                                          // 0.563 -> 0.553 s) | "fifo" (the reference simulator's
                                          // default) | "seeded-random" | "lowest-id"
    bool elide_input_offloads = true;  // an evicted *input* is never modified: skip its D2H and
                                       // reload from the input's own host (or HBM staging) copy
    bool poll = true;                // "completion": "poll" (spin on cudaEventQuery) | "callback"
                                     // (cudaLaunchHostFunc -> queue -> condition variable)
    bool alias_device_inputs = true;  // "device_inputs": "alias" -> with device residency the
                                      // Input vertex is zero-cost (reference: simulator.cpp:66-67):
                                      // generation-0 readers use the HBM staging copy in place;
                                      // "copy" -> a D2D copy into the placement at dispatch
    bool all_timestamps = false;      // "timestamps": "traced" -> runs without a trace use timing-free
                                      // completion events and programmatic dependent launch (a
                                      // timing event between two kernels costs ~3 us and blocks PDL);
                                      // "all" -> every run records per-vertex timestamps
    bool pdl = true;                  // "pdl": programmatic dependent launch between consecutive
                                      // compute-stream kernels of untimed runs (each kernel's
                                      // prologue overlaps its predecessor's tail; paired A/B on the
                                      // 7B step: 49.72 vs 50.00 ms, tools/ab_exec_cfg.py)
    bool graph = false;               // "execution": "events" (the host event loop) | "graph" (untimed
                                      // runs replay the memgraph as one CUDA graph whose node
                                      // dependencies are the memgraph edges; traced runs stay on the
                                      // host loop)
    bool zero_copy_gathers = true;    // "zero_copy_gathers": host-resident inputs read only as the
                                      // table of embedding kernels stay in mapped pinned memory and
                                      // the kernel gathers its rows over PCIe (the Input vertex
                                      // copies nothing; a reload of such an input still copies)
};
ExecConfig parse_exec_config(const std::string& text);

struct RunStats {
    std::int64_t vertices = 0, kernel_launches = 0;
    std::int64_t h2d_bytes = 0, d2h_bytes = 0, p2p_bytes = 0, d2d_bytes = 0, d2h_elided_bytes = 0;
    double flops = 0, makespan_s = 0, wall_s = 0;
    double kernel_time_s = 0, kernel_busy_s = 0, copy_time_s = 0, exposed_transfer_s = 0;
    double exposed_transfer_gpu_s = 0;  // same, per physical GPU (devices sharing a GPU cover each other)
    std::int64_t zero_copy_bytes = 0;     // bytes kernels read over PCIe from mapped host inputs
    // host event loop: time spent dispatching (ready-list ordering, resource
    // accounting, launch/copy API calls) vs waiting for the next completion
    double host_dispatch_s = 0, host_wait_s = 0;
    double host_launch_s = 0;  // part of host_dispatch_s inside the CUDA launch / copy / event calls
    // device-timed span of the run: max over GPUs of (t0 event recorded after the
    // pre-run synchronize -> end event recorded after the last vertex), no
    // per-vertex timestamps needed
    double device_makespan_s = 0;
    std::int64_t graph_nodes = 0;  // > 0: the run was a CUDA graph launch of this many vertex nodes
    std::string to_json() const;
};

class Executor {
  public:
    Executor(const std::string& memgraph_json, const std::string& taskgraph_json, const ExecConfig& cfg);
    ~Executor();
    void set_input(VertexId id, const void* src, std::size_t bytes, bool from_device);
    ExecutionTrace run(const SchedulerPolicy& pol, std::uint64_t seed, bool want_trace = true);
    ExecutionTrace last_trace();
    void get_output(VertexId id, void* host, std::size_t bytes);
    void* placement_ptr(VertexId id);
    const RunStats& stats() const;
    // The reference's compare_policies (simulator.cpp:391-417) on hardware:
    // `trials` paired runs of this memgraph, event-driven vs make_fixed_order,
    // alternating which policy goes first; makespan = device_makespan_s; trial t
    // uses seed mix64(seed + t); same summary schema and bootstrap (2000
    // resamples) as the simulator's.
    ComparisonSummary compare_policies(std::int64_t trials, std::uint64_t seed);
    TieBreak default_tie_break() const;
    struct Impl;

  private:
    std::unique_ptr<Impl> impl_;
};

}  // namespace tn
