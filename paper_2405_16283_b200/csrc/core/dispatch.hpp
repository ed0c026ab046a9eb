// The event-driven dispatch contract, shared by the virtual-time simulator
// (drop-in for the reference simulate()) and the CUDA executor.
//
// Reference: proj/src/simulator.cpp:108-344 (Dispatcher) and
// proj/include/memplan/simulator.hpp:22-61 (profile, policy, trace types).
// A vertex dispatches once every memgraph predecessor finished and its
// resources are free (simulator.cpp:167-177):
//   kernel   -> a free stream on its device + the device's compute token
//   transfer -> a free stream on the destination device
//   offload  -> a free stream + the device's host_out (D2H) channel
//   reload   -> a free stream + the device's host_in (H2D) channel
//   input    -> nothing (reference) | a stream when the executor materialises
//               inputs, plus host_in when they come from pinned host memory
//               (SURVEY hard part 3)
// The ready list is re-ordered before every dispatch by the tie-break
// (simulator.cpp:200-219) and the sweep restarts after each dispatch.
#pragma once

#include <algorithm>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "types.hpp"

namespace tn {

enum class NoiseKind : std::uint8_t { None, Uniform, Lognormal };
struct NoiseSpec {
    NoiseKind kind = NoiseKind::None;
    double param = 0.0;
};

struct DeviceProfile {
    std::int32_t streams_per_device = 5;
    double kernel_multiplier = 1.0;
    double d2d_bandwidth = 1.0;
    double host_link_bandwidth = 1.0;
    double link_latency = 0.0;
    NoiseSpec noise;
    std::uint64_t seed = 0;
};

enum class SchedulerKind : std::uint8_t { EventDriven, FixedOrder };
// PlanOrder (an extension, not in the reference simulator): ready vertices are
// taken in the memgraph's total order, so a copy engine loads the tensor the
// plan needs first rather than the one that became ready first.
enum class TieBreak : std::uint8_t { Fifo, SeededRandom, LowestId, PlanOrder };

struct SchedulerPolicy {
    SchedulerKind kind = SchedulerKind::EventDriven;
    TieBreak tie_break = TieBreak::Fifo;
};

TieBreak tie_break_from_string(const std::string& s);
SchedulerKind scheduler_kind_from_string(const std::string& s);

struct TraceRow {
    VertexId vertex = 0;
    double start = 0.0;
    double end = 0.0;
    DeviceId device = 0;
    std::int32_t stream = -1;
};

struct ExecutionTrace {
    std::vector<TraceRow> rows;  // dispatch order
    double makespan = 0.0;
    std::vector<double> busy_time;
    std::vector<double> idle_time;
    std::vector<std::int64_t> peak_live;
    std::int64_t host_bytes_transferred = 0;
    std::string to_json() const;
    std::string to_csv() const;
};

std::uint64_t mix64(std::uint64_t x);

// Fills makespan / busy / idle / peak_live / host bytes from rows
// (simulator.cpp:274-343).
void finalize_trace(const MemGraph& m, const MemoryMap& map, ExecutionTrace& t);

// Resource model (simulator.cpp:115-197) with two executor knobs:
// `compute_tokens` (reference: 1) and `inputs_use_host_in`.
class Resources {
  public:
    // kernels_take_stream = false (executor: kernels run in order on a per-device
    // compute stream) keeps the generic stream slots for copies, so a backlog of
    // ready input copies cannot hold off a ready kernel.
    Resources(int devices, int streams_per_device, int compute_tokens, bool inputs_take_stream,
              bool inputs_use_host_in = true, bool kernels_take_stream = true)
        : streams_(streams_per_device), inputs_(inputs_take_stream), inputs_host_(inputs_use_host_in),
          kernels_(kernels_take_stream), devs_(devices) {
        for (auto& d : devs_) {
            d.free_mask.assign((streams_per_device + 63) / 64, 0);
            for (int i = 0; i < streams_per_device; ++i) d.free_mask[i / 64] |= 1ULL << (i % 64);
            d.nfree = streams_per_device;
            d.compute = compute_tokens;
        }
    }
    bool holds_nothing(const MemVertex& v) const { return v.op == MemOpKind::Input && !inputs_; }
    bool slotless(const MemVertex& v) const { return v.op == MemOpKind::Kernel && !kernels_; }
    bool free(const MemVertex& v) const {
        const Dev& d = devs_[v.device];
        switch (v.op) {
            case MemOpKind::Input: return !inputs_ || (d.nfree > 0 && (!inputs_host_ || d.host_in));
            case MemOpKind::Kernel: return (!kernels_ || d.nfree > 0) && d.compute > 0;
            case MemOpKind::Transfer: return d.nfree > 0;
            case MemOpKind::Offload: return d.nfree > 0 && d.host_out;
            case MemOpKind::Reload: return d.nfree > 0 && d.host_in;
        }
        return false;
    }
    std::int32_t acquire(const MemVertex& v) {
        if (holds_nothing(v)) return -1;
        Dev& d = devs_[v.device];
        if (slotless(v)) {
            d.compute--;
            return -1;
        }
        std::int32_t s = -1;
        for (size_t w = 0; w < d.free_mask.size(); ++w)
            if (d.free_mask[w]) {
                int b = __builtin_ctzll(d.free_mask[w]);
                d.free_mask[w] &= ~(1ULL << b);
                s = static_cast<std::int32_t>(w * 64 + b);
                break;
            }
        d.nfree--;
        if (v.op == MemOpKind::Kernel) d.compute--;
        if (v.op == MemOpKind::Offload) d.host_out = false;
        if (v.op == MemOpKind::Reload || (v.op == MemOpKind::Input && inputs_host_)) d.host_in = false;
        return s;
    }
    void release(const MemVertex& v, std::int32_t s) {
        if (holds_nothing(v)) return;
        Dev& d = devs_[v.device];
        if (slotless(v)) {
            d.compute++;
            return;
        }
        d.free_mask[s / 64] |= 1ULL << (s % 64);
        d.nfree++;
        if (v.op == MemOpKind::Kernel) d.compute++;
        if (v.op == MemOpKind::Offload) d.host_out = true;
        if (v.op == MemOpKind::Reload || (v.op == MemOpKind::Input && inputs_host_)) d.host_in = true;
    }

  private:
    struct Dev {
        std::vector<std::uint64_t> free_mask;
        int nfree = 0;
        int compute = 1;
        bool host_out = true, host_in = true;
    };
    int streams_;
    bool inputs_, inputs_host_, kernels_;
    std::vector<Dev> devs_;
};

// Ready list + tie-break (simulator.cpp:135-219). FIFO entries arrive with
// non-decreasing ready time and increasing arrival, so the list is always
// FIFO-sorted and the reference's per-dispatch sort is the identity;
// LowestId keeps the list id-sorted on insert; SeededRandom re-sorts by id and
// reshuffles with the run's mt19937_64 before every sweep, exactly like the
// reference, because the shuffle consumes the shared generator.
class ReadyList {
  public:
    struct Entry {
        double ready_time;
        std::int64_t arrival;
        VertexId vertex;
        std::int32_t vidx;
    };
    ReadyList(TieBreak tb, std::uint64_t seed) : tb_(tb), rng_(mix64(seed)) {}
    // PlanOrder: rank[vidx] = position of vertex vidx in the memgraph's total order.
    void set_rank(std::vector<std::int32_t> rank) { rank_ = std::move(rank); }
    void push(VertexId id, std::int32_t vidx, double t) {
        Entry e{t, arrivals_++, id, vidx};
        if (tb_ == TieBreak::PlanOrder) {
            const std::vector<std::int32_t>& r = rank_;
            auto key = [&r](const Entry& x) { return r.empty() ? x.vidx : r[static_cast<size_t>(x.vidx)]; };
            auto it = std::upper_bound(v_.begin(), v_.end(), e,
                                       [&key](const Entry& a, const Entry& b) { return key(a) < key(b); });
            v_.insert(it, e);
        } else if (tb_ == TieBreak::LowestId) {
            auto it = std::upper_bound(v_.begin(), v_.end(), e,
                                       [](const Entry& a, const Entry& b) { return a.vertex < b.vertex; });
            v_.insert(it, e);
        } else {
            v_.push_back(e);
        }
    }
    // Reorders for a sweep; returns true when a restart from 0 is required
    // after every dispatch (SeededRandom).
    bool sort() {
        if (tb_ != TieBreak::SeededRandom) return false;
        std::sort(v_.begin(), v_.end(), [](const Entry& a, const Entry& b) { return a.vertex < b.vertex; });
        std::shuffle(v_.begin(), v_.end(), rng_);
        return true;
    }
    std::vector<Entry>& entries() { return v_; }
    void erase(size_t i) { v_.erase(v_.begin() + static_cast<std::ptrdiff_t>(i)); }
    bool empty() const { return v_.empty(); }
    size_t size() const { return v_.size(); }

  private:
    TieBreak tb_;
    std::mt19937_64 rng_;
    std::vector<Entry> v_;
    std::vector<std::int32_t> rank_;
    std::int64_t arrivals_ = 0;
};

// rank[vidx] = position in m.total_order (empty when the memgraph has none).
inline std::vector<std::int32_t> plan_rank(const MemGraph& m) {
    std::vector<std::int32_t> r;
    if (m.total_order.size() != m.vertices.size()) return r;
    r.assign(m.vertices.size(), 0);
    for (size_t i = 0; i < m.total_order.size(); ++i) r[static_cast<size_t>(m.idx(m.total_order[i]))] = static_cast<std::int32_t>(i);
    return r;
}

// Successor CSR and in-degrees of a memgraph, by vertex index.
struct GraphIndex {
    std::vector<std::int32_t> indeg, succ_start, succ;
    explicit GraphIndex(const MemGraph& m);
};

// The dispatch loop. Backend provides:
//   void launch(std::int32_t vidx, std::int32_t stream, double now);
//   bool idle() const;                       // nothing in flight
//   std::int32_t wait_next(double& now);      // blocks for one completion
template <class Backend>
void dispatch_loop(const MemGraph& m, Resources& res, ReadyList& ready, Backend& be) {
    GraphIndex gi(m);
    const size_t V = m.vertices.size();
    std::vector<std::int32_t> pending = gi.indeg;
    std::vector<std::int32_t> held(V, -1);
    for (size_t i = 0; i < V; ++i)
        if (pending[i] == 0) ready.push(m.vertices[i].id, static_cast<std::int32_t>(i), 0.0);
    double now = 0.0;
    size_t done = 0;
    while (done < V) {
        // Dispatch greedily until nothing fits.
        size_t i = 0;
        bool restart = ready.sort();
        while (i < ready.size()) {
            auto& e = ready.entries()[i];
            const MemVertex& v = m.vertices[e.vidx];
            if (!res.free(v)) {
                ++i;
                continue;
            }
            std::int32_t vidx = e.vidx;
            std::int32_t s = res.acquire(v);
            held[vidx] = s;
            ready.erase(i);
            be.launch(vidx, s, now);
            if (restart) {
                ready.sort();
                i = 0;
            }
        }
        if (be.idle()) {
            std::string msg = "simulation deadlock: " + std::to_string(ready.size()) +
                              " vertices ready but blocked, none in flight; frontier:";
            for (const auto& r : ready.entries()) msg += " " + std::to_string(r.vertex);
            throw DeadlockError(msg);
        }
        std::int32_t vidx = be.wait_next(now);
        res.release(m.vertices[vidx], held[vidx]);
        done++;
        for (std::int32_t a = gi.succ_start[vidx]; a < gi.succ_start[vidx + 1]; ++a) {
            std::int32_t w = gi.succ[a];
            if (--pending[w] == 0) ready.push(m.vertices[w].id, w, now);
        }
    }
}

// Lookahead variant for hardware backends (executor config "lookahead": 1).
// A kernel whose not-yet-completed predecessors are all kernels of its own
// device that are already running or queued on that device's compute token
// is dispatched immediately behind them (device-side event wait) instead of
// after a host round trip; at most `lookahead` kernels wait per device. The
// compute token still serialises kernels per device (reference semantics,
// simulator.cpp:171,184), every other op dispatches exactly as in
// dispatch_loop, and the GPU enforces every edge, so outputs are unchanged.
// Backend additionally provides:
//   void launch_after(std::int32_t vidx, std::int32_t stream, std::int32_t after, double now);
template <class Backend>
void dispatch_loop_lookahead(const MemGraph& m, Resources& res, ReadyList& ready, Backend& be, int lookahead) {
    GraphIndex gi(m);
    const size_t V = m.vertices.size();
    const int D = m.device_count;
    std::vector<std::int32_t> npc = gi.indeg, npd = gi.indeg;  // not completed / not dispatched preds
    std::vector<std::int32_t> held(V, -1);
    std::vector<char> queued_in_ready(V, 0), dispatched(V, 0);
    std::vector<std::int32_t> holder(D, -1);          // kernel owning the compute token
    std::vector<std::vector<std::int32_t>> waiting(D);  // kernels dispatched behind the holder
    // preds by vertex (for the early-dispatch check)
    std::vector<std::int32_t> pstart(V + 1, 0), preds;
    for (size_t u = 0; u < V; ++u)
        for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a) pstart[gi.succ[a] + 1]++;
    for (size_t i = 0; i < V; ++i) pstart[i + 1] += pstart[i];
    preds.resize(gi.succ.size());
    {
        std::vector<std::int32_t> fill(pstart.begin(), pstart.end() - 1);
        for (size_t u = 0; u < V; ++u)
            for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a)
                preds[fill[gi.succ[a]]++] = static_cast<std::int32_t>(u);
    }
    std::vector<char> done(V, 0);
    auto tail_of = [&](int d) { return waiting[d].empty() ? holder[d] : waiting[d].back(); };
    auto can_chain = [&](std::int32_t v) {
        const MemVertex& x = m.vertices[v];
        if (x.op != MemOpKind::Kernel || holder[x.device] < 0) return false;
        if (static_cast<int>(waiting[x.device].size()) >= lookahead) return false;
        for (std::int32_t k = pstart[v]; k < pstart[v + 1]; ++k) {
            const std::int32_t p = preds[k];
            if (done[p]) continue;
            const MemVertex& y = m.vertices[p];
            if (!dispatched[p] || y.op != MemOpKind::Kernel || y.device != x.device) return false;
        }
        return true;
    };
    auto push = [&](std::int32_t w, double t) {
        if (queued_in_ready[w]) return;
        queued_in_ready[w] = 1;
        ready.push(m.vertices[w].id, w, t);
    };
    for (size_t i = 0; i < V; ++i)
        if (npc[i] == 0) push(static_cast<std::int32_t>(i), 0.0);
    double now = 0.0;
    size_t ndone = 0;
    while (ndone < V) {
        size_t i = 0;
        bool restart = ready.sort();
        while (i < ready.size()) {
            auto& e = ready.entries()[i];
            const std::int32_t v = e.vidx;
            const MemVertex& x = m.vertices[v];
            bool go = false, chain = false;
            if (npc[v] == 0) {
                if (x.op == MemOpKind::Kernel) go = holder[x.device] < 0 && res.free(x);
                else go = res.free(x);
            } else {
                chain = can_chain(v) && res.free(x);
                go = chain;
            }
            if (!go) {
                ++i;
                continue;
            }
            const std::int32_t s = res.acquire(x);
            held[v] = s;
            dispatched[v] = 1;
            ready.erase(i);
            if (x.op == MemOpKind::Kernel && !chain) {
                holder[x.device] = v;
                be.launch(v, s, now);
            } else if (chain) {
                const std::int32_t after = tail_of(x.device);
                waiting[x.device].push_back(v);
                be.launch_after(v, s, after, now);
            } else {
                be.launch(v, s, now);
            }
            for (std::int32_t a = gi.succ_start[v]; a < gi.succ_start[v + 1]; ++a) {
                const std::int32_t w = gi.succ[a];
                if (--npd[w] == 0 && npc[w] > 0 && m.vertices[w].op == MemOpKind::Kernel) push(w, now);
            }
            if (restart) {
                ready.sort();
                i = 0;
            }
        }
        if (be.idle()) {
            std::string msg = "simulation deadlock: " + std::to_string(ready.size()) +
                              " vertices ready but blocked, none in flight; frontier:";
            for (const auto& r : ready.entries()) msg += " " + std::to_string(r.vertex);
            throw DeadlockError(msg);
        }
        const std::int32_t u = be.wait_next(now);
        const MemVertex& y = m.vertices[u];
        res.release(y, held[u]);
        done[u] = 1;
        ndone++;
        if (y.op == MemOpKind::Kernel) {
            auto& wq = waiting[y.device];
            if (holder[y.device] == u) {
                // hand the token down the chain (skipping kernels already seen done)
                holder[y.device] = -1;
                while (!wq.empty()) {
                    const std::int32_t nx = wq.front();
                    wq.erase(wq.begin());
                    if (!done[nx]) {
                        holder[y.device] = nx;
                        break;
                    }
                }
            } else {
                auto it = std::find(wq.begin(), wq.end(), u);
                if (it != wq.end()) wq.erase(it);
            }
        }
        for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a) {
            const std::int32_t w = gi.succ[a];
            if (--npc[w] == 0 && !dispatched[w]) push(w, now);
        }
    }
}

// --- virtual-time simulator (drop-in for the reference) ------------------------
double sample_duration(const MemVertex& v, const DeviceProfile& p, std::uint64_t draw_seed);
MemGraph make_fixed_order(const MemGraph& m);
MemGraph make_fixed_order(const MemGraph& m, const std::vector<VertexId>& order);
ExecutionTrace simulate(const MemGraph& m, const MemoryMap& map, const DeviceProfile& p,
                        const SchedulerPolicy& policy, std::uint64_t seed);

struct PolicyStats {
    double mean = 0.0, ci_low = 0.0, ci_high = 0.0;
    std::vector<double> makespans;
};
struct ComparisonSummary {
    PolicyStats event_driven, fixed_order;
    double speedup_mean = 0.0, speedup_ci_low = 0.0, speedup_ci_high = 0.0;
    std::int64_t trials = 0;
    std::string to_json() const;
};
PolicyStats bootstrap_stats(const std::vector<double>& samples, std::uint64_t seed);
ComparisonSummary compare_policies(const MemGraph& m, const MemoryMap& map, const DeviceProfile& p,
                                   std::int64_t trials, std::uint64_t seed);
// The summary of paired makespans (event-driven ev[t], fixed-order fx[t]):
// speedup (f - e) / f per pair, each series bootstrapped as in compare_policies.
ComparisonSummary summarize_pairs(const std::vector<double>& ev, const std::vector<double>& fx, std::uint64_t seed);

std::string serialize_profile(const DeviceProfile& p);
DeviceProfile parse_profile(const std::string& text);


// Device-dependency variant (executor config "dependencies": "device"): a
// vertex becomes a candidate as soon as every predecessor has been
// DISPATCHED; the backend makes it wait on the device for the predecessors
// that have not completed (CUDA events; kernel -> kernel on one device is
// ordered by the compute stream), so the host round trip between a copy and
// the kernel that consumes it (or the offload of a freshly produced tile)
// leaves the critical path. Resources are the reference's (stream slots,
// host_in / host_out per device, held from dispatch to completion); kernels
// of a device run in order on its compute stream, at most 1 + `lookahead`
// in flight. Each sweep first dispatches candidates whose predecessors have
// all completed (tie-break order), then the early ones. Outputs are
// unchanged: every memgraph edge is enforced on the GPU.
// Backend additionally provides:
//   void launch_waits(std::int32_t vidx, std::int32_t stream, const std::int32_t* waits, int n, double now);
template <class Backend>
void dispatch_loop_device_deps(const MemGraph& m, Resources& res, ReadyList& ready, Backend& be, int lookahead) {
    GraphIndex gi(m);
    const size_t V = m.vertices.size();
    const int D = m.device_count;
    std::vector<std::int32_t> npc = gi.indeg, npd = gi.indeg;
    std::vector<std::int32_t> held(V, -1), kq(D, 0);
    std::vector<char> done(V, 0);
    std::vector<std::int32_t> pstart(V + 1, 0), preds;
    for (size_t u = 0; u < V; ++u)
        for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a) pstart[gi.succ[a] + 1]++;
    for (size_t i = 0; i < V; ++i) pstart[i + 1] += pstart[i];
    preds.resize(gi.succ.size());
    {
        std::vector<std::int32_t> fill(pstart.begin(), pstart.end() - 1);
        for (size_t u = 0; u < V; ++u)
            for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a)
                preds[fill[gi.succ[a]]++] = static_cast<std::int32_t>(u);
    }
    const int kmax = 1 + std::max(0, lookahead);
    std::vector<std::int32_t> waits;
    for (size_t i = 0; i < V; ++i)
        if (npd[i] == 0) ready.push(m.vertices[i].id, static_cast<std::int32_t>(i), 0.0);
    double now = 0.0;
    size_t ndone = 0;
    while (ndone < V) {
        bool restart = ready.sort();
        for (int pass = 0; pass < 2; ++pass) {
            size_t i = 0;
            while (i < ready.size()) {
                const std::int32_t v = ready.entries()[i].vidx;
                const MemVertex& x = m.vertices[v];
                const bool early = npc[v] > 0;
                // Inputs (aliased ones complete at dispatch on a shared marker
                // stream) are never dispatched early.
                bool go = early == (pass == 1) && !(early && x.op == MemOpKind::Input) && res.free(x);
                if (go && x.op == MemOpKind::Kernel) go = kq[x.device] < kmax;
                if (!go) {
                    ++i;
                    continue;
                }
                held[v] = res.acquire(x);
                ready.erase(i);
                if (x.op == MemOpKind::Kernel) kq[x.device]++;
                waits.clear();
                for (std::int32_t k = pstart[v]; k < pstart[v + 1]; ++k) {
                    const std::int32_t p = preds[k];
                    if (done[p]) continue;
                    const MemVertex& y = m.vertices[p];
                    if (x.op == MemOpKind::Kernel && y.op == MemOpKind::Kernel && y.device == x.device) continue;
                    waits.push_back(p);
                }
                be.launch_waits(v, held[v], waits.data(), static_cast<int>(waits.size()), now);
                for (std::int32_t a = gi.succ_start[v]; a < gi.succ_start[v + 1]; ++a) {
                    const std::int32_t w = gi.succ[a];
                    if (--npd[w] == 0) ready.push(m.vertices[w].id, w, now);
                }
                if (restart) {
                    ready.sort();
                    i = 0;
                }
            }
        }
        if (be.idle()) {
            std::string msg = "simulation deadlock: " + std::to_string(ready.size()) +
                              " vertices ready but blocked, none in flight; frontier:";
            for (const auto& r : ready.entries()) msg += " " + std::to_string(r.vertex);
            throw DeadlockError(msg);
        }
        const std::int32_t u = be.wait_next(now);
        const MemVertex& y = m.vertices[u];
        res.release(y, held[u]);
        if (y.op == MemOpKind::Kernel) kq[y.device]--;
        done[u] = 1;
        ndone++;
        for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a) --npc[gi.succ[a]];
    }
}

}  // namespace tn
