// The CUDA executor: runs a memgraph for real on B200s, behind the same
// dispatch contract as the reference simulator (proj/src/simulator.cpp:108-344).
//
// Layout: one cudaMalloc arena of exactly capacities[d] bytes per memgraph
// device; every placement is arena[d] + offset (no allocation while running,
// PAPER.md:175). Offload/reload slots and input tensors live in a pinned host
// pool (cudaHostAlloc). Per device: `streams_per_device` non-blocking streams
// (reference default 5, simulator.hpp:23); copy engines are picked by the
// driver from the copy direction.
//
// Event loop (dispatch_loop in core/dispatch.hpp): a vertex dispatches when
// all memgraph predecessors have completed and its resources are free. Each
// launch is followed by cudaLaunchHostFunc; the callback (driver thread, no
// CUDA calls) pushes the vertex into a completion queue that wakes the loop.
// Per-vertex start/end cudaEvents give the trace times.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <unordered_set>

#include <nlohmann/json.hpp>

#include "../core/dispatch.hpp"
#include "../core/planner.hpp"
#include "../kernels/kernels.hpp"
#include "executor.hpp"
#include "ops.hpp"

namespace tn {

using json = nlohmann::json;

#define TN_CUDA(call)                                                                                     \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess)                                                                            \
            throw CudaError(std::string(#call) + " failed: " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")");                                              \
    } while (0)

namespace {

struct HostBuf {
    void* p = nullptr;
    std::size_t bytes = 0;
};

void* pinned_alloc(std::size_t bytes) {
    void* p = nullptr;
    TN_CUDA(cudaHostAlloc(&p, std::max<std::size_t>(bytes, 1), cudaHostAllocPortable));
    return p;
}

}  // namespace

struct Executor::Impl {
    // --- inputs ----------------------------------------------------------------
    MemGraph m;
    MemoryMap map;
    TaskGraph tg;
    std::unordered_map<VertexId, OpDesc> ops;
    ExecConfig cfg;

    // --- device state ----------------------------------------------------------
    int D = 1;
    std::vector<int> ordinal;       // logical device -> CUDA ordinal
    std::vector<int> num_sms;
    std::vector<char*> arena;       // per logical device
    std::vector<std::vector<cudaStream_t>> streams;
    std::vector<cudaStream_t> marker;  // per logical device: timestamps of instant vertices
    std::vector<cudaStream_t> compute;  // per logical device: every kernel when compute_tokens == 1, so a
                                        // lookahead chain is plain stream order (no cross-stream event wait)
    std::vector<std::vector<k::GemmWorkspace>> gws;  // per device x stream: stream-K GEMM scratch
    std::vector<cudaEvent_t> t0;    // per logical device
    std::vector<cudaEvent_t> tend;  // per logical device (owner of its GPU): end of the run
    std::vector<cudaEvent_t> ev_start, ev_end;  // per memgraph vertex index (timing events)
    std::vector<cudaEvent_t> ev_done;           // timing-free completion events (untimed runs)
    bool timed = true;                          // this run records ev_start / ev_end
    cudaEvent_t done_event(std::int32_t v) const { return timed ? ev_end[v] : ev_done[v]; }

    // --- host pool ---------------------------------------------------------------
    std::unordered_map<VertexId, HostBuf> inputs;  // taskgraph input id -> pinned bytes
    std::unordered_map<VertexId, HostBuf> staged;  // input id -> HBM staging copy (device residency)
    std::unordered_map<VertexId, HostBuf> slots;   // evicted root id -> pinned slot
    std::unordered_map<VertexId, char*> zero_copy;  // input id -> device view of its mapped pinned buffer
    std::unordered_map<VertexId, char*> alias;     // Input mem id -> its staging copy (aliased inputs)
    bool aliased_inputs() const { return cfg.inputs_on_device && cfg.alias_device_inputs; }

    // --- per-vertex launch programs ------------------------------------------------
    struct Instr {
        MemOpKind op = MemOpKind::Kernel;
        int dev = 0;
        int src_dev = 0;
        char* dst = nullptr;
        const char* src = nullptr;
        void* host = nullptr;  // offload/reload slot, input buffer
        std::size_t bytes = 0;
        VertexId input_id = -1;   // Input vertices, and offload/reload of an evicted input root
        bool elided = false;      // offload of an unmodified input: no copy
        bool instant = false;     // aliased Input: completes at dispatch, no stream, no copy
        bool timeless = false;    // instant with no in-edges: no device timestamps (trace time 0)
        // instant (non-timeless) predecessors: their marker event is waited on
        // device, so the trace's start >= each predecessor's end on every edge
        std::vector<std::int32_t> instant_preds;
        const OpDesc* op_desc = nullptr;
        std::vector<const char*> argp;  // resolved argument pointers
        std::unique_ptr<k::GemmPlan> gemm;
        std::unique_ptr<k::AttnPlan> attn;
        std::unique_ptr<k::AttnBwdPlan> attn_bwd;
        void* scratch = nullptr;  // per-vertex device scratch (xent_loss row losses), outside the arena
    };
    std::vector<Instr> prog;

    // --- completion queue ------------------------------------------------------------
    struct CbCtx {
        Impl* self;
        std::int32_t vidx;
    };
    std::vector<CbCtx> cb;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::int32_t> completed;
    std::atomic<int> callback_errors{0};

    // --- per run ---------------------------------------------------------------------
    std::vector<std::int32_t> dispatched;  // vidx in dispatch order
    std::vector<std::int32_t> stream_of;
    RunStats last;
    int cur_dev = -1;

    void set_device(int logical) {
        int o = ordinal[logical];
        if (o != cur_dev) {
            TN_CUDA(cudaSetDevice(o));
            cur_dev = o;
        }
    }

    char* ptr_of(VertexId mem_id) {
        if (!alias.empty()) {
            auto a = alias.find(mem_id);
            if (a != alias.end()) return a->second;
        }
        auto it = map.placements.find(mem_id);
        if (it == map.placements.end())
            throw Error("memgraph vertex " + std::to_string(mem_id) + " has no placement");
        const Placement& p = it->second;
        if (p.device < 0 || p.device >= D) throw Error("placement of " + std::to_string(mem_id) + " names unknown device");
        return arena[p.device] + p.offset;
    }
    std::int64_t size_of(VertexId mem_id) const { return map.placements.at(mem_id).size; }

    static void CUDART_CB on_done(void* data) {
        auto* c = static_cast<CbCtx*>(data);
        {
            std::lock_guard<std::mutex> g(c->self->mu);
            c->self->completed.push_back(c->vidx);
        }
        c->self->cv.notify_one();
    }

    void build();
    void prepare_kernel(Instr& in, const MemVertex& v, const std::vector<std::pair<VertexId, VertexId>>& data_in);
    void launch(std::int32_t vidx, std::int32_t stream, std::int32_t after = -1, const std::int32_t* waits = nullptr,
                int nwaits = 0);
    void issue(std::int32_t vidx, cudaStream_t s, std::int32_t stream);

    // --- graph mode ("execution": "graph") ------------------------------------------
    // The memgraph as ONE CUDA graph: a node per vertex (its copy / kernel
    // launches captured in isolation on the device's capture stream, added as
    // a child-graph node) whose dependencies are exactly the vertex's memgraph
    // in-edges. The GPU then resolves the dependencies itself: every vertex
    // starts when its predecessors have finished (the event-driven contract,
    // without a host round trip or a host API call per vertex). Built on the
    // first untimed run of each policy, replayed afterwards.
    struct GraphCache {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t x = nullptr;
        RunStats counters;  // per-run launch / byte counters (static for a graph)
        std::int64_t nodes = 0;
    };
    GraphCache graphs[2];           // [0] the memgraph, [1] its make_fixed_order form
    std::vector<cudaStream_t> cap;  // per logical device: capture stream
    bool capturing = false;
    std::string graph_error;        // why graph mode fell back to the host loop (empty: it did not)
    void drop_graphs();
    void build_graph(const MemGraph& g, GraphCache& gc);
    bool run_graph(const SchedulerPolicy& pol);
    // The CUDA stream a vertex runs on, as a dense lane id (device-major):
    // work on one lane completes in launch order, so completion polling only
    // ever needs to query the oldest in-flight vertex of each lane.
    int lanes() const { return D * (cfg.streams_per_device + 1); }
    int lane_of(std::int32_t vidx, std::int32_t stream) const {
        const Instr& in = prog[vidx];
        const bool on_compute = in.op == MemOpKind::Kernel && cfg.compute_tokens == 1;
        return in.dev * (cfg.streams_per_device + 1) + (on_compute ? cfg.streams_per_device : stream < 0 ? 0 : stream);
    }
    void run(const SchedulerPolicy& pol, std::uint64_t seed, ExecutionTrace* trace);
    ExecutionTrace build_trace();
    std::unique_ptr<MemGraph> last_graph;  // fixed-order graph of the last run
    ~Impl();
};

// ------------------------------------------------------------------ build ---
void Executor::Impl::build() {
    if (map.mode != MemoryMode::Byte) throw Error("the CUDA executor needs a byte-mode memgraph");
    D = m.device_count;
    if (static_cast<int>(map.capacities.size()) != D) throw Error("capacities must list one entry per device");
    int ngpu = 0;
    TN_CUDA(cudaGetDeviceCount(&ngpu));
    if (ngpu < 1) throw CudaError("no CUDA device visible");
    ordinal.resize(D);
    for (int d = 0; d < D; ++d) {
        ordinal[d] = d < static_cast<int>(cfg.devices.size()) ? cfg.devices[d] : d % ngpu;
        if (ordinal[d] < 0 || ordinal[d] >= ngpu) throw Error("device map names CUDA ordinal out of range");
    }
    num_sms.resize(D);
    arena.assign(D, nullptr);
    streams.resize(D);
    marker.assign(D, nullptr);
    compute.assign(D, nullptr);
    cap.assign(D, nullptr);
    t0.resize(D);
    tend.resize(D);
    for (int d = 0; d < D; ++d) {
        set_device(d);
        TN_CUDA(cudaDeviceGetAttribute(&num_sms[d], cudaDevAttrMultiProcessorCount, ordinal[d]));
        TN_CUDA(cudaMalloc(reinterpret_cast<void**>(&arena[d]), std::max<std::int64_t>(map.capacities[d], 256)));
        streams[d].resize(cfg.streams_per_device);
        for (auto& s : streams[d]) TN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        TN_CUDA(cudaStreamCreateWithFlags(&marker[d], cudaStreamNonBlocking));
        TN_CUDA(cudaStreamCreateWithFlags(&compute[d], cudaStreamNonBlocking));
        TN_CUDA(cudaStreamCreateWithFlags(&cap[d], cudaStreamNonBlocking));
        // One time origin per physical GPU: memgraph devices that share a GPU
        // share t0, so cross-device edges compare on one clock.
        int first = d;
        for (int e = 0; e < d; ++e)
            if (ordinal[e] == ordinal[d]) {
                first = e;
                break;
            }
        if (first == d) {
            TN_CUDA(cudaEventCreate(&t0[d]));
            TN_CUDA(cudaEventCreate(&tend[d]));
        } else {
            t0[d] = t0[first];
            tend[d] = tend[first];
        }
    }
    // Peer access for every pair of distinct GPUs a transfer connects.
    for (const auto& v : m.vertices) {
        if (v.op != MemOpKind::Transfer) continue;
        if (v.src_device < 0 || v.src_device >= D) throw Error("transfer with unknown src_device");
        int a = ordinal[v.device], b = ordinal[v.src_device];
        if (a == b) continue;
        int can = 0;
        TN_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
        if (can) {
            TN_CUDA(cudaSetDevice(a));
            cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TN_CUDA(e);
            cudaGetLastError();
            cur_dev = a;
        }
    }

    // Data in-edges per vertex, edge order.
    std::unordered_map<VertexId, std::vector<std::pair<VertexId, VertexId>>> data_in;  // to -> (from, root)
    std::unordered_map<VertexId, bool> has_in_edge;
    for (const auto& e : m.edges) has_in_edge[e.to] = true;
    for (const auto& e : m.edges) {
        if (e.kind != EdgeKind::Data) continue;
        const MemVertex& f = m.at(e.from);
        data_in[e.to].push_back({e.from, f.origin.ref});
    }
    // Placement bounds.
    for (const auto& [id, p] : map.placements) {
        if (p.device < 0 || p.device >= D || p.offset < 0 || p.size < 0 || p.offset + p.size > map.capacities[p.device])
            throw Error("placement of " + std::to_string(id) + " exceeds its device arena");
    }

    // Aliased device inputs: one HBM staging buffer per input, sized to its
    // placement (tail zeroed), allocated up front so every reader's pointer
    // (and TMA descriptor) is fixed at build time; tn_exec_set_input fills it.
    if (aliased_inputs()) {
        for (const auto& v : m.vertices) {
            if (v.op != MemOpKind::Input) continue;
            HostBuf& b = staged[v.origin.ref];
            set_device(v.device);
            b.bytes = static_cast<std::size_t>(std::max<std::int64_t>(size_of(v.id), 1));
            TN_CUDA(cudaMalloc(&b.p, b.bytes));
            TN_CUDA(cudaMemset(b.p, 0, b.bytes));
            alias[v.id] = static_cast<char*>(b.p);
        }
    }

    // Zero-copy gather tables (host residency): an input whose only readers
    // are embedding kernels (as their table) keeps its bytes in mapped pinned
    // memory sized to its placement; its Input vertices complete at dispatch
    // and readers resolve to the device view, so only the gathered rows cross
    // PCIe (seq * dim * 2 bytes instead of the whole vocab table).
    if (!cfg.inputs_on_device && cfg.zero_copy_gathers) {
        std::unordered_map<VertexId, int> table_uses, other_uses;
        for (const auto& [kid, op] : ops)
            for (size_t k = 0; k < op.args.size(); ++k)
                (op.type == OpType::Embedding && k == 1 ? table_uses : other_uses)[op.args[k]]++;
        for (const auto& v : m.vertices) {
            if (v.op != MemOpKind::Input) continue;
            const VertexId r = v.origin.ref;
            if (!table_uses.count(r) || other_uses.count(r)) continue;
            auto zc = zero_copy.find(r);
            if (zc == zero_copy.end()) {
                HostBuf& b = inputs[r];
                b.bytes = static_cast<std::size_t>(std::max<std::int64_t>(size_of(v.id), 1));
                TN_CUDA(cudaHostAlloc(&b.p, b.bytes, cudaHostAllocPortable | cudaHostAllocMapped));
                std::memset(b.p, 0, b.bytes);
                void* dp = nullptr;
                TN_CUDA(cudaHostGetDevicePointer(&dp, b.p, 0));
                zc = zero_copy.emplace(r, static_cast<char*>(dp)).first;
            }
            alias[v.id] = zc->second;
        }
    }

    const size_t V = m.vertices.size();
    prog.resize(V);
    cb.resize(V);
    ev_start.resize(V);
    ev_end.resize(V);
    ev_done.resize(V);
    for (size_t i = 0; i < V; ++i) {
        const MemVertex& v = m.vertices[i];
        Instr& in = prog[i];
        cb[i] = {this, static_cast<std::int32_t>(i)};
        in.op = v.op;
        in.dev = v.device;
        if (v.device < 0 || v.device >= D) throw Error("vertex " + std::to_string(v.id) + " on unknown device");
        set_device(v.device);
        TN_CUDA(cudaEventCreate(&ev_start[i]));
        TN_CUDA(cudaEventCreate(&ev_end[i]));
        TN_CUDA(cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming));
        const auto& din = data_in[v.id];
        switch (v.op) {
            case MemOpKind::Input: {
                in.dst = ptr_of(v.id);
                in.bytes = static_cast<std::size_t>(size_of(v.id));
                in.input_id = v.origin.ref;
                in.instant = aliased_inputs() || zero_copy.count(v.origin.ref) > 0;
                in.timeless = in.instant && !has_in_edge[v.id];
                break;
            }
            case MemOpKind::Offload: {
                if (din.size() != 1) throw Error("offload " + std::to_string(v.id) + " needs exactly one data source");
                in.src = ptr_of(din[0].first);
                in.bytes = static_cast<std::size_t>(v.size);
                HostBuf& s = slots[v.origin.ref];
                s.bytes = std::max(s.bytes, in.bytes);
                break;
            }
            case MemOpKind::Reload: {
                in.dst = ptr_of(v.id);
                in.bytes = static_cast<std::size_t>(std::min<std::int64_t>(v.size, size_of(v.id)));
                HostBuf& s = slots[v.origin.ref];
                s.bytes = std::max(s.bytes, in.bytes);
                break;
            }
            case MemOpKind::Transfer: {
                if (din.size() != 1) throw Error("transfer " + std::to_string(v.id) + " needs exactly one data source");
                in.src = ptr_of(din[0].first);
                in.src_dev = map.placements.at(din[0].first).device;
                in.dst = ptr_of(v.id);
                in.bytes = static_cast<std::size_t>(std::min(size_of(v.id), size_of(din[0].first)));
                break;
            }
            case MemOpKind::Kernel: prepare_kernel(in, v, din); break;
        }
    }
    {
        std::unordered_map<VertexId, std::int32_t> vidx;
        for (size_t i = 0; i < V; ++i) vidx[m.vertices[i].id] = static_cast<std::int32_t>(i);
        for (const auto& e : m.edges) {
            const std::int32_t f = vidx.at(e.from), t = vidx.at(e.to);
            if (prog[f].instant && !prog[f].timeless && !prog[t].instant) prog[t].instant_preds.push_back(f);
        }
    }
    // Pinned offload slots (one per evicted root, reused across generations:
    // generation g+1's offload data-depends on generation g's reload,
    // compiler.cpp:353-361).
    // Evicted inputs: their bytes are the input tensor itself, so the offload
    // copies nothing and the reload reads the input's host / staging copy.
    if (cfg.elide_input_offloads && cfg.materialize_inputs) {
        for (size_t i = 0; i < V; ++i) {
            const MemVertex& v = m.vertices[i];
            if (v.op != MemOpKind::Offload && v.op != MemOpKind::Reload) continue;
            const TaskVertex* root = tg.find(v.origin.ref);
            if (!root || root->kind != VertexKind::Input) continue;
            prog[i].input_id = v.origin.ref;
            prog[i].elided = v.op == MemOpKind::Offload;
        }
        for (size_t i = 0; i < V; ++i)
            if (prog[i].input_id >= 0 && m.vertices[i].op != MemOpKind::Input) slots.erase(m.vertices[i].origin.ref);
    }
    for (auto& [root, s] : slots) s.p = pinned_alloc(s.bytes);
    // Stream-K GEMM scratch, one per stream of each device (sized to the
    // largest plan on that device).
    gws.assign(D, std::vector<k::GemmWorkspace>(cfg.streams_per_device));
    for (int d = 0; d < D; ++d) {
        std::size_t need = 0;
        for (size_t i = 0; i < V; ++i)
            if (prog[i].gemm && prog[i].dev == d) need = std::max(need, prog[i].gemm->ws_bytes);
        if (!need) continue;
        set_device(d);
        for (auto& w : gws[d]) {
            TN_CUDA(cudaMalloc(&w.p, need));
            TN_CUDA(cudaMemset(w.p, 0, need));
            w.bytes = need;
            w.counter_count = 4096;  // split-K tile counters (zero between launches: the reducer resets them)
            TN_CUDA(cudaMalloc(&w.counters, w.counter_count * sizeof(unsigned)));
            TN_CUDA(cudaMemset(w.counters, 0, w.counter_count * sizeof(unsigned)));
        }
    }
    for (size_t i = 0; i < V; ++i) {
        const MemVertex& v = m.vertices[i];
        if ((v.op == MemOpKind::Offload || v.op == MemOpKind::Reload) && prog[i].input_id < 0)
            prog[i].host = slots.at(v.origin.ref).p;
    }
}

void Executor::Impl::prepare_kernel(Instr& in, const MemVertex& v,
                                    const std::vector<std::pair<VertexId, VertexId>>& din) {
    auto it = ops.find(v.origin.ref);
    if (it == ops.end()) throw Error("kernel vertex " + std::to_string(v.id) + " has no op payload");
    const OpDesc& op = it->second;
    in.op_desc = &op;
    in.dst = ptr_of(v.id);
    const std::int64_t out_bytes = size_of(v.id);
    std::vector<std::int64_t> arg_bytes;
    for (VertexId a : op.args) {
        const char* p = nullptr;
        std::int64_t sz = 0;
        for (const auto& [src, root] : din)
            if (root == a) {
                p = ptr_of(src);
                sz = size_of(src);
                break;
            }
        if (!p)
            throw Error("kernel " + std::to_string(v.id) + ": argument " + std::to_string(a) +
                        " is not a data predecessor in the memgraph");
        in.argp.push_back(p);
        arg_bytes.push_back(sz);
    }
    auto need_args = [&](size_t lo, size_t hi) {
        if (op.args.size() < lo || op.args.size() > hi)
            throw Error("kernel " + std::to_string(v.id) + " (" + to_string(op.type) + "): wrong argument count");
    };
    auto fits = [&](std::int64_t bytes, std::int64_t cap, const char* what) {
        if (bytes < 0 || bytes > cap)
            throw Error("kernel " + std::to_string(v.id) + " (" + to_string(op.type) + "): " + what +
                        " extent " + std::to_string(bytes) + " exceeds its region of " + std::to_string(cap) + " bytes");
    };
    auto es = [](int dt) { return static_cast<std::int64_t>(k::dtype_size(dt)); };
    switch (op.type) {
        case OpType::Gemm: {
            need_args(2, op.norm_out ? 4 : 3);
            k::GemmArgs g;
            g.M = static_cast<int>(op.M);
            g.N = static_cast<int>(op.N);
            g.K = static_cast<int>(op.K);
            g.batch = static_cast<int>(op.batch);
            g.lda = op.lda ? op.lda : op.K;
            g.ldb = op.ldb ? op.ldb : op.K;
            const std::int64_t n_out = op.epilogue == 1 ? op.N / 2 : op.N;
            g.ldc = op.ldc ? op.ldc : n_out;
            g.epi = op.epilogue;
            g.tile = op.tile;
            g.ksplit = op.ksplit == 1 ? -1 : op.ksplit;  // op: 0 automatic, 1 off, n > 1 forced
            g.split = op.split;
            if (op.split && op.in_dtype != k::F32) throw Error("gemm precision 3xtf32 needs f32 inputs");
            if (op.epilogue == 1 && (op.N % 256 != 0 || op.args.size() != 2))
                throw Error("gemm swiglu epilogue needs N % 256 == 0 and no residual");
            if (op.epilogue == 2 && (op.N != 3 * op.heads * 128 || op.args.size() != 3 || op.batch != 1))
                throw Error("gemm qkv_rope epilogue needs N = 3*heads*128, args [x, w, rope_table], batch 1");
            g.sa = op.sa;
            g.sb = op.sb;
            g.sc = op.sc;
            g.alpha = static_cast<float>(op.alpha);
            g.in_dtype = op.in_dtype;
            g.out_dtype = op.out_dtype;
            g.causal = op.causal;
            if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.batch <= 0) throw Error("gemm with empty shape");
            const std::int64_t ei = es(op.in_dtype), eo = es(op.out_dtype);
            auto extent = [](std::int64_t off, int batch, std::int64_t bs, std::int64_t rows, std::int64_t ld,
                             std::int64_t cols) { return off + (batch - 1) * bs + (rows - 1) * ld + cols; };
            g.a_mn = op.a_mn;
            g.b_mn = op.b_mn;
            if (op.a_mn && !op.lda) g.lda = op.M;  // MN-major: [K, M] / [K, N] row pitch
            if (op.b_mn && !op.ldb) g.ldb = op.N;
            if ((op.a_mn || op.b_mn) && (op.in_dtype != k::BF16 || op.epilogue != 0 || op.norm_out))
                throw Error("gemm MN-major operands need bf16 inputs and the plain epilogue");
            fits((op.a_mn ? extent(op.a_off, g.batch, g.sa, g.K, g.lda, g.M) : extent(op.a_off, g.batch, g.sa, g.M, g.lda, g.K)) * ei,
                 arg_bytes[0], "A");
            fits((op.b_mn ? extent(op.b_off, g.batch, g.sb, g.K, g.ldb, g.N) : extent(op.b_off, g.batch, g.sb, g.N, g.ldb, g.K)) * ei,
                 arg_bytes[1], "B");
            if (op.epilogue == 2) fits(3 * op.heads * 128 * op.M * 2, out_bytes, "C (packed q|k|vT)");
            else fits(extent(op.c_off, g.batch, g.sc, g.M, g.ldc, n_out) * eo, out_bytes, "C");
            g.A = in.argp[0] + op.a_off * ei;
            g.B = in.argp[1] + op.b_off * ei;
            g.C = in.dst + op.c_off * eo;
            if (op.epilogue == 2) {
                fits(op.M * 64 * 2 * 4, arg_bytes[2], "rope_table");
                g.rope = in.argp[2];
                g.heads = static_cast<int>(op.heads);
            } else if (op.args.size() >= 3) {
                fits(extent(op.r_off, g.batch, g.sc, g.M, g.ldc, g.N) * eo, arg_bytes[2], "R");
                g.R = in.argp[2] + op.r_off * eo;
            }
            if (op.norm_out) {  // [x | h | P] output, gamma = last argument
                if (op.args.size() != 4 || op.epilogue != 0 || op.batch != 1 || op.out_dtype != k::BF16 ||
                    g.ldc != op.N || op.N % 32 != 0)
                    throw Error("gemm norm_out needs args [A, B, R, gamma], bf16 out, batch 1, dense C, N % 32 == 0");
                fits(op.N * 2, arg_bytes[3], "gamma");
                fits(op.c_off * eo + 2 * op.M * op.N * 2 + (op.N / 32) * op.M * 4, out_bytes, "C (x | h | P)");
                g.no_g = in.argp[3];
                g.no_P = reinterpret_cast<float*>(in.dst + op.c_off * eo + 2 * op.M * op.N * 2);
            }
            if (op.rs_arg >= 0) {
                if (op.rs_arg >= static_cast<int>(op.args.size()) || op.rs_dim <= 0 || op.rs_dim % 32 != 0 || op.rs_ld <= 0)
                    throw Error("gemm row scale needs rs_arg < #args, rs_dim % 32 == 0, rs_ld > 0");
                if (op.rs_ld < op.rs_dim / 32) throw Error("gemm row scale: rs_ld < rs_dim / 32");
                fits(op.rs_off + ((op.rs_row0 + op.M - 1) * op.rs_ld + op.rs_dim / 32) * 4, arg_bytes[op.rs_arg],
                     "row-scale sums P");
                g.rs_P = reinterpret_cast<const float*>(in.argp[op.rs_arg] + op.rs_off);
                g.rs_ld = static_cast<int>(op.rs_ld);
                g.rs_row0 = static_cast<int>(op.rs_row0);
                g.rs_chunks = static_cast<int>(op.rs_dim / 32);
                g.rs_inv_dim = 1.0f / static_cast<float>(op.rs_dim);
                g.rs_eps = static_cast<float>(op.eps);
            }
            in.gemm = std::make_unique<k::GemmPlan>();
            if (k::gemm_prepare(g, in.gemm.get(), num_sms[v.device]) == cudaErrorNotSupported)
                throw Error("gemm norm_out needs the CTA-pair tcgen05 path with 16-byte aligned operands");
            if (op.epilogue == 2 && in.gemm->path == 1)
                throw Error("gemm qkv_rope epilogue needs a tcgen05-eligible shape (M >= 128, aligned operands)");
            break;
        }
        case OpType::RmsNorm:
            need_args(2, 2);
            fits(op.rows * op.cols * 2, arg_bytes[0], "x");
            fits(op.cols * 2, arg_bytes[1], "w");
            fits(op.rows * op.cols * 2, out_bytes, "y");
            break;
        case OpType::Softmax:
            need_args(1, 1);
            fits(op.batch * op.rows * op.cols * 4, arg_bytes[0], "S");
            fits(op.batch * op.rows * op.cols * 2, out_bytes, "P");
            break;
        case OpType::Rope:
            need_args(2, 2);
            if (op.hd % 2) throw Error("rope needs an even head dim");
            fits(((op.seq - 1) * op.ld + op.col_off + op.heads * op.hd) * 2, arg_bytes[0], "src");
            fits(op.seq * (op.hd / 2) * 2 * 4, arg_bytes[1], "table");
            fits(op.heads * op.seq * op.hd * 2, out_bytes, "out");
            break;
        case OpType::Transpose:
            need_args(1, 1);
            fits(op.batch * op.rows * op.cols * es(op.out_dtype), arg_bytes[0], "x");
            fits(op.batch * op.rows * op.cols * es(op.out_dtype), out_bytes, "out");
            break;
        case OpType::RmsNormBwd:
            need_args(3, 3);
            fits(op.rows * op.cols * 2, arg_bytes[0], "x");
            fits(op.cols * 2, arg_bytes[1], "w");
            fits(op.rows * op.cols * 2, arg_bytes[2], "dy");
            fits(op.rows * op.cols * 2, out_bytes, "dx");
            break;
        case OpType::SwigluBwd:
            need_args(2, 2);
            fits(op.rows * op.cols * 4, arg_bytes[0], "gu");
            fits(op.rows * op.cols * 2, arg_bytes[1], "da");
            fits(op.rows * op.cols * 4, out_bytes, "dgu");
            break;
        case OpType::SoftmaxBwd:
            need_args(2, 2);
            fits(op.batch * op.rows * op.cols * 2, arg_bytes[0], "P");
            fits(op.batch * op.rows * op.cols * es(op.in_dtype), arg_bytes[1], "dP");
            fits(op.batch * op.rows * op.cols * 2, out_bytes, "dS");
            break;
        case OpType::XentGrad:
        case OpType::XentLoss:
            need_args(2, 2);
            fits(op.rows * op.vocab * es(op.in_dtype), arg_bytes[0], "logits");
            fits(op.rows * 4, arg_bytes[1], "targets");
            if (op.type == OpType::XentGrad) {
                fits(op.rows * op.vocab * es(op.out_dtype), out_bytes, "grad");
            } else {
                fits(4, out_bytes, "loss");
                set_device(v.device);
                TN_CUDA(cudaMalloc(&in.scratch, static_cast<size_t>(op.rows) * 4 + 256));
            }
            break;
        case OpType::TransposeHeads:
            need_args(1, 1);
            fits(((op.seq - 1) * op.ld + op.col_off + op.heads * op.hd) * 2, arg_bytes[0], "src");
            fits(op.heads * op.seq * op.hd * 2, out_bytes, "out");
            break;
        case OpType::SiluMul:
            need_args(1, 1);
            fits(op.rows * op.cols * 2 * 2, arg_bytes[0], "gu");
            fits(op.rows * op.cols * 2, out_bytes, "out");
            break;
        case OpType::Sum:
            need_args(1, 16);
            if (!op.offs.empty() && op.offs.size() != op.args.size()) throw Error("sum: offs must list one offset per arg");
            for (size_t i = 0; i < op.args.size(); ++i) {
                const std::int64_t off = op.offs.empty() ? 0 : op.offs[i];
                fits((off + op.count) * es(op.in_dtype), arg_bytes[i], "part");
                in.argp[i] += off * es(op.in_dtype);
            }
            fits(op.count * es(op.out_dtype), out_bytes, "out");
            break;
        case OpType::Concat:
            need_args(1, 64);
            for (size_t i = 0; i < op.args.size(); ++i) fits(op.count * es(op.out_dtype), arg_bytes[i], "part");
            fits(static_cast<std::int64_t>(op.args.size()) * op.count * es(op.out_dtype), out_bytes, "out");
            break;
        case OpType::Embedding:
            need_args(op.norm_out ? 3 : 2, op.norm_out ? 3 : 2);
            fits(op.seq * 4, arg_bytes[0], "tokens");
            fits(op.vocab * op.dim * 2, arg_bytes[1], "table");
            fits(op.seq * op.dim * 2 * (op.norm_out ? 2 : 1) + (op.norm_out ? op.seq * (op.dim / 32) * 4 : 0), out_bytes,
                 "out");
            if (op.norm_out) {
                if (op.dim % 32 != 0) throw Error("embedding norm_out needs dim % 32 == 0");
                fits(op.dim * 2, arg_bytes[2], "gamma");
            }
            break;
        case OpType::Cast:
            need_args(1, 1);
            fits(op.count * es(op.in_dtype), arg_bytes[0], "x");
            fits(op.count * es(op.out_dtype), out_bytes, "out");
            break;
        case OpType::RowStats:
            need_args(1, 1);
            fits(op.rows * op.cols * 2, arg_bytes[0], "S");
            fits(op.rows * 8, out_bytes, "stats");
            break;
        case OpType::StatsCombine:
            need_args(1, 64);
            for (size_t i = 0; i < op.args.size(); ++i) fits(op.rows * 8, arg_bytes[i], "stats");
            fits(op.rows * 8, out_bytes, "stats");
            break;
        case OpType::SoftmaxApply:
            need_args(2, 2);
            fits(op.rows * op.cols * 2, arg_bytes[0], "S");
            fits(op.rows * 8, arg_bytes[1], "stats");
            fits(op.rows * op.cols * 2, out_bytes, "P");
            break;
        case OpType::Attention: {
            need_args(1, 3);
            if (op.args.size() == 2)
                throw Error("kernel " + std::to_string(v.id) +
                            " (attention): takes one packed tensor (q_off/k_off/v_off) or three arguments [q, k, vT]");
            if (op.hd <= 0 || op.hd > 256 || op.seq <= 0 || op.heads <= 0) throw Error("attention: bad shape");
            const std::int64_t ldo = op.ldo ? op.ldo : op.heads * op.hd;
            const std::int64_t sec = op.heads * op.seq * op.hd;
            const size_t iq = 0, ik = op.args.size() == 3 ? 1 : 0, iv = op.args.size() == 3 ? 2 : 0;
            fits((op.q_off + sec) * 2, arg_bytes[iq], "q");
            fits((op.k_off + sec) * 2, arg_bytes[ik], "k");
            fits((op.v_off + sec) * 2, arg_bytes[iv], "vt");
            fits(((op.seq - 1) * ldo + op.heads * op.hd) * 2, out_bytes, "out");
            if (op.lse) fits(op.seq * ldo * 2 + op.heads * op.seq * 4, out_bytes, "out (o + lse)");
            k::AttnArgs aa;
            aa.q = in.argp[iq] + op.q_off * 2;
            aa.k = in.argp[ik] + op.k_off * 2;
            aa.vt = in.argp[iv] + op.v_off * 2;
            aa.out = in.dst;
            aa.heads = static_cast<int>(op.heads);
            aa.seq = static_cast<int>(op.seq);
            aa.hd = static_cast<int>(op.hd);
            aa.ldo = ldo;
            aa.scale = static_cast<float>(op.scale);
            aa.causal = op.causal;
            if (op.lse) aa.lse = reinterpret_cast<float*>(in.dst + op.seq * ldo * 2);
            in.attn = std::make_unique<k::AttnPlan>();
            TN_CUDA(k::attention_prepare(aa, in.attn.get()));
            break;
        }
        case OpType::AttentionBwd: {
            need_args(5, 6);
            if (op.hd != 128 || op.seq <= 0 || op.seq % 128 != 0 || op.heads <= 0)
                throw Error("kernel " + std::to_string(v.id) + " (attention_bwd): needs hd 128 and seq % 128 == 0");
            const std::int64_t sec = op.heads * op.seq * op.hd, w = op.heads * op.hd;
            const std::int64_t ldo = op.ldo ? op.ldo : w, vld = op.v_ld ? op.v_ld : w, dld = op.do_ld ? op.do_ld : w;
            fits((op.q_off + sec) * 2, arg_bytes[0], "q");
            fits((op.k_off + sec) * 2, arg_bytes[1], "k");
            fits((op.v_off + (op.seq - 1) * vld + w) * 2, arg_bytes[2], "v");
            fits(op.seq * ldo * 2 + op.heads * op.seq * 4, arg_bytes[3], "o_lse");
            fits(((op.seq - 1) * dld + w) * 2, arg_bytes[4], "dO");
            fits(op.seq * 3 * w * 2 + op.heads * op.seq * 4, out_bytes, "out (dq|dk|dv + D)");
            if (op.args.size() == 6) fits(op.seq * op.hd * 4, arg_bytes[5], "rope table");
            k::AttnBwdArgs ab;
            ab.q = in.argp[0] + op.q_off * 2;
            ab.k = in.argp[1] + op.k_off * 2;
            ab.v = in.argp[2] + op.v_off * 2;
            ab.ldv = vld;
            ab.o = in.argp[3];
            ab.ldo = ldo;
            ab.lse = reinterpret_cast<const float*>(in.argp[3] + op.seq * ldo * 2);
            ab.dout = in.argp[4];
            ab.lddo = dld;
            ab.dq = in.dst;
            ab.dk = in.dst + w * 2;
            ab.dv = in.dst + 2 * w * 2;
            ab.ldg = 3 * w;
            ab.D = reinterpret_cast<float*>(in.dst + op.seq * 3 * w * 2);
            if (op.args.size() == 6) ab.rope = reinterpret_cast<const float*>(in.argp[5]);
            ab.heads = static_cast<int>(op.heads);
            ab.seq = static_cast<int>(op.seq);
            ab.hd = static_cast<int>(op.hd);
            ab.scale = static_cast<float>(op.scale);
            ab.causal = op.causal;
            in.attn_bwd = std::make_unique<k::AttnBwdPlan>();
            if (k::attention_bwd_prepare(ab, in.attn_bwd.get()) != cudaSuccess)
                throw Error("kernel " + std::to_string(v.id) + " (attention_bwd): operands not 16-byte aligned");
            break;
        }
    }
}

// ----------------------------------------------------------------- launch ---
void Executor::Impl::launch(std::int32_t vidx, std::int32_t stream, std::int32_t after, const std::int32_t* waits,
                            int nwaits) {
    Instr& in = prog[vidx];
    set_device(in.dev);
    if (in.timeless) return;  // zero-cost input with nothing to wait for: trace time 0
    const bool on_compute = in.op == MemOpKind::Kernel && cfg.compute_tokens == 1;
    cudaStream_t s = in.instant ? marker[in.dev]
                     : on_compute ? compute[in.dev]
                                  : streams[in.dev][stream < 0 ? 0 : stream];  // inputs hold no stream when not materialised
    // lookahead: run behind `after` (same stream when both are on the compute stream)
    if (after >= 0 && !(on_compute && prog[after].op == MemOpKind::Kernel && prog[after].dev == in.dev))
        TN_CUDA(cudaStreamWaitEvent(s, done_event(after), 0));
    // An instant predecessor completed at dispatch on the host, but its marker
    // timestamp is recorded on another stream: order this vertex behind it.
    for (std::int32_t p : in.instant_preds) TN_CUDA(cudaStreamWaitEvent(s, done_event(p), 0));
    // device-dependency dispatch: predecessors still running elsewhere
    for (int k = 0; k < nwaits; ++k)
        if (!prog[waits[k]].timeless) TN_CUDA(cudaStreamWaitEvent(s, done_event(waits[k]), 0));
    if (timed) TN_CUDA(cudaEventRecord(ev_start[vidx], s));
    issue(vidx, s, stream);
    TN_CUDA(cudaEventRecord(done_event(vidx), s));
    // instant vertices complete through the backend's instant queue at
    // dispatch; a host callback as well would complete them twice
    if (!cfg.poll && !in.instant) TN_CUDA(cudaLaunchHostFunc(s, &Impl::on_done, &cb[vidx]));
}

// The vertex's own work on stream `s` (no timing / completion events): the
// copy or kernel launch(es) of one memgraph vertex. Also what graph mode
// captures, one vertex at a time.
void Executor::Impl::issue(std::int32_t vidx, cudaStream_t s, std::int32_t stream) {
    Instr& in = prog[vidx];
    const bool on_compute = in.op == MemOpKind::Kernel && cfg.compute_tokens == 1;
    switch (in.op) {
        case MemOpKind::Input: {
            if (in.instant) break;  // readers use the staging copy in place
            if (cfg.inputs_on_device) {
                auto it = staged.find(in.input_id);
                if (it == staged.end() || !it->second.p)
                    throw Error("input " + std::to_string(in.input_id) + " has no data (tn_exec_set_input)");
                const std::size_t n = std::min(in.bytes, it->second.bytes);
                TN_CUDA(cudaMemcpyAsync(in.dst, it->second.p, n, cudaMemcpyDeviceToDevice, s));
                last.d2d_bytes += static_cast<std::int64_t>(n);
                break;
            }
            auto it = inputs.find(in.input_id);
            if (it == inputs.end() || !it->second.p)
                throw Error("input " + std::to_string(in.input_id) + " has no data (tn_exec_set_input)");
            TN_CUDA(cudaMemcpyAsync(in.dst, it->second.p, std::min(in.bytes, it->second.bytes), cudaMemcpyHostToDevice, s));
            last.h2d_bytes += static_cast<std::int64_t>(std::min(in.bytes, it->second.bytes));
            break;
        }
        case MemOpKind::Offload:
            if (in.elided) {
                last.d2h_elided_bytes += static_cast<std::int64_t>(in.bytes);
                break;
            }
            TN_CUDA(cudaMemcpyAsync(in.host, in.src, in.bytes, cudaMemcpyDeviceToHost, s));
            last.d2h_bytes += static_cast<std::int64_t>(in.bytes);
            break;
        case MemOpKind::Reload:
            if (in.input_id >= 0) {  // reload of an evicted input: from its own copy
                const bool dev_copy = cfg.inputs_on_device;
                auto& pool = dev_copy ? staged : inputs;
                auto it = pool.find(in.input_id);
                if (it == pool.end() || !it->second.p)
                    throw Error("input " + std::to_string(in.input_id) + " has no data (tn_exec_set_input)");
                const std::size_t n = std::min(in.bytes, it->second.bytes);
                TN_CUDA(cudaMemcpyAsync(in.dst, it->second.p, n, dev_copy ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
                (dev_copy ? last.d2d_bytes : last.h2d_bytes) += static_cast<std::int64_t>(n);
                break;
            }
            TN_CUDA(cudaMemcpyAsync(in.dst, in.host, in.bytes, cudaMemcpyHostToDevice, s));
            last.h2d_bytes += static_cast<std::int64_t>(in.bytes);
            break;
        case MemOpKind::Transfer:
            if (ordinal[in.src_dev] == ordinal[in.dev]) {
                TN_CUDA(cudaMemcpyAsync(in.dst, in.src, in.bytes, cudaMemcpyDeviceToDevice, s));
                last.d2d_bytes += static_cast<std::int64_t>(in.bytes);
            } else {
                TN_CUDA(cudaMemcpyPeerAsync(in.dst, ordinal[in.dev], in.src, ordinal[in.src_dev], in.bytes, s));
                last.p2p_bytes += static_cast<std::int64_t>(in.bytes);
            }
            break;
        case MemOpKind::Kernel: {
            const OpDesc& op = *in.op_desc;
            const auto& a = in.argp;
            struct PdlScope {  // PDL for this launch only (untimed runs, compute stream)
                explicit PdlScope(bool on) { k::set_pdl(on); }
                ~PdlScope() { k::set_pdl(false); }
            } pdl_scope(!timed && cfg.pdl && on_compute && !capturing);
            switch (op.type) {
                case OpType::Gemm:
                    TN_CUDA(k::gemm_launch(*in.gemm, s, &gws[in.dev][stream < 0 ? 0 : stream]));
                    last.flops += k::gemm_flops(in.gemm->args);
                    break;
                case OpType::RmsNorm:
                    TN_CUDA(k::rmsnorm(a[0], a[1], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols),
                                       static_cast<float>(op.eps), s));
                    break;
                case OpType::Softmax:
                    TN_CUDA(k::softmax(a[0], in.dst, static_cast<int>(op.batch), static_cast<int>(op.rows),
                                       static_cast<int>(op.cols), static_cast<float>(op.scale), op.causal, s));
                    break;
                case OpType::Rope:
                    TN_CUDA(k::rope(a[0], a[1], in.dst, static_cast<int>(op.seq), op.ld, op.col_off,
                                    static_cast<int>(op.heads), static_cast<int>(op.hd), s, op.inverse, op.tokens_out));
                    break;
                case OpType::Transpose:
                    TN_CUDA(k::transpose(a[0], in.dst, static_cast<int>(op.batch), static_cast<int>(op.rows),
                                         static_cast<int>(op.cols), k::dtype_size(op.out_dtype), s));
                    break;
                case OpType::RmsNormBwd:
                    TN_CUDA(k::rmsnorm_bwd(a[0], a[1], a[2], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols),
                                           static_cast<float>(op.eps), s));
                    break;
                case OpType::SwigluBwd:
                    TN_CUDA(k::swiglu_bwd(a[0], a[1], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols), s));
                    break;
                case OpType::SoftmaxBwd:
                    TN_CUDA(k::softmax_bwd(a[0], a[1], op.in_dtype, in.dst, static_cast<int>(op.batch),
                                           static_cast<int>(op.rows), static_cast<int>(op.cols), op.causal, s));
                    break;
                case OpType::XentGrad:
                    TN_CUDA(k::xent(a[0], op.in_dtype, a[1], in.dst, op.out_dtype, static_cast<int>(op.rows),
                                    static_cast<int>(op.vocab), static_cast<float>(op.scale), 1, nullptr, s));
                    break;
                case OpType::XentLoss:
                    TN_CUDA(k::xent(a[0], op.in_dtype, a[1], in.dst, k::F32, static_cast<int>(op.rows),
                                    static_cast<int>(op.vocab), static_cast<float>(op.scale), 0, in.scratch, s));
                    break;
                case OpType::TransposeHeads:
                    TN_CUDA(k::transpose_heads(a[0], in.dst, static_cast<int>(op.seq), op.ld, op.col_off,
                                               static_cast<int>(op.heads), static_cast<int>(op.hd), s));
                    break;
                case OpType::SiluMul:
                    TN_CUDA(k::silu_mul(a[0], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols), s));
                    break;
                case OpType::Sum: {
                    std::vector<const void*> ps(a.begin(), a.end());
                    TN_CUDA(k::sum_n(ps.data(), static_cast<int>(ps.size()), op.in_dtype, in.dst, op.out_dtype,
                                     op.count, s));
                    break;
                }
                case OpType::Embedding:
                    if (op.args.size() > 1) {
                        auto zc = zero_copy.find(op.args[1]);
                        if (zc != zero_copy.end() && a[1] == zc->second) last.zero_copy_bytes += op.seq * op.dim * 2;
                    }
                    if (op.norm_out)
                        TN_CUDA(k::embedding_norm(a[0], a[1], a[2], in.dst, static_cast<int>(op.seq),
                                                  static_cast<int>(op.dim), static_cast<int>(op.vocab), s));
                    else
                        TN_CUDA(k::embedding(a[0], a[1], in.dst, static_cast<int>(op.seq), static_cast<int>(op.dim),
                                             static_cast<int>(op.vocab), s));
                    break;
                case OpType::Cast:
                    TN_CUDA(k::cast(a[0], op.in_dtype, in.dst, op.out_dtype, op.count, s));
                    break;
                case OpType::Concat: {
                    std::vector<const void*> ps(a.begin(), a.end());
                    TN_CUDA(k::concat(ps.data(), static_cast<int>(ps.size()), op.count * k::dtype_size(op.out_dtype),
                                      in.dst, s));
                    break;
                }
                case OpType::RowStats:
                    TN_CUDA(k::rowstats(a[0], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols), op.causal, s));
                    break;
                case OpType::StatsCombine: {
                    std::vector<const void*> ps(a.begin(), a.end());
                    TN_CUDA(k::stats_combine(ps.data(), static_cast<int>(ps.size()), in.dst, static_cast<int>(op.rows), s));
                    break;
                }
                case OpType::SoftmaxApply:
                    TN_CUDA(k::softmax_apply(a[0], a[1], in.dst, static_cast<int>(op.rows), static_cast<int>(op.cols),
                                             op.causal, s));
                    break;
                case OpType::Attention:
                    TN_CUDA(k::attention_launch(*in.attn, s));
                    last.flops += k::attention_flops(in.attn->args);
                    break;
                case OpType::AttentionBwd:
                    TN_CUDA(k::attention_bwd_launch(*in.attn_bwd, s));
                    last.flops += k::attention_bwd_flops(in.attn_bwd->args);
                    last.kernel_launches++;  // attn_bwd_prep + attention_bwd_kernel
                    break;
            }
            last.kernel_launches++;
            break;
        }
    }
}

// -------------------------------------------------------------------- run ---
namespace {

class CudaBackend {
  public:
    explicit CudaBackend(Executor::Impl& x)
        : x_(x), start_(std::chrono::steady_clock::now()), lanes_(x.lanes()) {}
    void launch(std::int32_t vidx, std::int32_t stream, double) {
        const auto t_in = std::chrono::steady_clock::now();
        x_.launch(vidx, stream);
        launch_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count();
        x_.dispatched.push_back(vidx);
        x_.stream_of[vidx] = stream;
        in_flight_++;
        if (x_.prog[vidx].instant) instant_.push_back(vidx);
        else if (x_.cfg.poll) track(vidx, stream);
    }
    void launch_waits(std::int32_t vidx, std::int32_t stream, const std::int32_t* waits, int n, double) {
        const auto t_in = std::chrono::steady_clock::now();
        x_.launch(vidx, stream, -1, waits, n);
        launch_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count();
        x_.dispatched.push_back(vidx);
        x_.stream_of[vidx] = stream;
        in_flight_++;
        if (x_.prog[vidx].instant) instant_.push_back(vidx);
        else if (x_.cfg.poll) track(vidx, stream);
    }
    void launch_after(std::int32_t vidx, std::int32_t stream, std::int32_t after, double) {
        const auto t_in = std::chrono::steady_clock::now();
        x_.launch(vidx, stream, after);
        launch_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count();
        x_.dispatched.push_back(vidx);
        x_.stream_of[vidx] = stream;
        in_flight_++;
        if (x_.cfg.poll) track(vidx, stream);
    }
    bool idle() const { return in_flight_ == 0; }
    double wait_s() const { return wait_s_; }
    double launch_s() const { return launch_s_; }
    std::int32_t wait_next(double& now) {
        const auto t_in = std::chrono::steady_clock::now();
        const std::int32_t v = wait_next_(now);
        wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count();
        return v;
    }

  private:
    std::int32_t wait_next_(double& now) {
        if (!instant_.empty()) {  // aliased inputs complete at dispatch
            const std::int32_t v = instant_.front();
            instant_.pop_front();
            in_flight_--;
            now = std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count();
            return v;
        }
        if (x_.cfg.poll) return poll_next(now);
        std::unique_lock<std::mutex> lk(x_.mu);
        if (x_.completed.empty()) {
            if (!x_.cv.wait_for(lk, std::chrono::seconds(x_.cfg.timeout_s), [&] { return !x_.completed.empty(); }))
                throw CudaError("executor timed out waiting for a completion (" + std::to_string(in_flight_) +
                                " vertices in flight)");
        }
        std::int32_t v = x_.completed.front();
        x_.completed.pop_front();
        lk.unlock();
        in_flight_--;
        now = std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count();
        return v;
    }

    void track(std::int32_t vidx, std::int32_t stream) {
        const int l = x_.lane_of(vidx, stream);
        if (lanes_[l].empty()) active_.push_back(l);
        lanes_[l].push_back(vidx);
    }

    // Spins over the lanes with work in flight, querying only the OLDEST
    // vertex of each (a stream completes in order), round-robin from where
    // the last completion was found; lower latency than a host-function
    // round trip and O(#busy streams) per sweep instead of O(#in flight).
    std::int32_t poll_next(double& now) {
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(x_.cfg.timeout_s);
        for (std::uint64_t spin = 0;; ++spin) {
            const size_t n = active_.size();
            for (size_t k = 0; k < n; ++k) {
                const size_t i = (rr_ + k) % n;
                const int l = active_[i];
                const std::int32_t v = lanes_[l].front();
                const int dev = x_.prog[v].dev;
                if (x_.ordinal[dev] != x_.cur_dev) x_.set_device(dev);
                cudaError_t e = cudaEventQuery(x_.done_event(v));
                if (e == cudaErrorNotReady) continue;
                if (e != cudaSuccess) throw CudaError(std::string("vertex failed on the device: ") + cudaGetErrorString(e));
                lanes_[l].pop_front();
                if (lanes_[l].empty()) {
                    active_[i] = active_.back();
                    active_.pop_back();
                }
                rr_ = active_.empty() ? 0 : i % active_.size();
                in_flight_--;
                now = std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count();
                return v;
            }
            if ((spin & 1023) == 1023 && std::chrono::steady_clock::now() > deadline)
                throw CudaError("executor timed out waiting for a completion (" + std::to_string(in_flight_) +
                                " vertices in flight)");
        }
    }

    Executor::Impl& x_;
    std::chrono::steady_clock::time_point start_;
    int in_flight_ = 0;
    double wait_s_ = 0, launch_s_ = 0;
    std::vector<std::deque<std::int32_t>> lanes_;  // in-flight vertices per stream, launch order
    std::vector<int> active_;                      // lanes with work in flight
    size_t rr_ = 0;
    std::deque<std::int32_t> instant_;
};

}  // namespace

void Executor::Impl::run(const SchedulerPolicy& pol, std::uint64_t seed, ExecutionTrace* trace) {
    const MemGraph* g = &m;
    MemGraph fixed;
    if (pol.kind == SchedulerKind::FixedOrder) {
        fixed = make_fixed_order(m);
        fixed.reindex();
        g = &fixed;
    }
    timed = trace != nullptr || cfg.all_timestamps;
    if (cfg.graph && !timed && run_graph(pol)) return;
    last = RunStats{};
    dispatched.clear();
    dispatched.reserve(g->vertices.size());
    stream_of.assign(g->vertices.size(), -1);
    completed.clear();
    for (int d = 0; d < D; ++d) {
        set_device(d);
        TN_CUDA(cudaDeviceSynchronize());
        bool owner = true;
        for (int e = 0; e < d; ++e) owner = owner && ordinal[e] != ordinal[d];
        if (owner) TN_CUDA(cudaEventRecord(t0[d], streams[d][0]));
    }
    auto wall0 = std::chrono::steady_clock::now();
    const bool chain = cfg.lookahead > 0 && cfg.compute_tokens == 1;
    Resources res(D, cfg.streams_per_device, chain || cfg.device_deps ? (1 << 30) : cfg.compute_tokens,
                  cfg.materialize_inputs && !aliased_inputs(), !cfg.inputs_on_device,
                  !((chain || cfg.device_deps) && cfg.compute_tokens == 1 && !cfg.kernel_slots));
    ReadyList ready(pol.tie_break, seed);
    if (pol.tie_break == TieBreak::PlanOrder) ready.set_rank(plan_rank(*g));
    CudaBackend be(*this);
    try {
        if (cfg.device_deps) dispatch_loop_device_deps(*g, res, ready, be, cfg.lookahead);
        else if (chain) dispatch_loop_lookahead(*g, res, ready, be, cfg.lookahead);
        else dispatch_loop(*g, res, ready, be);
        last.host_wait_s = be.wait_s();
        last.host_launch_s = be.launch_s();
        last.host_dispatch_s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count() - last.host_wait_s;
    } catch (...) {
        for (int d = 0; d < D; ++d) {
            cudaSetDevice(ordinal[d]);
            cudaDeviceSynchronize();
        }
        cur_dev = -1;
        throw;
    }
    for (int d = 0; d < D; ++d) {
        set_device(d);
        TN_CUDA(cudaDeviceSynchronize());
    }
    last.device_makespan_s = 0;
    for (int d = 0; d < D; ++d) {
        if (t0[d] == nullptr || (d > 0 && std::find(ordinal.begin(), ordinal.begin() + d, ordinal[d]) != ordinal.begin() + d))
            continue;  // one clock per physical GPU
        set_device(d);
        TN_CUDA(cudaEventRecord(tend[d], streams[d][0]));
        TN_CUDA(cudaEventSynchronize(tend[d]));
        float ms = 0;
        TN_CUDA(cudaEventElapsedTime(&ms, t0[d], tend[d]));
        last.device_makespan_s = std::max(last.device_makespan_s, ms * 1e-3);
    }
    last.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    last.vertices = static_cast<std::int64_t>(dispatched.size());
    last_graph = g == &m ? nullptr : std::make_unique<MemGraph>(std::move(fixed));
    if (trace) *trace = build_trace();
}

// Trace of the most recent run from its device timestamps (seconds since the
// device's t0 event), plus the derived timing stats.
ExecutionTrace Executor::Impl::build_trace() {
    if (!timed)
        throw Error("the last run recorded no timestamps (untimed run): run with a trace or config "
                    "\"timestamps\": \"all\"");
    const MemGraph* g = last_graph ? last_graph.get() : &m;
    ExecutionTrace t;
    t.rows.reserve(dispatched.size());
    double kernel_s = 0, copy_s = 0;
    std::vector<std::vector<std::pair<double, double>>> kspans(D), cspans(D);
    for (std::int32_t vidx : dispatched) {
        const MemVertex& v = g->vertices[vidx];
        float a = 0, b = 0;
        if (!prog[vidx].timeless) {
            TN_CUDA(cudaEventElapsedTime(&a, t0[v.device], ev_start[vidx]));
            TN_CUDA(cudaEventElapsedTime(&b, t0[v.device], ev_end[vidx]));
        }
        double s = a * 1e-3, e = std::max(a, b) * 1e-3;
        // kernels that hold no generic stream slot run on the compute stream: its id is streams_per_device
        const std::int32_t st = stream_of[vidx] < 0 && v.op == MemOpKind::Kernel ? cfg.streams_per_device : stream_of[vidx];
        t.rows.push_back({v.id, s, e, v.device, st});
        if (v.op == MemOpKind::Kernel) {
            kernel_s += e - s;
            kspans[v.device].push_back({s, e});
        } else {
            copy_s += e - s;
            cspans[v.device].push_back({s, e});
        }
    }
    finalize_trace(*g, map, t);
    // Exposed transfer time: instants where a copy runs on a device and no
    // kernel does (union arithmetic per device).
    auto unite = [](std::vector<std::pair<double, double>>& sp) {
        std::sort(sp.begin(), sp.end());
        std::vector<std::pair<double, double>> out;
        for (auto& x : sp) {
            if (!out.empty() && x.first <= out.back().second) out.back().second = std::max(out.back().second, x.second);
            else out.push_back(x);
        }
        return out;
    };
    auto exposed_of = [&](std::vector<std::pair<double, double>> ks, std::vector<std::pair<double, double>> cs,
                          double* busy) {
        auto K = unite(ks), C = unite(cs);
        for (auto& kk : K) *busy += kk.second - kk.first;
        double ex = 0;
        size_t j = 0;
        for (auto& c : C) {
            double covered = 0;
            while (j < K.size() && K[j].second <= c.first) ++j;
            for (size_t q = j; q < K.size() && K[q].first < c.second; ++q)
                covered += std::min(c.second, K[q].second) - std::max(c.first, K[q].first);
            ex += (c.second - c.first) - covered;
        }
        return ex;
    };
    double exposed = 0, busy_k = 0, exposed_gpu = 0, busy_gpu = 0;
    for (int d = 0; d < D; ++d) exposed += exposed_of(kspans[d], cspans[d], &busy_k);
    // The same per physical GPU: memgraph devices sharing a GPU cover each
    // other's copies (times share one origin per GPU).
    std::map<int, std::pair<std::vector<std::pair<double, double>>, std::vector<std::pair<double, double>>>> per_gpu;
    for (int d = 0; d < D; ++d) {
        auto& pg = per_gpu[ordinal[d]];
        pg.first.insert(pg.first.end(), kspans[d].begin(), kspans[d].end());
        pg.second.insert(pg.second.end(), cspans[d].begin(), cspans[d].end());
    }
    for (auto& [gpu, pg] : per_gpu) exposed_gpu += exposed_of(pg.first, pg.second, &busy_gpu);
    last.makespan_s = t.makespan;
    last.kernel_time_s = kernel_s;
    last.copy_time_s = copy_s;
    last.kernel_busy_s = busy_k;
    last.exposed_transfer_s = exposed;
    last.exposed_transfer_gpu_s = exposed_gpu;
    return t;
}

Executor::Impl::~Impl() {
    for (int d = 0; d < D && d < static_cast<int>(ordinal.size()); ++d) {
        cudaSetDevice(ordinal[d]);
        cudaDeviceSynchronize();
    }
    for (size_t i = 0; i < ev_start.size(); ++i) {
        if (ev_start[i]) cudaEventDestroy(ev_start[i]);
        if (ev_end[i]) cudaEventDestroy(ev_end[i]);
        if (ev_done[i]) cudaEventDestroy(ev_done[i]);
    }
    for (int d = 0; d < static_cast<int>(t0.size()); ++d) {
        bool owner = true;
        for (int e = 0; e < d; ++e) owner = owner && t0[e] != t0[d];
        if (t0[d] && owner) cudaEventDestroy(t0[d]);
        if (d < static_cast<int>(tend.size()) && tend[d] && owner) cudaEventDestroy(tend[d]);
    }
    for (auto& ss : streams)
        for (auto s : ss)
            if (s) cudaStreamDestroy(s);
    drop_graphs();
    for (auto s : marker)
        if (s) cudaStreamDestroy(s);
    for (auto s : cap)
        if (s) cudaStreamDestroy(s);
    for (auto s : compute)
        if (s) cudaStreamDestroy(s);
    for (auto& ws : gws)
        for (auto& w : ws) {
            if (w.p) cudaFree(w.p);
            if (w.counters) cudaFree(w.counters);
        }
    for (auto p : arena)
        if (p) cudaFree(p);
    for (auto& [id, b] : inputs)
        if (b.p) cudaFreeHost(b.p);
    for (auto& [id, b] : staged)
        if (b.p) cudaFree(b.p);
    for (auto& in : prog)
        if (in.scratch) cudaFree(in.scratch);
    for (auto& [id, b] : slots)
        if (b.p) cudaFreeHost(b.p);
}

// -------------------------------------------------------------- graph mode ---
void Executor::Impl::drop_graphs() {
    for (auto& gc : graphs) {
        if (gc.x) cudaGraphExecDestroy(gc.x);
        if (gc.g) cudaGraphDestroy(gc.g);
        gc = GraphCache{};
    }
}

void Executor::Impl::build_graph(const MemGraph& g, GraphCache& gc) {
    for (const auto& in : prog)
        if (in.gemm && (in.gemm->sk_tiles > 0 || in.gemm->ksplit > 1))  // per-stream partial-sum workspaces
            throw Error("graph execution does not support stream-K / split-K GEMM tiles");
    const size_t V = g.vertices.size();
    GraphIndex gi(g);
    std::vector<std::vector<std::int32_t>> preds(V);
    for (size_t u = 0; u < V; ++u)
        for (std::int32_t a = gi.succ_start[u]; a < gi.succ_start[u + 1]; ++a)
            preds[gi.succ[a]].push_back(static_cast<std::int32_t>(u));
    // a topological order: the build's total order (every edge points forward)
    std::vector<std::int32_t> order;
    if (g.total_order.size() == V) {
        for (VertexId id : g.total_order) order.push_back(g.idx(id));
    } else {
        std::vector<std::int32_t> deg = gi.indeg;
        for (size_t i = 0; i < V; ++i)
            if (!deg[i]) order.push_back(static_cast<std::int32_t>(i));
        for (size_t k = 0; k < order.size(); ++k)
            for (std::int32_t a = gi.succ_start[order[k]]; a < gi.succ_start[order[k] + 1]; ++a)
                if (--deg[gi.succ[a]] == 0) order.push_back(gi.succ[a]);
    }
    if (order.size() != V) throw Error("graph execution needs an acyclic memgraph");
    TN_CUDA(cudaGraphCreate(&gc.g, 0));
    std::vector<cudaGraphNode_t> node(V, nullptr);
    const RunStats saved = last;
    last = RunStats{};
    capturing = true;
    try {
        std::vector<cudaGraphNode_t> deps;
        for (std::int32_t v : order) {
            deps.clear();
            for (std::int32_t p : preds[v])
                if (node[p]) deps.push_back(node[p]);
            std::sort(deps.begin(), deps.end());
            deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
            const Instr& in = prog[v];
            if (in.instant) {  // no device work: a join point for its in-edges, if any
                if (!deps.empty()) TN_CUDA(cudaGraphAddEmptyNode(&node[v], gc.g, deps.data(), deps.size()));
                continue;
            }
            set_device(in.dev);
            cudaGraph_t child = nullptr;
            TN_CUDA(cudaStreamBeginCapture(cap[in.dev], cudaStreamCaptureModeThreadLocal));
            try {
                issue(v, cap[in.dev], 0);
            } catch (...) {
                cudaStreamEndCapture(cap[in.dev], &child);
                if (child) cudaGraphDestroy(child);
                throw;
            }
            TN_CUDA(cudaStreamEndCapture(cap[in.dev], &child));
            size_t nn = 0;
            TN_CUDA(cudaGraphGetNodes(child, nullptr, &nn));
            if (nn == 0) TN_CUDA(cudaGraphAddEmptyNode(&node[v], gc.g, deps.data(), deps.size()));
            else TN_CUDA(cudaGraphAddChildGraphNode(&node[v], gc.g, deps.data(), deps.size(), child));
            cudaGraphDestroy(child);
            gc.nodes++;
        }
        set_device(0);
        TN_CUDA(cudaGraphInstantiate(&gc.x, gc.g, 0));
    } catch (...) {
        capturing = false;
        last = saved;
        if (gc.g) cudaGraphDestroy(gc.g);
        gc = GraphCache{};
        throw;
    }
    capturing = false;
    gc.counters = last;
    gc.counters.vertices = static_cast<std::int64_t>(V);
    last = saved;
}

// One untimed run as a graph launch; false (host loop instead) when the
// graph cannot be built for this memgraph (the reason is kept in graph_error).
bool Executor::Impl::run_graph(const SchedulerPolicy& pol) {
    if (!graph_error.empty()) return false;
    GraphCache& gc = graphs[pol.kind == SchedulerKind::FixedOrder ? 1 : 0];
    const auto w0 = std::chrono::steady_clock::now();
    if (!gc.x) {
        try {
            if (pol.kind == SchedulerKind::FixedOrder) {
                MemGraph fixed = make_fixed_order(m);
                fixed.reindex();
                build_graph(fixed, gc);
            } else {
                build_graph(m, gc);
            }
        } catch (const CudaError& e) {
            graph_error = e.what();
            cudaGetLastError();
            cur_dev = -1;
            return false;
        }
    }
    for (int d = 0; d < D; ++d) {
        set_device(d);
        TN_CUDA(cudaDeviceSynchronize());
    }
    set_device(0);
    cudaStream_t o = streams[0][0];
    const auto w1 = std::chrono::steady_clock::now();
    TN_CUDA(cudaEventRecord(t0[0], o));
    TN_CUDA(cudaGraphLaunch(gc.x, o));
    TN_CUDA(cudaEventRecord(tend[0], o));
    const auto w2 = std::chrono::steady_clock::now();
    TN_CUDA(cudaEventSynchronize(tend[0]));
    const auto w3 = std::chrono::steady_clock::now();
    float ms = 0;
    TN_CUDA(cudaEventElapsedTime(&ms, t0[0], tend[0]));
    last = gc.counters;
    last.device_makespan_s = ms * 1e-3;
    last.host_dispatch_s = std::chrono::duration<double>(w2 - w1).count();
    last.host_wait_s = std::chrono::duration<double>(w3 - w2).count();
    last.wall_s = std::chrono::duration<double>(w3 - w0).count();
    last.graph_nodes = gc.nodes;
    last_graph.reset();
    return true;
}

// ------------------------------------------------------------- public API ---
namespace {
// Every public entry point starts from the thread's real current device (the
// caller may have switched devices since the last call) and hands it back
// unchanged on exit.
struct DeviceGuard {
    int& cached;
    int saved = -1;
    explicit DeviceGuard(int& cur) : cached(cur) {
        if (cudaGetDevice(&saved) != cudaSuccess) saved = -1;
        cached = -1;
    }
    ~DeviceGuard() {
        if (saved >= 0) cudaSetDevice(saved);
        cached = -1;
    }
};
}  // namespace

Executor::Executor(const std::string& memgraph_json, const std::string& taskgraph_json, const ExecConfig& cfg)
    : impl_(std::make_unique<Impl>()) {
    DeviceGuard dg(impl_->cur_dev);
    auto [m, map] = parse_memgraph(memgraph_json);
    impl_->m = std::move(m);
    impl_->map = std::move(map);
    impl_->tg = parse_taskgraph(taskgraph_json);
    impl_->ops = parse_ops(taskgraph_json);
    impl_->cfg = cfg;
    if (cfg.streams_per_device < 1) throw Error("streams_per_device must be >= 1");
    if (cfg.compute_tokens < 1) throw Error("compute_tokens must be >= 1");
    impl_->build();
}

Executor::~Executor() {
    if (impl_) {
        DeviceGuard dg(impl_->cur_dev);
        impl_.reset();
    }
}

void Executor::set_input(VertexId id, const void* host, std::size_t bytes, bool from_device) {
    DeviceGuard dg(impl_->cur_dev);
    const TaskVertex* v = impl_->tg.find(id);
    if (!v || v->kind != VertexKind::Input) throw Error("vertex " + std::to_string(id) + " is not a taskgraph input");
    if (bytes > static_cast<std::size_t>(v->output_size))
        throw Error("input " + std::to_string(id) + ": " + std::to_string(bytes) + " bytes exceed output_size " +
                    std::to_string(v->output_size));
    if (impl_->aliased_inputs()) {
        HostBuf& b = impl_->staged.at(id);  // fixed at build: readers hold its address
        if (bytes > b.bytes) throw Error("input " + std::to_string(id) + " exceeds its placement");
        impl_->set_device(v->device);
        TN_CUDA(cudaMemcpy(b.p, host, bytes, from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        return;
    }
    if (impl_->cfg.inputs_on_device) {
        HostBuf& b = impl_->staged[id];
        impl_->set_device(v->device);
        if (!b.p || b.bytes != bytes) {
            if (b.p) cudaFree(b.p);
            b.p = nullptr;
            TN_CUDA(cudaMalloc(&b.p, std::max<std::size_t>(bytes, 1)));
            b.bytes = bytes;
            impl_->drop_graphs();
        }
        TN_CUDA(cudaMemcpy(b.p, host, bytes, from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        return;
    }
    HostBuf& b = impl_->inputs[id];
    if (impl_->zero_copy.count(id)) {  // fixed mapped buffer: kernels hold its device view
        if (bytes > b.bytes) throw Error("input " + std::to_string(id) + " exceeds its placement");
    } else if (!b.p || b.bytes != bytes) {
        if (b.p) cudaFreeHost(b.p);
        b.p = pinned_alloc(bytes);
        b.bytes = bytes;
        impl_->drop_graphs();  // captured copies hold the old buffer's address
    }
    if (from_device) TN_CUDA(cudaMemcpy(b.p, host, bytes, cudaMemcpyDeviceToHost));
    else std::memcpy(b.p, host, bytes);
}

ExecutionTrace Executor::run(const SchedulerPolicy& pol, std::uint64_t seed, bool want_trace) {
    DeviceGuard dg(impl_->cur_dev);
    ExecutionTrace t;
    impl_->run(pol, seed, want_trace ? &t : nullptr);
    return t;
}

ExecutionTrace Executor::last_trace() {
    if (impl_->dispatched.empty()) throw Error("no run to trace yet");
    DeviceGuard dg(impl_->cur_dev);
    return impl_->build_trace();
}

void Executor::get_output(VertexId id, void* host, std::size_t bytes) {
    auto it = impl_->map.placements.find(id);
    if (it == impl_->map.placements.end()) throw Error("vertex " + std::to_string(id) + " has no placement");
    if (bytes > static_cast<std::size_t>(it->second.size))
        throw Error("requested " + std::to_string(bytes) + " bytes from a region of " + std::to_string(it->second.size));
    DeviceGuard dg(impl_->cur_dev);
    impl_->set_device(it->second.device);
    TN_CUDA(cudaMemcpy(host, impl_->ptr_of(id), bytes, cudaMemcpyDeviceToHost));
}

void* Executor::placement_ptr(VertexId id) { return impl_->ptr_of(id); }

const RunStats& Executor::stats() const { return impl_->last; }

TieBreak Executor::default_tie_break() const { return impl_->cfg.tie_break; }

ComparisonSummary Executor::compare_policies(std::int64_t trials, std::uint64_t seed) {
    if (trials < 1) throw Error("compare_policies: trials must be >= 1");
    DeviceGuard dg(impl_->cur_dev);
    const SchedulerPolicy ev{SchedulerKind::EventDriven, impl_->cfg.tie_break};
    const SchedulerPolicy fx{SchedulerKind::FixedOrder, TieBreak::Fifo};
    impl_->run(ev, seed, nullptr);  // warm both paths (fixed-order graph, caches, clocks)
    impl_->run(fx, seed, nullptr);
    std::vector<double> e(trials), f(trials);
    for (std::int64_t t = 0; t < trials; ++t) {
        const std::uint64_t ts = mix64(seed + static_cast<std::uint64_t>(t));
        const bool ev_first = (t % 2) == 0;  // alternate to cancel drift (clocks, power)
        for (int k = 0; k < 2; ++k) {
            const bool is_ev = (k == 0) == ev_first;
            impl_->run(is_ev ? ev : fx, ts, nullptr);
            (is_ev ? e : f)[t] = impl_->last.device_makespan_s;
        }
    }
    return summarize_pairs(e, f, seed);
}

std::string RunStats::to_json() const {
    json j;
    j["vertices"] = vertices;
    j["kernel_launches"] = kernel_launches;
    j["h2d_bytes"] = h2d_bytes;
    j["d2h_bytes"] = d2h_bytes;
    j["d2h_elided_bytes"] = d2h_elided_bytes;
    j["p2p_bytes"] = p2p_bytes;
    j["d2d_bytes"] = d2d_bytes;
    j["flops"] = flops;
    j["makespan_s"] = makespan_s;
    j["wall_s"] = wall_s;
    j["kernel_time_s"] = kernel_time_s;
    j["kernel_busy_s"] = kernel_busy_s;
    j["copy_time_s"] = copy_time_s;
    j["exposed_transfer_s"] = exposed_transfer_s;
    j["exposed_transfer_gpu_s"] = exposed_transfer_gpu_s;
    j["zero_copy_bytes"] = zero_copy_bytes;
    j["host_dispatch_s"] = host_dispatch_s;
    j["host_wait_s"] = host_wait_s;
    j["host_launch_s"] = host_launch_s;
    j["device_makespan_s"] = device_makespan_s;
    j["graph_nodes"] = graph_nodes;
    return j.dump();
}

ExecConfig parse_exec_config(const std::string& text) {
    ExecConfig c;
    if (text.empty()) return c;
    json j;
    try {
        j = json::parse(text);
        if (j.contains("devices")) c.devices = j["devices"].get<std::vector<int>>();
        c.streams_per_device = j.value("streams_per_device", c.streams_per_device);
        c.compute_tokens = j.value("compute_tokens", c.compute_tokens);
        c.lookahead = j.value("lookahead", c.lookahead);
        c.kernel_slots = j.value("kernel_slots", c.kernel_slots);
        const std::string deps = j.value("dependencies", std::string("host"));
        if (deps != "host" && deps != "device") throw ParseError("dependencies must be host or device");
        c.device_deps = deps == "device";
        c.elide_input_offloads = j.value("elide_input_offloads", c.elide_input_offloads);
        c.materialize_inputs = j.value("materialize_inputs", c.materialize_inputs);
        c.timeout_s = j.value("timeout_s", c.timeout_s);
        if (j.contains("tie_break")) c.tie_break = tie_break_from_string(j["tie_break"].get<std::string>());
        const std::string comp = j.value("completion", std::string("poll"));
        if (comp != "poll" && comp != "callback") throw ParseError("completion must be poll or callback");
        c.poll = comp == "poll";
        c.zero_copy_gathers = j.value("zero_copy_gathers", c.zero_copy_gathers);
        c.pdl = j.value("pdl", c.pdl);
        const std::string ex = j.value("execution", std::string("events"));
        if (ex != "events" && ex != "graph") throw ParseError("execution must be events or graph");
        c.graph = ex == "graph";
        const std::string ts = j.value("timestamps", std::string("traced"));
        if (ts != "traced" && ts != "all") throw ParseError("timestamps must be traced or all");
        c.all_timestamps = ts == "all";
        const std::string res = j.value("input_residency", std::string("host"));
        if (res != "host" && res != "device") throw ParseError("input_residency must be host or device");
        c.inputs_on_device = res == "device";
        const std::string di = j.value("device_inputs", std::string("alias"));
        if (di != "alias" && di != "copy") throw ParseError("device_inputs must be alias or copy");
        c.alias_device_inputs = di == "alias";
    } catch (const json::exception& e) {
        throw ParseError(std::string("invalid executor config: ") + e.what());
    }
    return c;
}

}  // namespace tn
