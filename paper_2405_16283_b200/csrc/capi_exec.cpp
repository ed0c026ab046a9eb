// C ABI of the CUDA executor (include/turnip.h, tn_exec_*).
#include <cstdlib>
#include <cstring>
#include <exception>

#include "../../include/turnip.h"
#include "exec/executor.hpp"

using namespace tn;

struct tn_exec {
    std::unique_ptr<Executor> x;
};

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

int tn_exec_create(const char* memgraph_json, const char* taskgraph_json, const char* config_json, tn_exec** out,
                   char** err) {
    return guarded(err, [&] {
        auto h = std::make_unique<tn_exec>();
        h->x = std::make_unique<Executor>(str(memgraph_json), str(taskgraph_json), parse_exec_config(str(config_json)));
        *out = h.release();
    });
}

int tn_exec_set_input(tn_exec* h, int64_t id, const void* host, size_t bytes, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        h->x->set_input(id, host, bytes, false);
    });
}

int tn_exec_set_input_device(tn_exec* h, int64_t id, const void* dev, size_t bytes, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        h->x->set_input(id, dev, bytes, true);
    });
}

int tn_exec_run(tn_exec* h, const char* policy, const char* tie_break, uint64_t seed, char** trace, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        SchedulerPolicy pol;
        pol.kind = scheduler_kind_from_string(str(policy, "event-driven"));
        const std::string tb = str(tie_break);
        pol.tie_break = tb.empty() ? h->x->default_tie_break() : tie_break_from_string(tb);
        auto t = h->x->run(pol, seed, trace != nullptr);
        if (trace) *trace = dup(t.to_json());
    });
}

int tn_exec_last_trace(tn_exec* h, char** trace, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        *trace = dup(h->x->last_trace().to_json());
    });
}

int tn_exec_get_output(tn_exec* h, int64_t id, void* host, size_t bytes, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        h->x->get_output(id, host, bytes);
    });
}

int tn_exec_placement_ptr(tn_exec* h, int64_t id, void** ptr, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        *ptr = h->x->placement_ptr(id);
    });
}

int tn_exec_stats(tn_exec* h, char** out, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        *out = dup(h->x->stats().to_json());
    });
}

int tn_exec_compare_policies(tn_exec* h, int64_t trials, uint64_t seed, char** summary_json, char** err) {
    return guarded(err, [&] {
        if (!h) throw Error("null executor handle");
        *summary_json = dup(h->x->compare_policies(trials, seed).to_json());
    });
}

void tn_exec_destroy(tn_exec* h) {
    try {
        delete h;
    } catch (...) {
    }
}

}  // extern "C"
