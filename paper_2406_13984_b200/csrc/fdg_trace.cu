// fdg_trace.cu -- lightweight device timeline: CUDA events recorded around
// every library launch when tracing is on (the counterpart of the reference's
// per-stage DurationCounter / ScopedTimer, common.hpp:240-260, at kernel
// granularity). Dumped as CSV: name,stream,start_ms,end_ms (relative to the
// first traced event). Off by default; zero cost when off.
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {

bool g_trace = false;

namespace {
struct Rec {
    const char* name;
    cudaStream_t st;
    cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t get_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

TraceScope::TraceScope(const char* name, cudaStream_t st) : name_(name), st_(st) {
    if (!g_trace) return;
    std::lock_guard<std::mutex> lk(g_mu);
    a_ = get_event();
    cudaEventRecord(a_, st);
}

TraceScope::~TraceScope() {
    if (!g_trace || !a_) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEvent_t b = get_event();
    cudaEventRecord(b, st_);
    g_recs.push_back({name_, st_, a_, b});
}

}  // namespace fdg

using namespace fdg;

extern "C" {

int fdg_trace_enable(int on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_trace = on != 0;
    if (g_trace) {
        for (auto& r : g_recs) {
            g_pool.push_back(r.a);
            g_pool.push_back(r.b);
        }
        g_recs.clear();
    }
    return FDG_OK;
}

int fdg_trace_dump(const char* path) {
    FDG_CUDA(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_mu);
    FILE* f = std::fopen(path, "w");
    if (!f) return fail(FDG_INVALID_ARG, std::string("trace: cannot open ") + path);
    std::fprintf(f, "name,stream,start_ms,end_ms\n");
    if (!g_recs.empty()) {
        cudaEvent_t t0 = g_recs.front().a;
        for (auto& r : g_recs) {
            float s = 0, e = 0;
            cudaEventElapsedTime(&s, t0, r.a);
            cudaEventElapsedTime(&e, t0, r.b);
            std::fprintf(f, "%s,%p,%.4f,%.4f\n", r.name, (void*)r.st, s, e);
        }
    }
    std::fclose(f);
    return FDG_OK;
}

}  // extern "C"
