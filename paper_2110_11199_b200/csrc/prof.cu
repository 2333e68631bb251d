#include "prof.hpp"

#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace ab {
constexpr size_t kTraceWords = 160 * 48 + 160 * 64 * 12 + 2 * 8 * 64 * 3;  // tc_core.cuh: stamps + per-item timeline
unsigned long long* g_trace_buf = nullptr;  // device buffer while tracing is on (tc_core.cuh)
int g_trace_skip = 0;                       // pair-kernel launches to skip before the traced one

// The buffer for exactly one launch: the (skip+1)-th pair-kernel launch after enabling.
unsigned long long* trace_take() {
    if (!g_trace_buf) return nullptr;
    if (g_trace_skip-- == 0) return g_trace_buf;
    return nullptr;
}

// Debug timeline control (see tc_core.cuh): enable, then read and clear.
void trace_enable(int on) {
    if (on) g_trace_skip = on - 1;
    if (on && !g_trace_buf) {
        AB_CUDA(cudaMalloc(&g_trace_buf, sizeof(unsigned long long) * kTraceWords));
        AB_CUDA(cudaMemset(g_trace_buf, 0, sizeof(unsigned long long) * kTraceWords));
        AB_CUDA(cudaDeviceSynchronize());  // legacy-stream memset vs the engine's non-blocking streams
    }
    if (!on && g_trace_buf) {
        AB_CUDA(cudaDeviceSynchronize());
        AB_CUDA(cudaFree(g_trace_buf));
        g_trace_buf = nullptr;
    }
}
void trace_read(unsigned long long* out, int n) {
    AB_CUDA(cudaDeviceSynchronize());
    if (!g_trace_buf) return;
    if (n > static_cast<int>(kTraceWords)) n = static_cast<int>(kTraceWords);
    AB_CUDA(cudaMemcpy(out, g_trace_buf, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
    AB_CUDA(cudaMemset(g_trace_buf, 0, sizeof(unsigned long long) * kTraceWords));
    AB_CUDA(cudaDeviceSynchronize());
}

bool g_prof_enabled = false;
std::vector<ProfRec>* g_prof_capture = nullptr;

namespace {
std::vector<ProfRec> g_eager;
std::vector<cudaEvent_t> g_pool;
double g_ms[PROF_NCAT], g_flops[PROF_NCAT], g_bytes[PROF_NCAT];
int64_t g_launches[PROF_NCAT];
std::mutex g_mu;
cudaEvent_t get_event() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e;
    AB_CUDA(cudaEventCreate(&e));
    return e;
}
std::vector<ProfRec>& target() { return g_prof_capture ? *g_prof_capture : g_eager; }
void add(const ProfRec& r) {
    float t = 0;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) { cudaGetLastError(); return; }
    if (r.cat < 0 || r.cat >= PROF_NCAT) return;
    g_ms[r.cat] += t; g_flops[r.cat] += r.flops; g_bytes[r.cat] += r.bytes; g_launches[r.cat] += 1;
}
}  // namespace

int prof_begin(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    ProfRec r{get_event(), get_event(), -1, 0, 0};
    // inside stream capture a plain record is only a dependency marker; External makes it a
    // real event-record node that fires on every replay
    AB_CUDA(cudaEventRecordWithFlags(r.a, s, g_prof_capture ? cudaEventRecordExternal : cudaEventRecordDefault));
    target().push_back(r);
    return static_cast<int>(target().size()) - 1;
}

void prof_end(int id, cudaStream_t s, int cat, double flops, double bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    ProfRec& r = target()[id];
    AB_CUDA(cudaEventRecordWithFlags(r.b, s, g_prof_capture ? cudaEventRecordExternal : cudaEventRecordDefault));
    r.cat = cat; r.flops = flops; r.bytes = bytes;
}

void prof_accumulate(const std::vector<ProfRec>& recs) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const auto& r : recs) add(r);
}

void prof_read(double* ms, double* flops, double* bytes, int64_t* launches, int ncat) {
    std::lock_guard<std::mutex> lk(g_mu);
    AB_CUDA(cudaDeviceSynchronize());
    for (auto& r : g_eager) {
        add(r);
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_eager.clear();
    for (int c = 0; c < ncat && c < PROF_NCAT; ++c) {
        ms[c] = g_ms[c]; flops[c] = g_flops[c]; bytes[c] = g_bytes[c]; launches[c] = g_launches[c];
    }
    for (int c = 0; c < PROF_NCAT; ++c) { g_ms[c] = 0; g_flops[c] = 0; g_bytes[c] = 0; g_launches[c] = 0; }
}

namespace {
std::map<std::string, int64_t> g_variants;
std::mutex g_var_mu;
}  // namespace

// __PRETTY_FUNCTION__ of note_kernel<T>() ends in "[with T = <type>]"; keep <type> without the
// namespace prefix.
void note_variant(const char* pretty) {
    std::string s(pretty);
    const auto at = s.find("T = ");
    if (at != std::string::npos) {
        s = s.substr(at + 4);
        const auto end = s.rfind(']');
        if (end != std::string::npos) s = s.substr(0, end);
        const auto semi = s.find(';');
        if (semi != std::string::npos) s = s.substr(0, semi);
    }
    for (const char* ns : {"ab::", "tc::", "{anonymous}::", "(anonymous namespace)::"})
        for (auto p = s.find(ns); p != std::string::npos; p = s.find(ns)) s.erase(p, std::strlen(ns));
    // nvcc names anonymous namespaces _GLOBAL__N__<hash>_<file>::
    for (auto p = s.find("_GLOBAL__N_"); p != std::string::npos; p = s.find("_GLOBAL__N_")) {
        const auto e = s.find("::", p);
        if (e == std::string::npos) break;
        s.erase(p, e + 2 - p);
    }
    std::lock_guard<std::mutex> lk(g_var_mu);
    ++g_variants[s];
}

void log_map_alignment(const char* where, const void* base, uint64_t inner, uint64_t outer, int64_t pitch_bytes) {
    static const bool on = std::getenv("ADPSGD_LOG_ALIGN") != nullptr;
    if (!on) return;
    const bool bad_pitch = pitch_bytes % 128 != 0, bad_base = reinterpret_cast<uintptr_t>(base) % 128 != 0;
    if (!bad_pitch && !bad_base) return;
    static std::mutex mu;
    static std::map<std::string, int> seen;
    const std::string key = std::string(where) + ":" + std::to_string(inner) + "x" + std::to_string(outer) + "/" +
                            std::to_string(pitch_bytes) + (bad_base ? "/base" : "");
    std::lock_guard<std::mutex> lk(mu);
    if (seen[key]++ == 0)
        std::fprintf(stderr, "[align] %s inner %llu outer %llu pitch %lld B%s%s\n", where,
                     static_cast<unsigned long long>(inner), static_cast<unsigned long long>(outer),
                     static_cast<long long>(pitch_bytes), bad_pitch ? " (pitch not 128B)" : "",
                     bad_base ? " (base not 128B)" : "");
}

std::string variants_string(bool reset) {
    std::lock_guard<std::mutex> lk(g_var_mu);
    std::string out;
    for (const auto& kv : g_variants) out += kv.first + "=" + std::to_string(kv.second) + ";";
    if (reset) g_variants.clear();
    return out;
}

}  // namespace ab
