#include "prof.hpp"

#include <mutex>
#include <vector>

#include "common.cuh"

namespace ab {

bool g_prof_enabled = false;

namespace {
struct Rec { cudaEvent_t a, b; int cat; double flops, bytes; bool done; };
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::mutex g_mu;
cudaEvent_t get_event() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e;
    AB_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

int prof_begin(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{get_event(), get_event(), 0, 0, 0, false};
    AB_CUDA(cudaEventRecord(r.a, s));
    g_recs.push_back(r);
    return static_cast<int>(g_recs.size()) - 1;
}

void prof_end(int id, cudaStream_t s, int cat, double flops, double bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    Rec& r = g_recs[id];
    AB_CUDA(cudaEventRecord(r.b, s));
    r.cat = cat; r.flops = flops; r.bytes = bytes; r.done = true;
}

void prof_read(double* ms, double* flops, double* bytes, int64_t* launches, int ncat) {
    std::lock_guard<std::mutex> lk(g_mu);
    AB_CUDA(cudaDeviceSynchronize());
    for (int c = 0; c < ncat; ++c) { ms[c] = 0; flops[c] = 0; bytes[c] = 0; launches[c] = 0; }
    for (auto& r : g_recs) {
        if (r.done && r.cat < ncat) {
            float t = 0;
            AB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            ms[r.cat] += t; flops[r.cat] += r.flops; bytes[r.cat] += r.bytes; launches[r.cat] += 1;
        }
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
}

}  // namespace ab
