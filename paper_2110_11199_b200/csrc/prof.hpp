// Live per-kernel-class timing with CUDA events (enabled by bench.py): each library
// launch is bracketed by an event pair on its own stream and tagged with its algorithmic
// FLOPs and bytes, so achieved TFLOP/s and GB/s per kernel class come from the launches
// being timed. Launches captured into a CUDA graph keep their event nodes; after every
// replay the graph's records are re-read (prof_accumulate).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace ab {

enum ProfCat {
    PROF_GEMM_REC_FWD = 0,  // recurrent step GEMM [x_t | h_{t-1}] x [W_ih | W_hh]^T (+ fused cell)
    PROF_GEMM_REC_BWD,      // BPTT dgrad dz_t W_hh (+ fused cell backward)
    PROF_GEMM_WGRAD,        // dW_ih, dW_hh, dW_proj, dW_out
    PROF_GEMM_DGRAD_X,      // dX = sum_d dZ_d W_ih_d, dY, dTop
    PROF_GEMM_OUT,          // projection / output-layer forward (+ fused softmax-CE)
    PROF_GEMM_SIMT,         // fp32 parity-mode GEMMs
    PROF_CELL,
    PROF_CE,
    PROF_REDUCE,
    PROF_GATHER,
    PROF_MIX,
    PROF_OTHER,
    PROF_NCAT
};

struct ProfRec { cudaEvent_t a, b; int cat; double flops, bytes; };

extern bool g_prof_enabled;
// While non-null, new records are appended here (graph capture) instead of the eager list.
extern std::vector<ProfRec>* g_prof_capture;

int prof_begin(cudaStream_t s);
void prof_end(int id, cudaStream_t s, int cat, double flops, double bytes);
// Adds the elapsed times of a (replayed, completed) record list to the accumulators.
void prof_accumulate(const std::vector<ProfRec>& recs);
// Synchronises the device, folds the eager records in, returns and clears the accumulators.
void prof_read(double* ms, double* flops, double* bytes, int64_t* launches, int ncat);

struct ProfScope {
    int id = -1;
    cudaStream_t s;
    int cat;
    double flops, bytes;
    ProfScope(cudaStream_t s_, int cat_, double flops_, double bytes_) : s(s_), cat(cat_), flops(flops_), bytes(bytes_) {
        if (g_prof_enabled) id = prof_begin(s);
    }
    ~ProfScope() {
        if (id >= 0) prof_end(id, s, cat, flops, bytes);
    }
};

// Kernel-variant registry: every tcgen05 launch site records the template instantiation it
// selected (host-side, at eager launch or graph capture), so tests can assert which kernel a
// shape exercised (adpsgd_kernel_variants).
void note_variant(const char* pretty_function);
template <class T> struct cta_pair;    // markers: tile on a CTA pair (cta_group::2) ...
template <class T> struct cta_single;  // ... or on one CTA
template <class T>
inline void note_kernel() { note_variant(__PRETTY_FUNCTION__); }
// "name=count;..." of every variant noted since the last reset.
std::string variants_string(bool reset);

// ADPSGD_LOG_ALIGN=1 (diagnosis): report TMA maps whose base or row pitch is not a whole number of
// 128-byte lines (every box row then straddles two lines), once per distinct shape.
void log_map_alignment(const char* where, const void* base, uint64_t inner, uint64_t outer, int64_t pitch_bytes);
}  // namespace ab
