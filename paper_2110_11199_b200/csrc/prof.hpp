// Live per-kernel-class timing with CUDA events (enabled by bench.py over its timed
// region): each library launch is bracketed by an event pair on its own stream and
// tagged with its algorithmic FLOPs and bytes, so achieved TFLOP/s and GB/s per kernel
// class come from the same launches that are being timed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ab {

enum ProfCat { PROF_GEMM_TC = 0, PROF_GEMM_SIMT, PROF_CELL, PROF_CE, PROF_REDUCE, PROF_GATHER, PROF_MIX, PROF_OTHER,
               PROF_NCAT };

extern bool g_prof_enabled;
int prof_begin(cudaStream_t s);
void prof_end(int id, cudaStream_t s, int cat, double flops, double bytes);
// Synchronises the device, accumulates and clears the records.
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

}  // namespace ab
