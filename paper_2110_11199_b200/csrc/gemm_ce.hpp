// Output layer fused with softmax cross-entropy (gemm_ce.cu), bf16 mode.
#pragma once

#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "gemm_lstm.hpp"

namespace ab {

struct CeArgs {
    const bf16* Y;          // [M x K] frames x proj (K-major)
    const bf16* W;          // W_out [N x K] bf16 shadow
    const float* bias;      // b_out [N] (fp32 master)
    const int32_t* labels;  // [M]
    int M, N, K;
    int ldY;                // row pitch of Y (>= K)
    float scale;            // 1 / (T * B)
    float2* part;           // [M x ceil(N/256)] scratch
    float* zlab;            // [M] scratch
    float* lse;             // [M] scratch
    float* row_loss;        // [M] out
    bf16* dlogits;          // [M x N] out
};

void ce_forward_backward(const CeArgs& a, cudaStream_t s);
int64_t ce_part_elems(int M, int N);

}  // namespace ab
