// Fused LSTM step kernels (gemm_lstm.cu): recurrent GEMM + cell forward, and BPTT
// dgrad + cell backward, both directions of a layer per launch. bf16 mode, H % 64 == 0.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <cstring>

#include "common.cuh"

namespace ab {

// Sync scratch of the persistent recurrent kernels (engine: pb_sync, 520 u32): the BPTT uses
// [0, 256) exchange epochs, [256, 512) per-(dir, row-block, CTA) step counters, [512] exit; the
// forward [384, 512) step counters, [513] exit. Each kernel needs 2 dirs x m_tiles x 2 counters.
constexpr int kPbSyncWords = 520;
constexpr int kBwdDepSlots = 256;
constexpr int kFwdDepSlots = 128;

using EncodeFnT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct LstmFwdDir {
    const bf16* x; int64_t ldx; int Kx;       // x_t rows [B x Kx]
    const bf16* w_ih; int64_t ld_wih;         // [4H x Kx]
    const bf16* h_prev; int64_t ld_hprev;     // h_{t-1} rows [B x H] (nullptr at the first step)
    const bf16* w_hh;                         // [4H x H]
    const float* bias;                        // [4H] (fp32 master)
    const float* c_prev;                      // [B x H] at ldc (nullptr at the first step)
    bf16* gates; float* c; bf16* h;           // outputs (row pitch ldg / ldc / ldh); gates i,f,g,o bf16
};

struct LstmBwdDir {
    const bf16* dz_src; int64_t ld_dz_src;    // dz_t [B x 4H] (A of the recurrent dgrad)
    const bf16* w_hh;                         // [4H x H]
    const float* dH;                          // dHout[t'] (+ d*H), row pitch lddh
    float* dc_rec;                            // [B x H]
    const bf16* gates; const float* c; const float* c_prev;   // at t' (c_prev may be nullptr)
    bf16* dz_dst;                             // dz_{t'}
};

void lstm_fwd_step(const LstmFwdDir* dirs, int ndirs, int B, int H, int ldg, int ldc, int ldh, cudaStream_t s);
// One layer's whole forward recurrence (both directions, all T steps) in one persistent kernel;
// returns false (nothing launched) when the shape is not eligible.
struct LstmFwdLayer {
    const bf16* x; int64_t ldx; int Kx;  // layer input [T*B x Kx] (row pitch ldx)
    const bf16* w_ih[2]; int64_t ld_wih; // [4H x Kx] per direction
    const bf16* w_hh[2];                 // [4H x H] per direction
    const float* bias[2];                // [4H] per direction (fp32 master)
    bf16* gates; int64_t ldg;            // [T*B x 2*4H] out
    float* c; int64_t ldc;               // [T*B x 2H] out
    bf16* h; int64_t ldh;                // [T*B x 2H] out (and the recurrent operand)
};
bool lstm_fwd_layer_persistent(const LstmFwdLayer& L, int ndirs, int B, int H, int T, cudaStream_t s, unsigned int* dep,
                               unsigned int* exit_ctr);

// One layer's whole BPTT recurrence (both directions, steps after the first cell backward) in one
// persistent kernel; returns false (nothing launched) when the shape is not eligible.
struct LstmBwdLayer {
    bf16* dZ; int64_t ld_dz;          // [T*B x 2*4H]: dz_{T-1} (dir 0) / dz_0 (dir 1) given, the rest produced
    const bf16* w_hh[2];              // [4H x H] per direction
    const bf16* w_hh_t[2] = {nullptr, nullptr};  // optional [H x 4H] transposes (32-unit BPTT tiles)
    const float* dH; int64_t lddh;    // [T*B x 2H]
    float* dc_rec[2];                 // [B x H] per direction (carries the first cell backward's dc)
    const bf16* gates; int64_t ldg;   // [T*B x 2*4H]
    const float* c; int64_t ldc;      // [T*B x 2H]
};
// true when the persistent BPTT will take 32-unit tiles and so wants LstmBwdLayer::w_hh_t
bool lstm_bwd_wants_whh_t(int ndirs, int B, int H);
bool lstm_bwd_layer_persistent(const LstmBwdLayer& L, int ndirs, int B, int H, int T, cudaStream_t s, float* sk_scratch,
                               unsigned int* sk_flags, unsigned int* dep, unsigned int* exit_ctr);

// sk_scratch / sk_flags: split-K exchange buffers (lstm_bwd_splitk_slots(..) x 64 KB fp32 and
// x 1 u32, flags zeroed once); nullptr disables the split-K variant.
int64_t lstm_bwd_splitk_slots(int ndirs, int B, int H);
void lstm_bwd_step(const LstmBwdDir* dirs, int ndirs, int B, int H, int lddh, int ldg, int ldc, int lddz,
                   cudaStream_t s, float* sk_scratch = nullptr, unsigned int* sk_flags = nullptr);

}  // namespace ab
