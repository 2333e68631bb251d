// GEMM front-end shared by the fp32 SIMT path (parity mode) and the tcgen05 bf16 path.
//
//   C[M,N] = alpha * sum_seg sum_k A_seg(m,k) B_seg(n,k)  (+ C if accumulate) (+ bias[n])
//
// A(m,k) = A[m*lda + k] (K-major) or A[k*lda + m] (MN-major); B(n,k) likewise. Up to two
// K segments accumulate into one output tile (used for [x_t | h_{t-1}] x [W_ih | W_hh]
// and for the two directions of dX = sum_d dZ_d W_ih_d).
#pragma once

#include "knobs.hpp"

#include <cstdint>

#include "common.cuh"

namespace ab {

struct GemmOperand {
    const void* ptr = nullptr;
    int64_t ld = 0;
    bool mn = false;  // MN-major (the non-reduction index is contiguous)
};

struct GemmSeg {
    GemmOperand a, b;
    int K = 0;
};

struct GemmArgs {
    int M = 0, N = 0;
    GemmSeg seg[2];
    int nseg = 1;
    void* C = nullptr;
    int64_t ldc = 0;
    bool c_bf16 = false;
    float alpha = 1.0f;
    bool accumulate = false;
    const float* bias = nullptr;
    int tag = 0;  // ProfCat of the tcgen05 launch (prof.hpp)
    // Column redirect: output columns n >= n_main go to extra[m] (used with a ones column in the
    // B operand so a weight-gradient GEMM also yields the bias gradient). n_main < 0: off.
    int n_main = -1;
    float* extra = nullptr;
    // Optional K-major copy of B's columns [256 * floor(n_main / 256), +16) as [16 rows x K] bf16
    // (row pitch ld_tail elements): lets <= 8 columns past the last full 256-wide tile ride on an
    // extra N = 16 MMA of that tile instead of a mostly empty extra n-tile (tcgen05 path only).
    const void* b_tail = nullptr;
    int64_t ld_tail = 0;
    // Fused SGD update (tcgen05 path, fp32 output, no accumulate): instead of storing the
    // gradient value x of element (m, n) of C [of extra[m]], store o = upd_w - lr * x to upd_o and
    // bf16(o) to upd_sh, each laid out exactly like C [like extra]; lr = *upd_lr (device scalar).
    const float* upd_w = nullptr;
    float* upd_o = nullptr;
    bf16* upd_sh = nullptr;
    const float* upd_xw = nullptr;
    float* upd_xo = nullptr;
    bf16* upd_xsh = nullptr;
    const float* upd_lr = nullptr;
};

// Stream-K scratch of the calling thread's engine (set before its GEMMs run; see gemm_tc.cu):
// ws >= (SMs/2) * 2 * 17 * 128 * 32 floats, flags >= SMs (+ 2 per split-K tile) u32 zeroed once.
// ws == nullptr: no stream-K.
struct GemmWorkspace {
    float* ws = nullptr;
    size_t floats = 0;
    unsigned int* flags = nullptr;
    size_t flag_count = 0;
};
void set_gemm_workspace(const GemmWorkspace& w);
const GemmWorkspace& gemm_workspace();
// Binds a workspace for the GEMMs issued in this scope and restores the previous binding on exit,
// so no thread keeps a pointer into an engine that has since been destroyed.
struct GemmWorkspaceScope {
    GemmWorkspace prev;
    explicit GemmWorkspaceScope(const GemmWorkspace& w) : prev(gemm_workspace()) { set_gemm_workspace(w); }
    ~GemmWorkspaceScope() { set_gemm_workspace(prev); }
    GemmWorkspaceScope(const GemmWorkspaceScope&) = delete;
    GemmWorkspaceScope& operator=(const GemmWorkspaceScope&) = delete;
};
bool gemm_wgrad_wide(int M, int N);  // see gemm_tc.cu  // tests: take the extra-column / stream-K kernels whenever the layout allows

// fp32 operands, fp32 or bf16 output, any majorness (gemm_simt.cu).
void gemm_simt(const GemmArgs& g, cudaStream_t s);
// bf16 operands, tcgen05 + TMA + TMEM, fp32 accumulate (gemm_tc.cu).
void gemm_tc(const GemmArgs& g, cudaStream_t s);

inline void gemm(bool bf16_mode, const GemmArgs& g, cudaStream_t s) {
    if (bf16_mode) gemm_tc(g, s); else gemm_simt(g, s);
}

}  // namespace ab
