// Pointwise / reduction / update kernels of the learner step (kernels.cu).
#pragma once

#include "common.cuh"

namespace ab {

// X[(t*B + b)*ldx + i] = feats[idx[b]][t][i] (i < I), 0 for I <= i < ldx; lab[t*B+b] = labels[idx[b]][t]
template <typename AT>
void launch_gather(const float* feats, const int32_t* labels, const int32_t* idx, int B, int T, int I, int ldx,
                   AT* X, int32_t* lab, cudaStream_t s, bool ones_col, AT* tail = nullptr, int tail_n0 = 0);

// LSTM cell forward for one (layer, direction, time step) over B rows (gate order i,f,g,o).
template <typename AT>
void launch_cell_fwd(const float* z, int ldz, const float* c_prev, int ldc, AT* gates, int ldg, float* c, AT* h,
                     int ldh, int B, int H, cudaStream_t s);

// LSTM cell backward (BPTT step): dz = d(loss)/d(pre-activations) at time t; dc_rec updated in place.
template <typename AT>
void launch_cell_bwd(const float* dH, int lddh, const float* dh_rec, float* dc_rec, bool first, const AT* gates,
                     int ldg, const float* c, const float* c_prev, int ldc, AT* dz, int lddz, int B, int H,
                     cudaStream_t s);

// out [cols x rows] = in [rows x cols]^T (bf16)
void launch_transpose_bf16(const bf16* in, bf16* out, int rows, int cols, cudaStream_t s);

// First BPTT cell backward (no recurrent term) of both directions in one vectorised launch;
// false (nothing launched) when the layout does not allow 16-byte accesses.
bool launch_cell_bwd_first2(const float* const dH[2], const bf16* const gates[2], const float* const c[2],
                            const float* const c_prev[2], bf16* const dz[2], float* const dc_rec[2], int lddh, int ldg,
                            int ldc, int lddz, int B, int H, cudaStream_t s);

// Softmax cross-entropy over rows of fp32 logits: row_loss[r] = lse - logit[label],
// dlogits = (softmax - onehot) * scale.
template <typename AT>
void launch_softmax_ce(const float* logits, const int32_t* labels, int R, int C, float scale, AT* dlogits,
                       float* row_loss, cudaStream_t s);

// out[n] = sum_r X[r*ld + n], deterministic two-pass (partials in ws, >= chunks*N floats).
template <typename AT>
void launch_colsum(const AT* X, int64_t ld, int R, int N, float* out, float* ws, int64_t ws_elems, cudaStream_t s);

// out[0] = scale * sum(x[0..n)) (single block, fixed order).
void launch_sum(const float* x, int n, float scale, float* out, cudaStream_t s);

void launch_sum_masked(const float* x, int T, int B, int valid, float* out, cudaStream_t s);
// p[r * ld + col] = v for r < rows (the constant ones column of the bias-folding trick)
void launch_fill_col_bf16(bf16* p, int64_t rows, int64_t ld, int col, float v, cudaStream_t s);
void launch_f32_to_bf16(const float* in, bf16* out, int64_t n, cudaStream_t s);
// rows x cols fp32 (ld_in) -> bf16 (ld_out), zero-filling columns [cols, ld_out).
void launch_pad_rows_bf16(const float* in, int64_t ld_in, bf16* out, int64_t ld_out, int rows, int cols,
                          cudaStream_t s);

// ---- mixing + update (fp32 master weights, optional bf16 shadow) ----
// FM/RM: w_out = (w + w_l + w_r) * (1/3) - lr * g     (chronos.cpp:256, engine.cpp:166)
void launch_mix3(int64_t n, const float* w, const float* wl, const float* wr, const float* g, float lr, float* w_out,
                 bf16* shadow, cudaStream_t s);
// D1D: w_out[j] = (sum_i w[i]) / L - lr * g[j] for every local learner j (engine.cpp:173-184);
// w_sum != nullptr supplies a precomputed sum (allreduce result) instead of the w[] table.
void launch_d1d(int64_t n, int L, const float* const* w_tab, const float* w_sum, int nloc, const float* const* g_tab,
                float lr, float* const* out_tab, bf16* const* shadow_tab, cudaStream_t s);
// out = sum_i tab[i] in learner order (the local part of a multi-rank weight / gradient sum)
void launch_sum_tab(int64_t n, int L, const float* const* tab, float* out, cudaStream_t s);
// SDPSGD: w_out[j] = w - lr * (sum_i g[i]) / L (engine.cpp:145-153); g_sum as for d1d.
void launch_sdpsgd(int64_t n, int L, const float* w, const float* const* g_tab, const float* g_sum, int nloc,
                   float lr, float* const* out_tab, bf16* const* shadow_tab, cudaStream_t s);
// Generic dense mixing: out[j] = sum_i T[i*L + col_j] w[i] - lr * g[j] (engine.cpp:199).
void launch_dense_mix(int64_t n, int L, const float* const* w_tab, const double* T, const int* cols, int nloc,
                      const float* const* g_tab, float lr, float* const* out_tab, bf16* const* shadow_tab,
                      cudaStream_t s);
// Upper triangle of the Gram of deviations from the learner mean (fp64), L <= 16.
// Gram of the deviations from the learner mean (fp64 sums, deterministic: per-block partials in
// `partial` (>= gram_partial_doubles()) reduced in block order).
void launch_gram(int64_t n, int L, const float* const* w_tab, double* G, double* partial, cudaStream_t s);
size_t gram_partial_doubles();
// max_j max_p |w_j[p] - w_0[p]| -> out (float, atomicMax on bits)
void launch_maxdiff(int64_t n, const float* a, const float* b, float* out, cudaStream_t s);

// Device synthetic dataset (hash-based, deterministic in (seed, n, t, i)).
void launch_synth(float* feats, int32_t* labels, int n_seg, int T, int I, int C, uint64_t seed, cudaStream_t s);

// ---- free-running async FM / RM: versioned publication ring (engine.cu Ctx::async_step) ----
// Each learner's model version v lives in slot v % 4 of its ring; its counter block holds
// [0] = last published version (release-stored at system scope once the slot is complete) and
// [1] = version being written (announced before the slot's first byte is overwritten).
struct AsyncPeers {
    const unsigned long long* ver[2];  // left / right neighbour counter blocks (CUDA-IPC mapped)
    const float* slots[2][4];          // their publication rings
};
struct AsyncSel {
    const float* ptr[2];  // chosen neighbour versions' slots
    long long ver[2];     // chosen versions
    int torn;             // a neighbour began overwriting a chosen slot before the mix finished
    int err;              // wait timed out
    long long wait_ns;    // time spent waiting for neighbours
};
// select (1 thread): per neighbour, wait (mode LOCKSTEP: until version >= k; BOUNDED: >= k - lag;
// FREE: never) with ld.acquire.sys, choose the version (LOCKSTEP: k, else the latest), then
// announce this learner's write of version k + 1.
void launch_async_select(const AsyncPeers& pe, int mode, long long k, long long lag, unsigned long long* my_ver,
                         AsyncSel* sel, unsigned long long timeout_ns, cudaStream_t s);
// FM/RM mix against the selected slots: w_out = (w + w_L + w_R) / 3 - lr g (+ bf16 shadow).
void launch_mix3_sel(int64_t n, const float* w, const AsyncSel* sel, const float* g, float lr, float* w_out,
                     bf16* shadow, cudaStream_t s);
// publish (1 thread): torn-read check against the neighbours' write announcements, then a
// release store of version k + 1 (only if nothing was torn; the host then retries the mix).
void launch_async_publish(const AsyncPeers& pe, AsyncSel* sel, unsigned long long* my_ver, long long k,
                          cudaStream_t s);

// Device-side delay (straggler hook): spins for ns nanoseconds.
void launch_delay(uint64_t ns, cudaStream_t s);

}  // namespace ab
