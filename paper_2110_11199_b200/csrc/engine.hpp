// Device-resident learner context behind the C ABI (engine.cu, capi.cu).
#pragma once

#include "gemm.hpp"

#include <cuda_runtime.h>

#include <deque>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "adpsgd_b200.h"
#include "common.cuh"
#include "model.hpp"
#include "prof.hpp"
#include "rng.hpp"

namespace ab {

class Comm;

// engine.hpp:67-72 (LearnerState): model (fp32 master in a ring of nbuf versions + bf16 shadow),
// history (GENERIC), sampling stream.
struct Learner {
    int gid = 0;
    // version v of the model lives in w[v % nbuf]: nbuf = 2 (double buffer) for the synchronous
    // strategies, 4 for free-running async FM/RM (the publication ring, chronos.cpp:258-259)
    float* w[4] = {nullptr, nullptr, nullptr, nullptr};
    // publication counters, device memory exported over CUDA IPC: [0] = last published version,
    // [1] = version being written (its slot is being overwritten); async FM/RM only
    unsigned long long* ver = nullptr;
    float* g = nullptr;
    bf16* shadow = nullptr;          // bf16 copy of the current model (GEMM operand)
    std::vector<bf16*> l1pad;        // layer-1 W_ih per direction, rows padded for TMA
    std::vector<float*> hist;        // lags 1..depth-1 (ModelHistory, engine.cpp:79-97)
    Rng rng{0};
    double straggle = 1.0;
    float last_compute_ms = 0.f;
    double delay_ms = 0.0;       // fixed extra time per step (emulated compute, straggler studies)
    bool delay_on_host = false;  // ... as a host sleep (processes sharing one GPU) or a device spin
};

struct Ctx {
    explicit Ctx(const adpsgd_config& c);
    ~Ctx();

    adpsgd_config cfg;
    Layout lay;
    int64_t D = 0;
    bool bf16_mode = false;
    int es = 4;  // activation element size
    int T = 0, B = 0, H = 0, nd = 1, I = 0, Ipad = 0, ndH = 0, nd4H = 0;
    int64_t TB = 0;
    bool fold_bias = false;  // bf16 mode: bias grads via a ones column (no colsum passes)
    bool fold_ih_ok = true;  // ... also for the input-weight GEMMs (else a vectorised column sum of dZ)
    int ldH = 0, ldY = 0;     // row pitch of the layer outputs / projection output
    int64_t k = 0;
    int history_depth = 1;
    int nbuf = 2;  // model versions per learner (Learner::w)
    int slot(int64_t v) const { return static_cast<int>(v % nbuf); }

    cudaStream_t s_main = nullptr, s_comm = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_mix = nullptr, ev_comp0 = nullptr, ev_comp1 = nullptr;
    double last_step_ms = 0, last_mix_ms = 0, last_gossip_bytes = 0;
    double last_comm_start_ms = -1, last_comm_end_ms = -1, last_compute_end_ms = -1;

    // dataset (device)
    float* feats = nullptr;
    int32_t* labels = nullptr;
    int n_seg = 0, train_count = 0;

    // workspace
    int32_t* idx_dev = nullptr;
    int32_t* ident_idx = nullptr;
    void* X0 = nullptr;
    void* X0tail = nullptr;  // bf16 [16 x T*B]: K-major copy of X0 columns [256, 264) (tail-column dW_ih MMA)
    bf16* whh_t[2] = {nullptr, nullptr};  // W_hh^T of the layer in BPTT (32-unit persistent BPTT tiles)
    int32_t* lab_step = nullptr;
    std::vector<void*> Hout;
    std::vector<void*> gates;  // gate activations i,f,g,o (activation type)
    std::vector<float*> cst;
    void* Y = nullptr;
    void* dY = nullptr;
    float* logits = nullptr;       // fp32 mode only
    float2* ce_part = nullptr;      // bf16 mode: fused CE scratch
    float* ce_zlab = nullptr;
    float* ce_lse = nullptr;
    float* sk_scratch = nullptr;      // split-K BPTT partial exchange (gemm_lstm.cu)
    unsigned int* sk_flags = nullptr;
    unsigned int* pb_sync = nullptr;   // persistent recurrent kernels' counters (layout: gemm_lstm.hpp kPbSyncWords)
    GemmWorkspace gemm_ws;             // stream-K scratch of the generic tcgen05 GEMMs
    void* dlogits = nullptr;
    float* row_loss = nullptr;
    float *dHa = nullptr, *dHb = nullptr;
    void* dZ = nullptr;
    float* zstep = nullptr;
    float *dh_rec = nullptr, *dc_rec = nullptr;
    float* colsum_ws = nullptr;
    int64_t ws_elems = 0;
    float* loss_dev = nullptr;
    float* scratch_f = nullptr;
    void* scratch_grad = nullptr;
    float* scratch_w = nullptr;  // evaluate() / gradient() probe weights (never IPC-exported)
    float* stage_feats = nullptr;
    int32_t* stage_labels = nullptr;
    // host-batch prefetch (one local learner): two staging slots filled on s_copy while the
    // previous step computes; step_host_batch consumes the oldest slot whose pointers match
    float* stage_feats2 = nullptr;
    int32_t* stage_labels2 = nullptr;
    cudaStream_t s_copy = nullptr;
    cudaEvent_t ev_stage[2] = {nullptr, nullptr};
    struct Prefetch {
        const float* f;
        const int32_t* l;
        int slot;
    };
    std::deque<Prefetch> prefetched;
    int next_slot = 0;
    void prefetch_host_batch(const float* f, const int32_t* l);
    float* h_loss = nullptr;
    int32_t* h_idx = nullptr;  // pinned sampling slots, B per local learner

    struct StepGraph {
        cudaGraphExec_t exec = nullptr;
        std::vector<ProfRec> prof;
        int64_t launches = 0;
    };
    std::map<int, StepGraph> graphs;
    std::vector<const std::vector<ProfRec>*> replayed_prof;
    bool use_graphs = true;
    bool use_fused_cell = true;

    std::vector<Learner> learners;
    std::unique_ptr<Comm> comm;
    std::vector<void*> allocations;

    void* alloc(size_t bytes);
    void h2d_sync(void* dst, const void* src, size_t bytes);
    void* alloc_scratch_grad();
    void refresh_shadow(Learner& ln, const float* w, cudaStream_t s);
    void refresh_pad(Learner& ln, const float* w, cudaStream_t s);
    void gather_batch(const float* feats_src, const int32_t* labels_src, const int32_t* idx, cudaStream_t s);
    void sample_indices(Learner& ln, int j);
    void compute_body(int j, int mode, const float* wpt, cudaStream_t s);
    void run_compute(int j, int mode, const float* wpt, cudaStream_t s, int parity = -1);
    int64_t async_run(int strategy, const double* durations, int64_t target, int ipe, const double* lr_per_epoch,
                      int n_epochs, int32_t* ev_learner, double* ev_time, adpsgd_async_record* rec = nullptr);
    std::vector<float*> pubs;  // coupled-async publications, 4 per learner
    void clear_graphs();
    // Single learner (SGD, engine.cpp:245-247): the weight-gradient GEMM epilogues apply the update
    // w[nxt] = w[cur] - lr g and refresh the bf16 shadow in place (the gradient is never stored).
    struct FusedUpd {
        const float* w = nullptr;  // w[cur] (flat, like the gradient)
        float* o = nullptr;        // w[nxt]
        bf16* sh = nullptr;        // the learner's bf16 shadow (updated in place)
        const float* lr = nullptr; // device scalar
    };
    void forward_backward(const Learner& ln, const float* master, float* grad, float* loss_slot, cudaStream_t s,
                          bool backward = true, const FusedUpd* fu = nullptr);
    bool fused_update_ok() const;
    bool fuse_now = false;      // compute_body: apply the fused update in this compute
    bool fused_done = false;    // mix_and_update: this step's update already happened
    float* lr_dev = nullptr;
    float* h_lr = nullptr;      // pinned
    // restore: the model learner 0's bf16 shadow is rebuilt from afterwards (default: its current buffer)
    double evaluate(const double* w, const int32_t* idx, int M, double* g_out, const float* restore = nullptr);
    void averaged_model(double* out);
    double consensus_distance();
    void gram(const std::vector<const float*>& models, int64_t begin, int64_t end, double* out);
    bool observe_coupled(adpsgd_async_record& r, const std::vector<int>& par, int64_t processed, int ipe);
    void consensus_gram(int64_t begin, int64_t end, double* out);
    void averaged_model_all(double* out);
    double* gram_dev = nullptr;
    void mix_and_update(double lr, const int32_t* taus);
    const float* grad_point(const Learner& ln, const int32_t* taus);
    const float* weight_ptr(int gid, int buf) const;
    void neighbours(int strategy, int l, int* left, int* right) const;
    bool is_local(int gid) const;
    void check_sync();
    void step(double lr, const int32_t* taus, float* loss_out, const float* host_feats, const int32_t* host_labels,
              const double* injected);
    void step_compute(double lr, const int32_t* taus, const float* host_feats, const int32_t* host_labels,
                      const double* injected);
    void step_mix(double lr, const int32_t* taus);
    void step_finish(float* loss_out, bool injected);
    const float* grad_ptr(int gid) const;
    double gradient(const double* w, const int32_t* idx, int M, double* g_out);
    void gossip_probe(int left, int right, int reps, double* out4);
    // free-running async FM / RM across processes (engine.cu async_*)
    int async_mode = -1;  // -1 off; ADPSGD_ASYNC_FREE / _LOCKSTEP / _BOUNDED
    int64_t async_lag = 0;
    double async_timeout_s = 60.0;
    void* async_sel = nullptr;       // device selection record (AsyncSel, kernels.cuh)
    void* async_sel_host = nullptr;  // pinned mirror
    void async_init(int mode, int64_t max_lag, double timeout_s);
    void async_step(double lr, float* loss_out, adpsgd_async_info* info);
    void host_delay(const Learner& ln);
    double extra_delay_ms(const Learner& ln) const;
    bool ipc_exported = false;
    float* probe_buf[2] = {nullptr, nullptr};
    bf16* probe_shadow = nullptr;
};

double consensus_from_gram(const double* G, int L);
void set_last_error(const std::string& s);
const char* last_error();

}  // namespace ab
