// ADPSGD learner-step engine for B200: device-resident context, BLSTM forward/backward
// orchestration over the GEMM + pointwise kernels, and the mixing/update of every
// strategy (SDPSGD, FM, RM, D1D, GENERIC). Exposed through the C ABI in
// include/adpsgd_b200.h.
//
// Reference correspondence (per-iteration semantics):
//   step_sdpsgd         /root/reference/proj/src/engine.cpp:136-154
//   step_adpsgd_mixing  engine.cpp:156-171 (FM: fixed ring; RM: permutation of iteration k)
//   step_d1d            engine.cpp:173-184
//   step_generic        engine.cpp:186-204 (history ring, ModelHistory engine.cpp:79-97)
//   L == 1 -> SGD       engine.cpp:245-247
//   init_learners       engine.cpp:99-116; sampling objectives.cpp:239-249
#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <queue>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "engine.hpp"
#include "knobs.hpp"
#include "gemm.hpp"
#include "gemm_ce.hpp"
#include "gemm_lstm.hpp"
#include "kernels.cuh"
#include "prof.hpp"
#include "rng.hpp"

namespace ab {


namespace {
thread_local std::string g_last_error;

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

void set_last_error(const std::string& s) { g_last_error = s; }
const char* last_error() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// Device memory arena (one cudaMalloc per buffer; freed at ctx destroy).
// ---------------------------------------------------------------------------
// Host -> device copy ordered on s_main and complete on return. (A plain cudaMemcpy from pageable
// memory runs on the legacy stream, which the non-blocking s_main does not wait for, and may
// return before its DMA has landed: kernels on s_main could read the previous contents.)
void Ctx::h2d_sync(void* dst, const void* src, size_t bytes) {
    AB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s_main));
    AB_CUDA(cudaStreamSynchronize(s_main));
}

void* Ctx::alloc(size_t bytes) {
    void* p = nullptr;
    AB_CUDA(cudaMalloc(&p, round_up(bytes ? bytes : 16, 256)));
    if (knobs().poison_alloc >= 0) AB_CUDA(cudaMemset(p, knobs().poison_alloc & 0xFF, round_up(bytes ? bytes : 16, 256)));
    allocations.push_back(p);
    return p;
}

Ctx::~Ctx() {
    cudaSetDevice(cfg.device);
    cudaDeviceSynchronize();
    comm.reset();
    clear_graphs();
    for (void* p : allocations) cudaFree(p);
    for (auto& e : ev_stage)
        if (e) cudaEventDestroy(e);
    if (s_copy) cudaStreamDestroy(s_copy);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_mix) cudaEventDestroy(ev_mix);
    if (ev_comp0) cudaEventDestroy(ev_comp0);
    if (ev_comp1) cudaEventDestroy(ev_comp1);
    if (s_comm) cudaStreamDestroy(s_comm);
    if (s_main) cudaStreamDestroy(s_main);
    if (h_loss) cudaFreeHost(h_loss);
    if (h_idx) cudaFreeHost(h_idx);
    if (h_lr) cudaFreeHost(h_lr);
}

static void validate_config(const adpsgd_config& c) {
    const auto& m = c.model;
    AB_CHECK(m.layers >= 1 && m.hidden >= 1 && m.input_dim >= 1 && m.classes >= 2 && m.unroll >= 1 && m.proj >= 0,
             ADPSGD_E_CONFIG, "invalid model description");
    AB_CHECK(c.learners >= 1, ADPSGD_E_CONFIG, "learners must be >= 1");                       // engine.cpp:61
    AB_CHECK(!((c.strategy == ADPSGD_FM || c.strategy == ADPSGD_RM) && c.learners != 1 && c.learners < 3),
             ADPSGD_E_CONFIG, "FM/RM mixing requires at least 3 learners");                    // engine.cpp:62-65
    AB_CHECK(c.batch >= 1, ADPSGD_E_CONFIG, "batch must be >= 1");                             // engine.cpp:66
    AB_CHECK(c.staleness_cap >= 0, ADPSGD_E_CONFIG, "staleness_cap must be >= 0");             // engine.cpp:68
    AB_CHECK(c.strategy >= 0 && c.strategy <= 4, ADPSGD_E_CONFIG, "unknown strategy");
    AB_CHECK(c.local_learners >= 1 && c.first_learner >= 0 && c.first_learner + c.local_learners <= c.learners,
             ADPSGD_E_CONFIG, "local learner range outside [0, learners)");
    AB_CHECK(c.precision == ADPSGD_PREC_FP32 || c.precision == ADPSGD_PREC_BF16, ADPSGD_E_CONFIG, "bad precision");
    if (c.precision == ADPSGD_PREC_BF16) {
        AB_CHECK(m.hidden % 8 == 0 && m.classes % 8 == 0 && m.proj % 8 == 0, ADPSGD_E_CONFIG,
                 "bf16 tensor-core path needs hidden, classes and proj to be multiples of 8 (TMA pitch)");
    }
}

Ctx::Ctx(const adpsgd_config& c) : cfg(c) {
    validate_config(c);
    lay = make_layout(c.model);
    D = lay.total;
    bf16_mode = c.precision == ADPSGD_PREC_BF16;
    es = bf16_mode ? 2 : 4;
    T = lay.T; B = c.batch; H = lay.H; nd = lay.nd; I = lay.I;
    reload_knobs();  // tuning / experiment switches (knobs.hpp), re-read per context
    fold_bias = bf16_mode && knobs().fold_bias;  // bias grads from a ones column of the wgrad B operands
    fold_ih_ok = knobs().fold_ih;
    Ipad = bf16_mode ? static_cast<int>(round_up(I + (fold_bias ? 1 : 0), 8)) : I;
    ldH = nd * H + (fold_bias ? 8 : 0);
    ldY = lay.P > 0 ? (fold_bias ? lay.P + 8 : lay.P) : 0;
    if (knobs().pitch_align > 1) {  // row pitches in whole 128-byte lines: every TMA box row is one line (-2..3 % step)
        ldH = static_cast<int>(round_up(ldH, knobs().pitch_align));
        if (ldY) ldY = static_cast<int>(round_up(ldY, knobs().pitch_align));
    }
    TB = static_cast<int64_t>(T) * B;
    ndH = nd * H;
    nd4H = nd * 4 * H;
    k = 0;
    history_depth = c.strategy == ADPSGD_GENERIC ? c.staleness_cap + 1 : 1;  // engine.cpp:216-217
    use_graphs = knobs().graphs;
    use_fused_cell = knobs().fused_cell;

    AB_CUDA(cudaSetDevice(c.device));
    AB_CUDA(cudaStreamCreateWithFlags(&s_main, cudaStreamNonBlocking));
    AB_CUDA(cudaStreamCreateWithFlags(&s_comm, cudaStreamNonBlocking));
    AB_CUDA(cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking));
    for (auto& e : ev_stage) AB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    AB_CUDA(cudaEventCreate(&ev0));
    AB_CUDA(cudaEventCreate(&ev1));
    AB_CUDA(cudaEventCreate(&ev_mix));
    AB_CUDA(cudaEventCreate(&ev_comp0));
    AB_CUDA(cudaEventCreate(&ev_comp1));
    AB_CUDA(cudaMallocHost(&h_loss, sizeof(float) * 64));
    AB_CUDA(cudaMallocHost(&h_idx, sizeof(int32_t) * static_cast<size_t>(B) * c.local_learners));

    // ---- workspace (shared by the local learners; they are computed in turn) ----
    idx_dev = static_cast<int32_t*>(alloc(sizeof(int32_t) * B));
    X0 = alloc(TB * Ipad * es);
    if (bf16_mode && lstm_bwd_wants_whh_t(nd, B, H))
        for (auto& p : whh_t) p = static_cast<bf16*>(alloc(static_cast<size_t>(4) * H * H * sizeof(bf16)));
    if (bf16_mode && Ipad > 256 && Ipad <= 264) {
        X0tail = alloc(16 * TB * sizeof(bf16));
        AB_CUDA(cudaMemsetAsync(X0tail, 0, 16 * TB * sizeof(bf16), s_main));
    }
    lab_step = static_cast<int32_t*>(alloc(sizeof(int32_t) * TB));
    for (int l = 0; l < lay.L; ++l) {
        Hout.push_back(alloc(TB * ldH * es));
        gates.push_back(alloc(TB * nd4H * es));  // gate activations in the activation type
        cst.push_back(static_cast<float*>(alloc(TB * ndH * sizeof(float))));
    }
    if (lay.P > 0) {
        Y = alloc(TB * ldY * es);
        dY = alloc(TB * lay.P * es);
    }
    if (fold_bias) {
        for (int l = 0; l < lay.L; ++l) launch_fill_col_bf16(static_cast<bf16*>(Hout[l]), TB, ldH, ndH, 1.0f, s_main);
        if (lay.P > 0) launch_fill_col_bf16(static_cast<bf16*>(Y), TB, ldY, lay.P, 1.0f, s_main);
    }
    if (bf16_mode) {
        ce_part = static_cast<float2*>(alloc(ce_part_elems(static_cast<int>(TB), lay.C) * sizeof(float2)));
        ce_zlab = static_cast<float*>(alloc(TB * sizeof(float)));
        ce_lse = static_cast<float*>(alloc(TB * sizeof(float)));
        {   // stream-K scratch: (SMs / 2) pairs x 2 CTAs x (16 + 1) chunks x 128 rows x 32 fp32
            gemm_ws.floats = static_cast<size_t>(num_sms() / 2) * 2 * 17 * 128 * 32;
            gemm_ws.ws = static_cast<float*>(alloc(gemm_ws.floats * sizeof(float)));
            gemm_ws.flag_count = static_cast<size_t>(num_sms()) + 2 * 128;  // + split-K tile counters
            gemm_ws.flags = static_cast<unsigned int*>(alloc(gemm_ws.flag_count * sizeof(unsigned int)));
            AB_CUDA(cudaMemsetAsync(gemm_ws.flags, 0, gemm_ws.flag_count * sizeof(unsigned int), s_main));
        }
        if (H % 128 == 0) {  // split-K (H % 256) and persistent (H % 128) BPTT exchange buffers
            const int64_t slots = lstm_bwd_splitk_slots(nd, B, H);
            // per CTA slot: 2 parities x up to 4 K-split blocks x 32 KB (persistent BPTT, KQ <= 4)
            sk_scratch = static_cast<float*>(alloc(static_cast<size_t>(slots) * 4 * 128 * 128 * sizeof(float)));
            sk_flags = static_cast<unsigned int*>(alloc(static_cast<size_t>(slots) * sizeof(unsigned int)));
            AB_CUDA(cudaMemsetAsync(sk_flags, 0, static_cast<size_t>(slots) * sizeof(unsigned int), s_main));
            pb_sync = static_cast<unsigned int*>(alloc(kPbSyncWords * sizeof(unsigned int)));
            AB_CUDA(cudaMemsetAsync(pb_sync, 0, kPbSyncWords * sizeof(unsigned int), s_main));  // layout: gemm_lstm.hpp
        }
    }
    if (!bf16_mode || knobs().unfused_ce) logits = static_cast<float*>(alloc(TB * lay.C * sizeof(float)));
    dlogits = alloc(TB * lay.C * es);
    row_loss = static_cast<float*>(alloc(TB * sizeof(float)));
    int max_in = std::max(lay.top, Ipad);
    dHa = static_cast<float*>(alloc(TB * max_in * sizeof(float)));
    dHb = static_cast<float*>(alloc(TB * max_in * sizeof(float)));
    dZ = alloc(TB * nd4H * es);
    zstep = static_cast<float*>(alloc(static_cast<size_t>(nd) * B * 4 * H * sizeof(float)));
    dh_rec = static_cast<float*>(alloc(static_cast<size_t>(nd) * B * H * sizeof(float)));
    dc_rec = static_cast<float*>(alloc(static_cast<size_t>(nd) * B * H * sizeof(float)));
    ws_elems = std::max<int64_t>(int64_t(128) * std::max<int64_t>(nd4H, lay.C), 1 << 20);
    colsum_ws = static_cast<float*>(alloc(ws_elems * sizeof(float)));
    loss_dev = static_cast<float*>(alloc(sizeof(float) * 64));
    lr_dev = static_cast<float*>(alloc(sizeof(float) * 4));
    AB_CUDA(cudaMallocHost(&h_lr, sizeof(float) * 4));
    scratch_f = static_cast<float*>(alloc(sizeof(float) * 16));
    // staging for host batches (end-to-end path)
    stage_feats = static_cast<float*>(alloc(static_cast<size_t>(B) * T * I * sizeof(float)));
    stage_labels = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * T * sizeof(int32_t)));
    stage_feats2 = static_cast<float*>(alloc(static_cast<size_t>(B) * T * I * sizeof(float)));
    stage_labels2 = static_cast<int32_t*>(alloc(static_cast<size_t>(B) * T * sizeof(int32_t)));
    ident_idx = static_cast<int32_t*>(alloc(sizeof(int32_t) * B));
    {
        std::vector<int32_t> id(B);
        for (int b = 0; b < B; ++b) id[b] = b;
        h2d_sync(ident_idx, id.data(), sizeof(int32_t) * B);
    }

    // ---- learners: w0 shared by all (engine.cpp:101-103), streams 0xB000 + global id ----
    std::vector<double> w0(D);
    {
        Rng init(derive_seed(c.seed, kInitStream));
        for (int64_t i = 0; i < D; ++i) w0[i] = 0.1 * init.next_gaussian();
    }
    std::vector<float> w0f(w0.begin(), w0.end());
    for (int j = 0; j < c.local_learners; ++j) {
        Learner ln;
        ln.gid = c.first_learner + j;
        ln.rng = Rng(derive_seed(c.seed, kLearnerStream + static_cast<uint64_t>(ln.gid)));
        for (int b = 0; b < 2; ++b) ln.w[b] = static_cast<float*>(alloc(D * sizeof(float)));
        ln.ver = static_cast<unsigned long long*>(alloc(4 * sizeof(unsigned long long)));
        AB_CUDA(cudaMemsetAsync(ln.ver, 0, 4 * sizeof(unsigned long long), s_main));
        ln.g = static_cast<float*>(alloc(D * sizeof(float)));
        if (bf16_mode) {
            ln.shadow = static_cast<bf16*>(alloc(D * sizeof(bf16)));
            for (int d = 0; d < nd; ++d)
                ln.l1pad.push_back(static_cast<bf16*>(alloc(static_cast<size_t>(4) * H * Ipad * sizeof(bf16))));
        }
        for (int h = 1; h < history_depth; ++h) ln.hist.push_back(static_cast<float*>(alloc(D * sizeof(float))));
        h2d_sync(ln.w[0], w0f.data(), D * sizeof(float));
        learners.push_back(std::move(ln));
    }
    for (auto& ln : learners) {
        refresh_shadow(ln, ln.w[0], s_main);
        for (float* h : ln.hist) AB_CUDA(cudaMemcpyAsync(h, ln.w[0], D * sizeof(float), cudaMemcpyDeviceToDevice, s_main));
    }
    AB_CUDA(cudaStreamSynchronize(s_main));
}

// bf16 shadow of the master weights + TMA-aligned padded copy of layer-1 W_ih.
void Ctx::refresh_shadow(Learner& ln, const float* w, cudaStream_t s) {
    if (!bf16_mode) return;
    launch_f32_to_bf16(w, ln.shadow, D, s);
    refresh_pad(ln, w, s);
}
void Ctx::refresh_pad(Learner& ln, const float* w, cudaStream_t s) {
    if (!bf16_mode) return;
    for (int d = 0; d < nd; ++d)
        launch_pad_rows_bf16(w + lay.dir[0][d].w_ih, I, ln.l1pad[d], Ipad, 4 * H, I, s);
}

// Weight views used as GEMM operands for a given master vector / shadow.
struct WView {
    const void* base;   // bf16 shadow (bf16 mode) or fp32 master
    const float* master;
    const Ctx* c;
    const Learner* ln;
    const void* at(int64_t off) const {
        return static_cast<const uint8_t*>(base) + off * c->es;
    }
    // layer-1 W_ih: padded bf16 copy in bf16 mode (ld = Ipad), flat in fp32 mode (ld = I)
    const void* wih(int l, int d, int64_t* ld) const {
        if (l == 0 && c->bf16_mode) { *ld = c->Ipad; return ln->l1pad[d]; }
        *ld = c->lay.in_dim[l];
        return at(c->lay.dir[l][d].w_ih);
    }
};

static inline const void* off_ptr(const void* p, int64_t elems, int es) {
    return static_cast<const uint8_t*>(p) + elems * es;
}
static inline void* off_ptr(void* p, int64_t elems, int es) { return static_cast<uint8_t*>(p) + elems * es; }

// Forward + backward of the BLSTM on the batch already gathered into X0 / lab_step.
// grad (fp32, flat layout) receives d(mean CE)/dw; loss_slot receives the mean CE.
void Ctx::forward_backward(const Learner& ln, const float* master, float* grad, float* loss_slot, cudaStream_t s,
                           bool backward, const FusedUpd* fu) {
    GemmWorkspaceScope ws_scope(gemm_ws);
    const bool bf = bf16_mode;
    WView W{bf ? static_cast<const void*>(ln.shadow) : static_cast<const void*>(master), master, this, &ln};
    const int G4 = 4 * H;
    const bool fused = bf && use_fused_cell && H % 64 == 0;

    // ---------------- forward ----------------
    for (int l = 0; l < lay.L; ++l) {
        const void* Xin = l == 0 ? X0 : Hout[l - 1];
        const int Kin = l == 0 ? Ipad : ndH;
        const int ldx = l == 0 ? Ipad : ldH;
        if (fused) {
            LstmFwdLayer FL;
            FL.x = static_cast<const bf16*>(Xin); FL.ldx = ldx; FL.Kx = Kin;
            for (int d = 0; d < nd; ++d) {
                int64_t ldw;
                FL.w_ih[d] = static_cast<const bf16*>(W.wih(l, d, &ldw));
                FL.ld_wih = ldw;
                FL.w_hh[d] = static_cast<const bf16*>(W.at(lay.dir[l][d].w_hh));
                FL.bias[d] = master + lay.dir[l][d].b;
            }
            FL.gates = static_cast<bf16*>(gates[l]); FL.ldg = nd4H;
            FL.c = cst[l]; FL.ldc = ndH;
            FL.h = static_cast<bf16*>(Hout[l]); FL.ldh = ldH;
            const bool persistent = pb_sync && lstm_fwd_layer_persistent(FL, nd, B, H, T, s, pb_sync + 512 - kFwdDepSlots, pb_sync + 513);
            for (int st = 0; !persistent && st < T; ++st) {
                LstmFwdDir dirs[2];
                for (int d = 0; d < nd; ++d) {
                    const int t = d == 0 ? st : T - 1 - st;
                    const int tp = d == 0 ? t - 1 : t + 1;
                    int64_t ldw;
                    LstmFwdDir& a = dirs[d];
                    a.x = static_cast<const bf16*>(off_ptr(Xin, static_cast<int64_t>(t) * B * ldx, es));
                    a.ldx = ldx;
                    a.Kx = Kin;
                    a.w_ih = static_cast<const bf16*>(W.wih(l, d, &ldw));
                    a.ld_wih = ldw;
                    a.h_prev = st > 0 ? static_cast<const bf16*>(off_ptr(Hout[l], static_cast<int64_t>(tp) * B * ldH + d * H, es)) : nullptr;
                    a.ld_hprev = ldH;
                    a.w_hh = static_cast<const bf16*>(W.at(lay.dir[l][d].w_hh));
                    a.bias = master + lay.dir[l][d].b;
                    a.c_prev = st > 0 ? cst[l] + static_cast<int64_t>(tp) * B * ndH + d * H : nullptr;
                    a.gates = static_cast<bf16*>(off_ptr(gates[l], static_cast<int64_t>(t) * B * nd4H + d * G4, es));
                    a.c = cst[l] + static_cast<int64_t>(t) * B * ndH + d * H;
                    a.h = static_cast<bf16*>(off_ptr(Hout[l], static_cast<int64_t>(t) * B * ldH + d * H, es));
                }
                lstm_fwd_step(dirs, nd, B, H, nd4H, ndH, ldH, s);
            }
            continue;
        }
        for (int st = 0; st < T; ++st) {
            for (int d = 0; d < nd; ++d) {
                const int t = d == 0 ? st : T - 1 - st;
                const int tp = d == 0 ? t - 1 : t + 1;
                GemmArgs g;
                g.M = B; g.N = G4;
                int64_t ldw;
                const void* wih = W.wih(l, d, &ldw);
                g.seg[0].a = {off_ptr(Xin, static_cast<int64_t>(t) * B * ldx, es), ldx, false};
                g.seg[0].b = {wih, ldw, false};
                g.seg[0].K = Kin;
                g.nseg = 1;
                if (st > 0) {
                    g.seg[1].a = {off_ptr(Hout[l], static_cast<int64_t>(tp) * B * ldH + d * H, es), ldH, false};
                    g.seg[1].b = {W.at(lay.dir[l][d].w_hh), H, false};
                    g.seg[1].K = H;
                    g.nseg = 2;
                }
                g.C = zstep + static_cast<int64_t>(d) * B * G4;
                g.tag = PROF_GEMM_REC_FWD;
                g.ldc = G4;
                g.bias = master + lay.dir[l][d].b;
                gemm(bf, g, s);
                const float* cprev = st > 0 ? cst[l] + static_cast<int64_t>(tp) * B * ndH + d * H : nullptr;
                void* gt = off_ptr(gates[l], static_cast<int64_t>(t) * B * nd4H + d * G4, es);
                float* ct = cst[l] + static_cast<int64_t>(t) * B * ndH + d * H;
                void* ht = off_ptr(Hout[l], static_cast<int64_t>(t) * B * ldH + d * H, es);
                if (bf)
                    launch_cell_fwd<bf16>(zstep + static_cast<int64_t>(d) * B * G4, G4, cprev, ndH, static_cast<bf16*>(gt), nd4H, ct,
                                          static_cast<bf16*>(ht), ldH, B, H, s);
                else
                    launch_cell_fwd<float>(zstep + static_cast<int64_t>(d) * B * G4, G4, cprev, ndH, static_cast<float*>(gt), nd4H, ct,
                                           static_cast<float*>(ht), ldH, B, H, s);
            }
        }
    }
    const void* top = Hout[lay.L - 1];
    const void* yin = top;
    const int oi = lay.out_in;
    const int ld_yin = lay.P > 0 ? ldY : ldH;
    if (lay.P > 0) {
        GemmArgs g;
        g.M = static_cast<int>(TB); g.N = lay.P;
        g.seg[0].a = {top, ldH, false};
        g.seg[0].b = {W.at(lay.w_proj), ndH, false};
        g.seg[0].K = ndH;
        g.C = Y; g.ldc = ldY; g.c_bf16 = bf;
        g.bias = master + lay.b_proj;
        g.tag = PROF_GEMM_OUT;
        gemm(bf, g, s);
        yin = Y;
    }
    const float scale = 1.0f / static_cast<float>(TB);
    if (bf && !knobs().unfused_ce) {
        // output GEMM fused with softmax-CE: no logits in HBM (gemm_ce.cu)
        CeArgs a;
        a.Y = static_cast<const bf16*>(yin);
        a.W = static_cast<const bf16*>(W.at(lay.w_out));
        a.bias = master + lay.b_out;
        a.labels = lab_step;
        a.M = static_cast<int>(TB); a.N = lay.C; a.K = oi; a.ldY = ld_yin;
        a.scale = scale;
        a.part = ce_part; a.zlab = ce_zlab; a.lse = ce_lse;
        a.row_loss = row_loss;
        a.dlogits = static_cast<bf16*>(dlogits);
        ce_forward_backward(a, s);
    } else {
        GemmArgs g;
        g.M = static_cast<int>(TB); g.N = lay.C;
        g.seg[0].a = {yin, ld_yin, false};
        g.seg[0].b = {W.at(lay.w_out), oi, false};
        g.seg[0].K = oi;
        g.C = logits; g.ldc = lay.C;
        g.bias = master + lay.b_out;
        g.tag = PROF_GEMM_OUT;
        gemm(bf, g, s);
        if (bf)
            launch_softmax_ce<bf16>(logits, lab_step, static_cast<int>(TB), lay.C, scale, static_cast<bf16*>(dlogits),
                                    row_loss, s);
        else
            launch_softmax_ce<float>(logits, lab_step, static_cast<int>(TB), lay.C, scale, static_cast<float*>(dlogits),
                                     row_loss, s);
    }
    launch_sum(row_loss, static_cast<int>(TB), scale, loss_slot, s);
    if (!backward) return;

    // ---------------- backward: output / projection ----------------
    auto colsum = [&](const void* X, int64_t ld, int R, int N, float* out) {
        if (bf) launch_colsum<bf16>(static_cast<const bf16*>(X), ld, R, N, out, colsum_ws, ws_elems, s);
        else launch_colsum<float>(static_cast<const float*>(X), ld, R, N, out, colsum_ws, ws_elems, s);
    };
    // fused SGD update: the weight-gradient GEMMs write w[nxt] and the shadow instead of the gradient
    auto upd = [&](GemmArgs& g) {
        if (!fu) return;
        const int64_t off = static_cast<float*>(g.C) - grad;
        g.upd_w = fu->w + off; g.upd_o = fu->o + off; g.upd_sh = fu->sh + off; g.upd_lr = fu->lr;
        if (g.extra) {
            const int64_t ox = g.extra - grad;
            g.upd_xw = fu->w + ox; g.upd_xo = fu->o + ox; g.upd_xsh = fu->sh + ox;
        }
    };
    // order: every GEMM that reads a weight's shadow runs before that weight's gradient GEMM (which,
    // fused, overwrites the shadow): dY before dW_out, dTop before dW_proj, dX before dW_ih / dW_hh
    auto dw_out = [&] {  // dW_out = dlogits^T Yin
        GemmArgs g;
        g.M = lay.C; g.N = oi + (fold_bias ? 1 : 0);
        g.seg[0].a = {dlogits, lay.C, true};
        g.seg[0].b = {yin, ld_yin, true};
        g.seg[0].K = static_cast<int>(TB);
        g.C = grad + lay.w_out; g.ldc = oi;
        if (fold_bias) { g.n_main = oi; g.extra = grad + lay.b_out; }  // ones column of Y -> db_out
        g.tag = PROF_GEMM_WGRAD;
        upd(g);
        gemm(bf, g, s);
        if (!fold_bias) colsum(dlogits, lay.C, static_cast<int>(TB), lay.C, grad + lay.b_out);
    };
    float* dHcur = dHa;
    float* dHnext = dHb;
    if (!fu) dw_out();
    if (lay.P > 0) {
        {   // dY = dlogits W_out  (bf16/fp32 activation type: it is a GEMM operand next)
            GemmArgs g;
            g.M = static_cast<int>(TB); g.N = lay.P;
            g.seg[0].a = {dlogits, lay.C, false};
            g.seg[0].b = {W.at(lay.w_out), lay.P, true};
            g.seg[0].K = lay.C;
            g.C = dY; g.ldc = lay.P; g.c_bf16 = bf;
            g.tag = PROF_GEMM_DGRAD_X;
            gemm(bf, g, s);
        }
        if (fu) dw_out();
        auto dtop = [&] {  // dTop = dY W_proj
            GemmArgs g;
            g.M = static_cast<int>(TB); g.N = ndH;
            g.seg[0].a = {dY, lay.P, false};
            g.seg[0].b = {W.at(lay.w_proj), ndH, true};
            g.seg[0].K = lay.P;
            g.C = dHcur; g.ldc = ndH;
            g.tag = PROF_GEMM_DGRAD_X;
            gemm(bf, g, s);
        };
        if (fu) dtop();
        {   // dW_proj = dY^T top
            GemmArgs g;
            g.M = lay.P; g.N = ndH + (fold_bias ? 1 : 0);
            g.seg[0].a = {dY, lay.P, true};
            g.seg[0].b = {top, ldH, true};
            g.seg[0].K = static_cast<int>(TB);
            g.C = grad + lay.w_proj; g.ldc = ndH;
            if (fold_bias) { g.n_main = ndH; g.extra = grad + lay.b_proj; }  // ones column of the top layer -> db_proj
            g.tag = PROF_GEMM_WGRAD;
            upd(g);
            gemm(bf, g, s);
        }
        if (!fold_bias) colsum(dY, lay.P, static_cast<int>(TB), lay.P, grad + lay.b_proj);
        if (!fu) dtop();
    } else {
        GemmArgs g;
        g.M = static_cast<int>(TB); g.N = ndH;
        g.seg[0].a = {dlogits, lay.C, false};
        g.seg[0].b = {W.at(lay.w_out), ndH, true};
        g.seg[0].K = lay.C;
        g.C = dHcur; g.ldc = ndH;
        g.tag = PROF_GEMM_DGRAD_X;
        gemm(bf, g, s);
        if (fu) dw_out();
    }

    // ---------------- backward: LSTM layers (BPTT) ----------------
    for (int l = lay.L - 1; l >= 0; --l) {
        const void* Xin = l == 0 ? X0 : Hout[l - 1];
        const int Kin = l == 0 ? Ipad : ndH;
        const int ldx = l == 0 ? Ipad : ldH;
        if (fused) {
            // BPTT: first cell backward unfused (no recurrent term), then one launch per step
            // doing dh_rec = dz_t W_hh for both directions with the next cell backward fused.
            const float* f_dh[2]; const bf16* f_g[2]; const float* f_c[2]; const float* f_cp[2]; bf16* f_dz[2]; float* f_dc[2];
            for (int d = 0; d < nd; ++d) {
                const int t = d == 0 ? T - 1 : 0;
                const int tp = d == 0 ? t - 1 : t + 1;
                f_dh[d] = dHcur + static_cast<int64_t>(t) * B * ndH + d * H;
                f_g[d] = static_cast<const bf16*>(off_ptr(gates[l], static_cast<int64_t>(t) * B * nd4H + d * G4, es));
                f_c[d] = cst[l] + static_cast<int64_t>(t) * B * ndH + d * H;
                f_cp[d] = T > 1 ? cst[l] + static_cast<int64_t>(tp) * B * ndH + d * H : nullptr;
                f_dz[d] = static_cast<bf16*>(off_ptr(dZ, static_cast<int64_t>(t) * B * nd4H + d * G4, es));
                f_dc[d] = dc_rec + static_cast<int64_t>(d) * B * H;
            }
            const bool first2 = nd == 2 && launch_cell_bwd_first2(f_dh, f_g, f_c, f_cp, f_dz, f_dc, ndH, nd4H, ndH, nd4H, B, H, s);
            for (int d = 0; d < nd && !first2; ++d) {
                const int t = d == 0 ? T - 1 : 0;
                const int tp = d == 0 ? t - 1 : t + 1;
                const float* cp = T > 1 ? cst[l] + static_cast<int64_t>(tp) * B * ndH + d * H : nullptr;
                launch_cell_bwd<bf16>(dHcur + static_cast<int64_t>(t) * B * ndH + d * H, ndH, nullptr,
                                      dc_rec + static_cast<int64_t>(d) * B * H, true,
                                      static_cast<const bf16*>(off_ptr(gates[l], static_cast<int64_t>(t) * B * nd4H + d * G4, es)), nd4H,
                                      cst[l] + static_cast<int64_t>(t) * B * ndH + d * H, cp, ndH,
                                      static_cast<bf16*>(off_ptr(dZ, static_cast<int64_t>(t) * B * nd4H + d * G4, es)),
                                      nd4H, B, H, s);
            }
            LstmBwdLayer PL;
            PL.dZ = static_cast<bf16*>(dZ); PL.ld_dz = nd4H;
            for (int d = 0; d < nd; ++d) {
                PL.w_hh[d] = static_cast<const bf16*>(W.at(lay.dir[l][d].w_hh));
                PL.dc_rec[d] = dc_rec + static_cast<int64_t>(d) * B * H;
                if (whh_t[d] && (knobs().bwd_u32 || knobs().bwd_kmajor)) {  // K-major copy for the BPTT B operand
                    launch_transpose_bf16(PL.w_hh[d], whh_t[d], G4, H, s);
                    PL.w_hh_t[d] = whh_t[d];
                }
            }
            PL.dH = dHcur; PL.lddh = ndH;
            PL.gates = static_cast<const bf16*>(gates[l]); PL.ldg = nd4H;
            PL.c = cst[l]; PL.ldc = ndH;
            const bool persistent = pb_sync && sk_scratch &&
                                    lstm_bwd_layer_persistent(PL, nd, B, H, T, s, sk_scratch, pb_sync, pb_sync + 512 - kBwdDepSlots, pb_sync + 512);
            for (int st = 0; !persistent && st + 1 < T; ++st) {
                LstmBwdDir dirs[2];
                for (int d = 0; d < nd; ++d) {
                    const int sf = T - 1 - st, sn = sf - 1;
                    const int t = d == 0 ? sf : T - 1 - sf;
                    const int tn = d == 0 ? sn : T - 1 - sn;
                    const int tnp = d == 0 ? tn - 1 : tn + 1;
                    LstmBwdDir& a = dirs[d];
                    a.dz_src = static_cast<const bf16*>(off_ptr(dZ, static_cast<int64_t>(t) * B * nd4H + d * G4, es));
                    a.ld_dz_src = nd4H;
                    a.w_hh = static_cast<const bf16*>(W.at(lay.dir[l][d].w_hh));
                    a.dH = dHcur + static_cast<int64_t>(tn) * B * ndH + d * H;
                    a.dc_rec = dc_rec + static_cast<int64_t>(d) * B * H;
                    a.gates = static_cast<const bf16*>(off_ptr(gates[l], static_cast<int64_t>(tn) * B * nd4H + d * G4, es));
                    a.c = cst[l] + static_cast<int64_t>(tn) * B * ndH + d * H;
                    a.c_prev = sn > 0 ? cst[l] + static_cast<int64_t>(tnp) * B * ndH + d * H : nullptr;
                    a.dz_dst = static_cast<bf16*>(off_ptr(dZ, static_cast<int64_t>(tn) * B * nd4H + d * G4, es));
                }
                lstm_bwd_step(dirs, nd, B, H, ndH, nd4H, ndH, nd4H, s, sk_scratch, sk_flags);
            }
        } else
        for (int st = 0; st < T; ++st) {
            const int sf = T - 1 - st;  // forward-order step index of this time
            for (int d = 0; d < nd; ++d) {
                const int t = d == 0 ? sf : T - 1 - sf;
                const int tp = d == 0 ? t - 1 : t + 1;
                float* dhr = dh_rec + static_cast<int64_t>(d) * B * H;
                float* dcr = dc_rec + static_cast<int64_t>(d) * B * H;
                const void* gt = off_ptr(gates[l], static_cast<int64_t>(t) * B * nd4H + d * G4, es);
                const float* ct = cst[l] + static_cast<int64_t>(t) * B * ndH + d * H;
                const float* cp = sf > 0 ? cst[l] + static_cast<int64_t>(tp) * B * ndH + d * H : nullptr;
                void* dzt = off_ptr(dZ, static_cast<int64_t>(t) * B * nd4H + d * G4, es);
                const float* dHt = dHcur + static_cast<int64_t>(t) * B * ndH + d * H;
                if (bf)
                    launch_cell_bwd<bf16>(dHt, ndH, dhr, dcr, st == 0, static_cast<const bf16*>(gt), nd4H, ct, cp, ndH, static_cast<bf16*>(dzt),
                                          nd4H, B, H, s);
                else
                    launch_cell_bwd<float>(dHt, ndH, dhr, dcr, st == 0, static_cast<const float*>(gt), nd4H, ct, cp, ndH,
                                           static_cast<float*>(dzt), nd4H, B, H, s);
                if (sf > 0) {  // dh_{prev} = dz_t W_hh
                    GemmArgs g;
                    g.M = B; g.N = H;
                    g.seg[0].a = {dzt, nd4H, false};
                    g.seg[0].b = {W.at(lay.dir[l][d].w_hh), H, true};
                    g.seg[0].K = G4;
                    g.C = dhr; g.ldc = H;
                    g.tag = PROF_GEMM_REC_BWD;
                    gemm(bf, g, s);
                }
            }
        }
        auto dgrad_x = [&] {
        if (l > 0) {  // dXin = sum_d dZ_d W_ih_d
                GemmArgs g;
                g.M = static_cast<int>(TB); g.N = Kin;
                for (int d = 0; d < nd; ++d) {
                    int64_t ldw;
                    const void* wih = W.wih(l, d, &ldw);
                    g.seg[d].a = {off_ptr(dZ, d * G4, es), nd4H, false};
                    g.seg[d].b = {wih, ldw, true};
                    g.seg[d].K = G4;
                }
                g.nseg = nd;
                g.C = dHnext; g.ldc = Kin;
                g.tag = PROF_GEMM_DGRAD_X;
                gemm(bf, g, s);
                std::swap(dHcur, dHnext);
            }
        };
        auto wgrads = [&] {
        for (int d = 0; d < nd; ++d) {
                const DirOff& o = lay.dir[l][d];
                // one-wave 256 x 512 tiles for dW_ih (the bias then by a column sum of dZ) when the
                // 256-wide tiles plus the ones column would need a second wave (gemm_wgrad_wide)
                const bool fold_ih = fold_bias && fold_ih_ok && !gemm_wgrad_wide(G4, lay.in_dim[l]);
                {   // dW_ih = dZ_d^T Xin
                    GemmArgs g;
                    g.M = G4; g.N = lay.in_dim[l] + (fold_ih ? 1 : 0);
                    g.seg[0].a = {off_ptr(dZ, d * G4, es), nd4H, true};
                    g.seg[0].b = {Xin, ldx, true};
                    g.seg[0].K = static_cast<int>(TB);
                    g.C = grad + o.w_ih; g.ldc = lay.in_dim[l];
                    if (fold_ih) { g.n_main = lay.in_dim[l]; g.extra = grad + o.b; }  // ones column of the input -> db
                    if (fold_ih && l == 0 && X0tail) { g.b_tail = X0tail; g.ld_tail = TB; }  // features 256.. + ones column
                    g.tag = PROF_GEMM_WGRAD;
                    upd(g);
                    gemm(bf, g, s);
                }
                if (T > 1) {  // dW_hh = sum_t dz_t^T h_prev(t)
                    GemmArgs g;
                    g.M = G4; g.N = H;
                    const int64_t a_row0 = d == 0 ? B : 0;
                    const int64_t b_row0 = d == 0 ? 0 : B;
                    g.seg[0].a = {off_ptr(dZ, a_row0 * nd4H + d * G4, es), nd4H, true};
                    g.seg[0].b = {off_ptr(Hout[l], b_row0 * ldH + d * H, es), ldH, true};
                    g.seg[0].K = static_cast<int>((T - 1) * static_cast<int64_t>(B));
                    g.C = grad + o.w_hh; g.ldc = H;
                    g.tag = PROF_GEMM_WGRAD;
                    upd(g);
                    gemm(bf, g, s);
                } else {
                    AB_CUDA(cudaMemsetAsync(grad + o.w_hh, 0, sizeof(float) * G4 * H, s));
                }
                if (!fold_ih) colsum(off_ptr(dZ, d * G4, es), nd4H, static_cast<int>(TB), G4, grad + o.b);
            }
        };
        // fused update: this layer's W_ih shadow is read by dX before its update (see upd)
        if (fu) { dgrad_x(); wgrads(); } else { wgrads(); dgrad_x(); }
    }
}

void Ctx::gather_batch(const float* feats_src, const int32_t* labels_src, const int32_t* idx, cudaStream_t s) {
    if (bf16_mode)
        launch_gather<bf16>(feats_src, labels_src, idx, B, T, I, Ipad, static_cast<bf16*>(X0), lab_step, s, fold_bias,
                            static_cast<bf16*>(X0tail), 256);
    else
        launch_gather<float>(feats_src, labels_src, idx, B, T, I, Ipad, static_cast<float*>(X0), lab_step, s, false);
}

// Host-side sampling of learner j's batch: M draws next_below(train_count)
// (objectives.cpp:239-249) from its own stream into learner j's pinned slot.
void Ctx::sample_indices(Learner& ln, int j) {
    AB_CHECK(feats != nullptr && train_count >= 1, ADPSGD_E_INVALID_STATE, "dataset has no training samples");
    int32_t* hb = h_idx + static_cast<int64_t>(j) * B;
    for (int b = 0; b < B; ++b) hb[b] = static_cast<int32_t>(ln.rng.next_below(static_cast<uint64_t>(train_count)));
}

// The update folds into the weight-gradient GEMM epilogues when this context is the only
// learner (every strategy is SGD, engine.cpp:245-247) and every gradient block comes from a
// tcgen05 GEMM (bf16 mode, bias gradients folded into the GEMMs, T > 1).
bool Ctx::fused_update_ok() const {
    if (!(knobs().fused_update && bf16_mode && cfg.learners == 1 && cfg.local_learners == 1 && !(comm && comm->multi())))
        return false;
    if (!fold_bias || !fold_ih_ok || T < 2) return false;
    for (int l = 0; l < lay.L; ++l)
        if (gemm_wgrad_wide(4 * H, lay.in_dim[l])) return false;  // its bias would come from a column sum
    return true;
}

// Queue the H2D copy of a host batch (layout of step_host_batch, one local learner) on the copy
// stream; the next step_host_batch with the same pointers waits on it instead of copying. The
// caller keeps the host memory unchanged until that step (pinned memory makes the copy async).
void Ctx::prefetch_host_batch(const float* f, const int32_t* l) {
    AB_CHECK(f && l, ADPSGD_E_INVALID_STATE, "null host batch");
    AB_CHECK(cfg.local_learners == 1, ADPSGD_E_CONFIG, "host-batch prefetch needs one local learner per context");
    AB_CHECK(prefetched.size() < 2, ADPSGD_E_INVALID_STATE, "at most two prefetched host batches in flight");
    AB_CUDA(cudaSetDevice(cfg.device));
    const int slot = next_slot;
    next_slot ^= 1;
    const size_t nf = static_cast<size_t>(B) * T * I;
    AB_CUDA(cudaMemcpyAsync(slot ? stage_feats2 : stage_feats, f, nf * sizeof(float), cudaMemcpyHostToDevice, s_copy));
    AB_CUDA(cudaMemcpyAsync(slot ? stage_labels2 : stage_labels, l, sizeof(int32_t) * B * T, cudaMemcpyHostToDevice, s_copy));
    AB_CUDA(cudaEventRecord(ev_stage[slot], s_copy));
    prefetched.push_back({f, l, slot});
}

// The learner's gradient computation as one replayable unit: batch upload + gather +
// BLSTM forward/backward. mode 0 = indices from the pinned slot into the device dataset,
// mode 1 / 2 = batch already staged in staging slot 0 / 1.
void Ctx::compute_body(int j, int mode, const float* wpt, cudaStream_t s) {
    Learner& ln = learners[j];
    if (mode == 0) {
        AB_CUDA(cudaMemcpyAsync(idx_dev, h_idx + static_cast<int64_t>(j) * B, sizeof(int32_t) * B,
                                cudaMemcpyHostToDevice, s));
        gather_batch(feats, labels, idx_dev, s);
    } else if (mode == 1) {
        gather_batch(stage_feats, stage_labels, ident_idx, s);
    } else {
        gather_batch(stage_feats2, stage_labels2, ident_idx, s);
    }
    if (fuse_now) {
        FusedUpd fu;
        fu.w = ln.w[slot(k)]; fu.o = ln.w[slot(k + 1)]; fu.sh = ln.shadow; fu.lr = lr_dev;
        forward_backward(ln, wpt, ln.g, loss_dev + j, s, true, &fu);
    } else {
        forward_backward(ln, wpt, ln.g, loss_dev + j, s);
    }
}

// Runs compute_body through a CUDA graph keyed by (learner, weight parity, mode, profiling):
// the first encounter runs eagerly (warms plan caches / attributes), the second captures,
// later ones replay — ~1000 launches per learner step become one graph launch.
void Ctx::run_compute(int j, int mode, const float* wpt, cudaStream_t s, int parity) {
    Learner& ln = learners[j];
    if (parity < 0) parity = slot(k);
    const bool lagged = wpt != ln.w[parity];
    if (lagged || !use_graphs) {
        compute_body(j, mode, wpt, s);
        return;
    }
    const int key = (((j * 4 + parity) * 3 + mode) * 2 + (g_prof_enabled ? 1 : 0)) * 2 + (fuse_now ? 1 : 0);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
        StepGraph sg;
        graphs.emplace(key, std::move(sg));
        compute_body(j, mode, wpt, s);  // eager warm-up run
        return;
    }
    StepGraph& sg = it->second;
    if (!sg.exec) {
        const int64_t launches0 = g_launch_count;
        std::vector<ProfRec>* prev = g_prof_capture;
        if (g_prof_enabled) g_prof_capture = &sg.prof;
        AB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            compute_body(j, mode, wpt, s);
        } catch (...) {
            cudaGraph_t gtmp;
            cudaStreamEndCapture(s, &gtmp);
            if (gtmp) cudaGraphDestroy(gtmp);
            g_prof_capture = prev;
            throw;
        }
        cudaGraph_t graph;
        AB_CUDA(cudaStreamEndCapture(s, &graph));
        g_prof_capture = prev;
        AB_CUDA(cudaGraphInstantiate(&sg.exec, graph, 0));
        AB_CUDA(cudaGraphDestroy(graph));
        sg.launches = g_launch_count - launches0;
        g_launch_count = launches0;
    }
    AB_CUDA(cudaGraphLaunch(sg.exec, s));
    g_launch_count += sg.launches;
    if (!sg.prof.empty()) replayed_prof.push_back(&sg.prof);
}

// chronos::coupled_async (chronos.cpp:178-299) on the device: learners iterate at their own
// rates (duration_l), each update averages the learner's model with its neighbours' latest
// publications strictly before its update time (chronos.cpp:171-176) — w <- (w + pl + pr)/3 -
// lr g (chronos.cpp:256) — and publishes the result (4 kept per learner, chronos.cpp:258-259).
// The event order is the reference's min-heap order; gradients, mixing and publication run on
// the GPU in that order. Returns the number of updates applied.
int64_t Ctx::async_run(int strategy, const double* durations, int64_t target, int ipe, const double* lr_per_epoch,
                       int n_epochs, int32_t* ev_learner, double* ev_time, adpsgd_async_record* rec) {
    AB_CHECK(strategy == ADPSGD_FM || strategy == ADPSGD_RM, ADPSGD_E_CONFIG, "coupled async runs FM or RM");
    AB_CHECK(!(comm && comm->multi()) && cfg.local_learners == cfg.learners, ADPSGD_E_CONFIG,
             "coupled async: every learner hosted by this context");
    const int L = cfg.learners;
    AB_CHECK(L >= 3, ADPSGD_E_CONFIG, "FM/RM mixing requires at least 3 learners");
    AB_CHECK(ipe >= 1 && n_epochs >= 1, ADPSGD_E_CONFIG, "ipe and lr table must be non-empty");
    AB_CHECK(feats != nullptr && train_count >= 1, ADPSGD_E_INVALID_STATE, "dataset has no training samples");
    AB_CUDA(cudaSetDevice(cfg.device));
    cudaStream_t s = s_main;
    constexpr int kPubs = 4;
    if (pubs.empty())
        for (int l = 0; l < L; ++l)
            for (int q = 0; q < kPubs; ++q) pubs.push_back(static_cast<float*>(alloc(D * sizeof(float))));
    struct Pub { double t; int slot; };
    std::vector<std::vector<Pub>> pl(L);  // oldest first
    AB_CHECK(nbuf == 2, ADPSGD_E_CONFIG, "coupled async replay runs on the double-buffered (synchronous) context");
    std::vector<int> par(L, slot(k));
    for (int l = 0; l < L; ++l) {
        AB_CUDA(cudaMemcpyAsync(pubs[l * kPubs], learners[l].w[par[l]], D * sizeof(float), cudaMemcpyDeviceToDevice, s));
        pl[l].push_back({0.0, 0});
    }
    using Entry = std::pair<double, int>;
    std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> q;
    std::vector<int64_t> round(L, 0);
    for (int l = 0; l < L; ++l) q.push({durations[l], l});
    auto before = [&](int l, double t) -> const float* {  // chronos.cpp:171-176
        for (auto it = pl[l].rbegin(); it != pl[l].rend(); ++it)
            if (it->t < t) return pubs[l * kPubs + it->slot];
        return pubs[l * kPubs + pl[l].front().slot];
    };
    int64_t processed = 0;
    std::vector<int32_t> map(L);
    while (processed < target) {
        const auto [t_done, l] = q.top();
        q.pop();
        Learner& ln = learners[l];
        const int64_t r = round[l];
        // lr_at(cfg.lr, r / ipe) of the learner's own round (chronos.cpp:216): no clamp -- a fast
        // learner can run past cfg.epochs x ipe rounds, so the caller sizes the table for `target`
        const int64_t ep = r / ipe;
        AB_CHECK(ep < n_epochs, ADPSGD_E_CONFIG,
                 "lr table covers " + std::to_string(n_epochs) + " epochs, round " + std::to_string(r) + " needs epoch " +
                     std::to_string(ep));
        const float lr = static_cast<float>(lr_per_epoch[ep]);
        AB_CUDA(cudaStreamSynchronize(s));  // pinned sampling slot reuse
        sample_indices(ln, l);
        run_compute(l, 0, ln.w[par[l]], s, par[l]);
        int left, right;
        if (strategy == ADPSGD_FM) {
            left = (l + L - 1) % L;
            right = (l + 1) % L;
        } else {
            permutation_for_iteration(cfg.seed, L, r, map.data());
            int pos = 0;
            for (int i = 0; i < L; ++i) if (map[i] == l) { pos = i; break; }
            left = map[(pos + L - 1) % L];
            right = map[(pos + 1) % L];
        }
        const int nxt = par[l] ^ 1;
        launch_mix3(D, ln.w[par[l]], before(left, t_done), before(right, t_done), ln.g, lr, ln.w[nxt],
                    bf16_mode ? ln.shadow : nullptr, s);
        refresh_pad(ln, ln.w[nxt], s);
        par[l] = nxt;
        // publish (keep 4): reuse the oldest slot
        int slot;
        if (static_cast<int>(pl[l].size()) < kPubs) {
            slot = static_cast<int>(pl[l].size());
        } else {
            slot = pl[l].front().slot;
            pl[l].erase(pl[l].begin());
        }
        AB_CUDA(cudaMemcpyAsync(pubs[l * kPubs + slot], ln.w[nxt], D * sizeof(float), cudaMemcpyDeviceToDevice, s));
        pl[l].push_back({t_done, slot});
        if (ev_learner) ev_learner[processed] = l;
        if (ev_time) ev_time[processed] = t_done;
        ++round[l];
        ++processed;
        q.push({t_done + durations[l], l});
        if (rec && observe_coupled(*rec, par, processed, ipe)) break;  // diverged
    }
    // leave every model in the context's current buffer
    for (int l = 0; l < L; ++l) {
        Learner& ln = learners[l];
        const int cur = slot(k);
        if (par[l] != cur) {
            AB_CUDA(cudaMemcpyAsync(ln.w[cur], ln.w[par[l]], D * sizeof(float), cudaMemcpyDeviceToDevice, s));
            refresh_shadow(ln, ln.w[cur], s);
        }
    }
    AB_CUDA(cudaStreamSynchronize(s));
    for (auto* recs : replayed_prof) prof_accumulate(*recs);
    replayed_prof.clear();
    return processed;
}

void Ctx::clear_graphs() {
    for (auto& kv : graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
}

// ---------------------------------------------------------------------------
// The iteration (engine.cpp:245-283)
// ---------------------------------------------------------------------------
void Ctx::mix_and_update(double lr_d, const int32_t* taus) {
    const float lr = static_cast<float>(lr_d);
    const int cur = slot(k), nxt = slot(k + 1);
    const int Lg = cfg.learners;
    const int nloc = cfg.local_learners;
    std::vector<const float*> wtab, gtab;
    std::vector<float*> otab;
    std::vector<bf16*> stab;
    for (auto& ln : learners) {
        gtab.push_back(ln.g);
        otab.push_back(ln.w[nxt]);
        stab.push_back(bf16_mode ? ln.shadow : nullptr);
    }
    cudaStream_t s = s_main;
    int strategy = cfg.strategy;
    if (Lg == 1) strategy = ADPSGD_SDPSGD;  // engine.cpp:245-247
    last_gossip_bytes = 0;

    if (fused_done) {
        // the weight-gradient GEMMs already wrote w[nxt] = w[cur] - lr g and the shadow
    } else if (strategy == ADPSGD_SDPSGD) {
        if (comm && comm->local_group) {
            // single-process group: every learner's gradient read in place (NVLink peer loads), in
            // learner order, once the other contexts' gradient computes have finished
            for (Ctx* o : comm->group_ctxs)
                if (o != this) AB_CUDA(cudaStreamWaitEvent(s, o->ev_mix, 0));
            std::vector<const float*> gall;
            for (int gid = 0; gid < Lg; ++gid) gall.push_back(grad_ptr(gid));
            launch_sdpsgd(D, Lg, learners[0].w[cur], gall.data(), nullptr, nloc, lr, otab.data(), stab.data(), s);
        } else if (comm && comm->multi()) {
            // gradient allreduce (sum over ranks of the local sums), then the shared update
            const float* gsum = comm->allreduce_sum_grads(*this, s);
            launch_sdpsgd(D, Lg, learners[0].w[cur], nullptr, gsum, nloc, lr, otab.data(), stab.data(), s);
        } else {
            launch_sdpsgd(D, Lg, learners[0].w[cur], gtab.data(), nullptr, nloc, lr, otab.data(), stab.data(), s);
        }
    } else if (strategy == ADPSGD_D1D) {
        if (comm && comm->multi() && comm->ipc_only) {
            // CUDA-IPC-only transport: the mean reads every learner's w_k directly (learner order,
            // as the local path); w_k is final because the caller separates steps on the host
            for (int gid = 0; gid < Lg; ++gid) wtab.push_back(weight_ptr(gid, cur));
            launch_d1d(D, Lg, wtab.data(), nullptr, nloc, gtab.data(), lr, otab.data(), stab.data(), s);
        } else if (comm && comm->multi()) {
            const float* wsum = comm->wait_weight_sum(*this, s);  // allreduce started before the compute
            launch_d1d(D, Lg, nullptr, wsum, nloc, gtab.data(), lr, otab.data(), stab.data(), s);
        } else {
            for (auto& ln : learners) wtab.push_back(ln.w[cur]);
            launch_d1d(D, Lg, wtab.data(), nullptr, nloc, gtab.data(), lr, otab.data(), stab.data(), s);
        }
    } else if (strategy == ADPSGD_FM || strategy == ADPSGD_RM) {
        const int mode = (comm && comm->multi()) ? comm->gossip_mode : 0;
        if (comm && comm->multi() && mode == 0) comm->pre_gossip(*this, s);
        for (int j = 0; j < nloc; ++j) {
            int left, right;
            neighbours(strategy, learners[j].gid, &left, &right);
            const float* wl = weight_ptr(left, cur);
            const float* wr = weight_ptr(right, cur);
            if (mode == 1) {  // pulled by the copy engines while the gradient was computed
                AB_CUDA(cudaStreamWaitEvent(s, comm->nb_ready, 0));
                wl = comm->nb_left(); wr = comm->nb_right();
            } else if (mode == 2) {  // NCCL send / recv baseline
                comm->sendrecv_neighbours(*this, j, left, right, s);
                wl = comm->nb_left(); wr = comm->nb_right();
            }
            if (!is_local(left)) last_gossip_bytes += D * 4.0;
            if (!is_local(right)) last_gossip_bytes += D * 4.0;
            launch_mix3(D, learners[j].w[cur], wl, wr, learners[j].g, lr, learners[j].w[nxt], stab[j], s);
        }
    } else {  // GENERIC: W T - lr G(tau-lagged), engine.cpp:186-204
        AB_CHECK(!(comm && comm->multi()), ADPSGD_E_CONFIG, "GENERIC staleness is single-process only");
        std::vector<double> Tm(static_cast<size_t>(Lg) * Lg, 0.0);
        const int kind = cfg.generic_mix;
        if (kind == ADPSGD_MIX_UNIFORM) {
            AB_CHECK(Lg >= 2, ADPSGD_E_INVALID_ORDER, "uniform mixing requires order >= 2");
            std::fill(Tm.begin(), Tm.end(), 1.0 / Lg);
        } else {
            AB_CHECK(Lg >= 3, ADPSGD_E_INVALID_ORDER, "ring mixing requires order >= 3");
            std::vector<double> f(static_cast<size_t>(Lg) * Lg, 0.0);
            for (int i = 0; i < Lg; ++i) {
                f[i * Lg + i] += 1.0 / 3.0;
                f[i * Lg + (i + 1) % Lg] += 1.0 / 3.0;
                f[i * Lg + (i + Lg - 1) % Lg] += 1.0 / 3.0;
            }
            if (kind == ADPSGD_MIX_FIXED) {
                Tm = f;
            } else {
                std::vector<int32_t> map(Lg);
                permutation_for_iteration(cfg.seed, Lg, k, map.data());
                for (int a = 0; a < Lg; ++a)
                    for (int b = 0; b < Lg; ++b) Tm[map[a] * Lg + map[b]] += f[a * Lg + b];
            }
        }
        for (auto& ln : learners) wtab.push_back(ln.w[cur]);
        std::vector<int> cols;
        for (auto& ln : learners) cols.push_back(ln.gid);
        launch_dense_mix(D, Lg, wtab.data(), Tm.data(), cols.data(), nloc, gtab.data(), lr, otab.data(), stab.data(), s);
        (void)taus;
    }
    if (bf16_mode)
        for (auto& ln : learners) refresh_pad(ln, ln.w[nxt], s);
    // ModelHistory push (engine.cpp:85-88): keep depth-1 older models for GENERIC.
    if (history_depth > 1) {
        for (auto& ln : learners) {
            // rotate: hist[0] <- w[cur] (the model before this update)
            float* oldest = ln.hist.back();
            for (size_t h = ln.hist.size() - 1; h > 0; --h) ln.hist[h] = ln.hist[h - 1];
            ln.hist[0] = oldest;
            AB_CUDA(cudaMemcpyAsync(oldest, ln.w[cur], D * sizeof(float), cudaMemcpyDeviceToDevice, s));
        }
    }
}

// Ring neighbours of global learner l at the current iteration: FM l-1 / l+1, RM from the
// seeded permutation of iteration k (chronos.cpp:227-235).
void Ctx::neighbours(int strategy, int l, int* left, int* right) const {
    const int Lg = cfg.learners;
    if (strategy == ADPSGD_FM) {
        *left = (l + Lg - 1) % Lg;
        *right = (l + 1) % Lg;
        return;
    }
    std::vector<int32_t> map(Lg);
    permutation_for_iteration(cfg.seed, Lg, k, map.data());
    int pos = 0;
    for (int i = 0; i < Lg; ++i) if (map[i] == l) { pos = i; break; }
    *left = map[(pos + Lg - 1) % Lg];
    *right = map[(pos + 1) % Lg];
}

const float* Ctx::weight_ptr(int gid, int buf) const {
    const int j = gid - cfg.first_learner;
    if (j >= 0 && j < cfg.local_learners) return learners[j].w[buf];
    AB_CHECK(comm != nullptr, ADPSGD_E_INVALID_STATE, "neighbour weights not mapped (call adpsgd_import_ipc)");
    return comm->peer_weight(gid, buf);
}
const float* Ctx::grad_ptr(int gid) const {
    const int j = gid - cfg.first_learner;
    if (j >= 0 && j < cfg.local_learners) return learners[j].g;
    AB_CHECK(comm != nullptr, ADPSGD_E_INVALID_STATE, "neighbour gradients not mapped");
    return comm->peer_grad(gid);
}
bool Ctx::is_local(int gid) const {
    return gid >= cfg.first_learner && gid < cfg.first_learner + cfg.local_learners;
}

// Model each learner evaluates its gradient at: its own model (FM/RM/D1D), the shared
// model (SDPSGD; identical on every learner), or the tau-lagged model (GENERIC).
const float* Ctx::grad_point(const Learner& ln, const int32_t* taus) {
    const int cur = slot(k);
    if (cfg.strategy == ADPSGD_GENERIC && cfg.learners > 1 && taus) {
        const int tau = taus[ln.gid];
        AB_CHECK(tau >= 0 && tau < history_depth, ADPSGD_E_STALENESS_OVERFLOW,
                 "staleness " + std::to_string(tau) + " exceeds history depth " + std::to_string(history_depth));
        if (tau > 0) return ln.hist[tau - 1];
    }
    return ln.w[cur];
}

void Ctx::check_sync() {
    // engine.cpp:139-144 — models must agree within 1e-12 before an SDPSGD step
    // (local learners; identical fp32 arithmetic keeps them bit-identical).
    const bool group = comm && comm->local_group && cfg.first_learner != 0;
    if (cfg.local_learners < 2 && !group) return;
    const int cur = slot(k);
    AB_CUDA(cudaMemsetAsync(scratch_f, 0, sizeof(float), s_main));
    for (int j = 1; j < cfg.local_learners; ++j) launch_maxdiff(D, learners[j].w[cur], learners[0].w[cur], scratch_f, s_main);
    if (group) launch_maxdiff(D, learners[0].w[cur], weight_ptr(0, cur), scratch_f, s_main);  // vs global learner 0
    float h = 0;
    AB_CUDA(cudaMemcpyAsync(&h, scratch_f, sizeof(float), cudaMemcpyDeviceToHost, s_main));
    AB_CUDA(cudaStreamSynchronize(s_main));
    AB_CHECK(!(h > 1e-12f), ADPSGD_E_SYNC_VIOLATION, "learner desynchronized before SDPSGD step");
}

void Ctx::step(double lr, const int32_t* taus, float* loss_out, const float* host_feats, const int32_t* host_labels,
               const double* injected) {
    step_compute(lr, taus, host_feats, host_labels, injected);
    step_mix(lr, taus);
    step_finish(loss_out, injected != nullptr);
}

// Phase 1 of an iteration: sampling, comm-stream starts, every local learner's gradient (graph
// replays) on s_main; returns without waiting (ev_mix marks the gradients done).
void Ctx::step_compute(double lr, const int32_t* taus, const float* host_feats, const int32_t* host_labels,
                       const double* injected) {
    AB_CUDA(cudaSetDevice(cfg.device));
    const int strategy = cfg.learners == 1 ? ADPSGD_SDPSGD : cfg.strategy;
    if (strategy == ADPSGD_SDPSGD) check_sync();
    if (strategy == ADPSGD_GENERIC && taus) {
        for (int l = 0; l < cfg.learners; ++l)
            AB_CHECK(taus[l] >= 0 && taus[l] < history_depth, ADPSGD_E_STALENESS_OVERFLOW,
                     "staleness " + std::to_string(taus[l]) + " exceeds history depth " + std::to_string(history_depth));
    }
    cudaStream_t s = s_main;
    if (!injected && !host_feats)
        for (int j = 0; j < cfg.local_learners; ++j) sample_indices(learners[j], j);
    // single learner: the update happens inside the gradient GEMMs (lr via a device scalar, so
    // the captured graph serves every step)
    fuse_now = !injected && fused_update_ok() && !(strategy == ADPSGD_GENERIC && taus && taus[0] > 0);
    fused_done = false;
    if (fuse_now) {
        *h_lr = static_cast<float>(lr);
        AB_CUDA(cudaMemcpyAsync(lr_dev, h_lr, sizeof(float), cudaMemcpyHostToDevice, s));
    }
    AB_CUDA(cudaEventRecord(ev0, s));
    // D1D: start the weight allreduce on the comm stream before the gradient compute
    if (strategy == ADPSGD_D1D && comm && comm->multi() && !comm->ipc_only) comm->start_weight_sum(*this, s);
    // FM / RM, gossip mode 1: the neighbours' w_k travel by copy engine while this learner computes
    if ((strategy == ADPSGD_FM || strategy == ADPSGD_RM) && comm && comm->multi() && comm->gossip_mode == 1) {
        AB_CHECK(cfg.local_learners == 1, ADPSGD_E_CONFIG, "gossip mode 1 (copy-engine prefetch) hosts one learner per rank");
        int left, right;
        neighbours(strategy, learners[0].gid, &left, &right);
        comm->prefetch_neighbours(*this, weight_ptr(left, slot(k)), weight_ptr(right, slot(k)), s);
    }
    for (int j = 0; j < cfg.local_learners; ++j) {
        Learner& ln = learners[j];
        if (injected) {
            std::vector<float> gf(injected + j * D, injected + (j + 1) * D);
            AB_CUDA(cudaMemcpyAsync(ln.g, gf.data(), D * sizeof(float), cudaMemcpyHostToDevice, s));
            AB_CUDA(cudaStreamSynchronize(s));
            continue;
        }
        int mode = 0;
        if (host_feats && !prefetched.empty() && cfg.local_learners == 1 && prefetched.front().f == host_feats &&
            prefetched.front().l == host_labels) {
            // staged by prefetch_host_batch while the previous step ran
            const int slot = prefetched.front().slot;
            prefetched.pop_front();
            AB_CUDA(cudaStreamWaitEvent(s, ev_stage[slot], 0));
            mode = 1 + slot;
        } else if (host_feats) {
            if (!prefetched.empty()) {  // a different batch than the one prefetched: drop the prefetches
                AB_CUDA(cudaStreamSynchronize(s_copy));
                prefetched.clear();
            }
            const size_t nf = static_cast<size_t>(B) * T * I;
            AB_CUDA(cudaMemcpyAsync(stage_feats, host_feats + j * nf, nf * sizeof(float), cudaMemcpyHostToDevice, s));
            AB_CUDA(cudaMemcpyAsync(stage_labels, host_labels + static_cast<size_t>(j) * B * T,
                                    sizeof(int32_t) * B * T, cudaMemcpyHostToDevice, s));
            mode = 1;
        }
        const float* wpt = grad_point(ln, taus);
        const bool lagged = wpt != ln.w[slot(k)];
        if (bf16_mode && lagged) refresh_shadow(ln, wpt, s);  // GENERIC: shadow of the lagged model
        const bool stretch = ln.straggle > 1.0 || ln.delay_ms > 0;
        if (stretch) AB_CUDA(cudaEventRecord(ev_comp0, s));
        run_compute(j, mode, wpt, s);
        if (stretch) {
            AB_CUDA(cudaEventRecord(ev_comp1, s));
            // emulated compute (delay_ms) plus the straggler's (factor - 1) x its last measured compute
            if (!ln.delay_on_host && extra_delay_ms(ln) > 0)
                launch_delay(static_cast<uint64_t>(extra_delay_ms(ln) * 1e6), s);
        }
        if (bf16_mode && lagged) refresh_shadow(ln, ln.w[slot(k)], s);
    }
    AB_CUDA(cudaEventRecord(ev_mix, s));
}

// Phase 2: the mixing + update of cfg.strategy (engine.cpp:136-204).
void Ctx::step_mix(double lr, const int32_t* taus) {
    AB_CUDA(cudaSetDevice(cfg.device));
    fused_done = fuse_now;
    fuse_now = false;
    mix_and_update(lr, taus);
    fused_done = false;
    AB_CUDA(cudaEventRecord(ev1, s_main));
}

// Phase 3: join, losses to the host, step statistics, host-side delays; k -> k + 1.
void Ctx::step_finish(float* loss_out, bool injected) {
    AB_CUDA(cudaSetDevice(cfg.device));
    cudaStream_t s = s_main;
    if (!injected && loss_out) {
        AB_CUDA(cudaMemcpyAsync(h_loss, loss_dev, sizeof(float) * cfg.local_learners, cudaMemcpyDeviceToHost, s));
    }
    AB_CUDA(cudaStreamSynchronize(s));
    for (auto* recs : replayed_prof) prof_accumulate(*recs);
    replayed_prof.clear();
    if (!injected && loss_out) std::memcpy(loss_out, h_loss, sizeof(float) * cfg.local_learners);
    float ms = 0, mms = 0;
    AB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    AB_CUDA(cudaEventElapsedTime(&mms, ev_mix, ev1));
    last_step_ms = ms;
    last_mix_ms = mms;
    last_compute_end_ms = ms - mms;
    last_comm_start_ms = last_comm_end_ms = -1;
    if (comm && comm->ar_pending) {  // the D1D weight allreduce on the comm stream (overlap evidence)
        float a = 0, b = 0;
        AB_CUDA(cudaEventElapsedTime(&a, ev0, comm->t_ar0));
        AB_CUDA(cudaEventElapsedTime(&b, ev0, comm->t_ar1));
        last_comm_start_ms = a;
        last_comm_end_ms = b;
        comm->ar_pending = false;
    }
    for (auto& ln : learners) {
        if (ln.straggle > 1.0 || ln.delay_ms > 0) {
            float cm = 0;
            if (cudaEventElapsedTime(&cm, ev_comp0, ev_comp1) == cudaSuccess) ln.last_compute_ms = cm;
        }
    }
    for (auto& ln : learners) host_delay(ln);
    ++k;
}

// Straggler hook (chronos.cpp:51-58): a learner's compute is stretched to factor x (measured
// compute + emulated compute); the emulated part alone for factor 1.
double Ctx::extra_delay_ms(const Learner& ln) const {
    const double measured = ln.last_compute_ms;  // events around the gradient compute only
    return ln.delay_ms + (ln.straggle - 1.0) * (measured + ln.delay_ms);
}

void Ctx::host_delay(const Learner& ln) {
    if (!ln.delay_on_host) return;
    const double ms = extra_delay_ms(ln);
    if (ms > 0) std::this_thread::sleep_for(std::chrono::microseconds(static_cast<int64_t>(ms * 1000.0)));
}

// ---------------------------------------------------------------------------
// Free-running asynchronous FM / RM across processes (chronos.cpp:171-176, 178-299 on real clocks)
// ---------------------------------------------------------------------------
void Ctx::async_init(int mode, int64_t max_lag, double timeout_s) {
    AB_CHECK(mode >= ADPSGD_ASYNC_FREE && mode <= ADPSGD_ASYNC_BOUNDED, ADPSGD_E_CONFIG, "unknown async mode");
    AB_CHECK(max_lag >= 0 && timeout_s > 0, ADPSGD_E_CONFIG, "async: max_lag >= 0 and timeout > 0 required");
    AB_CHECK(cfg.strategy == ADPSGD_FM || cfg.strategy == ADPSGD_RM, ADPSGD_E_CONFIG, "async runs FM or RM");
    AB_CHECK(cfg.learners >= 3, ADPSGD_E_CONFIG, "FM/RM mixing requires at least 3 learners");
    AB_CHECK(cfg.local_learners == 1, ADPSGD_E_CONFIG, "async: one learner per context (process)");
    AB_CHECK(!ipc_exported, ADPSGD_E_INVALID_STATE, "async: call adpsgd_async_init before adpsgd_export_ipc");
    AB_CUDA(cudaSetDevice(cfg.device));
    AB_CUDA(cudaStreamSynchronize(s_main));
    Learner& ln = learners[0];
    if (nbuf == 2) {
        const int old = slot(k);
        ln.w[2] = static_cast<float*>(alloc(D * sizeof(float)));
        ln.w[3] = static_cast<float*>(alloc(D * sizeof(float)));
        nbuf = 4;
        if (slot(k) != old)
            AB_CUDA(cudaMemcpyAsync(ln.w[slot(k)], ln.w[old], D * sizeof(float), cudaMemcpyDeviceToDevice, s_main));
        clear_graphs();  // graphs are keyed by slot
    }
    const unsigned long long v[2] = {static_cast<unsigned long long>(k), static_cast<unsigned long long>(k)};
    h2d_sync(ln.ver, v, sizeof(v));
    if (!async_sel) {
        async_sel = alloc(sizeof(AsyncSel));
        AB_CUDA(cudaMallocHost(&async_sel_host, sizeof(AsyncSel)));
    }
    async_mode = mode;
    async_lag = max_lag;
    async_timeout_s = timeout_s;
}

void Ctx::async_step(double lr_d, float* loss_out, adpsgd_async_info* info) {
    AB_CHECK(async_mode >= 0, ADPSGD_E_INVALID_STATE, "async: call adpsgd_async_init first");
    AB_CHECK(comm != nullptr, ADPSGD_E_INVALID_STATE, "async: neighbours not mapped (adpsgd_comm_init / import_ipc)");
    AB_CUDA(cudaSetDevice(cfg.device));
    cudaStream_t s = s_main;
    Learner& ln = learners[0];
    const int cur = slot(k), nxt = slot(k + 1);
    const float lr = static_cast<float>(lr_d);
    sample_indices(ln, 0);
    AB_CUDA(cudaEventRecord(ev0, s));
    const bool stretch = ln.straggle > 1.0 || ln.delay_ms > 0;
    if (stretch) AB_CUDA(cudaEventRecord(ev_comp0, s));
    run_compute(0, 0, ln.w[cur], s, cur);
    if (stretch) {
        AB_CUDA(cudaEventRecord(ev_comp1, s));
        if (!ln.delay_on_host && extra_delay_ms(ln) > 0) launch_delay(static_cast<uint64_t>(extra_delay_ms(ln) * 1e6), s);
    }
    AB_CUDA(cudaEventRecord(ev_mix, s));
    int nb[2];
    neighbours(cfg.strategy, ln.gid, &nb[0], &nb[1]);  // RM: permutation of the learner's own round k
    AsyncPeers pe;
    for (int side = 0; side < 2; ++side) {
        AB_CHECK(!is_local(nb[side]), ADPSGD_E_INVALID_STATE, "async: neighbours live in other processes");
        pe.ver[side] = comm->peer_ver(nb[side]);
        for (int q = 0; q < 4; ++q) pe.slots[side][q] = comm->peer_weight(nb[side], q);
    }
    AsyncSel* sel = static_cast<AsyncSel*>(async_sel);
    AsyncSel* hsel = static_cast<AsyncSel*>(async_sel_host);
    const auto timeout_ns = static_cast<unsigned long long>(async_timeout_s * 1e9);
    int retries = 0;
    for (;;) {
        launch_async_select(pe, async_mode, k, async_lag, ln.ver, sel, timeout_ns, s);
        launch_mix3_sel(D, ln.w[cur], sel, ln.g, lr, ln.w[nxt], bf16_mode ? ln.shadow : nullptr, s);
        if (retries == 0 && knobs().async_hold_ms > 0)  // tests: widen the read window of the first attempt
            launch_delay(static_cast<uint64_t>(knobs().async_hold_ms) * 1000000ull, s);
        launch_async_publish(pe, sel, ln.ver, k, s);
        AB_CUDA(cudaMemcpyAsync(hsel, sel, sizeof(AsyncSel), cudaMemcpyDeviceToHost, s));
        AB_CUDA(cudaStreamSynchronize(s));
        AB_CHECK(!hsel->err, ADPSGD_E_INVALID_STATE,
                 "async: timed out waiting for neighbour versions (learner " + std::to_string(ln.gid) + ", round " +
                     std::to_string(k) + ")");
        if (!hsel->torn) break;
        AB_CHECK(++retries < 1000, ADPSGD_E_INVALID_STATE, "async: neighbour slots overwritten on every retry");
    }
    refresh_pad(ln, ln.w[nxt], s);
    AB_CUDA(cudaEventRecord(ev1, s));
    if (loss_out) AB_CUDA(cudaMemcpyAsync(h_loss, loss_dev, sizeof(float), cudaMemcpyDeviceToHost, s));
    AB_CUDA(cudaStreamSynchronize(s));
    for (auto* recs : replayed_prof) prof_accumulate(*recs);
    replayed_prof.clear();
    if (loss_out) *loss_out = h_loss[0];
    float ms = 0, mms = 0;
    AB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    AB_CUDA(cudaEventElapsedTime(&mms, ev_mix, ev1));
    last_step_ms = ms;
    last_mix_ms = mms;
    last_gossip_bytes = 8.0 * D * (retries + 1);
    if (stretch) {
        float cm = 0;
        if (cudaEventElapsedTime(&cm, ev_comp0, ev_comp1) == cudaSuccess) ln.last_compute_ms = cm;
    }
    if (info) {
        info->version = k + 1;
        info->left_version = hsel->ver[0];
        info->right_version = hsel->ver[1];
        info->left = nb[0];
        info->right = nb[1];
        info->retries = retries;
        info->reserved = 0;
        info->wait_ms = hsel->wait_ns * 1e-6;
        info->step_ms = ms;
    }
    host_delay(ln);
    ++k;
}

double Ctx::gradient(const double* w, const int32_t* idx, int M, double* g_out) {
    return evaluate(w, idx, M, g_out);
}

// Loss (and, if g_out != nullptr, gradient) at w over the given segments, chunked by the
// context batch B (the last chunk wraps); the mean is over all frames (objectives.cpp:144-157).
double Ctx::evaluate(const double* w, const int32_t* idx, int M, double* g_out, const float* restore) {
    AB_CHECK(!g_out || M == B, ADPSGD_E_DIMENSION, "gradient(): M must equal the context batch");
    AB_CHECK(M >= 1, ADPSGD_E_INVALID_STATE, "batch size must be >= 1");
    AB_CHECK(feats != nullptr, ADPSGD_E_INVALID_STATE, "dataset has no training samples");
    AB_CUDA(cudaSetDevice(cfg.device));
    cudaStream_t s = s_main;
    Learner& ln = learners[0];
    // evaluate at w in a private scratch buffer (w[nxt] is exported over CUDA IPC: a peer may still
    // be reading it); the learner's bf16 shadow is restored after
    if (!scratch_w) scratch_w = static_cast<float*>(alloc(D * sizeof(float)));
    std::vector<float> wf(w, w + D);
    AB_CUDA(cudaMemcpyAsync(scratch_w, wf.data(), D * sizeof(float), cudaMemcpyHostToDevice, s));
    AB_CUDA(cudaStreamSynchronize(s));  // wf is pageable and goes out of scope
    refresh_shadow(ln, scratch_w, s);
    double result = 0.0;
    if (g_out) {
        AB_CUDA(cudaMemcpyAsync(idx_dev, idx, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
        gather_batch(feats, labels, idx_dev, s);
        float* gtmp = static_cast<float*>(alloc_scratch_grad());
        forward_backward(ln, scratch_w, gtmp, loss_dev + 63, s, true);
        std::vector<float> gh(D);
        float lh = 0;
        AB_CUDA(cudaMemcpyAsync(gh.data(), gtmp, D * sizeof(float), cudaMemcpyDeviceToHost, s));
        AB_CUDA(cudaMemcpyAsync(&lh, loss_dev + 63, sizeof(float), cudaMemcpyDeviceToHost, s));
        AB_CUDA(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < D; ++i) g_out[i] = gh[i];
        result = lh;
    } else {
        // loss only, in chunks of B segments; the padded tail of the last chunk is masked out
        double total = 0.0;
        std::vector<int32_t> chunk(B);
        for (int start = 0; start < M; start += B) {
            const int valid = std::min(B, M - start);
            for (int b = 0; b < B; ++b) chunk[b] = idx[start + (b < valid ? b : 0)];
            AB_CUDA(cudaMemcpyAsync(idx_dev, chunk.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
            gather_batch(feats, labels, idx_dev, s);
            forward_backward(ln, scratch_w, nullptr, loss_dev + 63, s, false);
            launch_sum_masked(row_loss, T, B, valid, loss_dev + 62, s);
            float part = 0;
            AB_CUDA(cudaMemcpyAsync(&part, loss_dev + 62, sizeof(float), cudaMemcpyDeviceToHost, s));
            AB_CUDA(cudaStreamSynchronize(s));
            total += part;
        }
        result = total / (static_cast<double>(M) * T);
    }
    refresh_shadow(ln, restore ? restore : ln.w[slot(k)], s);
    AB_CUDA(cudaStreamSynchronize(s));
    return result;
}

// The coupled run's record (chronos.cpp:271-289) on the models the replay currently holds
// (learner l's model is w[par[l]]). Returns true when the divergence rule stops the run.
bool Ctx::observe_coupled(adpsgd_async_record& r, const std::vector<int>& par, int64_t processed, int ipe) {
    const int L = cfg.learners;
    if (processed % L == 0) {
        const int64_t kk = processed / L - 1;
        double c = 0.0;
        if (L >= 2) {
            std::vector<const float*> wt;
            for (int l = 0; l < L; ++l) wt.push_back(learners[l].w[par[l]]);
            std::vector<double> G(static_cast<size_t>(L) * L);
            gram(wt, 0, D, G.data());
            c = consensus_from_gram(G.data(), L);
        }
        if (r.consensus && kk < r.cap_iters) r.consensus[kk] = c;
        r.n_iters = kk + 1;
    }
    if (processed % (static_cast<int64_t>(L) * ipe) != 0) return false;
    const int epoch = static_cast<int>(processed / (static_cast<int64_t>(L) * ipe)) - 1;
    // averaged_model (engine.cpp:124-128) of the current models, fp64 in learner order
    std::vector<double> avg(D, 0.0);
    std::vector<float> f(D);
    AB_CUDA(cudaStreamSynchronize(s_main));
    for (int l = 0; l < L; ++l) {
        AB_CUDA(cudaMemcpy(f.data(), learners[l].w[par[l]], D * sizeof(float), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < D; ++i) avg[i] += f[i];
    }
    for (int64_t i = 0; i < D; ++i) avg[i] /= static_cast<double>(L);
    const float* keep = learners[0].w[par[0]];
    const double nan = std::numeric_limits<double>::quiet_NaN();
    const double h = r.n_heldout > 0 ? evaluate(avg.data(), r.heldout_idx, r.n_heldout, nullptr, keep) : nan;
    const double t = r.n_train > 0 ? evaluate(avg.data(), r.train_idx, r.n_train, nullptr, keep) : nan;
    if (epoch < r.cap_epochs) {
        if (r.heldout) r.heldout[epoch] = h;
        if (r.train) r.train[epoch] = t;
    }
    r.n_epochs = epoch + 1;
    if (!std::isfinite(h) || h > 10.0 * r.initial_heldout) {
        r.diverged_epoch = epoch;
        return true;
    }
    return false;
}

// engine.cpp:124-128 (averaged_model) over the local learners, fp64 on the host.
void Ctx::averaged_model(double* out) {
    AB_CUDA(cudaSetDevice(cfg.device));
    AB_CUDA(cudaStreamSynchronize(s_main));
    std::vector<float> f(D);
    std::fill(out, out + D, 0.0);
    for (auto& ln : learners) {
        AB_CUDA(cudaMemcpyAsync(f.data(), ln.w[slot(k)], D * sizeof(float), cudaMemcpyDeviceToHost, s_main));
        AB_CUDA(cudaStreamSynchronize(s_main));
        for (int64_t i = 0; i < D; ++i) out[i] += f[i];
    }
    for (int64_t i = 0; i < D; ++i) out[i] /= static_cast<double>(learners.size());
}

// mixing.cpp:159-180: ||W (I - 11^T/L)||_2 = sqrt(lambda_max(G)), G the Gram of the
// deviations of the local learners' models from their mean (device kernel, fp64 sums).
double Ctx::consensus_distance() {
    AB_CUDA(cudaSetDevice(cfg.device));
    const int L = cfg.local_learners;
    if (L < 2) return 0.0;
    std::vector<const float*> wt;
    for (auto& ln : learners) wt.push_back(ln.w[slot(k)]);
    std::vector<double> G(static_cast<size_t>(L) * L);
    gram(wt, 0, D, G.data());
    return consensus_from_gram(G.data(), L);
}

// Gram of the deviations from the learner mean over parameters [begin, end) of the given models.
void Ctx::gram(const std::vector<const float*>& models, int64_t begin, int64_t end, double* out) {
    const int L = static_cast<int>(models.size());
    if (!gram_dev) gram_dev = static_cast<double*>(alloc(sizeof(double) * (16 * 16 + gram_partial_doubles())));
    std::vector<const float*> wt;
    for (const float* w : models) wt.push_back(w + begin);
    launch_gram(end - begin, L, wt.data(), gram_dev, gram_dev + 16 * 16, s_main);
    AB_CUDA(cudaMemcpyAsync(out, gram_dev, sizeof(double) * L * L, cudaMemcpyDeviceToHost, s_main));
    AB_CUDA(cudaStreamSynchronize(s_main));
    for (int a = 0; a < L; ++a)
        for (int b = 0; b < a; ++b) out[a * L + b] = out[b * L + a];
}

// The shard [begin, end) of the consensus Gram over ALL global learners: local ones and peers
// mapped over NVLink (CUDA IPC). Ranks sum their shards (a small allreduce), then
// consensus_from_gram -- the multi-rank form of mixing.cpp:159-180.
void Ctx::consensus_gram(int64_t begin, int64_t end, double* out) {
    AB_CHECK(0 <= begin && begin <= end && end <= D, ADPSGD_E_DIMENSION, "consensus shard outside [0, D)");
    AB_CUDA(cudaSetDevice(cfg.device));
    std::vector<const float*> wt;
    for (int gid = 0; gid < cfg.learners; ++gid) wt.push_back(weight_ptr(gid, slot(k)));
    const int L = cfg.learners;
    if (end == begin) {
        std::fill(out, out + static_cast<size_t>(L) * L, 0.0);
        return;
    }
    gram(wt, begin, end, out);
}

// largest eigenvalue of the symmetric PSD L x L Gram by cyclic Jacobi (exact enough for L <= 16)
double consensus_from_gram(const double* G, int L) {
    std::vector<double> A(G, G + static_cast<size_t>(L) * L);
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0;
        for (int p = 0; p < L; ++p)
            for (int q = p + 1; q < L; ++q) off += A[p * L + q] * A[p * L + q];
        if (off < 1e-30) break;
        for (int p = 0; p < L; ++p)
            for (int q = p + 1; q < L; ++q) {
                const double apq = A[p * L + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double theta = (A[q * L + q] - A[p * L + p]) / (2 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
                const double c = 1 / std::sqrt(t * t + 1), sn = t * c;
                for (int r = 0; r < L; ++r) {
                    const double arp = A[r * L + p], arq = A[r * L + q];
                    A[r * L + p] = c * arp - sn * arq;
                    A[r * L + q] = sn * arp + c * arq;
                }
                for (int r = 0; r < L; ++r) {
                    const double apr = A[p * L + r], aqr = A[q * L + r];
                    A[p * L + r] = c * apr - sn * aqr;
                    A[q * L + r] = sn * apr + c * aqr;
                }
            }
    }
    double lam = 0;
    for (int p = 0; p < L; ++p) lam = std::max(lam, A[p * L + p]);
    return std::sqrt(std::max(0.0, lam));
}

// engine.cpp:124-128 averaged_model over ALL global learners (mapped peers included), fp64
// accumulation in learner order on the host.
void Ctx::averaged_model_all(double* out) {
    AB_CUDA(cudaSetDevice(cfg.device));
    AB_CUDA(cudaStreamSynchronize(s_main));
    std::vector<float> f(D);
    std::fill(out, out + D, 0.0);
    for (int gid = 0; gid < cfg.learners; ++gid) {
        AB_CUDA(cudaMemcpyAsync(f.data(), weight_ptr(gid, slot(k)), D * sizeof(float), cudaMemcpyDeviceToHost, s_main));
        AB_CUDA(cudaStreamSynchronize(s_main));
        for (int64_t i = 0; i < D; ++i) out[i] += f[i];
    }
    for (int64_t i = 0; i < D; ++i) out[i] /= static_cast<double>(cfg.learners);
}

// Bandwidth of the gossip data path at this context's model size: the fused mix kernel (22 B per
// parameter: w, w_L, w_R, g read, w' written fp32, the bf16 shadow) and the copy-engine pull of
// both neighbours, each timed over `reps` calls with CUDA events on s_main. Scratch outputs only.
void Ctx::gossip_probe(int left, int right, int reps, double* out) {
    AB_CUDA(cudaSetDevice(cfg.device));
    cudaStream_t s = s_main;
    AB_CUDA(cudaStreamSynchronize(s));
    if (!probe_buf[0]) {
        for (auto& p : probe_buf) p = static_cast<float*>(alloc(D * sizeof(float)));
        probe_shadow = static_cast<bf16*>(alloc(D * sizeof(bf16)));
        AB_CUDA(cudaMemsetAsync(probe_buf[0], 0, D * sizeof(float), s));
    }
    if (!scratch_w) scratch_w = static_cast<float*>(alloc(D * sizeof(float)));
    const int cur = slot(k);
    const Learner& ln = learners[0];
    // stand-ins at N = 1: the learner's spare weight buffer and its gradient buffer (distinct
    // 4 D-byte streams, so nothing is served from L2)
    const float* wl = left >= 0 ? weight_ptr(left, cur) : ln.w[slot(k + 1)];
    const float* wr = right >= 0 ? weight_ptr(right, cur) : probe_buf[0];
    const double nv = (left >= 0 && !is_local(left) ? 4.0 * D : 0.0) + (right >= 0 && !is_local(right) ? 4.0 * D : 0.0);
    launch_mix3(D, ln.w[cur], wl, wr, ln.g, 0.0f, scratch_w, probe_shadow, s);  // warm
    AB_CUDA(cudaEventRecord(ev0, s));
    for (int r = 0; r < reps; ++r) launch_mix3(D, ln.w[cur], wl, wr, ln.g, 0.0f, scratch_w, probe_shadow, s);
    AB_CUDA(cudaEventRecord(ev1, s));
    AB_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    AB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    out[0] = ms / reps;
    out[1] = nv;
    AB_CUDA(cudaEventRecord(ev0, s));
    for (int r = 0; r < reps; ++r) {
        AB_CUDA(cudaMemcpyAsync(scratch_w, wl, D * sizeof(float), cudaMemcpyDeviceToDevice, s));
        AB_CUDA(cudaMemcpyAsync(probe_buf[1], wr, D * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
    AB_CUDA(cudaEventRecord(ev1, s));
    AB_CUDA(cudaStreamSynchronize(s));
    AB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    out[2] = ms / reps;
    out[3] = 22.0 * D;
}

void* Ctx::alloc_scratch_grad() {
    if (!scratch_grad) scratch_grad = alloc(D * sizeof(float));
    return scratch_grad;
}

}  // namespace ab
