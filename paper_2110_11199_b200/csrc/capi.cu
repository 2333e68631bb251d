// extern "C" boundary (include/adpsgd_b200.h). Every entry point converts library
// exceptions into adpsgd_status codes and records the message for adpsgd_last_error().
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <vector>

#include "adpsgd_b200.h"
#include "comm.hpp"
#include "engine.hpp"
#include "gemm.hpp"
#include "kernels.cuh"
#include "prof.hpp"
#include "rng.hpp"

using namespace ab;

struct adpsgd_ctx {
    ab::Ctx* impl;
};

namespace {
template <typename F>
int guard(F&& f) {
    try {
        f();
        return ADPSGD_OK;
    } catch (const ab::Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return ADPSGD_E_CUDA;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ADPSGD_E_INVALID_STATE;
    }
}
// Stream-K / split-K scratch of the standalone adpsgd_gemm entry point: one per device, owned by
// the library for the life of the process (the engines bind their own; see GemmWorkspaceScope).
const GemmWorkspace& standalone_gemm_workspace() {
    static std::mutex mu;
    static std::map<int, GemmWorkspace> per_dev;
    int dev = 0;
    AB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it == per_dev.end()) {
        GemmWorkspace w;
        w.floats = static_cast<size_t>(num_sms() / 2) * 2 * 17 * 128 * 32;
        w.flag_count = static_cast<size_t>(num_sms()) + 2 * 128;
        AB_CUDA(cudaMalloc(&w.ws, w.floats * sizeof(float)));
        AB_CUDA(cudaMalloc(&w.flags, w.flag_count * sizeof(unsigned int)));
        AB_CUDA(cudaMemset(w.flags, 0, w.flag_count * sizeof(unsigned int)));
        it = per_dev.emplace(dev, w).first;
    }
    return it->second;
}
Ctx& C_(adpsgd_ctx* c) {
    AB_CHECK(c && c->impl, ADPSGD_E_INVALID_STATE, "null context");
    return *c->impl;
}
}  // namespace

extern "C" {

int64_t adpsgd_param_count(const adpsgd_model_desc* m) { return m ? make_layout(*m).total : -1; }

int adpsgd_permutation_for_iteration(uint64_t seed, int32_t L, int64_t k, int32_t* mapping) {
    return guard([&] {
        AB_CHECK(L >= 1, ADPSGD_E_INVALID_ORDER, "permutation requires order >= 1");  // mixing.cpp:65-68
        permutation_for_iteration(seed, L, k, mapping);
    });
}

int adpsgd_pairing(int32_t strategy, uint64_t seed, int32_t L, int64_t k, int32_t* mapping, int32_t* lr) {
    return guard([&] {
        AB_CHECK(L >= 3, ADPSGD_E_INVALID_ORDER, "ring pairing requires order >= 3");  // mixing.cpp:36-39
        std::vector<int32_t> map(L);
        if (strategy == ADPSGD_RM) permutation_for_iteration(seed, L, k, map.data());
        else for (int i = 0; i < L; ++i) map[i] = i;
        if (mapping) std::memcpy(mapping, map.data(), sizeof(int32_t) * L);
        // learner map[a] sits at ring position a (mixing.cpp:97-101, chronos.cpp:229-234)
        for (int a = 0; a < L; ++a) {
            const int l = map[a];
            lr[2 * l] = map[(a + L - 1) % L];
            lr[2 * l + 1] = map[(a + 1) % L];
        }
    });
}

double adpsgd_lr_at(double base, double peak, int32_t warmup, double anneal_factor, int32_t anneal_start, int32_t epoch) {
    // engine.cpp:45-58
    if (epoch < 0) return -1.0;
    double lr = (warmup > 0 && epoch < warmup) ? base + (peak - base) * static_cast<double>(epoch) / warmup : peak;
    if (epoch >= anneal_start) lr = peak * std::pow(anneal_factor, epoch - anneal_start);
    return lr;
}

const char* adpsgd_last_error(void) { return last_error(); }

const char* adpsgd_build_info(void) {
    return "libadpsgd_b200: sm_100a; tcgen05/TMA/TMEM bf16 GEMM + fp32 SIMT parity GEMM; NCCL via dlopen";
}

int adpsgd_ctx_create(const adpsgd_config* cfg, adpsgd_ctx** out) {
    return guard([&] {
        AB_CHECK(cfg && out, ADPSGD_E_CONFIG, "null argument");
        *out = nullptr;
        auto* c = new adpsgd_ctx{nullptr};
        try {
            c->impl = new Ctx(*cfg);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int adpsgd_ctx_destroy(adpsgd_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        delete ctx->impl;
        delete ctx;
    });
}

int adpsgd_set_dataset(adpsgd_ctx* ctx, const float* feats, const int32_t* labels, int32_t n_seg, int32_t train_count) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(n_seg >= 1 && train_count >= 1 && train_count <= n_seg, ADPSGD_E_INVALID_STATE,
                 "dataset has no training samples");
        AB_CUDA(cudaSetDevice(c.cfg.device));
        const size_t nf = static_cast<size_t>(n_seg) * c.T * c.I;
        if (c.n_seg < n_seg) {
            c.feats = static_cast<float*>(c.alloc(nf * sizeof(float)));
            c.labels = static_cast<int32_t*>(c.alloc(static_cast<size_t>(n_seg) * c.T * sizeof(int32_t)));
        }
        c.clear_graphs();
        AB_CUDA(cudaStreamSynchronize(c.s_main));  // no step still reading the old dataset
        c.h2d_sync(c.feats, feats, nf * sizeof(float));
        c.h2d_sync(c.labels, labels, static_cast<size_t>(n_seg) * c.T * sizeof(int32_t));
        c.n_seg = n_seg;
        c.train_count = train_count;
    });
}

int adpsgd_synth_dataset(adpsgd_ctx* ctx, int32_t n_seg, int32_t train_count, uint64_t seed) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(n_seg >= 1 && train_count >= 1 && train_count <= n_seg, ADPSGD_E_INVALID_STATE,
                 "dataset has no training samples");
        AB_CUDA(cudaSetDevice(c.cfg.device));
        if (c.n_seg < n_seg) {
            c.feats = static_cast<float*>(c.alloc(static_cast<size_t>(n_seg) * c.T * c.I * sizeof(float)));
            c.labels = static_cast<int32_t*>(c.alloc(static_cast<size_t>(n_seg) * c.T * sizeof(int32_t)));
        }
        c.clear_graphs();
        launch_synth(c.feats, c.labels, n_seg, c.T, c.I, c.lay.C, seed, c.s_main);
        AB_CUDA(cudaStreamSynchronize(c.s_main));
        c.n_seg = n_seg;
        c.train_count = train_count;
    });
}

int adpsgd_get_dataset(adpsgd_ctx* ctx, float* feats, int32_t* labels) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(c.feats, ADPSGD_E_INVALID_STATE, "no dataset");
        AB_CUDA(cudaMemcpyAsync(feats, c.feats, static_cast<size_t>(c.n_seg) * c.T * c.I * sizeof(float), cudaMemcpyDeviceToHost, c.s_main));
        AB_CUDA(cudaMemcpyAsync(labels, c.labels, static_cast<size_t>(c.n_seg) * c.T * sizeof(int32_t), cudaMemcpyDeviceToHost, c.s_main));
        AB_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

int adpsgd_set_weights(adpsgd_ctx* ctx, int32_t j, const double* w, int64_t n) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(j >= 0 && j < c.cfg.local_learners, ADPSGD_E_DIMENSION, "local learner out of range");
        AB_CHECK(n == c.D, ADPSGD_E_DIMENSION, "weight vector length != parameter count");
        AB_CUDA(cudaSetDevice(c.cfg.device));
        std::vector<float> f(w, w + n);
        Learner& ln = c.learners[j];
        const int cur = c.slot(c.k);
        AB_CUDA(cudaStreamSynchronize(c.s_main));
        c.h2d_sync(ln.w[cur], f.data(), n * sizeof(float));
        c.refresh_shadow(ln, ln.w[cur], c.s_main);
        AB_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

int adpsgd_get_weights(adpsgd_ctx* ctx, int32_t j, double* w, int64_t n) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(j >= 0 && j < c.cfg.local_learners, ADPSGD_E_DIMENSION, "local learner out of range");
        AB_CHECK(n == c.D, ADPSGD_E_DIMENSION, "weight vector length != parameter count");
        AB_CUDA(cudaSetDevice(c.cfg.device));
        std::vector<float> f(n);
        AB_CUDA(cudaMemcpyAsync(f.data(), c.learners[j].w[c.slot(c.k)], n * sizeof(float), cudaMemcpyDeviceToHost, c.s_main));
        AB_CUDA(cudaStreamSynchronize(c.s_main));
        for (int64_t i = 0; i < n; ++i) w[i] = f[i];
    });
}

int adpsgd_step(adpsgd_ctx* ctx, double lr, const int32_t* taus, float* loss_out) {
    return guard([&] { C_(ctx).step(lr, taus, loss_out, nullptr, nullptr, nullptr); });
}

int adpsgd_step_host_batch(adpsgd_ctx* ctx, double lr, const float* feats, const int32_t* labels, float* loss_out) {
    return guard([&] {
        AB_CHECK(feats && labels, ADPSGD_E_INVALID_STATE, "null host batch");
        C_(ctx).step(lr, nullptr, loss_out, feats, labels, nullptr);
    });
}

int adpsgd_prefetch_host_batch(adpsgd_ctx* ctx, const float* feats, const int32_t* labels) {
    return guard([&] { C_(ctx).prefetch_host_batch(feats, labels); });
}

int adpsgd_step_injected(adpsgd_ctx* ctx, double lr, const int32_t* taus, const double* grads) {
    return guard([&] {
        AB_CHECK(grads, ADPSGD_E_INVALID_STATE, "null gradients");
        C_(ctx).step(lr, taus, nullptr, nullptr, nullptr, grads);
    });
}

int adpsgd_gradient(adpsgd_ctx* ctx, const double* w, const int32_t* idx, int32_t M, double* g_out, double* loss_out) {
    return guard([&] {
        double l = C_(ctx).gradient(w, idx, M, g_out);
        if (loss_out) *loss_out = l;
    });
}

int adpsgd_set_straggler(adpsgd_ctx* ctx, int32_t j, double factor) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(j >= 0 && j < c.cfg.local_learners, ADPSGD_E_CONFIG, "straggler learner_id out of range");
        AB_CHECK(factor >= 1.0, ADPSGD_E_CONFIG, "slowdown factor must be >= 1");  // chronos.cpp:47
        c.learners[j].straggle = factor;
    });
}

int adpsgd_get_stats(adpsgd_ctx* ctx, adpsgd_perf* out) {
    return guard([&] {
        Ctx& c = C_(ctx);
        out->last_step_ms = c.last_step_ms;
        out->last_mix_ms = c.last_mix_ms;
        out->gossip_bytes = c.last_gossip_bytes;
        out->steps = c.k;
        out->kernel_launches = g_launch_count;
        out->comm_start_ms = c.last_comm_start_ms;
        out->comm_end_ms = c.last_comm_end_ms;
        out->compute_end_ms = c.last_compute_end_ms;
    });
}

int64_t adpsgd_iteration(adpsgd_ctx* ctx) { return ctx && ctx->impl ? ctx->impl->k : -1; }

int adpsgd_set_iteration(adpsgd_ctx* ctx, int64_t k) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(k >= 0, ADPSGD_E_INVALID_STATE, "iteration must be >= 0");
        AB_CHECK(((k ^ c.k) & 1) == 0, ADPSGD_E_INVALID_STATE, "iteration parity must be preserved");
        c.k = k;
    });
}

int adpsgd_consensus_distance(adpsgd_ctx* ctx, double* out) {
    return guard([&] { *out = C_(ctx).consensus_distance(); });
}

int adpsgd_eval_loss(adpsgd_ctx* ctx, const double* w, const int32_t* idx, int32_t M, double* loss_out) {
    return guard([&] { *loss_out = C_(ctx).evaluate(w, idx, M, nullptr); });
}

int adpsgd_consensus_gram(adpsgd_ctx* ctx, int64_t begin, int64_t end, double* gram) {
    return guard([&] { C_(ctx).consensus_gram(begin, end, gram); });
}

int adpsgd_consensus_from_gram(const double* gram, int32_t L, double* out) {
    return guard([&] {
        AB_CHECK(gram && out && L >= 1 && L <= 16, ADPSGD_E_DIMENSION, "consensus_from_gram: 1 <= L <= 16");
        *out = consensus_from_gram(gram, L);
    });
}

int adpsgd_averaged_model_all(adpsgd_ctx* ctx, double* out, int64_t n) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(n == c.D, ADPSGD_E_DIMENSION, "averaged model length != parameter count");
        c.averaged_model_all(out);
    });
}

int adpsgd_averaged_model(adpsgd_ctx* ctx, double* out, int64_t n) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(n == c.D, ADPSGD_E_DIMENSION, "weight vector length != parameter count");
        c.averaged_model(out);
    });
}

int adpsgd_async_run(adpsgd_ctx* ctx, int32_t strategy, const double* durations, int64_t target, int32_t ipe,
                     const double* lr_per_epoch, int32_t n_epochs, int32_t* event_learner, double* event_time,
                     int64_t* processed) {
    return guard([&] {
        AB_CHECK(durations && lr_per_epoch, ADPSGD_E_CONFIG, "null durations / lr table");
        for (int l = 0; l < C_(ctx).cfg.learners; ++l)
            AB_CHECK(durations[l] > 0.0, ADPSGD_E_CONFIG, "cluster profile: compute_time must be > 0");
        const int64_t n = C_(ctx).async_run(strategy, durations, target, ipe, lr_per_epoch, n_epochs, event_learner,
                                            event_time);
        if (processed) *processed = n;
    });
}

int adpsgd_async_run_record(adpsgd_ctx* ctx, int32_t strategy, const double* durations, int64_t target, int32_t ipe,
                            const double* lr_per_epoch, int32_t n_epochs, int32_t* event_learner, double* event_time,
                            adpsgd_async_record* record, int64_t* processed) {
    return guard([&] {
        AB_CHECK(durations && lr_per_epoch && record, ADPSGD_E_CONFIG, "null durations / lr table / record");
        for (int l = 0; l < C_(ctx).cfg.learners; ++l)
            AB_CHECK(durations[l] > 0.0, ADPSGD_E_CONFIG, "cluster profile: compute_time must be > 0");
        AB_CHECK(record->n_heldout >= 0 && record->n_train >= 0 && (record->n_heldout == 0 || record->heldout_idx) &&
                     (record->n_train == 0 || record->train_idx),
                 ADPSGD_E_CONFIG, "record: index lists");
        for (int i = 0; i < record->n_heldout; ++i)
            AB_CHECK(record->heldout_idx[i] >= 0 && record->heldout_idx[i] < C_(ctx).n_seg, ADPSGD_E_DIMENSION,
                     "record: held-out index outside the dataset");
        for (int i = 0; i < record->n_train; ++i)
            AB_CHECK(record->train_idx[i] >= 0 && record->train_idx[i] < C_(ctx).n_seg, ADPSGD_E_DIMENSION,
                     "record: train index outside the dataset");
        record->n_iters = 0;
        record->n_epochs = 0;
        record->diverged_epoch = -1;
        const int64_t n = C_(ctx).async_run(strategy, durations, target, ipe, lr_per_epoch, n_epochs, event_learner,
                                            event_time, record);
        if (processed) *processed = n;
    });
}

int adpsgd_nccl_unique_id(void* out128) { return guard([&] { Comm::unique_id(out128); }); }

int adpsgd_comm_init(adpsgd_ctx* ctx, int32_t rank, int32_t world, const void* id) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CUDA(cudaSetDevice(c.cfg.device));
        c.comm = std::make_unique<Comm>(c, rank, world, id);
    });
}

int64_t adpsgd_ipc_handle_size(adpsgd_ctx* ctx) {
    return ctx && ctx->impl ? static_cast<int64_t>(ctx->impl->cfg.local_learners) * Comm::ipc_record_bytes() : -1;
}

int adpsgd_export_ipc(adpsgd_ctx* ctx, void* out, int64_t size) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(c.comm, ADPSGD_E_INVALID_STATE, "adpsgd_comm_init first");
        c.comm->export_ipc(c, out, size);
        c.ipc_exported = true;
    });
}

int adpsgd_import_ipc(adpsgd_ctx* ctx, int32_t rank, int32_t first, int32_t count, const void* h, int64_t size) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(c.comm, ADPSGD_E_INVALID_STATE, "adpsgd_comm_init first");
        AB_CUDA(cudaSetDevice(c.cfg.device));
        c.comm->import_ipc(rank, first, count, h, size);
    });
}

int adpsgd_set_gossip_mode(adpsgd_ctx* ctx, int32_t mode) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(mode >= 0 && mode <= 2, ADPSGD_E_CONFIG, "gossip mode must be 0, 1 or 2");
        AB_CHECK(c.comm, ADPSGD_E_INVALID_STATE, "adpsgd_comm_init first");
        c.comm->gossip_mode = mode;
    });
}

int adpsgd_group_link(adpsgd_ctx* const* ctxs, int32_t n) {
    return guard([&] {
        AB_CHECK(ctxs && n >= 1, ADPSGD_E_CONFIG, "group: at least one context");
        std::vector<Ctx*> cs;
        for (int i = 0; i < n; ++i) cs.push_back(&C_(ctxs[i]));
        std::sort(cs.begin(), cs.end(), [](const Ctx* a, const Ctx* b) { return a->cfg.first_learner < b->cfg.first_learner; });
        const adpsgd_config& c0 = cs[0]->cfg;
        int next = 0;
        for (Ctx* c : cs) {
            AB_CHECK(c->cfg.first_learner == next, ADPSGD_E_CONFIG, "group: contexts must host contiguous learner ranges from 0");
            next += c->cfg.local_learners;
            AB_CHECK(std::memcmp(&c->cfg.model, &c0.model, sizeof(c0.model)) == 0 && c->cfg.strategy == c0.strategy &&
                         c->cfg.learners == c0.learners && c->cfg.batch == c0.batch && c->cfg.seed == c0.seed &&
                         c->cfg.precision == c0.precision && c->k == cs[0]->k && c->nbuf == cs[0]->nbuf,
                     ADPSGD_E_CONFIG, "group: contexts differ in model / strategy / learners / batch / seed / precision / iteration");
            AB_CHECK(!c->comm, ADPSGD_E_INVALID_STATE, "group: context already has a communicator");
        }
        AB_CHECK(next == c0.learners, ADPSGD_E_CONFIG, "group: contexts must host all cfg.learners learners");
        for (Ctx* a : cs)
            for (Ctx* b : cs)
                if (a->cfg.device != b->cfg.device) {
                    AB_CUDA(cudaSetDevice(a->cfg.device));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(b->cfg.device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else AB_CUDA(e);
                }
        for (size_t i = 0; i < cs.size(); ++i) {
            Ctx* c = cs[i];
            c->comm = std::make_unique<Comm>(*c, static_cast<int>(i), static_cast<int>(cs.size()), Comm::LocalGroupTag{});
            c->comm->group_ctxs = cs;
            for (Ctx* o : cs)
                if (o != c) c->comm->link_local(*o);
        }
    });
}

int adpsgd_group_step(adpsgd_ctx* const* ctxs, int32_t n, double lr, float* loss_out) {
    return guard([&] {
        AB_CHECK(ctxs && n >= 1, ADPSGD_E_CONFIG, "group: at least one context");
        std::vector<Ctx*> cs;
        for (int i = 0; i < n; ++i) cs.push_back(&C_(ctxs[i]));
        for (Ctx* c : cs)
            AB_CHECK(n == 1 || (c->comm && c->comm->local_group && static_cast<int>(c->comm->group_ctxs.size()) == n),
                     ADPSGD_E_INVALID_STATE, "group: adpsgd_group_link these contexts first");
        for (Ctx* c : cs) c->step_compute(lr, nullptr, nullptr, nullptr, nullptr);  // all GPUs compute concurrently
        for (Ctx* c : cs) c->step_mix(lr, nullptr);
        std::vector<float> part(64);
        for (Ctx* c : cs) {
            c->step_finish(part.data(), false);
            if (loss_out)
                for (int j = 0; j < c->cfg.local_learners; ++j) loss_out[c->cfg.first_learner + j] = part[j];
        }
    });
}

int adpsgd_async_init(adpsgd_ctx* ctx, int32_t mode, int32_t max_lag, double timeout_s) {
    return guard([&] { C_(ctx).async_init(mode, max_lag, timeout_s); });
}

int adpsgd_async_step(adpsgd_ctx* ctx, double lr, float* loss_out, adpsgd_async_info* info) {
    return guard([&] { C_(ctx).async_step(lr, loss_out, info); });
}

int adpsgd_set_step_delay(adpsgd_ctx* ctx, int32_t j, double ms, int32_t on_host) {
    return guard([&] {
        Ctx& c = C_(ctx);
        AB_CHECK(j >= 0 && j < c.cfg.local_learners, ADPSGD_E_DIMENSION, "local learner out of range");
        AB_CHECK(ms >= 0, ADPSGD_E_CONFIG, "step delay must be >= 0");
        c.learners[j].delay_ms = ms;
        c.learners[j].delay_on_host = on_host != 0;
    });
}

int adpsgd_gossip_probe(adpsgd_ctx* ctx, int32_t left, int32_t right, int32_t reps, double* out4) {
    return guard([&] {
        AB_CHECK(out4 && reps >= 1, ADPSGD_E_INVALID_STATE, "gossip probe: out4 and reps >= 1 required");
        C_(ctx).gossip_probe(left, right, reps, out4);
    });
}

int adpsgd_barrier(adpsgd_ctx* ctx) {
    return guard([&] {
        Ctx& c = C_(ctx);
        if (!c.comm) return;
        c.comm->barrier(c.s_main);
        AB_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

int adpsgd_profile_enable(int32_t on) {
    return guard([&] { g_prof_enabled = on != 0; });
}

int adpsgd_kernel_variants(char* out, size_t n, int32_t reset) {
    return guard([&] {
        const std::string v = variants_string(reset != 0);
        if (out && n) {
            const size_t m = v.size() < n - 1 ? v.size() : n - 1;
            std::memcpy(out, v.data(), m);
            out[m] = 0;
        }
    });
}

int adpsgd_profile_read(double* ms, double* flops, double* bytes, int64_t* launches, int32_t ncat) {
    return guard([&] { prof_read(ms, flops, bytes, launches, ncat < PROF_NCAT ? ncat : PROF_NCAT); });
}

}  // extern "C"
namespace ab { void trace_enable(int); void trace_read(unsigned long long*, int); }
extern "C" {
// Debug: device timeline of the CTA-pair tcgen05 kernels (160 CTAs x 32 globaltimer stamps).
int adpsgd_debug_buffer(adpsgd_ctx* ctx, int32_t which, void* out, size_t bytes) {
    return guard([&] {
        ab::Ctx& c = C_(ctx);
        AB_CUDA(cudaSetDevice(c.cfg.device));
        AB_CUDA(cudaStreamSynchronize(c.s_main));
        const void* src = nullptr;
        size_t n = 0;
        const size_t TB = static_cast<size_t>(c.TB);
        if (which == 0) { src = c.X0; n = TB * c.Ipad * c.es; }
        else if (which >= 1 && which <= c.lay.L) { src = c.Hout[which - 1]; n = TB * c.ldH * c.es; }
        else if (which == 100) { src = c.Y; n = TB * c.ldY * c.es; }
        else if (which == 101) { src = c.row_loss; n = TB * sizeof(float); }
        else if (which == 102) { src = c.learners[0].shadow; n = static_cast<size_t>(c.D) * 2; }
        else if (which == 103) { src = c.learners[0].g; n = static_cast<size_t>(c.D) * sizeof(float); }
        else if (which >= 200 && which < 200 + c.lay.L) { src = c.cst[which - 200]; n = TB * c.ndH * sizeof(float); }
        else if (which >= 300 && which < 300 + c.lay.L) { src = c.gates[which - 300]; n = TB * c.nd4H * c.es; }
        AB_CHECK(src != nullptr, ADPSGD_E_INVALID_STATE, "debug_buffer: no such buffer");
        AB_CUDA(cudaMemcpyAsync(out, src, bytes < n ? bytes : n, cudaMemcpyDeviceToHost, c.s_main));
        AB_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

// Device address range of an engine buffer (diagnosis: mapping sanitizer reports to buffers).
// which: as adpsgd_debug_buffer, plus 400 / 401 = the two BPTT dH ping-pong buffers.
int adpsgd_debug_buffer_range(adpsgd_ctx* ctx, int32_t which, uint64_t* addr, uint64_t* bytes) {
    return guard([&] {
        ab::Ctx& c = C_(ctx);
        const size_t TB = static_cast<size_t>(c.TB);
        const void* src = nullptr;
        size_t n = 0;
        if (which == 0) { src = c.X0; n = TB * c.Ipad * c.es; }
        else if (which >= 1 && which <= c.lay.L) { src = c.Hout[which - 1]; n = TB * c.ldH * c.es; }
        else if (which >= 200 && which < 200 + c.lay.L) { src = c.cst[which - 200]; n = TB * c.ndH * sizeof(float); }
        else if (which >= 300 && which < 300 + c.lay.L) { src = c.gates[which - 300]; n = TB * c.nd4H * c.es; }
        else if (which == 400 || which == 401) { src = which == 400 ? c.dHa : c.dHb; n = TB * c.ndH * sizeof(float); }
        AB_CHECK(src != nullptr, ADPSGD_E_INVALID_STATE, "debug_buffer_range: no such buffer");
        *addr = reinterpret_cast<uint64_t>(src);
        *bytes = n;
    });
}

int adpsgd_debug_trace(int32_t enable, uint64_t* out, int32_t n) {
    return guard([&] {
        if (out) ab::trace_read(reinterpret_cast<unsigned long long*>(out), n);
        ab::trace_enable(enable);
    });
}

int adpsgd_gemm(int32_t bf, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_mn, const void* B,
                int64_t ldb, int32_t b_mn, void* Cout, int64_t ldc, int32_t c_bf16, float alpha, int32_t accumulate,
                const float* bias, void* stream) {
    return guard([&] {
        GemmArgs g;
        g.M = M; g.N = N;
        g.seg[0].a = {A, lda, a_mn != 0};
        g.seg[0].b = {B, ldb, b_mn != 0};
        g.seg[0].K = K;
        g.C = Cout; g.ldc = ldc; g.c_bf16 = c_bf16 != 0;
        g.alpha = alpha; g.accumulate = accumulate != 0; g.bias = bias;
        GemmWorkspaceScope ws_scope(standalone_gemm_workspace());
        gemm(bf != 0, g, static_cast<cudaStream_t>(stream));
    });
}

int adpsgd_mix_update(int64_t n, const float* w, const float* wl, const float* wr, const float* g, float lr, float* out,
                      void* shadow, void* stream) {
    return guard([&] {
        launch_mix3(n, w, wl, wr, g, lr, out, static_cast<bf16*>(shadow), static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
