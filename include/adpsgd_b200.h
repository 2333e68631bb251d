/*
 * adpsgd_b200.h — C ABI of the B200-native ADPSGD learner step.
 *
 * Drop-in boundary for the reference's per-learner step API
 * (/root/reference/proj/include/adpsgd/engine.hpp:85-105) and its loss/gradient
 * plugin (/root/reference/proj/include/adpsgd/objectives.hpp:45-69). Plain pointers
 * and sizes only; every entry point returns an adpsgd_status that the C++/Python
 * shims map 1:1 onto the reference's exception types (errors.hpp:9-46).
 *
 * Implemented by libadpsgd_b200.so (paper_2110_11199_b200/csrc), sm_100a only.
 */
#ifndef ADPSGD_B200_H
#define ADPSGD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:9-46, in declaration order; CUDA/NCCL failures are additional. */
typedef enum adpsgd_status {
    ADPSGD_OK = 0,
    ADPSGD_E_INVALID_ORDER = 1,       /* InvalidOrderError      (mixing.cpp:36-39, 81-84) */
    ADPSGD_E_DIMENSION = 2,           /* DimensionError         (engine.cpp:158-160)      */
    ADPSGD_E_OUT_OF_REGIME = 3,       /* OutOfRegimeError                                 */
    ADPSGD_E_NUMERICAL = 4,           /* NumericalError                                   */
    ADPSGD_E_SYNC_VIOLATION = 5,      /* SyncViolationError     (engine.cpp:139-144)      */
    ADPSGD_E_STALENESS_OVERFLOW = 6,  /* StalenessOverflowError (engine.cpp:90-96)        */
    ADPSGD_E_INVALID_STATE = 7,       /* InvalidStateError      (objectives.cpp:240-241)  */
    ADPSGD_E_CONFIG = 8,              /* ConfigError            (engine.cpp:60-77)        */
    ADPSGD_E_CUDA = 9,
    ADPSGD_E_NCCL = 10
} adpsgd_status;

/* engine.hpp:17 — Strategy enum, same order. */
typedef enum adpsgd_strategy {
    ADPSGD_SDPSGD = 0,
    ADPSGD_FM = 1,
    ADPSGD_RM = 2,
    ADPSGD_D1D = 3,
    ADPSGD_GENERIC = 4
} adpsgd_strategy;

/* mixing.hpp:13 — MixKind (generic-staleness mixing matrix). */
typedef enum adpsgd_mix_kind { ADPSGD_MIX_FIXED = 0, ADPSGD_MIX_RANDOM = 1, ADPSGD_MIX_UNIFORM = 2 } adpsgd_mix_kind;

/* GEMM operand precision of the learner step. FP32 = SIMT fp32 GEMMs (parity mode);
 * BF16 = tcgen05 bf16 x bf16 -> fp32 (TMEM) GEMMs. Master weights, cell state, gate
 * activations, the update and the mixing are fp32 in both modes. */
typedef enum adpsgd_precision { ADPSGD_PREC_FP32 = 0, ADPSGD_PREC_BF16 = 1 } adpsgd_precision;

/* BLSTM acoustic model. proj = 0 means no projection layer. */
typedef struct adpsgd_model_desc {
    int32_t layers;
    int32_t hidden;        /* cells per direction */
    int32_t bidirectional; /* 0 or 1 */
    int32_t input_dim;
    int32_t proj;
    int32_t classes;
    int32_t unroll;        /* T, frames per segment */
} adpsgd_model_desc;

typedef struct adpsgd_config {
    adpsgd_model_desc model;
    int32_t precision;        /* adpsgd_precision */
    int32_t strategy;         /* adpsgd_strategy (engine.hpp:36) */
    int32_t learners;         /* global L (engine.hpp:37) */
    int32_t first_learner;    /* global id of this context's first learner */
    int32_t local_learners;   /* learners hosted by this context (same device) */
    int32_t batch;            /* M segments per learner per step (engine.hpp:38) */
    int32_t device;
    int32_t generic_mix;      /* adpsgd_mix_kind, GENERIC only */
    int32_t staleness_cap;    /* GENERIC only (engine.hpp:44) */
    uint64_t seed;            /* run seed (engine.hpp:41) */
} adpsgd_config;

typedef struct adpsgd_perf {
    double last_step_ms;      /* device time of the last step (CUDA events) */
    double last_mix_ms;       /* device time of the mixing/update phase */
    double gossip_bytes;      /* bytes pulled from neighbours in the last step */
    int64_t steps;            /* global iteration counter k */
    int64_t kernel_launches;  /* this library's kernel launches so far */
    /* D1D across ranks: device times (ms after the step's start) at which the weight allreduce on
     * the comm stream started and finished, and at which the gradient compute finished; -1 when
     * no allreduce ran in the last step. comm_end <= compute_end means the allreduce was hidden. */
    double comm_start_ms;
    double comm_end_ms;
    double compute_end_ms;
} adpsgd_perf;

typedef struct adpsgd_ctx adpsgd_ctx;

/* ---- pure host helpers (bit-exact with rng.hpp / mixing.cpp / engine.cpp) ---- */
int64_t adpsgd_param_count(const adpsgd_model_desc* m);
/* engine.cpp:130-134 — mapping[L] for iteration k. */
int adpsgd_permutation_for_iteration(uint64_t seed, int32_t learners, int64_t k, int32_t* mapping);
/* (left, right) of every learner for FM (l±1) or RM (chronos.cpp:224-235): left_right[2*l+{0,1}]. */
int adpsgd_pairing(int32_t strategy, uint64_t seed, int32_t learners, int64_t k, int32_t* mapping,
                   int32_t* left_right);
double adpsgd_lr_at(double base_lr, double peak_lr, int32_t warmup_epochs, double anneal_factor,
                    int32_t anneal_start_epoch, int32_t epoch);
const char* adpsgd_last_error(void);
const char* adpsgd_build_info(void);

/* ---- context lifecycle ---- */
int adpsgd_ctx_create(const adpsgd_config* cfg, adpsgd_ctx** out);
int adpsgd_ctx_destroy(adpsgd_ctx* ctx);
/* Device-resident dataset: feats [n_seg][T][input_dim] fp32, labels [n_seg][T] int32.
 * Segments [0, train_count) are the training split (objectives.hpp:24-32). */
int adpsgd_set_dataset(adpsgd_ctx* ctx, const float* feats, const int32_t* labels, int32_t n_seg,
                       int32_t train_count);
/* Deterministic synthetic SWB-shaped dataset generated on the device. */
int adpsgd_synth_dataset(adpsgd_ctx* ctx, int32_t n_seg, int32_t train_count, uint64_t seed);
int adpsgd_get_dataset(adpsgd_ctx* ctx, float* feats, int32_t* labels);
/* fp64 host mirrors of learner weights (init_learners, engine.cpp:99-116, runs at create). */
int adpsgd_set_weights(adpsgd_ctx* ctx, int32_t local_learner, const double* w, int64_t n);
int adpsgd_get_weights(adpsgd_ctx* ctx, int32_t local_learner, double* w, int64_t n);

/* ---- the per-learner step ---- */
/* One iteration k of cfg.strategy for every local learner: sample M segments from the
 * learner's stream (engine.cpp:17-21), BLSTM forward/backward on the device, then the
 * mixing+update (engine.cpp:136-204). loss_out[local_learners] = batch-mean CE (nullable).
 * taus (GENERIC) = per-global-learner staleness, nullable. */
int adpsgd_step(adpsgd_ctx* ctx, double lr, const int32_t* taus, float* loss_out);
/* Same step, batch supplied by the caller in HOST memory: feats [local][M][T][input_dim],
 * labels [local][M][T]; copied H2D inside (the end-to-end path). */
int adpsgd_step_host_batch(adpsgd_ctx* ctx, double lr, const float* feats, const int32_t* labels,
                           float* loss_out);
/* Data-loader prefetch for the host-batch step (one local learner per context): queue the H2D
 * copy of a batch on a copy stream so it overlaps the current step; the next
 * adpsgd_step_host_batch with the same two pointers uses it instead of copying. At most two
 * batches in flight; the caller keeps the host memory unchanged until that step. */
int adpsgd_prefetch_host_batch(adpsgd_ctx* ctx, const float* feats, const int32_t* labels);
/* Gradient-injection step: grads [local_learners][D] fp64 replace the LSTM gradient. */
int adpsgd_step_injected(adpsgd_ctx* ctx, double lr, const int32_t* taus, const double* grads);
/* Objective::gradient adapter (objectives.hpp:50-51): loss and gradient at w over the
 * given segment indices, computed on the device; does not touch learner state. */
int adpsgd_gradient(adpsgd_ctx* ctx, const double* w, const int32_t* idx, int32_t M, double* g_out,
                    double* loss_out);
/* Straggler hook (chronos.cpp:51-58): local learner's step is stretched by factor >= 1
 * with a device-side delay of (factor-1) x its measured compute time. */
int adpsgd_set_straggler(adpsgd_ctx* ctx, int32_t local_learner, double factor);
int adpsgd_get_stats(adpsgd_ctx* ctx, adpsgd_perf* out);
int64_t adpsgd_iteration(adpsgd_ctx* ctx);
int adpsgd_set_iteration(adpsgd_ctx* ctx, int64_t k);
/* Consensus distance ||W (I - 11^T/L)||_2 over the local learners (mixing.cpp:159-180),
 * Gram of the deviations reduced on the device. */
int adpsgd_consensus_distance(adpsgd_ctx* ctx, double* out);
/* Mean frame cross-entropy at w over M segments (any M; heldout / full-train evaluation,
 * objectives.hpp:55-56, engine.cpp:291-293). Forward only, on the device. */
int adpsgd_eval_loss(adpsgd_ctx* ctx, const double* w, const int32_t* idx, int32_t M, double* loss_out);
/* engine.cpp:124-128 averaged_model over the local learners (fp64 host vector). */
int adpsgd_averaged_model(adpsgd_ctx* ctx, double* out, int64_t n);
/* Multi-rank consensus distance (mixing.cpp:159-180 with one learner per GPU): the L x L Gram
 * (row-major, L = cfg.learners) of every global learner's deviation from the learner mean over
 * parameters [begin, end) -- local models and peers mapped over NVLink (adpsgd_import_ipc). Each
 * rank computes its shard, the shards are summed across ranks, then adpsgd_consensus_from_gram. */
int adpsgd_consensus_gram(adpsgd_ctx* ctx, int64_t begin, int64_t end, double* gram);
/* sqrt(largest eigenvalue) of a symmetric PSD L x L Gram (L <= 16). */
int adpsgd_consensus_from_gram(const double* gram, int32_t L, double* out);
/* averaged_model over ALL global learners (mapped peers included), fp64, learner order. */
int adpsgd_averaged_model_all(adpsgd_ctx* ctx, double* out, int64_t n);

/* chronos::coupled_async (chronos.cpp:178-299) on the device: FM/RM learners iterate at their
 * own rates (durations[l] seconds per update = max(compute_l x straggler_l, comm_pairwise),
 * chronos.cpp:51-58, 207), each update mixing with the neighbours' latest publications strictly
 * before its time; `target` updates in the reference's event order. lr of update round r is
 * lr_per_epoch[r / ipe] (no clamp, chronos.cpp:216: a fast learner can run past cfg.epochs x ipe
 * rounds, so the table must cover (target - 1) / ipe + 1 epochs, else ADPSGD_E_CONFIG).
 * event_learner / event_time (nullable, length target) receive the event log. */
int adpsgd_async_run(adpsgd_ctx* ctx, int32_t strategy, const double* durations, int64_t target, int32_t ipe,
                     const double* lr_per_epoch, int32_t n_epochs, int32_t* event_learner, double* event_time,
                     int64_t* processed);

/* The RunRecord of a coupled run (chronos.cpp:271-289): after every L updates the consensus
 * distance of the learners' current models (mixing.cpp:159-180); after every L x ipe updates the
 * held-out and full-train loss of their average, and the divergence rule (non-finite, or more than
 * 10 x initial_heldout, engine.cpp:291-299) that stops the run. Inputs first, then outputs. */
typedef struct adpsgd_async_record {
    const int32_t* heldout_idx; /* segments of the held-out split (may be NULL with n_heldout 0) */
    int32_t n_heldout;
    const int32_t* train_idx;   /* segments of the full training split */
    int32_t n_train;
    double initial_heldout;     /* held-out loss of the initial averaged model */
    double* consensus;          /* out [cap_iters]: k = updates / L - 1 */
    int64_t cap_iters;
    double* heldout;            /* out [cap_epochs] */
    double* train;              /* out [cap_epochs] */
    int32_t cap_epochs;
    int64_t n_iters;            /* out: consensus points written */
    int32_t n_epochs;           /* out: epoch points written */
    int32_t diverged_epoch;     /* out: -1, or the epoch whose held-out loss diverged (run stopped) */
} adpsgd_async_record;
int adpsgd_async_run_record(adpsgd_ctx* ctx, int32_t strategy, const double* durations, int64_t target, int32_t ipe,
                            const double* lr_per_epoch, int32_t n_epochs, int32_t* event_learner, double* event_time,
                            adpsgd_async_record* record, int64_t* processed);

/* ---- single-process multi-GPU drop-in (engine.cpp:212-304 drives all L learners from one process) ----
 * Link n contexts that together host learners [0, L) (typically one context per GPU, each with the same
 * config but its own device / first_learner / local_learners): every context then reads the others'
 * weights (and, for SDPSGD, gradients) in place -- direct NVLink peer loads after
 * cudaDeviceEnablePeerAccess, no IPC, no NCCL. */
int adpsgd_group_link(adpsgd_ctx* const* ctxs, int32_t n);
/* One iteration k of every linked context, the GPUs running concurrently: all gradient computes are
 * launched, then all mixes / updates (SDPSGD's waits on the other contexts' gradients by CUDA events),
 * then all are joined. loss_out[cfg.learners] (nullable) in global learner order. */
int adpsgd_group_step(adpsgd_ctx* const* ctxs, int32_t n, double lr, float* loss_out);

/* ---- free-running asynchronous FM / RM across processes (one learner per process) ----
 * chronos::coupled_async's semantics on real clocks (chronos.cpp:171-176, 237-259): every learner
 * iterates at its own rate with no barrier, mixing with its ring neighbours' latest *published*
 * models -- w <- (w + p_L + p_R)/3 - lr g, chronos.cpp:256 -- and publishing the result into a ring
 * of 4 versioned buffers (4 publications kept, chronos.cpp:258-259) exported over CUDA IPC. Version
 * counters are device memory read with ld.acquire.sys / written with st.release.sys; a reader whose
 * chosen slot a neighbour started overwriting before its mix finished (torn read) redoes the mix.
 * RM pairs by the learner's own round (chronos.cpp:228). */
typedef enum adpsgd_async_mode {
    ADPSGD_ASYNC_FREE = 0,      /* latest publication, never wait (the paper's asynchronous ADPSGD) */
    ADPSGD_ASYNC_LOCKSTEP = 1,  /* exactly the neighbours' version k (waits): equals synchronous FM/RM */
    ADPSGD_ASYNC_BOUNDED = 2    /* latest publication, waiting until it is >= k - max_lag */
} adpsgd_async_mode;

typedef struct adpsgd_async_info {
    int64_t version;        /* this learner's model version after the step (its round count) */
    int64_t left_version;   /* neighbour versions mixed with */
    int64_t right_version;
    int32_t left, right;    /* global ids of the neighbours */
    int32_t retries;        /* torn-read retries of the mix */
    int32_t reserved;
    double wait_ms;         /* device time the select kernel waited for neighbours */
    double step_ms;         /* device time of the whole step */
} adpsgd_async_info;

/* Switch this context (one local learner, FM or RM) to the 4-slot publication ring; call before
 * adpsgd_export_ipc. timeout_s bounds every wait for a neighbour (ADPSGD_E_INVALID_STATE on expiry). */
int adpsgd_async_init(adpsgd_ctx* ctx, int32_t mode, int32_t max_lag, double timeout_s);
/* One free-running iteration of this learner: sample, forward/backward, select neighbour versions,
 * mix + update into the next slot, publish. info (nullable) describes what was mixed. */
int adpsgd_async_step(adpsgd_ctx* ctx, double lr, float* loss_out, adpsgd_async_info* info);
/* Fixed extra time per step for a local learner (emulated compute for straggler studies), as a
 * device spin after the gradient (on_host = 0) or a host sleep after the step (on_host = 1, for
 * processes sharing one GPU). The straggler factor (adpsgd_set_straggler) then stretches measured
 * compute + this delay, on the same side. */
int adpsgd_set_step_delay(adpsgd_ctx* ctx, int32_t local_learner, double ms, int32_t on_host);

/* ---- multi-process (one process per GPU) ---- */
/* NCCL communicator over all ranks; nccl_id = 128-byte ncclUniqueId from rank 0.
 * nccl_id = NULL: CUDA-IPC-only transport (FM / RM / D1D by peer reads; no device barrier, so the caller
 * separates steps with a host barrier) for ranks that share one GPU, where NCCL refuses
 * duplicate devices. */
int adpsgd_nccl_unique_id(void* out128);
int adpsgd_comm_init(adpsgd_ctx* ctx, int32_t rank, int32_t world, const void* nccl_id128);
/* CUDA IPC handles of this context's weight buffers, for peer (NVLink P2P) gossip pulls. */
int64_t adpsgd_ipc_handle_size(adpsgd_ctx* ctx);
int adpsgd_export_ipc(adpsgd_ctx* ctx, void* out, int64_t size);
int adpsgd_import_ipc(adpsgd_ctx* ctx, int32_t rank, int32_t rank_first_learner,
                      int32_t rank_local_learners, const void* handles, int64_t size);
/* Gossip transport for FM/RM: 0 = direct peer loads inside the fused mix kernel,
 * 1 = copy-engine prefetch overlapped with compute, 2 = NCCL send/recv (baseline). */
int adpsgd_set_gossip_mode(adpsgd_ctx* ctx, int32_t mode);
/* Gossip bandwidth probe (bench): `reps` timed runs (CUDA events) of the fused FM/RM mix kernel reading
 * global learners `left` and `right`'s current weights -- local, or peers mapped over NVLink P2P --
 * and of a copy-engine pull of both, into scratch buffers (learner state untouched). left = right = -1:
 * two local stand-in buffers (the N = 1, HBM-only figure). out[0] = mix ms per call, out[1] = neighbour
 * bytes per call that crossed NVLink, out[2] = copy ms per call (both neighbours), out[3] = HBM +
 * NVLink bytes the mix kernel moves per call. */
int adpsgd_gossip_probe(adpsgd_ctx* ctx, int32_t left, int32_t right, int32_t reps, double* out4);
int adpsgd_barrier(adpsgd_ctx* ctx);

/* ---- live kernel profiling (CUDA events around every library launch) ---- */
/* Kernel classes: tcgen05 GEMMs 0 recurrent fwd, 1 BPTT dgrad, 2 weight grads, 3 input dgrad,
 * 4 output/projection fwd; 5 SIMT GEMM, 6 LSTM cell, 7 softmax-CE, 8 reductions, 9 batch
 * gather, 10 mixing/update/shadow, 11 other. */
#define ADPSGD_PROF_NCAT 12
int adpsgd_profile_enable(int32_t on);
/* Synchronises the device; returns per-class device ms, algorithmic FLOPs, algorithmic
 * bytes and launch counts accumulated since the last read, then clears them. */
int adpsgd_profile_read(double* ms, double* flops, double* bytes, int64_t* launches, int32_t ncat);

/* Kernel variants selected so far (tcgen05 template instantiations, host-side record at eager launch or
 * graph capture): "name=count;..." written to out (NUL-terminated, truncated to n bytes); reset != 0
 * clears the record. Lets tests assert which kernel a shape exercised. */
int adpsgd_kernel_variants(char* out, size_t n, int32_t reset);

/* Debug: device timeline of the CTA-pair tensor-core kernels (160 CTAs x 32 globaltimer stamps). */
int adpsgd_debug_trace(int32_t enable, uint64_t* out, int32_t n);
/* Diagnosis: copy an internal activation buffer of learner 0 to host (which: 0 = X0, 1 + l = layer
 * l output H, 100 = Y, 101 = row_loss, 102 = bf16 shadow, 103 = last fp32 gradient, 200 + l = layer l cell state c,
 * 300 + l = layer l gates); bytes clipped to the buffer. */
int adpsgd_debug_buffer(adpsgd_ctx* ctx, int32_t which, void* out, size_t bytes);
/* Diagnosis: device address and size of an engine buffer (which as adpsgd_debug_buffer; 400 / 401 =
 * the BPTT dH ping-pong buffers), to attribute sanitizer reports. */
int adpsgd_debug_buffer_range(adpsgd_ctx* ctx, int32_t which, uint64_t* addr, uint64_t* bytes);

/* ---- kernel-level entry points (tests / benchmarks; device pointers) ---- */
/* C[M,N] = alpha * sum_k A(m,k) B(n,k) (+ C if accumulate) (+ bias[n]).
 * A(m,k) = a_mn ? A[k*lda+m] : A[m*lda+k]; B likewise. bf16 = 1: A,B bf16, tcgen05;
 * bf16 = 0: fp32 SIMT. c_bf16 selects the output type. */
int adpsgd_gemm(int32_t bf16, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_mn,
                const void* B, int64_t ldb, int32_t b_mn, void* Cout, int64_t ldc, int32_t c_bf16,
                float alpha, int32_t accumulate, const float* bias, void* stream);
/* w_out = (w_self + w_left + w_right)/3 - lr*g, also writes a bf16 shadow (nullable). */
int adpsgd_mix_update(int64_t n, const float* w_self, const float* w_left, const float* w_right,
                      const float* g, float lr, float* w_out, void* shadow_bf16, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADPSGD_B200_H */
